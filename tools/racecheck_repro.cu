// racecheck_repro.cu -- minimal reproducer for the racecheck reports on the
// persistent kernel (profiles/sanitizer): a double-buffered producer /
// consumer over shared memory where the producer is a bulk copy (TMA unit)
// completing on an mbarrier and the consumer releases the buffer through a
// second mbarrier -- the exact protocol of worker.cuh's epilogue-input ring.
// The program is correct (the result is checked on the host), yet
// compute-sanitizer --tool racecheck reports a race between the bulk copy's
// write and the consumer's read: racecheck does not model the ordering an
// mbarrier's complete_tx / try_wait establishes for async-proxy writes.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o racecheck_repro racecheck_repro.cu
// run:   compute-sanitizer --tool racecheck ./racecheck_repro
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

constexpr int N = 2048;   // floats per chunk (8 KiB)

__global__ void ring(const float *src, float *out, int chunks) {
  __shared__ alignas(128) float buf[2][N];
  __shared__ uint64_t full[2], empty[2];
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; b++) { mbar_init(&full[b], 1); mbar_init(&empty[b], 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {                       // producer: one bulk copy per chunk
    for (int i = 0; i < chunks; i++) {
      const int b = i & 1;
      mbar_wait(&empty[b], ((i >> 1) & 1) ^ 1);   // the consumer released this buffer
      mbar_expect_tx(&full[b], N * 4);
      bulk_g2s(buf[b], src + (size_t)i * N, N * 4, &full[b]);
    }
  } else if (threadIdx.x >= 32 && threadIdx.x < 64) {   // consumer warp
    const int lane = threadIdx.x - 32;
    float s = 0.f;
    for (int i = 0; i < chunks; i++) {
      const int b = i & 1;
      mbar_wait(&full[b], (i >> 1) & 1);      // the chunk has landed
      for (int k = lane; k < N; k += 32) s += buf[b][k];
      __syncwarp();
      mbar_arrive(&empty[b]);                 // hand the buffer back (32 arrivals)
    }
    out[lane] = s;
  }
}

int main() {
  const int chunks = 64;
  std::vector<float> h((size_t)chunks * N);
  double want = 0;
  for (size_t i = 0; i < h.size(); i++) { h[i] = (float)(i % 7); want += h[i]; }
  float *src, *out;
  cudaMalloc(&src, h.size() * 4);
  cudaMalloc(&out, 32 * 4);
  cudaMemcpy(src, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  ring<<<1, 64>>>(src, out, chunks);
  float o[32];
  cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
  double got = 0;
  for (float x : o) got += x;
  printf("sum %.0f, expected %.0f: %s\n", got, want, got == want ? "OK" : "WRONG");
  return got == want ? 0 : 1;
}
