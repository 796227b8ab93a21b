// Microbenchmark: how bulk copies overlap inside one SM's TMA unit.  Issue K
// 16 KiB cp.async.bulk copies back to back (own mbarrier each, or one shared
// barrier), then wait for all; time per burst on an L2-resident and on an
// HBM-resident (> L2) source.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o burst_bench burst_bench.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// lanes = 1: thread 0 issues all K copies; lanes = K: lane k issues copy k
__global__ void __launch_bounds__(32, 1) burst_lanes(const uint8_t *src, uint64_t src_bytes, int K, int CHB, int reps,
                                                     unsigned long long *out_ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[16];
  const int l = threadIdx.x;
  if (l < 16) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[l])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const uint64_t nch = src_bytes / CHB;
  uint64_t tot = 0;
  for (int r = 0; r < reps; r++) {
    __syncwarp();
    const uint64_t t0 = gt();
    if (l < K) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[l])), "r"(CHB));
      const uint64_t c = ((uint64_t)blockIdx.x * 104729 + (uint64_t)r * 7919 + l * 31) % nch;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(smem + l * CHB)), "l"(src + c * CHB), "r"(CHB), "r"(sa(&bar[l])) : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(sa(&bar[l])), "r"(r & 1));
    }
    __syncwarp();
    tot += gt() - t0;
  }
  if (l == 0) out_ns[blockIdx.x] = tot / reps;
}

__global__ void __launch_bounds__(32, 1) burst(const uint8_t *src, uint64_t src_bytes, int K, int CHB, int shared_bar,
                                               int reps, unsigned long long *out_ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < 16; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const uint64_t nch = src_bytes / CHB;
  uint64_t tot = 0;
  for (int r = 0; r < reps; r++) {
    const uint64_t t0 = gt();
    if (shared_bar) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[0])), "r"(K * CHB));
    for (int k = 0; k < K; k++) {
      uint64_t *b = shared_bar ? &bar[0] : &bar[k];
      if (!shared_bar) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(CHB));
      const uint64_t c = ((uint64_t)blockIdx.x * 104729 + (uint64_t)r * 7919 + k * 31) % nch;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(smem + k * CHB)), "l"(src + c * CHB), "r"(CHB), "r"(sa(b)) : "memory");
    }
    for (int k = 0; k < (shared_bar ? 1 : K); k++) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(sa(&bar[k])), "r"(r & 1));
    }
    tot += gt() - t0;
  }
  out_ns[blockIdx.x] = tot / reps;
}

int main() {
  for (uint64_t bytes : {32ull << 20, 4ull << 30}) {
    uint8_t *src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    unsigned long long *d, h[160];
    cudaMalloc(&d, 160 * 8);
    cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(burst_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int CHB : {16384, 32768})
      for (int K : {1, 2, 4, 6}) {
        burst_lanes<<<1, 32, 200 * 1024>>>(src, bytes, K, CHB, 50, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("src %s lanes-issue copy %5d B x %d: %7.3f us per burst (%6.1f GB/s per SM)\n",
               bytes > (1ull << 30) ? "HBM" : "L2 ", CHB, K, h[0] / 1e3, (double)K * CHB / h[0]);
      }
    for (int grid : {1})
      for (int shared_bar : {0, 1})
        for (int CHB : {8192, 16384, 32768})
          for (int K : {1, 2, 4, 6}) {
            if (K * CHB > 192 * 1024) continue;
            burst<<<grid, 32, 200 * 1024>>>(src, bytes, K, CHB, shared_bar, 50, d);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < grid; i++) avg += h[i];
            avg /= grid;
            printf("src %s grid %3d %s copy %5d B x %d: %7.3f us per burst (%6.1f GB/s per SM) %s\n",
                   bytes > (1ull << 30) ? "HBM" : "L2 ", grid, shared_bar ? "1 bar " : "K bars", CHB, K, avg / 1e3,
                   (double)K * CHB / avg, e ? cudaGetErrorString(e) : "");
          }
    cudaFree(src);
    cudaFree(d);
  }
  return 0;
}
