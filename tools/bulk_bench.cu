// Microbenchmark: per-SM throughput of global->shared async copies on B200.
// Compares cp.async.bulk (non-tensor, what the worker's operand loader
// issues) with cp.async.bulk.tensor.2d (TMA with a tensor map), for an
// L2-resident source, PIPE stages in flight, 1 CTA or one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bulk_bench bulk_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <int MODE, int PIPE, int CH, int SPIN = 0>
__global__ void __launch_bounds__(32, 1) bench(const __grid_constant__ CUtensorMap tmap, const uint8_t *src,
                                               uint64_t src_bytes, int iters, unsigned long long *out_ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[PIPE];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < PIPE; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const uint64_t nchunks = src_bytes / CH;
  const uint64_t t0 = gt();
  for (int i = 0; i < iters + PIPE; i++) {
    const int s = i % PIPE;
    if (i >= PIPE) {   // wait for the copy issued PIPE iterations ago
      const uint32_t par = ((i / PIPE) - 1) & 1;
      uint32_t ok = 0;
      if (SPIN)   // non-blocking test_wait spin
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(sa(&full[s])), "r"(par));
      else
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(sa(&full[s])), "r"(par));
    }
    if (i >= iters) continue;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(CH));
    const uint64_t c = ((uint64_t)blockIdx.x * 7919 + (uint64_t)i * 13) % nchunks;
    uint8_t *dst = smem + s * CH;
    if (MODE == 0) {          // one bulk copy per 16 KiB
      for (int q = 0; q < CH / 16384; q++)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(dst + q * 16384)), "l"(src + c * CH + q * 16384), "r"(16384), "r"(sa(&full[s])) : "memory");
    } else {                  // one 2D tensor box (128 B x 128 rows) per 16 KiB
      for (int q = 0; q < CH / 16384; q++) {
        const int row = (int)((c * CH + q * 16384) / 128);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(sa(dst + q * 16384)), "l"(&tmap), "r"(0), "r"(row), "r"(sa(&full[s])) : "memory");
      }
    }
  }
  out_ns[blockIdx.x] = gt() - t0;
}

template <int MODE, int PIPE, int CH, int SPIN = 0>
void run(const CUtensorMap &tm, const uint8_t *src, uint64_t bytes, int grid, const char *name) {
  unsigned long long *d_ns;
  cudaMalloc(&d_ns, grid * 8);
  const int iters = 4000, smem = PIPE * CH;
  cudaFuncSetAttribute(bench<MODE, PIPE, CH, SPIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<MODE, PIPE, CH, SPIN><<<grid, 32, smem>>>(tm, src, bytes, iters, d_ns);   // warm
  bench<MODE, PIPE, CH, SPIN><<<grid, 32, smem>>>(tm, src, bytes, iters, d_ns);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[1024];
  cudaMemcpy(h, d_ns, grid * 8, cudaMemcpyDeviceToHost);
  double mx = 0, sum = 0;
  for (int i = 0; i < grid; i++) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
  const double per_sm = (double)iters * CH / (sum / grid);   // bytes per ns = GB/s
  printf("%-28s grid %3d PIPE %d CH %6d: per-SM %7.1f GB/s  chip %8.1f GB/s  %s\n", name, grid, PIPE, CH, per_sm,
         (double)iters * CH * grid / mx, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d_ns);
}

int main() {
  const uint64_t bytes = 32ull << 20;   // L2-resident source
  uint8_t *src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  PFN_cuTensorMapEncodeTiled enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t gdim[2] = {128, bytes / 128};
  cuuint64_t gstr[1] = {128};
  cuuint32_t box[2] = {128, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, src, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("tensor map encode: %d\n", (int)r);
  for (int grid : {1, 148}) {
    run<0, 4, 32768, 1>(tm, src, bytes, grid, "bulk 16K x2 test_wait");
    run<0, 6, 65536, 0>(tm, src, bytes, grid, "bulk 16K x4");
    run<0, 3, 65536, 1>(tm, src, bytes, grid, "bulk 16K x4 test_wait");
    run<0, 2, 32768>(tm, src, bytes, grid, "bulk 16K x2");
    run<0, 4, 32768>(tm, src, bytes, grid, "bulk 16K x2");
    run<0, 6, 32768>(tm, src, bytes, grid, "bulk 16K x2");
    run<1, 2, 32768>(tm, src, bytes, grid, "tensor 16K x2");
    run<1, 4, 32768>(tm, src, bytes, grid, "tensor 16K x2");
    run<1, 6, 32768>(tm, src, bytes, grid, "tensor 16K x2");
    run<0, 4, 16384>(tm, src, bytes, grid, "bulk 16K");
    run<1, 4, 16384>(tm, src, bytes, grid, "tensor 16K");
  }
  return 0;
}
