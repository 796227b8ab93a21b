// salus_kernel.cu — the persistent Salus execution-service kernel.
//
// One CTA per SM, launched cooperatively in clusters of 2 (CTA pairs on one
// TPC, all co-resident).  CTA 0's first warp is the scheduler
// (scheduler.cuh) and its cluster partner (CTA 1) exits at once; every
// other cluster is a worker pair (worker.cuh).  The kernel lives for the
// whole trace: "a singleton execution service which consolidates all GPU
// accesses".
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include "salus_dev.h"
#include "scheduler.cuh"
#include "worker.cuh"

namespace salus {

__global__ void __launch_bounds__(WORKER_THREADS, 1) salus_persistent_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (blockIdx.x == 0) {
    if (threadIdx.x < 32) {
      Sched s(P, *reinterpret_cast<SchedShared *>(smem_raw));
      s.run();
    }
    return;
  }
  if (blockIdx.x == 1) return;   // the scheduler's cluster partner
  run_worker(P, smem_raw);
}

size_t kernel_smem_bytes() {
  size_t w = sizeof(WorkerSmem);   // base is 1 KiB-aligned (checked in run_worker)
  size_t s = sizeof(SchedShared) + 16;
  return w > s ? w : s;
}

static cudaLaunchConfig_t pair_config(uint32_t grid, size_t smem, cudaStream_t stream,
                                      cudaLaunchAttribute (&attrs)[2], bool cooperative) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(WORKER_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeCooperative;
  attrs[1].val.cooperative = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = cooperative ? 2 : 1;
  return cfg;
}

// Launch on `stream`; returns cudaError_t as int.  `grid` (even) CTAs were
// checked co-resident by max_coresident_grid.
int launch_persistent(const Params &P, uint32_t grid, cudaStream_t stream) {
  const size_t smem = kernel_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(salus_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  cudaLaunchAttribute attrs[2];
  // SALUS_COOP=0 (diagnostics, e.g. under ncu, whose replay refuses
  // cooperative cluster launches): plain cluster launch; `grid` still fits
  // one wave (max_coresident_grid), so all CTAs are resident together.
  const char *coop = getenv("SALUS_COOP");
  const bool cooperative = !(coop && coop[0] == '0');
  cudaLaunchConfig_t cfg = pair_config(grid, smem, stream, attrs, cooperative);
  e = cudaLaunchKernelEx(&cfg, salus_persistent_kernel, P);
  return (int)e;
}

// Co-resident grid: 2 x the number of CTA pairs that fit at once.
int max_coresident_grid(int device, int *grid) {
  (void)device;
  const size_t smem = kernel_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(salus_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  cudaLaunchAttribute attrs[2];
  cudaLaunchConfig_t cfg = pair_config(2, smem, 0, attrs, false);
  int clusters = 0;
  e = cudaOccupancyMaxActiveClusters(&clusters, (void *)salus_persistent_kernel, &cfg);
  if (e != cudaSuccess) return (int)e;
  *grid = 2 * clusters;
  return 0;
}

}  // namespace salus
