// salus_kernel.cu — the persistent Salus execution-service kernel.
//
// One CTA per SM, launched cooperatively (all CTAs co-resident).  CTA 0's
// first warp is the scheduler (scheduler.cuh); CTAs 1..N are workers
// (worker.cuh).  The kernel lives for the whole trace: "a singleton
// execution service which consolidates all GPU accesses".
#include <cuda_runtime.h>
#include <stdio.h>
#include "salus_dev.h"
#include "scheduler.cuh"
#include "worker.cuh"

namespace salus {

__global__ void __launch_bounds__(WORKER_THREADS, 1) salus_persistent_kernel(Params P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (blockIdx.x == 0) {
    if (threadIdx.x < 32) {
      Sched s(P, *reinterpret_cast<SchedShared *>(smem_raw));
      s.run();
    }
    return;
  }
  run_worker(P, smem_raw);
}

size_t kernel_smem_bytes() {
  size_t w = sizeof(WorkerSmem) + 1024;
  size_t s = sizeof(SchedShared) + 16;
  return w > s ? w : s;
}

// Launch on `stream`; returns cudaError_t as int.
int launch_persistent(const Params &P, uint32_t grid, cudaStream_t stream) {
  const size_t smem = kernel_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(salus_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  void *args[] = {const_cast<Params *>(&P)};
  e = cudaLaunchCooperativeKernel((const void *)salus_persistent_kernel, dim3(grid), dim3(WORKER_THREADS), args,
                                  smem, stream);
  return (int)e;
}

int max_coresident_grid(int device, int *grid) {
  int sms = 0, per_sm = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return (int)e;
  const size_t smem = kernel_smem_bytes();
  e = cudaFuncSetAttribute(salus_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, salus_persistent_kernel, WORKER_THREADS, smem);
  if (e != cudaSuccess) return (int)e;
  *grid = sms * (per_sm > 0 ? 1 : 0);
  return 0;
}

}  // namespace salus
