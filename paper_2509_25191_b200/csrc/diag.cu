// Diagnostic-build-only helpers for tools/ (compiled empty into the product library).
#ifdef VX_DIAG
#include "../../include/vx_api.h"
#include "common.cuh"
#include "host_util.h"

namespace vx {
// Occupies `ctas` SMs for `cycles` SM clocks with `smem` bytes of shared memory each: stands in for an
// NCCL transfer kernel (which holds its SMs for the transfer) in tools/bench_ring_step.py.
__global__ void sm_hog_kernel(long long cycles) {
  extern __shared__ unsigned char s[];
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 0 && cycles < 0) s[0] = 1;
}
}  // namespace vx

extern "C" int vx_diag_sm_hog(int ctas, long long cycles, int smem, void* stream) {
  using namespace vx;
  cudaError_t e = cudaFuncSetAttribute(sm_hog_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return fail_cuda(e, "sm_hog attr");
  sm_hog_kernel<<<ctas, 512, smem, reinterpret_cast<cudaStream_t>(stream)>>>(cycles);
  VX_CHECK_LAUNCH("sm_hog launch");
  return VX_OK;
}
#endif
