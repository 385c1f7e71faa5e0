// Batched epipolar residual / gradient kernels of the Global Alignment stage.
//
// Replaces the reference's per-pair native loops pkg/src/epialign/_kernels_cy.pyx:26-54
// (pair_residuals) and :57-116 (pair_accumulate), which the aligner calls once per image
// pair from a host thread pool (pkg/src/epialign/aligner.py:190-207, :209-278).  Here one
// launch covers every pair: one CTA per pair, threads strided over its correspondences,
// fp64 arithmetic with the reference's formulas and thresholds (LINE_NORMAL_EPS = 1e-12,
// GRAD_DEADZONE = 1e-9), deterministic fixed-order block reductions.
#include "../../include/vx_api.h"
#include "epipolar.cuh"
#include "host_util.h"

namespace vx {

__global__ void __launch_bounds__(EPI_THREADS) epipolar_residuals_kernel(
    const double* __restrict__ F, const int64_t* __restrict__ off, const double* __restrict__ xi,
    const double* __restrict__ xj, int mode, double* __restrict__ e, int32_t* __restrict__ n_deg) {
  const int p = blockIdx.x;
  double f[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) f[q] = F[9 * p + q];
  int deg = 0;
  for (int64_t m = off[p] + threadIdx.x; m < off[p + 1]; m += EPI_THREADS) e[m] = epi_residual(f, xi, xj, m, mode, deg);
  __shared__ int sdeg[EPI_THREADS / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) deg += __shfl_xor_sync(0xffffffff, deg, o);
  if ((threadIdx.x & 31) == 0) sdeg[threadIdx.x >> 5] = deg;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < EPI_THREADS / 32; ++w) t += sdeg[w];
    n_deg[p] = t;
  }
}

// out[p] = {loss_sum, weight_sum, G00..G22}
__global__ void __launch_bounds__(EPI_THREADS) epipolar_accumulate_kernel(
    const double* __restrict__ F, const int64_t* __restrict__ off, const double* __restrict__ xi,
    const double* __restrict__ xj, const double* __restrict__ w, int mode, double* __restrict__ out,
    int32_t* __restrict__ n_skipped) {
  const int p = blockIdx.x;
  double f[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) f[q] = F[9 * p + q];
  double acc[11];
#pragma unroll
  for (int q = 0; q < 11; ++q) acc[q] = 0.0;
  int skipped = 0;
  epi_accumulate<EPI_THREADS>(f, xi, xj, w, off[p], off[p + 1], mode, acc, skipped);
  __shared__ double red[EPI_THREADS / 32][12];
  epi_block_reduce<EPI_THREADS>(acc, skipped, red);
  if (threadIdx.x < 11) out[11 * (int64_t)p + threadIdx.x] = red[0][threadIdx.x];
  else if (threadIdx.x == 11) n_skipped[p] = int32_t(red[0][11]);
}

}  // namespace vx

extern "C" int vx_epipolar_residuals(const double* F, const int64_t* offsets, const double* xy_i, const double* xy_j,
                                     int num_pairs, int mode, double* e, int32_t* n_deg, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(num_pairs >= 0 && (mode == 0 || mode == 1), "vx_epipolar_residuals: bad args");
  if (num_pairs == 0) return VX_OK;
  VX_CHECK_ARG(F && offsets && xy_i && xy_j && e && n_deg, "vx_epipolar_residuals: null pointer");
  epipolar_residuals_kernel<<<num_pairs, EPI_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      F, offsets, xy_i, xy_j, mode, e, n_deg);
  VX_CHECK_LAUNCH("epipolar residuals launch");
  return VX_OK;
}

extern "C" int vx_epipolar_accumulate(const double* F, const int64_t* offsets, const double* xy_i, const double* xy_j,
                                      const double* w, int num_pairs, int mode, double* out, int32_t* n_skipped,
                                      void* stream) {
  using namespace vx;
  VX_CHECK_ARG(num_pairs >= 0 && (mode == 0 || mode == 1), "vx_epipolar_accumulate: bad args");
  if (num_pairs == 0) return VX_OK;
  VX_CHECK_ARG(F && offsets && xy_i && xy_j && w && out && n_skipped, "vx_epipolar_accumulate: null pointer");
  epipolar_accumulate_kernel<<<num_pairs, EPI_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      F, offsets, xy_i, xy_j, w, mode, out, n_skipped);
  VX_CHECK_LAUNCH("epipolar accumulate launch");
  return VX_OK;
}
