// Batched epipolar residual / gradient kernels of the Global Alignment stage.
//
// Replaces the reference's per-pair native loops pkg/src/epialign/_kernels_cy.pyx:26-54
// (pair_residuals) and :57-116 (pair_accumulate), which the aligner calls once per image
// pair from a host thread pool (pkg/src/epialign/aligner.py:190-207, :209-278).  Here one
// launch covers every pair: one CTA per pair, threads strided over its correspondences,
// fp64 arithmetic with the reference's formulas and thresholds (LINE_NORMAL_EPS = 1e-12,
// GRAD_DEADZONE = 1e-9), deterministic fixed-order block reductions.
#include <math.h>

#include "../../include/vx_api.h"
#include "common.cuh"
#include "host_util.h"

namespace vx {

constexpr double LINE_EPS = 1e-12;
constexpr double DEADZONE = 1e-9;
constexpr int EPI_THREADS = 128;

VX_DEVICE double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}

__global__ void __launch_bounds__(EPI_THREADS) epipolar_residuals_kernel(
    const double* __restrict__ F, const int64_t* __restrict__ off, const double* __restrict__ xi,
    const double* __restrict__ xj, int mode, double* __restrict__ e, int32_t* __restrict__ n_deg) {
  const int p = blockIdx.x;
  const double* f = F + 9 * p;
  const double f00 = f[0], f01 = f[1], f02 = f[2], f10 = f[3], f11 = f[4], f12 = f[5], f20 = f[6], f21 = f[7],
               f22 = f[8];
  int deg = 0;
  for (int64_t m = off[p] + threadIdx.x; m < off[p + 1]; m += EPI_THREADS) {
    const double u = xi[2 * m], v = xi[2 * m + 1];
    const double l0 = f00 * u + f01 * v + f02;
    const double l1 = f10 * u + f11 * v + f12;
    const double l2 = f20 * u + f21 * v + f22;
    const double s = xj[2 * m] * l0 + xj[2 * m + 1] * l1 + l2;
    if (mode == 0) {
      e[m] = fabs(s);
    } else {
      const double n = sqrt(l0 * l0 + l1 * l1);
      if (n < LINE_EPS) {
        e[m] = NAN;
        ++deg;
      } else {
        e[m] = fabs(s) / n;
      }
    }
  }
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
  const double* f = F + 9 * p;
  const double f00 = f[0], f01 = f[1], f02 = f[2], f10 = f[3], f11 = f[4], f12 = f[5], f20 = f[6], f21 = f[7],
               f22 = f[8];
  double acc[11];
#pragma unroll
  for (int q = 0; q < 11; ++q) acc[q] = 0.0;
  int skipped = 0;
  for (int64_t m = off[p] + threadIdx.x; m < off[p + 1]; m += EPI_THREADS) {
    const double u = xi[2 * m], v = xi[2 * m + 1];
    const double up = xj[2 * m], vp = xj[2 * m + 1];
    const double l0 = f00 * u + f01 * v + f02;
    const double l1 = f10 * u + f11 * v + f12;
    const double l2 = f20 * u + f21 * v + f22;
    const double s = up * l0 + vp * l1 + l2;
    double n, err;
    if (mode == 0) {
      n = 1.0;
      err = fabs(s);
    } else {
      n = sqrt(l0 * l0 + l1 * l1);
      if (n < LINE_EPS) {
        ++skipped;
        continue;
      }
      err = fabs(s) / n;
    }
    const double wk = w[m];
    acc[0] += wk * err;
    acc[1] += wk;
    if (err < DEADZONE) continue;
    const double sgn = s > 0 ? 1.0 : (s < 0 ? -1.0 : 0.0);
    const double c1 = wk * sgn / n;
    acc[2] += c1 * up * u;
    acc[3] += c1 * up * v;
    acc[4] += c1 * up;
    acc[5] += c1 * vp * u;
    acc[6] += c1 * vp * v;
    acc[7] += c1 * vp;
    acc[8] += c1 * u;
    acc[9] += c1 * v;
    acc[10] += c1;
    if (mode == 1) {
      const double c2 = wk * fabs(s) / (n * n * n);
      acc[2] -= c2 * l0 * u;
      acc[3] -= c2 * l0 * v;
      acc[4] -= c2 * l0;
      acc[5] -= c2 * l1 * u;
      acc[6] -= c2 * l1 * v;
      acc[7] -= c2 * l1;
    }
  }
  __shared__ double sacc[EPI_THREADS / 32][12];
#pragma unroll
  for (int q = 0; q < 11; ++q) acc[q] = warp_sum(acc[q]);
#pragma unroll
  for (int o = 16; o; o >>= 1) skipped += __shfl_xor_sync(0xffffffff, skipped, o);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int q = 0; q < 11; ++q) sacc[threadIdx.x >> 5][q] = acc[q];
    sacc[threadIdx.x >> 5][11] = double(skipped);
  }
  __syncthreads();
  if (threadIdx.x < 12) {
    double t = 0.0;
    for (int wq = 0; wq < EPI_THREADS / 32; ++wq) t += sacc[wq][threadIdx.x];
    if (threadIdx.x < 11) out[11 * (int64_t)p + threadIdx.x] = t;
    else n_skipped[p] = int32_t(t);
  }
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
