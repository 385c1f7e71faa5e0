// Per-correspondence epipolar arithmetic shared by the batched GA kernels (epipolar.cu) and the
// on-device optimiser (ga.cu).  Formulas and thresholds follow pkg/src/epialign/_kernels_cy.pyx
// (:26-54 residuals, :57-116 accumulate); compile with -fmad=false like the reference's x86 code.
#pragma once
#include <math.h>

#include "common.cuh"

namespace vx {

constexpr double EPI_LINE_EPS = 1e-12;  // _kernels_cy.pyx:12
constexpr double EPI_DEADZONE = 1e-9;   // _kernels_cy.pyx:13
constexpr int EPI_THREADS = 128;

VX_DEVICE double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}

// residual of correspondence m under F (row-major 3x3); NaN + ++deg for degenerate lines
VX_DEVICE double epi_residual(const double* f, const double* __restrict__ xi, const double* __restrict__ xj,
                              int64_t m, int mode, int& deg) {
  const double u = xi[2 * m], v = xi[2 * m + 1];
  const double l0 = f[0] * u + f[1] * v + f[2];
  const double l1 = f[3] * u + f[4] * v + f[5];
  const double l2 = f[6] * u + f[7] * v + f[8];
  const double s = xj[2 * m] * l0 + xj[2 * m + 1] * l1 + l2;
  if (mode == 0) return fabs(s);
  const double n = sqrt(l0 * l0 + l1 * l1);
  if (n < EPI_LINE_EPS) {
    ++deg;
    return NAN;
  }
  return fabs(s) / n;
}

// one correspondence's contribution to acc = {loss_sum, weight_sum, G00..G22}; branch-free so that
// several correspondences' loads can be in flight (skipped lines / dead-zone entries add exact zeros)
template <int MODE>
VX_DEVICE void epi_accum_one(const double* f, double2 xi, double2 xj, double wk, double acc[11], int& skipped) {
  constexpr int mode = MODE;
  const double u = xi.x, v = xi.y, up = xj.x, vp = xj.y;
  const double l0 = f[0] * u + f[1] * v + f[2];
  const double l1 = f[3] * u + f[4] * v + f[5];
  const double l2 = f[6] * u + f[7] * v + f[8];
  const double s = up * l0 + vp * l1 + l2;
  const double n = mode == 0 ? 1.0 : sqrt(l0 * l0 + l1 * l1);
  const bool ok = !(n < EPI_LINE_EPS);
  skipped += ok ? 0 : 1;
  // one reciprocal instead of three divisions: per-term rounding differs from the reference's
  // |s|/n, w*sgn/n, w*|s|/n^3 by an ulp, far inside the tolerance of the sums
  const double rn = 1.0 / n;
  const double as = fabs(s);
  const double err = as * rn;
  acc[0] += ok ? wk * err : 0.0;
  acc[1] += ok ? wk : 0.0;
  const bool grad = ok && !(err < EPI_DEADZONE);
  const double sgn = s > 0 ? 1.0 : (s < 0 ? -1.0 : 0.0);
  const double c1 = grad ? wk * sgn * rn : 0.0;
  // dL/dF-hat += (c1 x' - c2 l') (u, v, 1)^T with l' = (l0, l1, 0): the reference's per-term
  // updates (_kernels_cy.pyx:96-113) factored into one outer product, FMA-accumulated
  double a0 = c1 * up, a1 = c1 * vp;
  if (mode == 1) {
    const double c2 = grad ? wk * as * (rn * rn * rn) : 0.0;
    a0 -= c2 * l0;
    a1 -= c2 * l1;
  }
  acc[2] = __fma_rn(a0, u, acc[2]);
  acc[3] = __fma_rn(a0, v, acc[3]);
  acc[4] += a0;
  acc[5] = __fma_rn(a1, u, acc[5]);
  acc[6] = __fma_rn(a1, v, acc[6]);
  acc[7] += a1;
  acc[8] = __fma_rn(c1, u, acc[8]);
  acc[9] = __fma_rn(c1, v, acc[9]);
  acc[10] += c1;
}

// acc over this thread's strided share of [begin, end), 16-byte loads
template <int THREADS, int UNROLL, int MODE>
VX_DEVICE void epi_accumulate_m(const double* f, const double* __restrict__ xi, const double* __restrict__ xj,
                                const double* __restrict__ w, int64_t begin, int64_t end, double acc[11],
                                int& skipped) {
  const double2* xi2 = reinterpret_cast<const double2*>(xi);
  const double2* xj2 = reinterpret_cast<const double2*>(xj);
  int64_t m = begin + threadIdx.x;
  // UNROLL correspondences per step with all their loads issued before any arithmetic
#pragma unroll 1
  for (; m + (UNROLL - 1) * THREADS < end; m += UNROLL * THREADS) {
    double2 a[UNROLL], b[UNROLL];
    double ww[UNROLL];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      a[k] = __ldg(xi2 + m + k * THREADS);
      b[k] = __ldg(xj2 + m + k * THREADS);
      ww[k] = __ldg(w + m + k * THREADS);
    }
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) epi_accum_one<MODE>(f, a[k], b[k], ww[k], acc, skipped);
  }
#pragma unroll 1
  for (; m < end; m += THREADS) epi_accum_one<MODE>(f, __ldg(xi2 + m), __ldg(xj2 + m), __ldg(w + m), acc, skipped);
}

template <int THREADS, int UNROLL = 2>
VX_DEVICE void epi_accumulate(const double* f, const double* __restrict__ xi, const double* __restrict__ xj,
                              const double* __restrict__ w, int64_t begin, int64_t end, int mode, double acc[11],
                              int& skipped) {
  if (mode == 0) epi_accumulate_m<THREADS, UNROLL, 0>(f, xi, xj, w, begin, end, acc, skipped);
  else epi_accumulate_m<THREADS, UNROLL, 1>(f, xi, xj, w, begin, end, acc, skipped);
}

// fixed-order block reduction of acc[11] + skipped; result valid in red[0][0..11] after the call
template <int THREADS>
VX_DEVICE void epi_block_reduce(double acc[11], int skipped, double (*red)[12]) {
#pragma unroll
  for (int q = 0; q < 11; ++q) acc[q] = warp_sum_d(acc[q]);
#pragma unroll
  for (int o = 16; o; o >>= 1) skipped += __shfl_xor_sync(0xffffffff, skipped, o);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int q = 0; q < 11; ++q) red[threadIdx.x >> 5][q] = acc[q];
    red[threadIdx.x >> 5][11] = double(skipped);
  }
  __syncthreads();
  if (threadIdx.x < 12) {
    double t = 0.0;
    for (int wq = 0; wq < THREADS / 32; ++wq) t += red[wq][threadIdx.x];
    red[0][threadIdx.x] = t;  // only row 0 is rewritten; rows 1.. were fully read above by this thread
  }
  __syncthreads();
}

}  // namespace vx
