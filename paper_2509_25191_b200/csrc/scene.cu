// Scene-level consumers of the predictions, fp64 except the dense map:
//   vx_matched_points    pkg/src/epialign/pointcloud.py:66-130 (sample_depth, select_matched_points)
//                        with geometry.py:341-348 (unproject): one CTA per image pair, one thread
//                        per correspondence; outputs are dense per correspondence and compacted
//                        by the caller in (pair, correspondence) order;
//   vx_unproject_depth   dense depth -> world-point maps of the VGGT outputs (fp32, HBM-bound:
//                        4 B read + 12 B written per pixel, 4 pixels per thread);
//   vx_select_pairs      pairing.py:88-109 over the upper triangle of the view-angle matrix;
//   vx_pairwise_errors   metrics.py:79-118 (relative rotation / translation-direction errors).
// Per-element formulas keep the reference's evaluation order (compiled with -fmad=false).
#include <math.h>

#include "../../include/vx_api.h"
#include "common.cuh"
#include "host_util.h"

namespace vx {

constexpr double ZERO_BASELINE_TOL = 1e-9;  // metrics.py:22
constexpr double RAD2DEG = 57.295779513082323;  // np.degrees factor 180/pi

template <typename T>
VX_DEVICE double depth_at(const T* d, int64_t idx) {
  return double(d[idx]);
}

// pointcloud.py:66-88
template <typename T>
VX_DEVICE double sample_depth(const T* d, int h, int w, double u, double v) {
  const double fu = floor(u), fv = floor(v);
  // clamp in double before converting so far-away samples cannot overflow the integer cast
  const double cu0 = fmin(fmax(fu, -1.0), double(w)), cv0 = fmin(fmax(fv, -1.0), double(h));
  const int x0 = int(cu0), y0 = int(cv0);
  const int xa = min(max(x0, 0), w - 1), xb = min(max(x0 + 1, 0), w - 1);
  const int ya = min(max(y0, 0), h - 1), yb = min(max(y0 + 1, 0), h - 1);
  const double q00 = depth_at(d, (int64_t)ya * w + xa), q01 = depth_at(d, (int64_t)ya * w + xb);
  const double q10 = depth_at(d, (int64_t)yb * w + xa), q11 = depth_at(d, (int64_t)yb * w + xb);
  if (q00 > 0 && q01 > 0 && q10 > 0 && q11 > 0) {
    const double fx = u - fu, fy = v - fv;
    const double top = q00 * (1 - fx) + q01 * fx;
    const double bot = q10 * (1 - fx) + q11 * fx;
    return top * (1 - fy) + bot * fy;
  }
  // Python round() on a float64: round half to even == rint in the default rounding mode
  const double ru = fmin(fmax(rint(u), 0.0), double(w - 1)), rv = fmin(fmax(rint(v), 0.0), double(h - 1));
  const double val = depth_at(d, (int64_t)int(rv) * w + int(ru));
  return val > 0 ? val : 0.0;
}

// geometry.py:341-348: R^T (z Kinv [u v 1]^T - t)
VX_DEVICE void unproject(double u, double v, double z, const double* R, const double* t, const double* Ki,
                         double* p) {
  double x[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) x[r] = z * (Ki[3 * r] * u + Ki[3 * r + 1] * v + Ki[3 * r + 2] * 1.0) - t[r];
#pragma unroll
  for (int c = 0; c < 3; ++c) p[c] = R[c] * x[0] + R[3 + c] * x[1] + R[6 + c] * x[2];
}

template <typename T>
__global__ void __launch_bounds__(128) matched_points_kernel(
    const T* __restrict__ depth, const int64_t* __restrict__ map_off, const int32_t* __restrict__ map_hw,
    const int32_t* __restrict__ slot, const double* __restrict__ R, const double* __restrict__ t,
    const double* __restrict__ Kinv, const int32_t* __restrict__ pair_ij, const int64_t* __restrict__ offsets,
    const double* __restrict__ xy_i, const double* __restrict__ xy_j, const double* __restrict__ w, double thr,
    double* __restrict__ points, double* __restrict__ gap, int8_t* __restrict__ state) {
  const int p = blockIdx.x;
  const int i = pair_ij[2 * p], j = pair_ij[2 * p + 1];
  const int si = slot[i], sj = slot[j];
  for (int64_t m = offsets[p] + threadIdx.x; m < offsets[p + 1]; m += blockDim.x) {
    if (!(w[m] > thr)) {  // strictly greater (pointcloud.py:114)
      state[m] = 0;
      continue;
    }
    const double ui = xy_i[2 * m], vi = xy_i[2 * m + 1], uj = xy_j[2 * m], vj = xy_j[2 * m + 1];
    const double zi = sample_depth(depth + map_off[si], map_hw[2 * si], map_hw[2 * si + 1], ui, vi);
    const double zj = sample_depth(depth + map_off[sj], map_hw[2 * sj], map_hw[2 * sj + 1], uj, vj);
    if (zi <= 0 || zj <= 0) {  // also NaN-free: sample_depth never returns NaN for finite maps
      state[m] = 2;
      continue;
    }
    if (!isfinite(zi) || !isfinite(zj)) {  // geometry.unproject raises InvalidDepth
      state[m] = 3;
      continue;
    }
    double a[3], b[3];
    unproject(ui, vi, zi, R + 9 * i, t + 3 * i, Kinv + 9 * i, a);
    unproject(uj, vj, zj, R + 9 * j, t + 3 * j, Kinv + 9 * j, b);
    const double d0 = a[0] - b[0], d1 = a[1] - b[1], d2 = a[2] - b[2];
    double* o = points + 6 * m;
    o[0] = a[0];
    o[1] = a[1];
    o[2] = a[2];
    o[3] = b[0];
    o[4] = b[1];
    o[5] = b[2];
    gap[m] = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    state[m] = 1;
  }
}

// dense world points: 4 consecutive pixels of the flattened H*W image per thread (16-byte depth load,
// three 16-byte point stores when H*W % 4 == 0, scalar tail otherwise)
__global__ void unproject_depth_kernel(const float* __restrict__ depth, int S, int H, int W,
                                       const float* __restrict__ extri, const float* __restrict__ intri,
                                       float* __restrict__ out) {
  const int s = blockIdx.y;
  const int HW = H * W;
  const float* E = extri + 12 * s;
  const float* K = intri + 9 * s;
  const float fx = K[0], fy = K[4], cx = K[2], cy = K[5];
  const float ifx = 1.0f / fx, ify = 1.0f / fy;
  const float r00 = E[0], r01 = E[1], r02 = E[2], t0 = E[3];
  const float r10 = E[4], r11 = E[5], r12 = E[6], t1 = E[7];
  const float r20 = E[8], r21 = E[9], r22 = E[10], t2 = E[11];
  const int q0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (q0 >= HW) return;
  const float* dp = depth + (int64_t)s * HW;
  float* op = out + 3 * ((int64_t)s * HW);
  const bool vec = (HW % 4 == 0);
  float z[4];
  if (vec) {
    const float4 d4 = __ldcs(reinterpret_cast<const float4*>(dp + q0));
    z[0] = d4.x;
    z[1] = d4.y;
    z[2] = d4.z;
    z[3] = d4.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) z[k] = q0 + k < HW ? dp[q0 + k] : 0.0f;
  }
  int v = q0 / W, u = q0 - v * W;
  float res[12];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float x0 = z[k] * ((float(u) - cx) * ifx) - t0;
    const float x1 = z[k] * ((float(v) - cy) * ify) - t1;
    const float x2 = z[k] - t2;
    res[3 * k + 0] = r00 * x0 + r10 * x1 + r20 * x2;
    res[3 * k + 1] = r01 * x0 + r11 * x1 + r21 * x2;
    res[3 * k + 2] = r02 * x0 + r12 * x1 + r22 * x2;
    if (++u == W) {
      u = 0;
      ++v;
    }
  }
  if (vec) {
    float4* o4 = reinterpret_cast<float4*>(op + 3 * (int64_t)q0);
    __stcs(o4 + 0, make_float4(res[0], res[1], res[2], res[3]));
    __stcs(o4 + 1, make_float4(res[4], res[5], res[6], res[7]));
    __stcs(o4 + 2, make_float4(res[8], res[9], res[10], res[11]));
  } else {
    for (int k = 0; k < 4; ++k)
      if (q0 + k < HW)
        for (int c = 0; c < 3; ++c) op[3 * ((int64_t)q0 + k) + c] = res[3 * k + c];
  }
}

VX_DEVICE int64_t tri_index(int64_t n, int64_t i, int64_t j) {  // (i < j) in row-major upper-triangle order
  return i * (2 * n - i - 1) / 2 + (j - i - 1);
}

// pairing.py:88-109: forward axis = third row of R
__global__ void select_pairs_kernel(const double* __restrict__ R, int n, double thr, int8_t* __restrict__ flag,
                                    double* __restrict__ angle) {
  const int i = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j <= i || j >= n) return;
  const double* zi = R + 9 * i + 6;
  const double* zj = R + 9 * j + 6;
  const double c = fmin(fmax(zi[0] * zj[0] + zi[1] * zj[1] + zi[2] * zj[2], -1.0), 1.0);
  const double a = acos(c) * RAD2DEG;
  const int64_t k = tri_index(n, i, j);
  angle[k] = a;
  flag[k] = a <= thr;
}

VX_DEVICE void rel_pose(const double* Ri, const double* ti, const double* Rj, const double* tj, double* dR,
                        double* dt) {  // geometry.py:261-269: (Ri^T Rj, Ri^T (tj - ti))
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) dR[3 * r + c] = Ri[r] * Rj[c] + Ri[3 + r] * Rj[3 + c] + Ri[6 + r] * Rj[6 + c];
  const double d[3] = {tj[0] - ti[0], tj[1] - ti[1], tj[2] - ti[2]};
#pragma unroll
  for (int r = 0; r < 3; ++r) dt[r] = Ri[r] * d[0] + Ri[3 + r] * d[1] + Ri[6 + r] * d[2];
}

VX_DEVICE void pose_errors(const double* Rp, const double* tp, const double* Rg, const double* tg, int i, int j,
                           int gi, int gj, double& rre, double& rte, uint8_t& flag) {
  double dRp[9], dtp[3], dRg[9], dtg[3];
  rel_pose(Rp + 9 * i, tp + 3 * i, Rp + 9 * j, tp + 3 * j, dRp, dtp);
  rel_pose(Rg + 9 * gi, tg + 3 * gi, Rg + 9 * gj, tg + 3 * gj, dRg, dtg);
  // trace(dRg^T dRp), diagonal entries summed in np.trace order
  double m[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) m[c] = dRg[c] * dRp[c] + dRg[3 + c] * dRp[3 + c] + dRg[6 + c] * dRp[6 + c];
  const double tr = m[0] + m[1] + m[2];
  rre = acos(fmin(fmax((tr - 1.0) / 2.0, -1.0), 1.0)) * RAD2DEG;
  const double na = sqrt(dtp[0] * dtp[0] + dtp[1] * dtp[1] + dtp[2] * dtp[2]);
  const double nb = sqrt(dtg[0] * dtg[0] + dtg[1] * dtg[1] + dtg[2] * dtg[2]);
  if (na < ZERO_BASELINE_TOL || nb < ZERO_BASELINE_TOL) {
    rte = 0.0;
    flag = 1;
    return;
  }
  const double c = fmin(fmax((dtp[0] * dtg[0] + dtp[1] * dtg[1] + dtp[2] * dtg[2]) / (na * nb), -1.0), 1.0);
  rte = acos(c) * RAD2DEG;
  flag = 0;
}

__global__ void pairwise_errors_kernel(const double* __restrict__ Rp, const double* __restrict__ tp,
                                       const double* __restrict__ Rg, const double* __restrict__ tg,
                                       const int32_t* __restrict__ gt_of, int n, int both, double* __restrict__ rre,
                                       double* __restrict__ rte, uint8_t* __restrict__ flag) {
  const int i = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j <= i || j >= n) return;
  const int64_t k = tri_index(n, i, j) * (both ? 2 : 1);
  pose_errors(Rp, tp, Rg, tg, i, j, gt_of[i], gt_of[j], rre[k], rte[k], flag[k]);
  if (both) pose_errors(Rp, tp, Rg, tg, j, i, gt_of[j], gt_of[i], rre[k + 1], rte[k + 1], flag[k + 1]);
}

}  // namespace vx

extern "C" int vx_matched_points(const void* depth, int depth_f32, const int64_t* map_offset, const int32_t* map_hw,
                                 const int32_t* slot, const double* R, const double* t, const double* Kinv,
                                 const int32_t* pair_ij, const int64_t* offsets, int n_pairs, const double* xy_i,
                                 const double* xy_j, const double* w, double threshold, double* points, double* gap,
                                 int8_t* state, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(n_pairs >= 0, "vx_matched_points: bad pair count");
  if (n_pairs == 0) return VX_OK;
  VX_CHECK_ARG(depth && map_offset && map_hw && slot && R && t && Kinv && pair_ij && offsets && xy_i && xy_j && w &&
                   points && gap && state,
               "vx_matched_points: null pointer");
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (depth_f32)
    matched_points_kernel<float><<<n_pairs, 128, 0, st>>>(static_cast<const float*>(depth), map_offset, map_hw, slot,
                                                          R, t, Kinv, pair_ij, offsets, xy_i, xy_j, w, threshold,
                                                          points, gap, state);
  else
    matched_points_kernel<double><<<n_pairs, 128, 0, st>>>(static_cast<const double*>(depth), map_offset, map_hw,
                                                           slot, R, t, Kinv, pair_ij, offsets, xy_i, xy_j, w,
                                                           threshold, points, gap, state);
  VX_CHECK_LAUNCH("matched points launch");
  return VX_OK;
}

extern "C" int vx_unproject_depth(const float* depth, int S, int H, int W, const float* extrinsic,
                                  const float* intrinsic, float* out, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(S >= 0 && H > 0 && W > 0 && S <= 65535 && (int64_t)H * W < (1ll << 31) - 4,
               "vx_unproject_depth: bad shape");
  if (S == 0) return VX_OK;
  VX_CHECK_ARG(depth && extrinsic && intrinsic && out, "vx_unproject_depth: null pointer");
  const int64_t quads = ((int64_t)H * W + 3) / 4;
  dim3 grid((unsigned)((quads + 255) / 256), S);
  unproject_depth_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(depth, S, H, W, extrinsic,
                                                                                  intrinsic, out);
  VX_CHECK_LAUNCH("unproject depth launch");
  return VX_OK;
}

extern "C" int vx_select_pairs(const double* R, int n, double threshold_deg, int8_t* flag, double* angle,
                               void* stream) {
  using namespace vx;
  VX_CHECK_ARG(n >= 0 && n <= 65535, "vx_select_pairs: bad frame count");
  if (n < 2) return VX_OK;
  VX_CHECK_ARG(R && flag && angle, "vx_select_pairs: null pointer");
  dim3 grid((n + 127) / 128, n);
  select_pairs_kernel<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(R, n, threshold_deg, flag, angle);
  VX_CHECK_LAUNCH("select pairs launch");
  return VX_OK;
}

extern "C" int vx_pairwise_errors(const double* Rp, const double* tp, const double* Rg, const double* tg,
                                  const int32_t* gt_of, int n, int order_invariant, double* rre, double* rte,
                                  uint8_t* zero_baseline, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(n >= 0 && n <= 65535, "vx_pairwise_errors: bad frame count");
  if (n < 2) return VX_OK;
  VX_CHECK_ARG(Rp && tp && Rg && tg && gt_of && rre && rte && zero_baseline, "vx_pairwise_errors: null pointer");
  dim3 grid((n + 127) / 128, n);
  pairwise_errors_kernel<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(Rp, tp, Rg, tg, gt_of, n,
                                                                                  order_invariant, rre, rte,
                                                                                  zero_baseline);
  VX_CHECK_LAUNCH("pairwise errors launch");
  return VX_OK;
}
