// Global-Alignment optimiser on the device.
//
// The reference runs every alignment iteration as a host loop over image pairs
// (pkg/src/epialign/aligner.py:209-278: per pair, numpy 3x3 algebra + the Cython sum over its
// correspondences, dispatched through a thread pool), then a per-frame chain rule and an Adam
// step in numpy (:264-277, :408-417).  Here one iteration is four launches and the whole
// 300-iteration loop is one CUDA graph:
//   ga_geom_kernel   one thread per pair: the pair's relative pose, essential and fundamental
//                    matrices from the decoded cameras (_pair_F, :176-185);
//   ga_pair_kernel   one CTA per pair: the weighted residual / dL/dF sums over its
//                    correspondences (_kernels_cy.pyx:57-116) -> 13 doubles of a 32-double payload;
//   ga_chain_kernel  one thread per pair: the chain rule back to the pair's two cameras
//                    (:232-257), kept out of the streaming kernel so that one stays lean, and
//                    the deterministic reduction of the loss / weight sums -> loss-trace entry;
//   ga_frame_kernel  one warp per frame: its payload entries (CSR, fixed-order reduction), rot6d
//                    backward (geometry.py:216-248), gradient / den, the Adam update, and the
//                    decode of the new parameters (aligner.py:160-174) for the next iteration.
// fp64 throughout, FMA contraction disabled (-fmad=false) like the reference's numpy/x86 code.
#include <algorithm>
#include <vector>

#include "../../include/vx_api.h"
#include "epipolar.cuh"
#include "host_util.h"

namespace vx {

constexpr double GA_F_NORM_EPS = 1e-15;  // aligner.py:43
constexpr double GA_PARALLEL_TOL = 1e-12;  // geometry.py:26
constexpr double GA_BETA1 = 0.9, GA_BETA2 = 0.999, GA_EPS = 1e-8;  // aligner.py:40-42
constexpr int GA_PAYLOAD = 32;
constexpr int GA_FRAME_THREADS = 128;  // 4 frames (one warp each) per CTA

constexpr int GA_CHAIN_THREADS = 64;

// payload layout (doubles)
enum {
  PL_LOSS = 0, PL_WSUM = 1, PL_SKIP = 2, PL_VALID = 3,
  PL_GH = 4,     // dL/dF-hat sums (pair kernel), overwritten by the chain-rule kernel with:
  PL_GRJ = 4,    // G_Rrel @ R_i, added to G_R[j]
  PL_GRI = 13,   // G_Rrel^T @ R_j, added to G_R[i]
  PL_GTI = 22,   // -R_ij^T g_trel, added to g_t[i]
  PL_GTJ = 25,   // g_trel, added to g_t[j]
  PL_GSI = 28, PL_GSJ = 29
};

// ---- 3x3 helpers (row-major), numpy evaluation order: c_ij = a_i0 b_0j + a_i1 b_1j + a_i2 b_2j ----
VX_DEVICE void mm(const double* a, const double* b, double* c) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}
VX_DEVICE void mmT(const double* a, const double* b, double* c) {  // a @ b^T
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      c[3 * i + j] = a[3 * i] * b[3 * j] + a[3 * i + 1] * b[3 * j + 1] + a[3 * i + 2] * b[3 * j + 2];
}
VX_DEVICE void mTm(const double* a, const double* b, double* c) {  // a^T @ b
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[3 * i + j] = a[i] * b[j] + a[3 + i] * b[3 + j] + a[6 + i] * b[6 + j];
}
VX_DEVICE void skew(const double* v, double* s) {
  s[0] = 0.0; s[1] = -v[2]; s[2] = v[1];
  s[3] = v[2]; s[4] = 0.0; s[5] = -v[0];
  s[6] = -v[1]; s[7] = v[0]; s[8] = 0.0;
}
VX_DEVICE double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
VX_DEVICE void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

// geometry.py:188-207; returns false on a degenerate encoding
VX_DEVICE bool rot6d_decode(const double* dr, double* R) {
  const double* a = dr;
  const double* b = dr + 3;
  const double na = sqrt(dot3(a, a));
  if (na <= GA_PARALLEL_TOL) return false;
  double b1[3], u[3], b2[3], b3[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) b1[q] = a[q] / na;
  const double d = dot3(b1, b);
#pragma unroll
  for (int q = 0; q < 3; ++q) u[q] = b[q] - d * b1[q];
  const double nu = sqrt(dot3(u, u));
  if (nu <= GA_PARALLEL_TOL) return false;
#pragma unroll
  for (int q = 0; q < 3; ++q) b2[q] = u[q] / nu;
  cross3(b1, b2, b3);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    R[3 * r] = b1[r];
    R[3 * r + 1] = b2[r];
    R[3 * r + 2] = b3[r];
  }
  return true;
}

// geometry.py:216-248
VX_DEVICE void rot6d_backward(const double* dr, const double* gR, double* out) {
  const double* a = dr;
  const double* b = dr + 3;
  const double na = sqrt(dot3(a, a));
  double b1[3], u[3], b2[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) b1[q] = a[q] / na;
  const double d = dot3(b1, b);
#pragma unroll
  for (int q = 0; q < 3; ++q) u[q] = b[q] - d * b1[q];
  const double nu = sqrt(dot3(u, u));
#pragma unroll
  for (int q = 0; q < 3; ++q) b2[q] = u[q] / nu;
  const double g1[3] = {gR[0], gR[3], gR[6]}, g2[3] = {gR[1], gR[4], gR[7]}, g3[3] = {gR[2], gR[5], gR[8]};
  double c[3], h1[3], h2[3], qv[3];
  cross3(b2, g3, c);
#pragma unroll
  for (int q = 0; q < 3; ++q) h1[q] = g1[q] + c[q];
  cross3(g3, b1, c);
#pragma unroll
  for (int q = 0; q < 3; ++q) h2[q] = g2[q] + c[q];
  const double h2b2 = dot3(h2, b2);
#pragma unroll
  for (int q = 0; q < 3; ++q) qv[q] = (h2[q] - h2b2 * b2[q]) / nu;
  const double qb1 = dot3(qv, b1);
#pragma unroll
  for (int q = 0; q < 3; ++q) out[3 + q] = qv[q] - qb1 * b1[q];
  const double b1b = dot3(b1, b);
#pragma unroll
  for (int q = 0; q < 3; ++q) h1[q] = h1[q] - qb1 * b[q] - b1b * qv[q];
  const double h1b1 = dot3(h1, b1);
#pragma unroll
  for (int q = 0; q < 3; ++q) out[q] = (h1[q] - h1b1 * b1[q]) / na;
}

// aligner.py:160-174 for frame f
VX_DEVICE void decode_frame(const vx_ga_problem& pb, int f, const double* prm) {
  double dR[9], R[9];
  if (!rot6d_decode(prm, dR)) {
    atomicOr(pb.status, 1);
#pragma unroll
    for (int q = 0; q < 9; ++q) dR[q] = (q % 4 == 0) ? 1.0 : 0.0;
  }
  mm(dR, pb.base_R + 9 * f, R);
#pragma unroll
  for (int q = 0; q < 9; ++q) pb.Rs[9 * f + q] = R[q];
#pragma unroll
  for (int q = 0; q < 3; ++q) pb.ts[3 * f + q] = pb.base_t[3 * f + q] + prm[6 + q];
  const double s = pb.dim == 10 ? exp(-prm[9]) : 1.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) pb.Kinv[9 * f + q] = (pb.dim == 10 && q < 6) ? pb.base_Kinv[9 * f + q] * s
                                                                           : pb.base_Kinv[9 * f + q];
}

__global__ void ga_decode_kernel(vx_ga_problem pb) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= pb.n_frames) return;
  double prm[10];
  for (int q = 0; q < pb.dim; ++q) prm[q] = pb.params[pb.dim * f + q];
  decode_frame(pb, f, prm);
}

struct PairGeom {
  double Rij[9], tij[3], E[9], Fh[9], r;
  int valid;
};

// aligner.py:176-185 (thread 0)
VX_DEVICE void pair_geometry(const vx_ga_problem& pb, int i, int j, PairGeom& g) {
  const double* Ri = pb.Rs + 9 * i;
  const double* Rj = pb.Rs + 9 * j;
  const double* ti = pb.ts + 3 * i;
  const double* tj = pb.ts + 3 * j;
  mmT(Rj, Ri, g.Rij);
#pragma unroll
  for (int q = 0; q < 3; ++q) g.tij[q] = tj[q] - (g.Rij[3 * q] * ti[0] + g.Rij[3 * q + 1] * ti[1] + g.Rij[3 * q + 2] * ti[2]);
  double S[9], T[9], F[9];
  skew(g.tij, S);
  mm(S, g.Rij, g.E);
  mTm(pb.Kinv + 9 * j, g.E, T);
  mm(T, pb.Kinv + 9 * i, F);
  double ss = 0.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) ss += F[q] * F[q];
  g.r = sqrt(ss);
  g.valid = !(g.r < GA_F_NORM_EPS);
#pragma unroll
  for (int q = 0; q < 9; ++q) g.Fh[q] = F[q] / g.r;
}

// geometry of every pair (thread per pair) -> geom[p] = (R_ij 9, t_ij 3, E 9, F/|F| 9, |F|, valid)
constexpr int GG_RIJ = 0, GG_TIJ = 9, GG_E = 12, GG_FH = 21, GG_R = 30, GG_VALID = 31;

__global__ void ga_geom_kernel(vx_ga_problem pb) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= pb.n_pairs) return;
  PairGeom g;
  pair_geometry(pb, pb.pair_ij[2 * p], pb.pair_ij[2 * p + 1], g);
  double* o = pb.geom + 32 * (int64_t)p;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    o[GG_RIJ + q] = g.Rij[q];
    o[GG_E + q] = g.E[q];
    o[GG_FH + q] = g.Fh[q];
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) o[GG_TIJ + q] = g.tij[q];
  o[GG_R] = g.r;
  o[GG_VALID] = g.valid;
}

__global__ void __launch_bounds__(EPI_THREADS) ga_residuals_kernel(vx_ga_problem pb, double* __restrict__ e,
                                                                   int32_t* __restrict__ deg_pair,
                                                                   int32_t* __restrict__ n_deg) {
  const int p = blockIdx.x;
  __shared__ PairGeom g;
  if (threadIdx.x == 0) pair_geometry(pb, pb.pair_ij[2 * p], pb.pair_ij[2 * p + 1], g);
  __syncthreads();
  const int64_t b = pb.offsets[p], en = pb.offsets[p + 1];
  double f[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) f[q] = g.Fh[q];
  int deg = 0;
  for (int64_t m = b + threadIdx.x; m < en; m += EPI_THREADS)
    e[m] = g.valid ? epi_residual(f, pb.xy_i, pb.xy_j, m, pb.mode, deg) : NAN;
  __shared__ int sdeg[EPI_THREADS / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) deg += __shfl_xor_sync(0xffffffff, deg, o);
  if ((threadIdx.x & 31) == 0) sdeg[threadIdx.x >> 5] = deg;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < EPI_THREADS / 32; ++w) t += sdeg[w];
    deg_pair[p] = g.valid ? 0 : 1;
    n_deg[p] = g.valid ? t : int32_t(en - b);
  }
}

// per-pair sums: payload[0..12] = (loss_sum, weight_sum, skipped, valid, dL/dF-hat row-major)
template <int MODE, int THREADS, int MINB, int UNROLL>
__global__ void __launch_bounds__(THREADS, MINB) ga_pair_kernel(vx_ga_problem pb) {
  const int p = blockIdx.x;
  __shared__ double red[THREADS / 32][12];
  const double* gg = pb.geom + 32 * (int64_t)p;
  const int64_t b = pb.offsets[p], en = pb.offsets[p + 1];
  double* pl = pb.payload + (int64_t)GA_PAYLOAD * p;
  if (gg[GG_VALID] == 0.0) {  // aligner.py:223-224: the whole pair is skipped
    if (threadIdx.x < GA_PAYLOAD) pl[threadIdx.x] = threadIdx.x == PL_SKIP ? double(en - b) : 0.0;
    return;
  }
  double f[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) f[q] = gg[GG_FH + q];
  double acc[11];
#pragma unroll
  for (int q = 0; q < 11; ++q) acc[q] = 0.0;
  int skipped = 0;
  epi_accumulate_m<THREADS, UNROLL, MODE>(f, pb.xy_i, pb.xy_j, pb.w, b, en, acc, skipped);
  epi_block_reduce<THREADS>(acc, skipped, red);
  if (threadIdx.x < 2) pl[threadIdx.x] = red[0][threadIdx.x];
  else if (threadIdx.x == 2) pl[PL_SKIP] = red[0][11];
  else if (threadIdx.x == 3) pl[PL_VALID] = 1.0;
  else if (threadIdx.x < 13) pl[PL_GH + threadIdx.x - 4] = red[0][threadIdx.x - 2];
}

// chain rule back to the pair's cameras (aligner.py:232-257) for a valid pair p; reads the G-hat
// sums and overwrites them with the contributions (payload layout above)
VX_DEVICE void chain_rule(const vx_ga_problem& pb, int p) {
  double* pl = pb.payload + (int64_t)GA_PAYLOAD * p;
  const int i = pb.pair_ij[2 * p], j = pb.pair_ij[2 * p + 1];
  const double* gg = pb.geom + 32 * (int64_t)p;
  PairGeom g;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    g.Rij[q] = gg[GG_RIJ + q];
    g.E[q] = gg[GG_E + q];
    g.Fh[q] = gg[GG_FH + q];
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) g.tij[q] = gg[GG_TIJ + q];
  g.r = gg[GG_R];
  double Gh[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) Gh[q] = pl[PL_GH + q];
  const double* Ki = pb.Kinv + 9 * i;
  const double* Kj = pb.Kinv + 9 * j;
  const double* Ri = pb.Rs + 9 * i;
  const double* Rj = pb.Rs + 9 * j;
  const double* ti = pb.ts + 3 * i;
  double vd = 0.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) vd += Gh[q] * g.Fh[q];
  double Graw[9], T[9], GE[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) Graw[q] = (Gh[q] - vd * g.Fh[q]) / g.r;
  mm(Kj, Graw, T);
  mmT(T, Ki, GE);
  double gsi = 0.0, gsj = 0.0;
  if (pb.dim == 10) {
    double GB[9], GA[9], U[9];
    mTm(g.E, Kj, U);  // E^T @ Kinv_j
    mm(U, Graw, GB);
    mmT(Graw, Ki, U);  // G_raw @ Kinv_i^T
    mmT(U, g.E, GA);   // ... @ E^T
    double s1 = 0.0, s2 = 0.0;
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 3; ++c) s1 += GB[3 * r + c] * Ki[3 * r + c];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 2; ++c) s2 += GA[3 * r + c] * Kj[3 * c + r];
    gsi = -s1;
    gsj = -s2;
  }
  double M[9];
  mmT(GE, g.Rij, M);
  const double gt[3] = {M[7] - M[5], M[2] - M[6], M[3] - M[1]};
  double S[9], GRrel[9], C[9];
  skew(g.tij, S);
  mTm(S, GE, GRrel);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) GRrel[3 * r + c] -= gt[r] * ti[c];
  mm(GRrel, Ri, C);
#pragma unroll
  for (int q = 0; q < 9; ++q) pl[PL_GRJ + q] = C[q];
  mTm(GRrel, Rj, C);
#pragma unroll
  for (int q = 0; q < 9; ++q) pl[PL_GRI + q] = C[q];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    pl[PL_GTI + q] = -(g.Rij[q] * gt[0] + g.Rij[3 + q] * gt[1] + g.Rij[6 + q] * gt[2]);
    pl[PL_GTJ + q] = gt[q];
  }
  pl[PL_GSI] = gsi;
  pl[PL_GSJ] = gsj;
}

// one thread per pair: the chain rule, then num / den / skipped over all pairs — per-block partials
// in fixed order, the last block to finish sums them in block order (deterministic) and writes the
// loss-trace entry.  scalars[4 + 3b ..] hold block b's partials, status[1] counts finished blocks.
__global__ void __launch_bounds__(GA_CHAIN_THREADS) ga_chain_kernel(vx_ga_problem pb, double* trace, int t,
                                                                    double* skipped_total) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0;
  if (p < pb.n_pairs) {
    const double* pl = pb.payload + (int64_t)GA_PAYLOAD * p;
    v0 = pl[PL_LOSS];
    v1 = pl[PL_WSUM];
    v2 = pl[PL_SKIP];
    if (pl[PL_VALID] != 0.0) chain_rule(pb, p);
  }
  __shared__ double s[3][GA_CHAIN_THREADS / 32];
  __shared__ int last;
  v0 = warp_sum_d(v0);
  v1 = warp_sum_d(v1);
  v2 = warp_sum_d(v2);
  if ((threadIdx.x & 31) == 0) {
    s[0][threadIdx.x >> 5] = v0;
    s[1][threadIdx.x >> 5] = v1;
    s[2][threadIdx.x >> 5] = v2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int w = 0; w < GA_CHAIN_THREADS / 32; ++w) {
      a += s[0][w];
      b += s[1][w];
      c += s[2][w];
    }
    double* part = pb.scalars + 4 + 3 * (int64_t)blockIdx.x;
    part[0] = a;
    part[1] = b;
    part[2] = c;
    __threadfence();
    const unsigned prev = atomicAdd(reinterpret_cast<unsigned*>(pb.status + 1), 1u);
    last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  v0 = v1 = v2 = 0.0;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += GA_CHAIN_THREADS) {
    const double* part = pb.scalars + 4 + 3 * (int64_t)k;
    v0 += __ldcg(part);
    v1 += __ldcg(part + 1);
    v2 += __ldcg(part + 2);
  }
  v0 = warp_sum_d(v0);
  v1 = warp_sum_d(v1);
  v2 = warp_sum_d(v2);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    s[0][threadIdx.x >> 5] = v0;
    s[1][threadIdx.x >> 5] = v1;
    s[2][threadIdx.x >> 5] = v2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double num = 0.0, den = 0.0, sk = 0.0;
    for (int w = 0; w < GA_CHAIN_THREADS / 32; ++w) {
      num += s[0][w];
      den += s[1][w];
      sk += s[2][w];
    }
    pb.scalars[0] = num;
    pb.scalars[1] = den;
    pb.scalars[2] = sk;
    if (!(den > 0.0)) atomicOr(pb.status, 2);
    if (trace) trace[t] = num / den;
    if (skipped_total) *skipped_total += sk;
    pb.status[1] = 0;  // re-arm the block counter for the next launch
  }
}

// per-frame reduction of payloads (one warp per frame: lanes strided over its entries, fixed-order
// shuffle tree), rot6d backward, / den; then the Adam step + decode (lane 0) unless grad_out is set
__global__ void __launch_bounds__(GA_FRAME_THREADS) ga_frame_kernel(vx_ga_problem pb, double* grad_out, double lr,
                                                                    const double* bc1, const double* bc2, int t) {
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (f >= pb.n_frames) return;
  const int dim = pb.dim;
  double GR[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, gt[3] = {0, 0, 0}, gs = 0.0;
  if (f != pb.gauge) {
    for (int e = pb.frame_ptr[f] + lane; e < pb.frame_ptr[f + 1]; e += 32) {
      const int ent = pb.frame_ent[e];
      const double* pl = pb.payload + (int64_t)GA_PAYLOAD * (ent >> 1);
      if (pl[PL_VALID] == 0.0) continue;
      const bool as_j = ent & 1;
      const double* gr = pl + (as_j ? PL_GRJ : PL_GRI);
      const double* gtt = pl + (as_j ? PL_GTJ : PL_GTI);
#pragma unroll
      for (int q = 0; q < 9; ++q) GR[q] += gr[q];
#pragma unroll
      for (int q = 0; q < 3; ++q) gt[q] += gtt[q];
      gs += pl[as_j ? PL_GSJ : PL_GSI];
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) GR[q] = warp_sum_d(GR[q]);
#pragma unroll
    for (int q = 0; q < 3; ++q) gt[q] = warp_sum_d(gt[q]);
    gs = warp_sum_d(gs);
  }
  if (lane != 0) return;
  double prm[10], g[10];
  for (int q = 0; q < dim; ++q) {
    prm[q] = pb.params[dim * f + q];
    g[q] = 0.0;
  }
  if (f != pb.gauge) {
    double GdR[9];
    mmT(GR, pb.base_R + 9 * f, GdR);
    rot6d_backward(prm, GdR, g);
#pragma unroll
    for (int q = 0; q < 3; ++q) g[6 + q] = gt[q];
    if (dim == 10) g[9] = gs;
    const double den = pb.scalars[1];
    for (int q = 0; q < dim; ++q) g[q] = g[q] / den;
  }
  if (grad_out) {
    for (int q = 0; q < dim; ++q) grad_out[dim * f + q] = g[q];
    return;
  }
  // aligner.py:412-417
  const double c1 = bc1[t], c2 = bc2[t];
  for (int q = 0; q < dim; ++q) {
    const double m = GA_BETA1 * pb.adam_m[dim * f + q] + (1.0 - GA_BETA1) * g[q];
    const double v = GA_BETA2 * pb.adam_v[dim * f + q] + (1.0 - GA_BETA2) * g[q] * g[q];
    pb.adam_m[dim * f + q] = m;
    pb.adam_v[dim * f + q] = v;
    const double mh = m / c1, vh = v / c2;
    prm[q] = prm[q] - lr * mh / (sqrt(vh) + GA_EPS);
    pb.params[dim * f + q] = prm[q];
  }
  decode_frame(pb, f, prm);
}

// adaptive weights (weighting.py:56-109)
__global__ void ga_hist_kernel(const double* __restrict__ e, int64_t K, const double* __restrict__ edges, int n_bins,
                               int64_t* __restrict__ counts) {
  const double lo = edges[0], hi = edges[n_bins];
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < K; m += (int64_t)gridDim.x * blockDim.x) {
    const double x = e[m];
    if (!isfinite(x)) continue;
    const double r = fmin(fmax(x, lo), hi);
    // np.histogram with explicit edges: bin = searchsorted(edges, r, 'right') - 1, last edge inclusive
    int a = 0, b = n_bins + 1;  // first index with edges[idx] > r, in [0, n_bins + 1]
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (edges[mid] > r) b = mid;
      else a = mid + 1;
    }
    int bin = a - 1;
    if (bin >= n_bins) bin = n_bins - 1;
    if (bin >= 0) atomicAdd(reinterpret_cast<unsigned long long*>(counts + bin), 1ull);
  }
}

constexpr int GA_W_THREADS = 1024;

__global__ void __launch_bounds__(GA_W_THREADS) ga_density_kernel(const double* __restrict__ e, int64_t K,
                                                                   const double* __restrict__ edges, int n_bins,
                                                                   const int64_t* __restrict__ counts,
                                                                   double* __restrict__ stats) {
  // single CTA: densities, then the mean density over every finite residual
  __shared__ double dens[256];
  __shared__ double red[2][GA_W_THREADS / 32];
  if (threadIdx.x == 0) {
    double raw_sum = 0.0;
    for (int q = 0; q < n_bins; ++q) raw_sum += counts[q] ? double(counts[q]) : 1e-6;
    const double width = (edges[n_bins] - edges[0]) / n_bins;
    for (int q = 0; q < n_bins; ++q) dens[q] = (counts[q] ? double(counts[q]) : 1e-6) / (raw_sum * width);
  }
  __syncthreads();
  const double lo = edges[0], hi = edges[n_bins];
  double s = 0.0, c = 0.0;
  for (int64_t m = threadIdx.x; m < K; m += GA_W_THREADS) {
    const double x = e[m];
    if (!isfinite(x)) continue;
    const double r = fmin(fmax(x, lo), hi);
    int a = 0, b = n_bins + 1;
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (edges[mid] > r) b = mid;
      else a = mid + 1;
    }
    const int bin = min(max(a - 1, 0), n_bins - 1);
    s += dens[bin];
    c += 1.0;
  }
  s = warp_sum_d(s);
  c = warp_sum_d(c);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s;
    red[1][threadIdx.x >> 5] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s = c = 0.0;
    for (int w = 0; w < GA_W_THREADS / 32; ++w) {
      s += red[0][w];
      c += red[1][w];
    }
    stats[0] = c > 0 ? s / c : NAN;
    stats[1] = c;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < n_bins; q += GA_W_THREADS) stats[2 + q] = dens[q];
}

__global__ void ga_weight_kernel(const double* __restrict__ e, int64_t K, const double* __restrict__ edges, int n_bins,
                                 const double* __restrict__ stats, double alpha, double* __restrict__ w) {
  const double lo = edges[0], hi = edges[n_bins];
  const double avg = stats[0];
  const double* dens = stats + 2;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < K; m += (int64_t)gridDim.x * blockDim.x) {
    const double x = e[m];
    if (!isfinite(x)) {
      w[m] = 0.0;
      continue;
    }
    const double r = fmin(fmax(x, lo), hi);
    int a = 0, b = n_bins + 1;
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (edges[mid] > r) b = mid;
      else a = mid + 1;
    }
    const int bin = min(max(a - 1, 0), n_bins - 1);
    w[m] = pow(dens[bin] / avg, alpha);
  }
}

static bool problem_ok(const vx_ga_problem* pb) {
  return pb && pb->n_frames > 0 && pb->n_pairs >= 0 && (pb->dim == 9 || pb->dim == 10) &&
         (pb->mode == 0 || pb->mode == 1) && pb->pair_ij && pb->offsets && pb->base_R && pb->base_t &&
         pb->base_Kinv && pb->params && pb->Rs && pb->ts && pb->Kinv && pb->status;
}

// 128 threads x 4 correspondences in flight per thread: the best of a shape sweep at 200 views /
// 12.9M correspondences (tools/sweep_ga.sh: 256x1 -> 182 us per evaluation, 128x2 -> 144, 128x4 -> 119)
constexpr int GA_PAIR_THREADS = 128, GA_PAIR_MINB = 3, GA_PAIR_UNROLL = 4;

template <int MODE>
static void launch_pair(const vx_ga_problem& pb, cudaStream_t st) {
  ga_pair_kernel<MODE, GA_PAIR_THREADS, GA_PAIR_MINB, GA_PAIR_UNROLL><<<pb.n_pairs, GA_PAIR_THREADS, 0, st>>>(pb);
}

static int frame_blocks(int n) { return (n + GA_FRAME_THREADS - 1) / GA_FRAME_THREADS; }
static int frame_warp_blocks(int n) { return (32 * n + GA_FRAME_THREADS - 1) / GA_FRAME_THREADS; }
static int chain_blocks(int p) { return std::max(1, (p + GA_CHAIN_THREADS - 1) / GA_CHAIN_THREADS); }

static uint64_t iteration_kernels(const vx_ga_problem& pb) { return pb.n_pairs > 0 ? 4 : 2; }

static void launch_iteration(const vx_ga_problem& pb, int t, double lr, const double* bc1, const double* bc2,
                             double* trace, double* skipped_total, cudaStream_t st) {
  if (pb.n_pairs > 0) {
    ga_geom_kernel<<<chain_blocks(pb.n_pairs), GA_CHAIN_THREADS, 0, st>>>(pb);
    if (pb.mode == 0) launch_pair<0>(pb, st);
    else launch_pair<1>(pb, st);
  }
  ga_chain_kernel<<<chain_blocks(pb.n_pairs), GA_CHAIN_THREADS, 0, st>>>(pb, trace, t, skipped_total);
  ga_frame_kernel<<<frame_warp_blocks(pb.n_frames), GA_FRAME_THREADS, 0, st>>>(pb, nullptr, lr, bc1, bc2, t);
}

}  // namespace vx

extern "C" int vx_ga_decode(const vx_ga_problem* pb, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(problem_ok(pb), "vx_ga_decode: bad problem");
  ga_decode_kernel<<<frame_blocks(pb->n_frames), GA_FRAME_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*pb);
  VX_CHECK_LAUNCH("ga decode launch");
  return VX_OK;
}

extern "C" int vx_ga_residuals(const vx_ga_problem* pb, double* e, int32_t* deg_pair, int32_t* n_deg, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(problem_ok(pb) && pb->xy_i && pb->xy_j, "vx_ga_residuals: bad problem");
  if (pb->n_pairs == 0) return VX_OK;
  VX_CHECK_ARG(e && deg_pair && n_deg, "vx_ga_residuals: null output");
  ga_residuals_kernel<<<pb->n_pairs, EPI_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*pb, e, deg_pair,
                                                                                                n_deg);
  VX_CHECK_LAUNCH("ga residuals launch");
  return VX_OK;
}

extern "C" int vx_ga_loss_grad(const vx_ga_problem* pb, double* grad, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(problem_ok(pb) && pb->w && pb->geom && pb->payload && pb->scalars && pb->frame_ptr && pb->frame_ent && grad,
               "vx_ga_loss_grad: bad problem");
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (pb->n_pairs > 0) {
    ga_geom_kernel<<<chain_blocks(pb->n_pairs), GA_CHAIN_THREADS, 0, st>>>(*pb);
    if (pb->mode == 0) launch_pair<0>(*pb, st);
    else launch_pair<1>(*pb, st);
  }
  ga_chain_kernel<<<chain_blocks(pb->n_pairs), GA_CHAIN_THREADS, 0, st>>>(*pb, nullptr, 0, nullptr);
  ga_frame_kernel<<<frame_warp_blocks(pb->n_frames), GA_FRAME_THREADS, 0, st>>>(*pb, grad, 0.0, nullptr, nullptr, 0);
  VX_CHECK_LAUNCH_N("ga loss/grad launch", iteration_kernels(*pb));
  return VX_OK;
}

extern "C" int vx_ga_adam(const vx_ga_problem* pb, int t0, int iters, double lr, const double* bc1, const double* bc2,
                          double* trace, double* skipped_total, int use_graph, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(problem_ok(pb) && pb->w && pb->geom && pb->payload && pb->scalars && pb->frame_ptr && pb->frame_ent &&
                   pb->adam_m && pb->adam_v && bc1 && bc2 && t0 >= 0 && iters >= 0,
               "vx_ga_adam: bad arguments");
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (iters == 0) return VX_OK;
  if (!use_graph) {
    for (int k = 0; k < iters; ++k) launch_iteration(*pb, t0 + k, lr, bc1, bc2, trace, skipped_total, st);
    VX_CHECK_LAUNCH_N("ga adam launch", (uint64_t)iters * iteration_kernels(*pb));
    return VX_OK;
  }
  // capture on a private stream (the caller's may be the legacy default stream), replay on the caller's
  cudaStream_t cap;
  cudaError_t err = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
  if (err != cudaSuccess) return fail_cuda(err, "ga capture stream");
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  err = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
  if (err == cudaSuccess) {
    for (int k = 0; k < iters; ++k) launch_iteration(*pb, t0 + k, lr, bc1, bc2, trace, skipped_total, cap);
    err = cudaStreamEndCapture(cap, &graph);
  }
  if (err == cudaSuccess) err = cudaGraphInstantiate(&exec, graph, 0);
  if (err == cudaSuccess) err = cudaGraphLaunch(exec, st);
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  cudaStreamDestroy(cap);
  if (err != cudaSuccess) return fail_cuda(err, "ga adam graph");
  count_launches((uint64_t)iters * iteration_kernels(*pb));
  return VX_OK;
}

extern "C" int vx_ga_adaptive_weights(const double* e, int64_t K, const double* edges, int n_bins, double alpha,
                                      double* w, int64_t* counts, double* out_stats, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(K >= 0 && n_bins > 0 && n_bins <= 256, "vx_ga_adaptive_weights: bad sizes");
  VX_CHECK_ARG(e && edges && w && counts && out_stats, "vx_ga_adaptive_weights: null pointer");
  auto st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t err = cudaMemsetAsync(counts, 0, sizeof(int64_t) * n_bins, st);
  if (err != cudaSuccess) return fail_cuda(err, "ga hist memset");
  const int blocks = (int)std::min<int64_t>((K + 255) / 256 + 1, 4 * (int64_t)num_sms());
  ga_hist_kernel<<<blocks, 256, 0, st>>>(e, K, edges, n_bins, counts);
  ga_density_kernel<<<1, GA_W_THREADS, 0, st>>>(e, K, edges, n_bins, counts, out_stats);
  ga_weight_kernel<<<blocks, 256, 0, st>>>(e, K, edges, n_bins, out_stats, alpha, w);
  VX_CHECK_LAUNCH_N("ga adaptive weights launch", 3);
  return VX_OK;
}
