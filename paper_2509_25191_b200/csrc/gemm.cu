// Persistent warp-specialised tcgen05 GEMM with fused VGGT epilogues (sm_100a).
//
//   D[M, N] = A[M, K] . B[N, K]^T, bf16 operands (K-major, TMA SWIZZLE_128B),
//   fp32 accumulators in TMEM (two BN-column buffers so the epilogue of tile t
//   overlaps the main loop of tile t+1).
//
// Warp roles (384 threads): w0 TMA producer, w1 tcgen05.mma issuer (one elected
// lane), w2 TMEM allocator, w4..w11 epilogue: thread i of warp 4+e owns TMEM lane /
// tile row 32(e%4)+i and half of the tile's columns, so per-row work such as the
// per-head q/k LayerNorm and RoPE of the qkv epilogue is entirely thread-local.
// (K=1024 GEMMs are epilogue-bound with 4 epilogue warps; 8 halve that time.)
//
// Replaces the upstream nn.Linear calls of the VGGT Block (SURVEY.md §8a a6, a9,
// a10) and the conv patch-embed (a2), with the norm/RoPE/LayerScale/residual
// element-wise ops fused into the epilogue.
#include "../../include/vx_api.h"
#include "common.cuh"
#include "host_util.h"
#include <stdlib.h>

namespace vx {

struct GemmArgs {
  int M, N, K;
  vx_epilogue ep;
  vx_spatial sp;
  int conv_cin_blocks;  // > 0: implicit 3x3 conv A addressing (K = 9 * cin_blocks * 64)
  int conv_w2;          // padded row length W + 2
};

constexpr int VX_EPI_SPATIAL = 6;
constexpr int VX_EPI_HEADOUT = 7;
// VX_EPI_RESID without the kept copy on 256-wide tiles (Attention.proj): the fp32 residual tile moves
// through shared memory with TMA loads / stores instead of per-lane global loads and stores
constexpr int VX_EPI_RESID_TMA = 8;

#ifndef VX_RT_NBOX
#define VX_RT_NBOX 2
#endif
constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 384;  // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4..w11 epilogue
constexpr int GEMM_EPI_WARPS = 8;  // two warps per TMEM lane quarter, each owning half of the tile columns

// HALO (implicit 3x3 conv with N <= 32, the DPT output head): one stage per 64 input channels holds
// the three 130-row bands of the tile's input rows (row shifts dy = 0, 1, 2 of the padded grid) and
// the 9 taps' B tiles; tap (dy, dx) reads band dy from row dx on, so the input is staged once per
// channel block instead of once per tap (9x less L2 -> shared traffic; 36 MMAs per stage)
constexpr int HALO_ROWS = GEMM_BM + 2;
constexpr int HALO_MAX_CB = 2;  // input channels <= 128 (the DPT output head: features / 2)
constexpr uint32_t HALO_BAND_BYTES = (HALO_ROWS * GEMM_BK * 2 + 1023) / 1024 * 1024;

template <int BN, bool CG2 = false, bool RT = false, bool HALO = false>
struct GemmCfg {
  // CG2 (CTA pair, cta_group::2): each CTA stages its 128 A rows and half of the B tile; RT (TMA
  // residual epilogue): 4 stages, leaving 64 KB for the residual boxes
  static constexpr int STAGES =
      HALO ? 3 : (RT ? (VX_RT_NBOX >= 4 ? 3 : 4) : (CG2 ? 6 : (BN == 256 ? 4 : (BN == 128 ? 6 : 8))));
  static constexpr uint32_t A_BYTES = HALO ? 3 * HALO_BAND_BYTES : GEMM_BM * GEMM_BK * 2;
  // HALO: the B (weight) tiles of all 9 taps x up to HALO_MAX_CB channel blocks stay resident
  static constexpr uint32_t B_BYTES = HALO ? 0 : (CG2 ? BN / 2 : BN) * GEMM_BK * 2;
  static constexpr uint32_t B_RES_BYTES = HALO ? 9 * HALO_MAX_CB * BN * GEMM_BK * 2 : 0;
  static constexpr uint32_t RING = STAGES * (A_BYTES + B_BYTES) + B_RES_BYTES;
  static constexpr uint32_t SMEM = RING + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static_assert(SMEM <= 227 * 1024, "GEMM stage ring exceeds the 227 KB smem per CTA");
};

// RESID epilogue transpose buffer: each epilogue warp stages its 32 x 32 fp32 accumulator block
// (stride 33: conflict-free row writes and column reads) so that the fp32 residual read-modify-
// write walks row segments with the 32 lanes on consecutive columns (one 128 B sector run per
// row) instead of 32 rows per instruction (32 half-used sectors)
constexpr uint32_t RESID_TILE_FLOATS = 32 * 33;
// RESID_TMA: per epilogue warp two 32 x 32 fp32 residual boxes (4 KB each, 128-byte swizzled rows),
// 1024-byte aligned after the barrier block
constexpr uint32_t RT_BOX_BYTES = 32 * 32 * 4;
constexpr int RT_NBOX = VX_RT_NBOX;  // boxes per epilogue warp (4: the warp's whole 32 x 128 tile share)
template <int EPI>
constexpr uint32_t epi_smem_bytes() {
  return EPI == VX_EPI_RESID ? GEMM_EPI_WARPS * RESID_TILE_FLOATS * 4
                             : (EPI == VX_EPI_RESID_TMA ? 1024 + GEMM_EPI_WARPS * RT_NBOX * RT_BOX_BYTES : 0);
}

// ---------------------------------------------------------------------------
// epilogues: one thread = one output row; columns processed 32 at a time
// ---------------------------------------------------------------------------
// the chunk's bias, loaded before the TMEM load so its latency overlaps it instead of
// serialising behind it (RESID has its own warp-transposed epilogue in gemm_kernel)
template <int EPI>
struct EpiPre {
  float4 b[8];
};

template <int EPI>
VX_DEVICE void epi_prefetch(const GemmArgs& a, int row, int col, EpiPre<EPI>& p) {
  const vx_epilogue& e = a.ep;
  if (e.bias) {
    const float4* b4 = reinterpret_cast<const float4*>(e.bias + col);
#pragma unroll
    for (int j = 0; j < 8; ++j) p.b[j] = __ldg(b4 + j);
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) p.b[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

template <int EPI>
VX_DEVICE void epi_chunk32(const GemmArgs& a, int row, int col, const uint32_t* r, const EpiPre<EPI>& pre) {
  const vx_epilogue& e = a.ep;
  float v[32];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    v[4 * j] = __uint_as_float(r[4 * j]) + pre.b[j].x;
    v[4 * j + 1] = __uint_as_float(r[4 * j + 1]) + pre.b[j].y;
    v[4 * j + 2] = __uint_as_float(r[4 * j + 2]) + pre.b[j].z;
    v[4 * j + 3] = __uint_as_float(r[4 * j + 3]) + pre.b[j].w;
  }
  if (row >= a.M) return;
  if constexpr (EPI == VX_EPI_BF16 || EPI == VX_EPI_GELU) {
    uint32_t w[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const float t0 = (EPI == VX_EPI_GELU) ? gelu_erf_fast(v[2 * u]) : v[2 * u];
      const float t1 = (EPI == VX_EPI_GELU) ? gelu_erf_fast(v[2 * u + 1]) : v[2 * u + 1];
      w[u] = pack_bf16(t0, t1);
    }
    store_64b(reinterpret_cast<__nv_bfloat16*>(e.out) + (size_t)row * e.ldo + col, w);
  } else if constexpr (EPI == VX_EPI_F32) {
    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(e.out) + (size_t)row * e.ldo + col);
#pragma unroll
    for (int j = 0; j < 8; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  } else if constexpr (EPI == VX_EPI_PATCH) {
    const int P = a.M / 1;  // unused
    (void)P;
    const int npatch = e.tokens_per_frame - e.patch_start;
    const int f = row / npatch, p = row - f * npatch;
    float4* dst = reinterpret_cast<float4*>(e.resid + ((size_t)f * e.tokens_per_frame + e.patch_start + p) * e.ldr + col);
#pragma unroll
    for (int j = 0; j < 8; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  }
}

// q/k/v head epilogue: D columns (one head) per call.
template <int D>
VX_DEVICE void epi_qkv_head(const GemmArgs& a, int row, int col, float* v) {
  const vx_epilogue& e = a.ep;
  const int C = e.embed_dim;
  const int gcol = col + e.col_offset;  // column of the whole [3C] q/k/v output (bias is sliced alike)
  const int which = gcol / C;
  const int h = (gcol - which * C) / D;
  if (e.bias) {
    const float4* b4 = reinterpret_cast<const float4*>(e.bias + col);
#pragma unroll
    for (int j = 0; j < D / 4; ++j) {
      float4 b = __ldg(b4 + j);
      v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
    }
  }
  if (row >= a.M) return;
  if (which < 2) {
    const float* nw = which == 0 ? e.qn_w : e.kn_w;
    const float* nb = which == 0 ? e.qn_b : e.kn_b;
    if (nw) {
      float mean = 0.f;
#pragma unroll
      for (int j = 0; j < D; ++j) mean += v[j];
      mean *= (1.0f / D);
      float var = 0.f;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        float d = v[j] - mean;
        var += d * d;
      }
      const float rstd = rsqrtf(var * (1.0f / D) + e.eps);
      const float4* w4 = reinterpret_cast<const float4*>(nw);
      const float4* b4 = reinterpret_cast<const float4*>(nb);
#pragma unroll
      for (int j = 0; j < D / 4; ++j) {  // 16-byte uniform loads of the affine parameters
        const float4 w = __ldg(w4 + j), b = __ldg(b4 + j);
        v[4 * j + 0] = (v[4 * j + 0] - mean) * rstd * w.x + b.x;
        v[4 * j + 1] = (v[4 * j + 1] - mean) * rstd * w.y + b.y;
        v[4 * j + 2] = (v[4 * j + 2] - mean) * rstd * w.z + b.z;
        v[4 * j + 3] = (v[4 * j + 3] - mean) * rstd * w.w + b.w;
      }
    }
    if (e.rope_cos) {
      const int t = row % e.tokens_per_frame;
      int py = 0, px = 0;
      if (t >= e.patch_start) {
        const int p = t - e.patch_start;
        py = p / e.grid_w + 1;
        px = p - (py - 1) * e.grid_w + 1;
      }
      constexpr int Q4 = D / 4;
      static_assert(Q4 % 4 == 0, "rope quarter must be a multiple of 4");
      const float4* cy = reinterpret_cast<const float4*>(e.rope_cos + py * Q4);
      const float4* sy = reinterpret_cast<const float4*>(e.rope_sin + py * Q4);
      const float4* cx = reinterpret_cast<const float4*>(e.rope_cos + px * Q4);
      const float4* sx = reinterpret_cast<const float4*>(e.rope_sin + px * Q4);
      auto rot = [&](int j0, const float4 c4, const float4 s4) {  // (x0, x1) = (v[j], v[j + Q4]) rotated
        const float cc[4] = {c4.x, c4.y, c4.z, c4.w}, ss[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float x0 = v[j0 + u], x1 = v[j0 + u + Q4];
          v[j0 + u] = x0 * cc[u] - x1 * ss[u];
          v[j0 + u + Q4] = x1 * cc[u] + x0 * ss[u];
        }
      };
#pragma unroll
      for (int j = 0; j < Q4 / 4; ++j) {  // y rotation on the first half, x rotation on the second
        rot(4 * j, __ldg(cy + j), __ldg(sy + j));
        rot(2 * Q4 + 4 * j, __ldg(cx + j), __ldg(sx + j));
      }
    }
  }
  __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(which == 0 ? e.q : (which == 1 ? e.k : e.v));
  // a head row is D * 2 = 64 or 128 bytes at a multiple of its size: 32-byte stores (whole sectors)
  __nv_bfloat16* dst = base + ((size_t)h * e.tokens_total + row) * D;
  if (which == 0 && e.q_scale != 0.f) {
#pragma unroll
    for (int j = 0; j < D; ++j) v[j] *= e.q_scale;
  }
#pragma unroll
  for (int j = 0; j < D / 16; ++j) {
    const float* w = v + 16 * j;
    st_global_v8(dst + 16 * j, pack_bf16(w[0], w[1]), pack_bf16(w[2], w[3]), pack_bf16(w[4], w[5]),
                 pack_bf16(w[6], w[7]), pack_bf16(w[8], w[9]), pack_bf16(w[10], w[11]), pack_bf16(w[12], w[13]),
                 pack_bf16(w[14], w[15]));
  }
}

// q/k/v scatter without qk-norm / RoPE (camera-head trunk, head_dim = e.head_dim, any multiple of
// 32): a 32-column chunk never straddles a head, so it goes straight to [H, T, head_dim]
VX_DEVICE void epi_qkv_scatter32(const GemmArgs& a, int row, int col, const uint32_t* r, const EpiPre<VX_EPI_QKV>& pre) {
  const vx_epilogue& e = a.ep;
  if (row >= a.M) return;
  const int C = e.embed_dim;
  const int gcol = col + e.col_offset;
  const int which = gcol / C;
  const int hc = gcol - which * C;
  const int h = hc / e.head_dim, off = hc - h * e.head_dim;
  __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(which == 0 ? e.q : (which == 1 ? e.k : e.v));
  const float qs = which == 0 && e.q_scale != 0.f ? e.q_scale : 1.0f;
  uint32_t w[16];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 bb = pre.b[j];
    w[2 * j] = pack_bf16((__uint_as_float(r[4 * j]) + bb.x) * qs, (__uint_as_float(r[4 * j + 1]) + bb.y) * qs);
    w[2 * j + 1] = pack_bf16((__uint_as_float(r[4 * j + 2]) + bb.z) * qs, (__uint_as_float(r[4 * j + 3]) + bb.w) * qs);
  }
  store_64b(base + ((size_t)h * e.tokens_total + row) * e.head_dim + off, w);
}

// ---------------------------------------------------------------------------
// spatial (DPT) epilogues
// ---------------------------------------------------------------------------
struct PixInfo {
  bool valid;
  int f, yo, xo;  // output pixel (before the shuffle offset)
};

VX_DEVICE PixInfo pix_of_row(const GemmArgs& a, int row) {
  const vx_spatial& sp = a.sp;
  PixInfo p;
  const int rw = sp.conv3x3 ? sp.W + 2 : sp.W;
  const int pf = sp.conv3x3 ? (sp.H + 2) * (sp.W + 2) : sp.H * sp.W;
  p.f = row / pf;
  const int rem = row - p.f * pf;
  const int y = rem / rw;
  const int x = rem - y * rw;
  p.valid = row < a.M && y < sp.H && x < sp.W;
  if (sp.subsample2) {
    p.valid = p.valid && ((y | x) & 1) == 0;
    p.yo = y >> 1;
    p.xo = x >> 1;
  } else {
    p.yo = y * sp.shuffle;
    p.xo = x * sp.shuffle;
  }
  return p;
}

VX_DEVICE int64_t pix_index(int f, int y, int x, int Ho, int Wo, int pad) {
  return pad ? ((int64_t)(f * (Ho + 2) + y + 1) * (Wo + 2) + x + 1) : ((int64_t)(f * Ho + y) * Wo + x);
}

VX_DEVICE void load8_bf16(const void* base, int64_t elem, float* o) {
  const uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(base) + elem);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __bfloat1622float2(h[k]);
    o[2 * k] = f.x;
    o[2 * k + 1] = f.y;
  }
}

VX_DEVICE void epi_spatial32(const GemmArgs& a, const PixInfo& pi, int col, const uint32_t* r) {
  const vx_spatial& sp = a.sp;
  const vx_epilogue& e = a.ep;
  const int s = sp.shuffle;
  const int Cout = a.N / (s * s);
  int c = col, yo = pi.yo, xo = pi.xo;
  if (s > 1) {
    const int ij = col / Cout;
    c = col - ij * Cout;
    yo += ij / s;
    xo += ij % s;
  }
  const int Ho = sp.subsample2 ? (sp.H + 1) / 2 : sp.H * s;
  const int Wo = sp.subsample2 ? (sp.W + 1) / 2 : sp.W * s;
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  if (e.bias) {
    const float4* b4 = reinterpret_cast<const float4*>(e.bias + c);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 b = __ldg(b4 + j);
      v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
    }
  }
  if (!pi.valid) return;
  float t[8];
  if (sp.pos) {
    const int64_t pe = ((int64_t)yo * Wo + xo) * Cout + c;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      load8_bf16(sp.pos, pe + 8 * q, t);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[8 * q + k] += t[k];
    }
  }
  if (sp.relu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
  }
  if (sp.res1) {
    const int64_t re = pix_index(pi.f, yo, xo, Ho, Wo, sp.res1_pad) * Cout + c;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      load8_bf16(sp.res1, re + 8 * q, t);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[8 * q + k] += t[k];
    }
  }
  if (sp.res2) {
    const int64_t re = pix_index(pi.f, yo, xo, Ho, Wo, sp.res2_pad) * Cout + c;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      load8_bf16(sp.res2, re + 8 * q, t);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[8 * q + k] += t[k];
    }
  }
  {
    uint32_t w[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) w[u] = pack_bf16(v[2 * u], v[2 * u + 1]);
    store_64b(reinterpret_cast<__nv_bfloat16*>(sp.out1) + pix_index(pi.f, yo, xo, Ho, Wo, sp.out1_pad) * Cout + c, w);
  }
  if (sp.out2) {
    uint32_t w[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) w[u] = pack_bf16(fmaxf(v[2 * u], 0.f), fmaxf(v[2 * u + 1], 0.f));
    store_64b(reinterpret_cast<__nv_bfloat16*>(sp.out2) + pix_index(pi.f, yo, xo, Ho, Wo, sp.out2_pad) * Cout + c, w);
  }
}

// DPT output head: relu(conv3x3 + b) (32 ch) -> fp32 1x1 (odim) -> activation
VX_DEVICE void epi_headout(const GemmArgs& a, const PixInfo& pi, const uint32_t* r) {
  const vx_spatial& sp = a.sp;
  const vx_epilogue& e = a.ep;
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = fmaxf(__uint_as_float(r[j]) + (e.bias ? __ldg(e.bias + j) : 0.f), 0.f);
  if (!pi.valid) return;
  const int od = sp.head_odim;
  const int64_t pix = ((int64_t)pi.f * sp.H + pi.yo) * sp.W + pi.xo;
  for (int k = 0; k < od; ++k) {
    float o = __ldg(sp.head_b + k);
#pragma unroll
    for (int j = 0; j < 32; ++j) o = fmaf(__ldg(sp.head_w + k * 32 + j), v[j], o);
    if (k == od - 1) {
      sp.head_conf[pix] = 1.0f + expf(o);
    } else {
      float pr;
      if (sp.head_act == 0) pr = expf(o);
      else pr = copysignf(expm1f(fabsf(o)), o);
      sp.head_pred[pix * (od - 1) + k] = pr;
    }
  }
}

// ---------------------------------------------------------------------------
// kernel
// ---------------------------------------------------------------------------
// MC: clusters of 2 CTAs on adjacent M tiles (same N tile); each CTA TMA-loads half of the
// B tile and multicasts it to both, halving the per-SM L2->SMEM traffic of the main loop
// (a 128x256 tile needs ~94 B/clk/SM from L2 otherwise — above the chip's L2 throughput).
// CG2: CTA pairs with cta_group::2 MMAs: a pair computes a 256 x BN tile; each CTA TMA-loads its
// 128 A rows and half of the B tile into its own smem (completion on the leader's barrier), the
// leader issues M = 256 MMAs reading both CTAs' smem, and each CTA's TMEM receives its 128 rows.
// Per-SM smem operand traffic per MMA drops from (128 + BN) to (128 + BN/2) rows.
template <int BN, int EPI, int HD, bool MC, bool CG2 = false>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmR, const GemmArgs args) {
  constexpr bool HALO = EPI == VX_EPI_HEADOUT;
  using Cfg = GemmCfg<BN, CG2, EPI == VX_EPI_RESID_TMA, HALO>;
  constexpr bool PAIRED = MC || CG2;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::RING);  // after the stages (+ resident B)
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  [[maybe_unused]] uint64_t* bres_full = tempty + 2;  // HALO: resident weight tiles landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 3);
  // offset from smem_raw (not the integer-aligned pointer) so the compiler keeps the shared state
  // space and emits LDS / STS for the transpose tile rather than generic LD / ST
  [[maybe_unused]] float* epi_buf = reinterpret_cast<float*>(smem_raw + (smem - smem_raw) + Cfg::RING + 256);
  // RESID_TMA: per-warp residual boxes and their TMA-load barriers
  [[maybe_unused]] float* rbox = reinterpret_cast<float*>(smem_raw + (smem - smem_raw) + Cfg::RING + 1024);
  [[maybe_unused]] uint64_t* rbar = reinterpret_cast<uint64_t*>(smem + Cfg::RING + 128);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int M = args.M, N = args.N, K = args.K;
  const int num_n = (N + BN - 1) / BN;
  const int num_m = (M + GEMM_BM - 1) / GEMM_BM;
  const int kblocks = K / GEMM_BK;
  // work decomposition: MC clusters walk (M-tile pair, N tile) units; otherwise single tiles
  const uint32_t crank = PAIRED ? cluster_ctarank() : 0;
  const int units = PAIRED ? ((num_m + 1) / 2) * num_n : num_m * num_n;
  const int unit0 = PAIRED ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int ustep = PAIRED ? int(gridDim.x >> 1) : int(gridDim.x);
  auto tile_mn = [&](int u, int& m_blk, int& n_blk) {
    const int mu = u / num_n;
    n_blk = u - mu * num_n;
    m_blk = PAIRED ? 2 * mu + int(crank) : mu;
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC ? 2 : 1);  // MC: released by both CTAs' MMA warps
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      // CG2: the leader's accumulator is released by both CTAs' epilogue warps
      mbar_init(&tempty[s], CG2 ? 2 * GEMM_EPI_WARPS : GEMM_EPI_WARPS);
    }
    if constexpr (EPI == VX_EPI_RESID_TMA)
      for (int i = 0; i < RT_NBOX * GEMM_EPI_WARPS; ++i) mbar_init(&rbar[i], 1);
    if constexpr (HALO) mbar_init(bres_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG2) tmem_alloc_cg2(tmem_slot, Cfg::TMEM_COLS);
    else tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIRED) cluster_sync();  // peer barriers initialised before any multicast / remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_b = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      [[maybe_unused]] const uint64_t pol_a = policy_evict_normal();
      for (int u = unit0; u < units; u += ustep) {
        int m_blk, n_blk;
        tile_mn(u, m_blk, n_blk);
        if constexpr (HALO) {
          if (u == unit0) {  // the weights of every (tap, channel block), once per CTA (N == BN: one N tile)
            mbar_expect_tx(bres_full, 9 * args.conv_cin_blocks * BN * GEMM_BK * 2);
            for (int cb = 0; cb < args.conv_cin_blocks; ++cb)
              for (int t = 0; t < 9; ++t)
                tma_load_2d_hint(sB + (cb * 9 + t) * (BN * GEMM_BK * 2), &tmB, bres_full,
                                 (t * args.conv_cin_blocks + cb) * GEMM_BK, 0, pol_b);
          }
          for (int cb = 0; cb < args.conv_cin_blocks; ++cb) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], 3 * HALO_ROWS * GEMM_BK * 2);
            for (int dy = 0; dy < 3; ++dy)
              tma_load_2d(sA + stage * Cfg::A_BYTES + dy * HALO_BAND_BYTES, &tmA, &full[stage], cb * GEMM_BK,
                          m_blk * GEMM_BM + dy * args.conv_w2);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          continue;
        }
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          int a_col = kb * GEMM_BK, a_row = m_blk * GEMM_BM;
          if (args.conv_cin_blocks > 0) {  // implicit 3x3 conv: tap t shifts the padded-grid row
            const int t = kb / args.conv_cin_blocks;
            a_col = (kb - t * args.conv_cin_blocks) * GEMM_BK;
            a_row += (t / 3) * args.conv_w2 + (t % 3);
          }
          if constexpr (CG2) {  // both CTAs' halves complete on the leader's full barrier
            if (crank == 0) mbar_expect_tx(&full[stage], 2 * (Cfg::A_BYTES + Cfg::B_BYTES));
            const uint32_t full0 = mapa_shared(smem_u32(&full[stage]), 0);
            tma_load_2d_cg2(sA + stage * Cfg::A_BYTES, &tmA, full0, a_col, a_row, pol_a);
            tma_load_2d_cg2(sB + stage * Cfg::B_BYTES, &tmB, full0, kb * GEMM_BK, n_blk * BN + int(crank) * (BN / 2),
                            pol_b);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          mbar_expect_tx(&full[stage], Cfg::A_BYTES + Cfg::B_BYTES);
          tma_load_2d(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], a_col, a_row);
          if constexpr (MC) {  // my half of the B tile, multicast to both CTAs of the pair
            tma_load_2d_mc(sB + stage * Cfg::B_BYTES + crank * (Cfg::B_BYTES / 2), &tmB, &full[stage], kb * GEMM_BK,
                           n_blk * BN + int(crank) * (BN / 2), 0x3, pol_b);
          } else {
            tma_load_2d_hint(sB + stage * Cfg::B_BYTES, &tmB, &full[stage], kb * GEMM_BK, n_blk * BN, pol_b);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (CG2 && crank != 0) {
      // the pair leader issues every MMA of the pair
    } else if (elect_one()) {
      constexpr uint32_t idesc = make_idesc_bf16(CG2 ? 2 * GEMM_BM : GEMM_BM, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = unit0; u < units; u += ustep) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        if constexpr (HALO) {
          if (u == unit0) mbar_wait(bres_full, 0);
          for (int cb = 0; cb < args.conv_cin_blocks; ++cb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA + stage * Cfg::A_BYTES);
            const uint32_t b0 = smem_u32(sB) + cb * 9 * (BN * GEMM_BK * 2);
#pragma unroll
            for (int t = 0; t < 9; ++t) {
              const int dy = t / 3, dx = t % 3;
              // band dy from row dx: the 128-byte swizzle is applied on absolute shared-memory address bits,
              // so a start that is a whole number of 128-byte rows into a swizzle atom needs no base offset
              const uint32_t at = a0 + dy * HALO_BAND_BYTES + dx * (GEMM_BK * 2);
              const uint32_t bt = b0 + t * (BN * GEMM_BK * 2);
#pragma unroll
              for (int k = 0; k < GEMM_BK / 16; ++k)
                mma_ss(d_tmem, make_sdesc(at + k * 32, 16, 1024, 2), make_sdesc(bt + k * 32, 16, 1024, 2), idesc,
                       (cb | t | k) != 0);
            }
            mma_commit(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          mma_commit(&tfull[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          continue;
        }
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            if constexpr (CG2)
              mma_ss_cg2(d_tmem, make_sdesc(a0 + k * 32, 16, 1024, 2), make_sdesc(b0 + k * 32, 16, 1024, 2), idesc,
                         (kb | k) != 0);
            else
              mma_ss(d_tmem, make_sdesc(a0 + k * 32, 16, 1024, 2), make_sdesc(b0 + k * 32, 16, 1024, 2), idesc,
                     (kb | k) != 0);
          }
          if constexpr (CG2) mma_commit_cg2_mc(&empty[stage], 0x3);  // stage free in both CTAs
          else if constexpr (MC) mma_commit_mc(&empty[stage], 0x3);  // stage free in both CTAs' producers
          else mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (CG2) mma_commit_cg2_mc(&tfull[acc], 0x3);  // both CTAs' epilogues
        else mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    [[maybe_unused]] uint32_t rph = 0;    // RESID_TMA: phase bit per residual box
    const int ew = (warp - 4) & 3;        // TMEM lane quarter
    // column half (a 32-wide tile is handled whole by warps 4..7; warps 8..11 only arrive)
    const int c_beg = BN <= 32 ? ((warp - 4) >> 2) * BN : ((warp - 4) >> 2) * (BN / 2);
    const int c_end = BN <= 32 ? BN : c_beg + BN / 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = unit0; u < units; u += ustep) {
      int m_blk, n_blk;
      tile_mn(u, m_blk, n_blk);
      // RESID: the first residual chunk of this tile is loaded before the accumulator wait, so its
      // latency overlaps the tile's main loop; later chunks are loaded one chunk ahead (below)
      [[maybe_unused]] float xpre[EPI == VX_EPI_RESID ? 32 : 1];
      [[maybe_unused]] const int rrow0 = m_blk * GEMM_BM + ew * 32;
      [[maybe_unused]] const int nrows = M - rrow0 < 32 ? M - rrow0 : 32;
      [[maybe_unused]] auto load_resid = [&](int col) {
        const float* xc = args.ep.resid + (size_t)rrow0 * args.ep.ldr + col + int(lane);
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) xpre[rr] = rr < nrows ? xc[(size_t)rr * args.ep.ldr] : 0.f;
      };
      if constexpr (EPI == VX_EPI_RESID) {
        if (n_blk * BN + c_beg < N) load_resid(n_blk * BN + c_beg);
      }
      // RESID_TMA: the warp's first two 32 x 32 residual boxes are requested before the accumulator
      // wait (their load overlaps the tile's main loop); later boxes reuse a buffer once its store has
      // read it
      [[maybe_unused]] const int wcol0 = n_blk * BN + c_beg;
      [[maybe_unused]] const int nbox = wcol0 < N ? ((N - wcol0 < c_end - c_beg ? N - wcol0 : c_end - c_beg) / 32) : 0;
      [[maybe_unused]] float* wbox = rbox + (warp - 4) * RT_NBOX * (RT_BOX_BYTES / 4);
      [[maybe_unused]] uint64_t* wbar = rbar + (warp - 4) * RT_NBOX;
      if constexpr (EPI == VX_EPI_RESID_TMA) {
        if (lane == 0) {
          bulk_wait_read<0>();  // the previous tile's stores have read the boxes
          for (int b = 0; b < RT_NBOX && b < nbox; ++b) {
            mbar_expect_tx(&wbar[b], RT_BOX_BYTES);
            tma_load_2d(wbox + b * (RT_BOX_BYTES / 4), &tmR, &wbar[b], wcol0 + 32 * b, rrow0);
          }
        }
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m_blk * GEMM_BM + ew * 32 + lane;
      const uint32_t taddr = tmem_base + (uint32_t(ew * 32) << 16) + acc * BN;
      if constexpr (EPI == VX_EPI_QKV && HD == 0) {
#pragma unroll 1
        for (int c0 = c_beg; c0 < c_end; c0 += 32) {
          const int col = n_blk * BN + c0;
          if (col >= N) break;
          EpiPre<EPI> pre;
          epi_prefetch<EPI>(args, row, col, pre);
          uint32_t r[32];
          tmem_ld32(taddr + c0, r);
          tmem_wait_ld();
          epi_qkv_scatter32(args, row, col, r, pre);
        }
      } else if constexpr (EPI == VX_EPI_QKV) {
#pragma unroll 1
        for (int c0 = c_beg; c0 < c_end; c0 += HD) {
          const int col = n_blk * BN + c0;
          if (col >= N) break;
          uint32_t r[HD];
#pragma unroll
          for (int u = 0; u < HD; u += 32) tmem_ld32(taddr + c0 + u, r + u);
          tmem_wait_ld();
          float v[HD];
#pragma unroll
          for (int j = 0; j < HD; ++j) v[j] = __uint_as_float(r[j]);
          epi_qkv_head<HD>(args, row, col, v);
        }
      } else if constexpr (EPI == VX_EPI_SPATIAL || EPI == VX_EPI_HEADOUT) {
        const PixInfo pi = pix_of_row(args, row);
#pragma unroll 1
        for (int c0 = c_beg; c0 < c_end; c0 += 32) {
          const int col = n_blk * BN + c0;
          if (col >= N) break;
          uint32_t r[32];
          tmem_ld32(taddr + c0, r);
          tmem_wait_ld();
          if constexpr (EPI == VX_EPI_SPATIAL) epi_spatial32(args, pi, col, r);
          else epi_headout(args, pi, r);
        }
      } else if constexpr (EPI == VX_EPI_RESID_TMA) {
        const vx_epilogue& e = args.ep;
#pragma unroll 1
        for (int cb = 0; cb < nbox; ++cb) {
          const int b = cb % RT_NBOX;
          float* box = wbox + b * (RT_BOX_BYTES / 4);
          const int col = wcol0 + 32 * cb;
          uint32_t r[32];
          tmem_ld32(taddr + c_beg + 32 * cb, r);
          mbar_wait(&wbar[b], (rph >> b) & 1);
          rph ^= 1u << b;
          tmem_wait_ld();
          // this thread's row of the box: 8 float4 at 128-byte-swizzled positions (conflict-free)
          float* rowp = box + lane * 32;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4* p4 = reinterpret_cast<float4*>(rowp + ((j ^ (lane & 7)) * 4));
            const float4 x = *p4;
            const float4 g = __ldg(reinterpret_cast<const float4*>(e.gamma + col) + j);
            const float4 bb = e.bias ? __ldg(reinterpret_cast<const float4*>(e.bias + col) + j)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            *p4 = make_float4(x.x + g.x * (__uint_as_float(r[4 * j + 0]) + bb.x),
                              x.y + g.y * (__uint_as_float(r[4 * j + 1]) + bb.y),
                              x.z + g.z * (__uint_as_float(r[4 * j + 2]) + bb.z),
                              x.w + g.w * (__uint_as_float(r[4 * j + 3]) + bb.w));
          }
          fence_proxy_async_smem();  // generic-proxy writes visible to the TMA store
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmR, box, col, rrow0);  // rows >= M are clipped by the tensor map
            bulk_commit();
            if (cb + RT_NBOX < nbox) {  // refill this buffer with box cb + NBOX once the store has read it
              bulk_wait_read<0>();
              mbar_expect_tx(&wbar[b], RT_BOX_BYTES);
              tma_load_2d(box, &tmR, &wbar[b], col + 32 * RT_NBOX, rrow0);
            }
          }
          __syncwarp();
        }
      } else if constexpr (EPI == VX_EPI_RESID) {
        float* tb = epi_buf + (warp - 4) * RESID_TILE_FLOATS;
        const vx_epilogue& e = args.ep;
        const int row0 = rrow0;
#pragma unroll 1
        for (int c0 = c_beg; c0 < c_end; c0 += 32) {
          const int col = n_blk * BN + c0;
          if (col >= N) break;
          const int cc = col + int(lane);
          float* xcol = e.resid + (size_t)row0 * e.ldr + cc;
          float x[32];
#pragma unroll
          for (int rr = 0; rr < 32; ++rr) x[rr] = xpre[rr];
          if (c0 + 32 < c_end && col + 32 < N) load_resid(col + 32);
          const float b = e.bias ? __ldg(e.bias + cc) : 0.f;
          const float g = __ldg(e.gamma + cc);
          uint32_t r[32];
          tmem_ld32(taddr + c0, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) tb[lane * 33 + j] = __uint_as_float(r[j]);
          __syncwarp();
          __nv_bfloat16* kcol = e.kept ? reinterpret_cast<__nv_bfloat16*>(e.kept) + (size_t)row0 * e.ldk + cc : nullptr;
#pragma unroll
          for (int rr = 0; rr < 32; ++rr) {
            if (rr < nrows) {
              const float xv = x[rr] + g * (tb[rr * 33 + lane] + b);
              xcol[(size_t)rr * e.ldr] = xv;
              if (kcol) kcol[(size_t)rr * e.ldk] = __float2bfloat16_rn(xv);
            }
          }
          __syncwarp();
        }
      } else {
#pragma unroll 1
        for (int c0 = c_beg; c0 < c_end; c0 += 32) {
          const int col = n_blk * BN + c0;
          if (col >= N) break;
          EpiPre<EPI> pre;
          epi_prefetch<EPI>(args, row, col, pre);
          uint32_t r[32];
          tmem_ld32(taddr + c0, r);
          tmem_wait_ld();
          epi_chunk32<EPI>(args, row, col, r, pre);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG2) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));  // the leader's barrier
        else mbar_arrive(&tempty[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  if constexpr (EPI == VX_EPI_RESID_TMA) {
    if (warp >= 4 && lane_id() == 0) bulk_wait<0>();  // residual stores complete before the CTA exits
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIRED) cluster_sync();  // no CTA leaves while its peer may still multicast / arrive
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG2) tmem_dealloc_cg2(tmem_base, Cfg::TMEM_COLS);
    else tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

template <int BN, int EPI, int HD, bool MC = false, bool CG2 = false>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& args, cudaStream_t st,
                       const CUtensorMap* tr = nullptr) {
  using Cfg = GemmCfg<BN, CG2, EPI == VX_EPI_RESID_TMA, EPI == VX_EPI_HEADOUT>;
  static const CUtensorMap no_map{};
  const CUtensorMap& trr = tr ? *tr : no_map;
  constexpr uint32_t SMEM = Cfg::SMEM + epi_smem_bytes<EPI>();
  static_assert(SMEM <= 227 * 1024, "GEMM stage ring + epilogue buffer exceed the 227 KB smem per CTA");
  auto kern = gemm_kernel<BN, EPI, HD, MC, CG2>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return fail_cuda(e, "gemm: cudaFuncSetAttribute");
    attr_set = true;
  }
  const int num_m = (args.M + GEMM_BM - 1) / GEMM_BM, num_n = (args.N + BN - 1) / BN;
  if constexpr (MC || CG2) {
    const int units = ((num_m + 1) / 2) * num_n;
    const int clusters = units < num_sms() / 2 ? units : num_sms() / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, trr, args);
    if (e != cudaSuccess) return fail_cuda(e, "gemm cluster launch");
  } else {
    const int tiles = num_m * num_n;
    const int grid = tiles < num_sms() ? tiles : num_sms();
    kern<<<grid, GEMM_THREADS, SMEM, st>>>(ta, tb, trr, args);
  }
  VX_CHECK_LAUNCH("gemm launch");
  return VX_OK;
}

template <int BN, bool MC = false, bool CG2 = false>
static int dispatch_epi(int epi, const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a, cudaStream_t st) {
  switch (epi) {
    case VX_EPI_BF16: return launch_gemm<BN, VX_EPI_BF16, 0, MC, CG2>(ta, tb, a, st);
    case VX_EPI_GELU: return launch_gemm<BN, VX_EPI_GELU, 0, MC, CG2>(ta, tb, a, st);
    case VX_EPI_RESID: return launch_gemm<BN, VX_EPI_RESID, 0, MC, CG2>(ta, tb, a, st);
    case VX_EPI_PATCH: return launch_gemm<BN, VX_EPI_PATCH, 0, MC, CG2>(ta, tb, a, st);
    case VX_EPI_F32: return launch_gemm<BN, VX_EPI_F32, 0, MC, CG2>(ta, tb, a, st);
    case VX_EPI_SPATIAL: return launch_gemm<BN, VX_EPI_SPATIAL, 0, MC, CG2>(ta, tb, a, st);
    case VX_EPI_QKV:
      if (!a.ep.qn_w && !a.ep.rope_cos) return launch_gemm<BN, VX_EPI_QKV, 0, MC, CG2>(ta, tb, a, st);
      if (a.ep.head_dim == 64) return launch_gemm<BN, VX_EPI_QKV, 64, MC, CG2>(ta, tb, a, st);
      if (a.ep.head_dim == 32) return launch_gemm<BN, VX_EPI_QKV, 32, MC, CG2>(ta, tb, a, st);
      set_error("vx_gemm: qkv epilogue needs head_dim 32 or 64 (got %d)", a.ep.head_dim);
      return VX_E_ARG;
  }
  set_error("vx_gemm: unknown epilogue %d", epi);
  return VX_E_ARG;
}

// CTA pairs for the large 256-wide-N GEMMs (enough M tiles to pair up): 1 = B-tile multicast
// with per-CTA M = 128 MMAs, 2 = cta_group::2 M = 256 MMAs
static int pair_mode(int BN, int M) {
#ifdef VX_DIAG
  static int env = [] {
    const char* e = getenv("VX_GEMM_PAIR");  // diagnostic build only: 0 single CTAs, 1 multicast pairs, 2 MMA pairs
    return e ? atoi(e) : 2;
  }();
#else
  constexpr int env = 2;
#endif
  return (BN == 256 && M >= 8 * GEMM_BM) ? env : 0;
}

}  // namespace vx

extern "C" int vx_gemm(int epi, const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K,
                       const vx_epilogue* ep, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(A && B && ep, "vx_gemm: null pointer");
  VX_CHECK_ARG(M > 0 && N > 0 && K > 0, "vx_gemm: empty problem M=%d N=%d K=%d", M, N, K);
  VX_CHECK_ARG(K % GEMM_BK == 0, "vx_gemm: K=%d must be a multiple of %d", K, GEMM_BK);
  VX_CHECK_ARG(N % 32 == 0, "vx_gemm: N=%d must be a multiple of 32", N);
  VX_CHECK_ARG(lda >= K && ldb >= K && lda % 8 == 0 && ldb % 8 == 0, "vx_gemm: bad lda/ldb");
  if (epi == VX_EPI_RESID) VX_CHECK_ARG(ep->resid && ep->gamma, "vx_gemm: resid epilogue needs resid+gamma");
  if (epi == VX_EPI_QKV) {
    VX_CHECK_ARG(ep->q && ep->k && ep->v, "vx_gemm: qkv epilogue needs q/k/v");
    VX_CHECK_ARG(ep->head_dim > 0 && ep->embed_dim % ep->head_dim == 0 && ep->col_offset >= 0 &&
                     ep->col_offset % ep->head_dim == 0 && N % ep->head_dim == 0 && ep->col_offset + N <= 3 * ep->embed_dim,
                 "vx_gemm: qkv columns [col_offset, col_offset + N) = [%d, %d) not head-aligned within 3C = %d",
                 ep->col_offset, ep->col_offset + N, 3 * ep->embed_dim);
    VX_CHECK_ARG(ep->head_dim % 32 == 0 || ep->qn_w || ep->rope_cos, "vx_gemm: qkv scatter needs head_dim %% 32 == 0");
    VX_CHECK_ARG(ep->tokens_total >= M, "vx_gemm: tokens_total < M");
  }
  if (epi == VX_EPI_PATCH) VX_CHECK_ARG(ep->resid && ep->tokens_per_frame > ep->patch_start, "vx_gemm: patch args");
  if (epi == VX_EPI_BF16 || epi == VX_EPI_GELU || epi == VX_EPI_F32) VX_CHECK_ARG(ep->out, "vx_gemm: null out");
  GemmArgs args = {};
  args.M = M;
  args.N = N;
  args.K = K;
  args.ep = *ep;
  // a single M tile (camera-head trunk, M = views) is bound by streaming the weights: 64-wide N
  // tiles spread that over up to 4x more SMs than 256-wide ones
  const bool plain_qkv = epi == VX_EPI_QKV && !ep->qn_w && !ep->rope_cos;
  const bool small_m = M <= GEMM_BM && N % 64 == 0 && (epi != VX_EPI_QKV || plain_qkv) && epi != VX_EPI_PATCH;
  const int BN = small_m ? 64 : ((N % 256 == 0 || N > 512) ? 256 : 128);
  const int pm = pair_mode(BN, M);
  CUtensorMap ta, tb;
  if (!make_tmap_2d_bf16(&ta, A, M, K, lda, GEMM_BM, GEMM_BK, 128)) return VX_E_ARG;
  if (!make_tmap_2d_bf16(&tb, B, N, K, ldb, pm ? BN / 2 : BN, GEMM_BK, 128)) return VX_E_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (small_m) {
    switch (epi) {
      case VX_EPI_BF16: return launch_gemm<64, VX_EPI_BF16, 0>(ta, tb, args, st);
      case VX_EPI_GELU: return launch_gemm<64, VX_EPI_GELU, 0>(ta, tb, args, st);
      case VX_EPI_RESID: return launch_gemm<64, VX_EPI_RESID, 0>(ta, tb, args, st);
      case VX_EPI_F32: return launch_gemm<64, VX_EPI_F32, 0>(ta, tb, args, st);
      case VX_EPI_QKV: return launch_gemm<64, VX_EPI_QKV, 0>(ta, tb, args, st);
      default: break;
    }
  }
  // proj (K = C) on CTA pairs: residual tile through TMA boxes (VX_EPI_RESID_TMA). Not for fc2 (K = 4C):
  // its main loop needs the 6-stage ring the boxes would take (measured 10-16% slower with 4 stages)
  if (epi == VX_EPI_RESID && !ep->kept && pm == 2 && K <= 2048 && (reinterpret_cast<uintptr_t>(ep->resid) & 15) == 0 &&
      ep->ldr % 4 == 0) {
    CUtensorMap tr;
    if (!make_tmap_2d(&tr, ep->resid, true, M, N, ep->ldr, 32, 32, 128)) return VX_E_ARG;
    return launch_gemm<256, VX_EPI_RESID_TMA, 0, false, true>(ta, tb, args, st, &tr);
  }
  if (pm == 2) return dispatch_epi<256, false, true>(epi, ta, tb, args, st);
#ifdef VX_DIAG
  if (pm) return dispatch_epi<256, true>(epi, ta, tb, args, st);  // B-tile multicast pairs (measured slower)
#endif
  return BN == 256 ? dispatch_epi<256>(epi, ta, tb, args, st) : dispatch_epi<128>(epi, ta, tb, args, st);
}

extern "C" int vx_gemm_spatial(const void* A, const void* B, int N, int K, const float* bias, const vx_spatial* sp,
                               void* stream) {
  using namespace vx;
  VX_CHECK_ARG(A && B && sp, "vx_gemm_spatial: null pointer");
  VX_CHECK_ARG(sp->out1 != nullptr || sp->head_odim > 0, "vx_gemm_spatial: no output");
  VX_CHECK_ARG(sp->F > 0 && sp->H > 0 && sp->W > 0, "vx_gemm_spatial: bad grid");
  VX_CHECK_ARG(K % GEMM_BK == 0 && N % 32 == 0, "vx_gemm_spatial: K %% 64, N %% 32 required (K=%d N=%d)", K, N);
  const int s = sp->shuffle < 1 ? 1 : sp->shuffle;
  VX_CHECK_ARG(N % (s * s) == 0 && (N / (s * s)) % 32 == 0, "vx_gemm_spatial: Cout must be a multiple of 32");
  VX_CHECK_ARG(!(sp->subsample2 && s > 1), "vx_gemm_spatial: subsample2 and shuffle are exclusive");
  if (sp->head_odim > 0) VX_CHECK_ARG(N == 32 && sp->head_w && sp->head_b && sp->head_pred && sp->head_conf &&
                                      sp->head_odim >= 2 && !sp->subsample2 && s == 1 && sp->conv3x3 &&
                                      K <= 9 * HALO_MAX_CB * GEMM_BK,
                                      "vx_gemm_spatial: fused head needs a 3x3 conv with N == 32, <= 128 input "
                                      "channels and head pointers");
  GemmArgs args = {};
  args.N = N;
  args.K = K;
  args.sp = *sp;
  args.sp.shuffle = s;
  args.ep.bias = bias;
  int64_t rows;
  if (sp->conv3x3) {
    VX_CHECK_ARG(K % (9 * GEMM_BK) == 0, "vx_gemm_spatial: conv3x3 needs Cin %% 64 == 0 (K=%d)", K);
    args.conv_cin_blocks = K / (9 * GEMM_BK);
    args.conv_w2 = sp->W + 2;
    rows = (int64_t)sp->F * (sp->H + 2) * (sp->W + 2);
  } else {
    rows = (int64_t)sp->F * sp->H * sp->W;
  }
  VX_CHECK_ARG(rows < (1ll << 31), "vx_gemm_spatial: too many rows");
  args.M = int(rows);
  const int BN = sp->head_odim > 0 ? 32 : ((N % 256 == 0 || N > 512) ? 256 : 128);
  const int64_t lda = sp->conv3x3 ? K / 9 : K;
  const int pm = pair_mode(BN, int(rows));
  CUtensorMap ta, tb;
  // the output head stages 130-row input bands (HALO)
  if (!make_tmap_2d_bf16(&ta, A, rows, lda, lda, sp->head_odim > 0 ? HALO_ROWS : GEMM_BM, GEMM_BK, 128))
    return VX_E_ARG;
  if (!make_tmap_2d_bf16(&tb, B, N, K, K, pm ? BN / 2 : BN, GEMM_BK, 128)) return VX_E_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int epi = sp->head_odim > 0 ? VX_EPI_HEADOUT : VX_EPI_SPATIAL;
  if (BN == 32) return launch_gemm<32, VX_EPI_HEADOUT, 0>(ta, tb, args, st);  // N == 32 output head
  if (pm == 2) return launch_gemm<256, VX_EPI_SPATIAL, 0, false, true>(ta, tb, args, st);
#ifdef VX_DIAG
  if (pm) return launch_gemm<256, VX_EPI_SPATIAL, 0, true>(ta, tb, args, st);
#endif
  return BN == 256 ? dispatch_epi<256>(epi, ta, tb, args, st) : dispatch_epi<128>(epi, ta, tb, args, st);
}
