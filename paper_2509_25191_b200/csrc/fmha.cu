// tcgen05/TMEM flash attention for VGGT frame and global attention (sm_100a).
//
// Replaces F.scaled_dot_product_attention in the upstream Attention.forward
// (frame blocks, batch S*16 sequences of 1374 tokens; a8:
// global blocks, 16 sequences of S*1374 tokens).  Non-causal, d in {32, 64}.
//
// One CTA = one work unit = 256 query rows (two 128-row Q tiles) of one
// (head, sequence); persistent grid over units, head-major so concurrently
// running CTAs share K/V through L2.
//
// Warp roles (384 threads):
//   w0      TMA producer: Q tiles once per unit, K/V tiles through a KST-stage ring
//   w1      tcgen05.mma issuer (one lane): S_i = Q_i K^T (SS), O_i += P_i V (TS, P in TMEM)
//   w2      TMEM allocator (512 columns: S0 | S1 | O0 | O1, P_i aliases S_i)
//   w4..w7  softmax + epilogue for Q tile 0, w8..w11 for Q tile 1
//           (thread = one query row = one TMEM lane: row max / sum are thread-local;
//            lazy O rescaling only when the running max grows by > 2^8)
//   (v4: each Q tile's 128 score columns are split over two warpgroups, 16 softmax warps in
//    total, partial row maxima exchanged through shared memory + a named barrier)
// MMA issue order per KV tile j:  PV_0(j), S_0(j+1), PV_1(j), S_1(j+1), so each
// softmax warpgroup's exp work overlaps the other tile's tensor-core work.
#include <math.h>
#include <stdlib.h>

#include "../../include/vx_api.h"
#include "common.cuh"
#include "host_util.h"

namespace vx {

struct AttnArgs {
  int H, nseq, Lq, Lk;
  int64_t Tq, Tk;
  int q_blocks, kv_tiles, units;
  float scale_log2;
  __nv_bfloat16* out;
  int64_t ldo;
  float* lse;
};

template <int D>
struct AttnCfg {
  static constexpr int KST = 3;
  static constexpr uint32_t ROW_BYTES = D * 2;
  static constexpr uint32_t TILE_BYTES = 128 * ROW_BYTES;
  static constexpr int SWIZZLE = D == 64 ? 128 : 64;
  static constexpr uint32_t LAYOUT = D == 64 ? 2 : 4;  // SWIZZLE_128B / SWIZZLE_64B
  static constexpr uint32_t SBO = 8 * ROW_BYTES;       // 8-row core-matrix group
  static constexpr uint32_t ONES_BYTES = 2048;  // 16 x 64 bf16 ones (row-sum B operand)
  static constexpr uint32_t SMEM = (2 + 2 * KST) * TILE_BYTES + ONES_BYTES + 1024 + 512 + 2048;
};

constexpr int ATTN_THREADS = 640;  // 4 control warps + 4 softmax warpgroups
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units

// EMU_PAIRS_OF_8: of every 8 exp pairs, this many use the FMA-pipe polynomial
template <int D, int EMU_PAIRS_OF_8>
__global__ void __launch_bounds__(ATTN_THREADS, 1)
    fmha_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using Cfg = AttnCfg<D>;
  constexpr int KST = Cfg::KST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                 // 2 tiles
  uint8_t* sK = sQ + 2 * Cfg::TILE_BYTES;             // KST tiles
  uint8_t* sV = sK + KST * Cfg::TILE_BYTES;           // KST tiles
  uint8_t* sOnes = sV + KST * Cfg::TILE_BYTES;        // 2 KB of bf16 1.0
  uint64_t* bar = reinterpret_cast<uint64_t*>(sOnes + Cfg::ONES_BYTES);
  uint64_t* q_full = bar;
  uint64_t* q_empty = bar + 1;
  uint64_t* k_full = bar + 2;
  uint64_t* k_empty = k_full + KST;
  uint64_t* v_full = k_empty + KST;
  uint64_t* v_empty = v_full + KST;
  uint64_t* s_full = v_empty + KST;  // [2]
  uint64_t* p_full = s_full + 2;     // [2]
  uint64_t* o_full = p_full + 2;     // [2]
  uint64_t* o_empty = o_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);
  float* xmax = reinterpret_cast<float*>(bar + 64);  // [2 tiles][2 halves][128 rows] partial maxima

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  if (warp == 3) {
    uint4* o4 = reinterpret_cast<uint4*>(sOnes);
    for (int i = lane; i < int(Cfg::ONES_BYTES / 16); i += 32) o4[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int per_head = a.nseq * a.q_blocks;
  const int nkv = a.kv_tiles;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t pol_kv = policy_evict_last();
      const uint64_t pol_q = policy_evict_first();
      uint32_t c = 0;  // global K/V tile counter
      uint32_t n = 0;  // local unit counter
      for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++n) {
        const int h = u / per_head;
        const int rem = u - h * per_head;
        const int s = rem / a.q_blocks;
        const int qb = rem - s * a.q_blocks;
        const int q_row = int(h * a.Tq + (int64_t)s * a.Lq + qb * 256);
        const int kv_row = int(h * a.Tk + (int64_t)s * a.Lk);
        mbar_wait(q_empty, (n & 1) ^ 1);
        mbar_expect_tx(q_full, 2 * Cfg::TILE_BYTES);
        tma_load_2d_hint(sQ, &tmQ, q_full, 0, q_row, pol_q);
        tma_load_2d_hint(sQ + Cfg::TILE_BYTES, &tmQ, q_full, 0, q_row + 128, pol_q);
        for (int j = 0; j < nkv; ++j, ++c) {
          const uint32_t st = c % KST, ph = (c / KST) & 1;
          mbar_wait(&k_empty[st], ph ^ 1);
          mbar_expect_tx(&k_full[st], Cfg::TILE_BYTES);
          tma_load_2d_hint(sK + st * Cfg::TILE_BYTES, &tmK, &k_full[st], 0, kv_row + 128 * j, pol_kv);
          mbar_wait(&v_empty[st], ph ^ 1);
          mbar_expect_tx(&v_full[st], Cfg::TILE_BYTES);
          tma_load_2d_hint(sV + st * Cfg::TILE_BYTES, &tmV, &v_full[st], 0, kv_row + 128 * j, pol_kv);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16(128, D, 0, 1);
      const uint32_t q0 = smem_u32(sQ), q1 = q0 + Cfg::TILE_BYTES;
      auto issue_qk = [&](uint32_t d_tmem, uint32_t qs, uint32_t ks) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k)
          mma_ss(d_tmem, make_sdesc(qs + k * 32, 16, Cfg::SBO, Cfg::LAYOUT),
                 make_sdesc(ks + k * 32, 16, Cfg::SBO, Cfg::LAYOUT), idesc_qk, k > 0);
      };
      constexpr uint32_t idesc_sum = make_idesc_bf16(128, 16, 0, 0);
      const uint64_t ones_desc = make_sdesc(smem_u32(sOnes), 16, 1024, 2);
      // O[:, 0:D] += P V ; O[:, D:D+16] += P 1 (row sums of the bf16 P, on the tensor core)
      auto issue_pv = [&](uint32_t d_tmem, uint32_t p_tmem, uint32_t vs, uint32_t acc) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          mma_ts(d_tmem, p_tmem + kk * 8, make_sdesc(vs + kk * 16 * Cfg::ROW_BYTES, 16, Cfg::SBO, Cfg::LAYOUT),
                 idesc_pv, (acc | kk) != 0);
          mma_ts(d_tmem + D, p_tmem + kk * 8, ones_desc, idesc_sum, (acc | kk) != 0);
        }
      };
      const uint32_t S0 = tmem, S1 = tmem + 128, O0 = tmem + 256, O1 = tmem + 384;
      uint32_t c = 0;
      uint32_t n = 0;
      uint32_t pph0 = 0, pph1 = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++n) {
        mbar_wait(q_full, n & 1);
        tc_fence_after();
        {
          const uint32_t st = c % KST, ph = (c / KST) & 1;
          mbar_wait(&k_full[st], ph);
          tc_fence_after();
          const uint32_t ks = smem_u32(sK + st * Cfg::TILE_BYTES);
          issue_qk(S0, q0, ks);
          mma_commit(&s_full[0]);
          issue_qk(S1, q1, ks);
          mma_commit(&s_full[1]);
          mma_commit(&k_empty[st]);
          if (nkv == 1) mma_commit(q_empty);
        }
        for (int j = 0; j < nkv; ++j, ++c) {
          const uint32_t st = c % KST, ph = (c / KST) & 1;
          const uint32_t vs = smem_u32(sV + st * Cfg::TILE_BYTES);
          const bool has_next = j + 1 < nkv;
          const uint32_t nst = (c + 1) % KST, nph = ((c + 1) / KST) & 1;
          const uint32_t nks = smem_u32(sK + nst * Cfg::TILE_BYTES);
          mbar_wait(&v_full[st], ph);
          // ---- tile 0
          if (j == 0) mbar_wait(&o_empty[0], (n & 1) ^ 1);
          mbar_wait(&p_full[0], pph0);
          pph0 ^= 1;
          tc_fence_after();
          issue_pv(O0, S0, vs, j > 0);
          if (!has_next) mma_commit(&o_full[0]);
          if (has_next) {
            mbar_wait(&k_full[nst], nph);
            tc_fence_after();
            issue_qk(S0, q0, nks);
            mma_commit(&s_full[0]);
          }
          // ---- tile 1
          if (j == 0) mbar_wait(&o_empty[1], (n & 1) ^ 1);
          mbar_wait(&p_full[1], pph1);
          pph1 ^= 1;
          tc_fence_after();
          issue_pv(O1, S1, vs, j > 0);
          mma_commit(&v_empty[st]);
          if (!has_next) mma_commit(&o_full[1]);
          if (has_next) {
            issue_qk(S1, q1, nks);
            mma_commit(&s_full[1]);
            mma_commit(&k_empty[nst]);
            if (j + 2 == nkv) mma_commit(q_empty);
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax / epilogue
    // 4 warpgroups: (tile, half) = Q tile 0/1 x score columns 0-63 / 64-127 of the same rows;
    // the two halves of a tile exchange their partial row maxima through shared memory.
    const int sw = warp - 4;
    const int tile = sw >> 3;
    const int half = (sw >> 2) & 1;
    const int wl = warp & 3;          // TMEM lane quarter
    const int r = wl * 32 + lane;     // row within the Q tile
    const uint32_t lane_off = uint32_t(wl * 32) << 16;
    const uint32_t S_addr = tmem + lane_off + tile * 128;
    const uint32_t O_addr = tmem + lane_off + 256 + tile * 128;
    float* my_max = xmax + (tile * 2 + half) * 128;
    const float* other_max = xmax + (tile * 2 + (half ^ 1)) * 128;
    const float sl2 = a.scale_log2;
    uint32_t sph = 0, oph = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
      const int h = u / per_head;
      const int rem = u - h * per_head;
      const int s = rem / a.q_blocks;
      const int qb = rem - s * a.q_blocks;
      const int q_local = qb * 256 + tile * 128 + r;
      float m_run = -INFINITY;
      for (int j = 0; j < nkv; ++j) {
        mbar_wait(&s_full[tile], sph);
        sph ^= 1;
        tc_fence_after();
        uint32_t sr[64];
        tmem_ld32(S_addr + 64 * half, sr);
        tmem_ld32(S_addr + 64 * half + 32, sr + 32);
        tmem_wait_ld();
        const int valid = a.Lk - 128 * j - 64 * half;
        if (valid < 64) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c >= valid) sr[c] = 0xff800000u;  // -inf
        }
        // partial row max over 64 columns: 4 independent FMNMX3 chains + tree
        float mq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) mq[u] = fmaxf(__uint_as_float(sr[u]), __uint_as_float(sr[u + 4]));
#pragma unroll
        for (int c = 8; c < 64; c += 8)
#pragma unroll
          for (int u = 0; u < 4; ++u) mq[u] = max3(mq[u], __uint_as_float(sr[c + u]), __uint_as_float(sr[c + 4 + u]));
        const float pmax = fmaxf(max3(mq[0], mq[1], mq[2]), mq[3]);
        my_max[r] = pmax;
        named_bar_sync(1 + tile, 256);   // both halves loaded S and published their maxima
        const float mx = fmaxf(pmax, other_max[r]);
        const float m_new = mx * sl2;
        const bool need = m_new > m_run + RESCALE_THRESHOLD;
        const float alpha = need ? ex2(m_run - m_new) : 1.0f;
        if (need) m_run = m_new;
        const uint64_t SL2 = f2_pack(sl2, sl2);
        const uint64_t NEGM = f2_pack(-m_run, -m_run);
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          // x = s * scale*log2(e) - m for two columns with one FFMA2
          const uint64_t x = f2_fma(f2_pack(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), SL2, NEGM);
          float x0, x1, p0, p1;
          f2_unpack(x, x0, x1);
          if ((c & 7) >= 8 - EMU_PAIRS_OF_8) {  // part of the exps on the FMA pipe
            ex2_poly2(x0, x1, p0, p1);
          } else {
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          pk[c] = pack_bf16(p0, p1);
        }
        // P (bf16 pairs) overwrites S columns [32*half, 32*half + 32): the other half has already
        // loaded its S columns (named barrier above)
        tmem_st32(S_addr + 32 * half, pk);
        // lazy O / row-sum correction (warp-uniform); PV(j-1) completed before s_full(j)
        if (__any_sync(0xffffffff, need) && j > 0) {
          if (half == 0) {
            uint32_t orr[D];
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += 32) tmem_ld32(O_addr + c0, orr + c0);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < D; ++c) orr[c] = __float_as_uint(__uint_as_float(orr[c]) * alpha);
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += 32) tmem_st32(O_addr + c0, orr + c0);
          } else {
            uint32_t orr[16];
            tmem_ld16(O_addr + D, orr);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 16; ++c) orr[c] = __float_as_uint(__uint_as_float(orr[c]) * alpha);
            tmem_st16(O_addr + D, orr);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[tile]);
      }
      // ---- epilogue: O[:, half*D/2 : +D/2] / l -> bf16
      mbar_wait(&o_full[tile], oph);
      oph ^= 1;
      tc_fence_after();
      constexpr int DH = D / 2;
      uint32_t orr[DH];
      uint32_t lr[16];
      if constexpr (DH == 32) {
        tmem_ld32(O_addr + half * DH, orr);
      } else {
        tmem_ld16(O_addr + half * DH, orr);
      }
      tmem_ld16(O_addr + D, lr);
      tmem_wait_ld();
      const float l_run = __uint_as_float(lr[0]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[tile]);
      if (q_local < a.Lq) {
        const float inv = 1.0f / l_run;
        const int64_t orow = (int64_t)s * a.Lq + q_local;
        uint4* dst = reinterpret_cast<uint4*>(a.out + orow * a.ldo + h * D + half * DH);
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) {
#define VX_O(i) (__uint_as_float(orr[8 * c + i]) * inv)
          dst[c] = make_uint4(pack_bf16(VX_O(0), VX_O(1)), pack_bf16(VX_O(2), VX_O(3)),
                              pack_bf16(VX_O(4), VX_O(5)), pack_bf16(VX_O(6), VX_O(7)));
#undef VX_O
        }
        if (a.lse && half == 0) a.lse[h * a.Tq + orow] = (m_run + __log2f(l_run)) * 0.69314718055994531f;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, int EMU>
static int launch_fmha(const void* q, const void* k, const void* v, const AttnArgs& args, cudaStream_t st) {
  using Cfg = AttnCfg<D>;
  CUtensorMap tq, tk, tv;
  if (!make_tmap_2d_bf16(&tq, q, (uint64_t)args.H * args.Tq, D, D, 128, D, Cfg::SWIZZLE)) return VX_E_ARG;
  if (!make_tmap_2d_bf16(&tk, k, (uint64_t)args.H * args.Tk, D, D, 128, D, Cfg::SWIZZLE)) return VX_E_ARG;
  if (!make_tmap_2d_bf16(&tv, v, (uint64_t)args.H * args.Tk, D, D, 128, D, Cfg::SWIZZLE)) return VX_E_ARG;
  auto kern = fmha_kernel<D, EMU>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return fail_cuda(e, "fmha: cudaFuncSetAttribute");
    attr_set = true;
  }
  const int grid = args.units < num_sms() ? args.units : num_sms();
  kern<<<grid, ATTN_THREADS, Cfg::SMEM, st>>>(tq, tk, tv, args);
  VX_CHECK_LAUNCH("fmha launch");
  return VX_OK;
}

}  // namespace vx

extern "C" int vx_attention(const void* q, const void* k, const void* v, void* out, int64_t ldo, float* lse, int D,
                            int H, int nseq, int Lq, int Lk, int64_t Tq, int64_t Tk, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(q && k && v && out, "vx_attention: null pointer");
  VX_CHECK_ARG(D == 32 || D == 64, "vx_attention: head_dim %d unsupported (32, 64)", D);
  VX_CHECK_ARG(H > 0 && nseq > 0 && Lq > 0 && Lk > 0, "vx_attention: empty problem");
  VX_CHECK_ARG((int64_t)nseq * Lq <= Tq && (int64_t)nseq * Lk <= Tk, "vx_attention: sequences exceed buffers");
  VX_CHECK_ARG((int64_t)H * Tq + 512 < (1ll << 31) && (int64_t)H * Tk + 512 < (1ll << 31),
               "vx_attention: too many rows for 32-bit TMA coordinates");
  VX_CHECK_ARG(ldo >= (int64_t)H * D && ldo % 8 == 0, "vx_attention: bad ldo");
  AttnArgs a;
  a.H = H;
  a.nseq = nseq;
  a.Lq = Lq;
  a.Lk = Lk;
  a.Tq = Tq;
  a.Tk = Tk;
  a.q_blocks = (Lq + 255) / 256;
  a.kv_tiles = (Lk + 127) / 128;
  a.units = H * nseq * a.q_blocks;
  a.scale_log2 = (1.0f / sqrtf(float(D))) * 1.4426950408889634f;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.ldo = ldo;
  a.lse = lse;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  static int emu = [] {
    const char* e = getenv("VX_FMHA_EMU");  // diagnostic: exp pairs (of 8) on the FMA pipe
    return e ? atoi(e) : 3;
  }();
  if (D == 64) {
    switch (emu) {
      case 0: return launch_fmha<64, 0>(q, k, v, a, st);
      case 2: return launch_fmha<64, 2>(q, k, v, a, st);
      case 3: return launch_fmha<64, 3>(q, k, v, a, st);
      case 5: return launch_fmha<64, 5>(q, k, v, a, st);
      case 4: return launch_fmha<64, 4>(q, k, v, a, st);
      default: return launch_fmha<64, 3>(q, k, v, a, st);
    }
  }
  return launch_fmha<32, 3>(q, k, v, a, st);
}
