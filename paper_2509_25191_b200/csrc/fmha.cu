// tcgen05/TMEM flash attention for VGGT frame and global attention (sm_100a).
//
// Replaces F.scaled_dot_product_attention in the upstream Attention.forward
// (frame blocks, batch S*16 sequences of 1374 tokens; a8:
// global blocks, 16 sequences of S*1374 tokens).  Non-causal, d in {32, 64}.
//
// One CTA = one work unit = NT 128-row Q tiles of one (head, sequence); persistent grid over
// units, head-major so concurrently running CTAs share K/V through L2.
//
// d = 64 (default): NT = 4 tiles x 48-wide KV tiles.  TMEM (512 columns) per Q tile i:
//   S_i [48 fp32, P_i bf16 written over it] | O_i [64 + 8 fp32].
// V is extended by a constant panel of ones, so the PV MMA also accumulates the row sums of P
// into O_i[:, 64] (same lazy rescaling as O; no FADD row sums); the PV MMA runs with N = 72.  With P aliased onto S the MMA
// issuer runs PV_i(j) then S_i(j+1) into the same columns (tcgen05 executes in issue order).
// Other shapes (d = 32 / 128, diagnostics): separate P columns, S(j+1) issued ahead of the softmax.
//
// Warp roles (128 + 128*NT threads):
//   w0      TMA producer: Q tiles once per unit, K/V tiles through a KST-stage ring
//   w1      tcgen05.mma issuer (one lane): S_i = Q_i K^T (SS), O_i += P_i V (TS: P from TMEM)
//   w2      TMEM allocator
//   w4..    softmax + epilogue: one warpgroup per Q tile; thread = one query row = one TMEM
//           lane owning all score columns of the KV tile (row max / sum thread-local).
// Softmax arithmetic: x = s*scale*log2e - m with FFMA2 (packed fp32x2), 2 of every 8 exp pairs
// on the FMA pipe (packed degree-2 polynomial), the rest on MUFU ex2; FMNMX3 max tree; lazy
// rescaling of O only when the running max grows by > 2^8.  Because m only moves past that
// threshold, the exps of a tile start with the running max and the tile max is computed alongside
// them (speculative; a warp with a row over the threshold redoes the tile).  The column mask of
// the last KV tile lives on a separate code path (BoolTag) so the common path carries none.
#include <math.h>
#include <stdlib.h>

#include <map>
#include <mutex>
#include <utility>

#include "../../include/vx_api.h"
#include "common.cuh"
#include "host_util.h"

#ifndef VX_FMHA_PSM
#define VX_FMHA_PSM 0
#endif
#ifndef VX_FMHA_W96
#define VX_FMHA_W96 0
#endif
#ifndef VX_FMHA_NOMAX_EMU  // exp pairs (of 8) on the FMA pipe in the max-free kernel
#define VX_FMHA_NOMAX_EMU 2
#endif
#ifndef VX_FMHA_ONES_ALL  // 1: the row-sum panel all ones (round-2 builds before the single ones column)
#define VX_FMHA_ONES_ALL 0
#endif
#ifndef VX_FMHA_NOMAX_W64  // max-free kernel with 64-wide KV tiles and FADD row sums
#define VX_FMHA_NOMAX_W64 0
#endif

namespace vx {

struct AttnArgs {
  int H, nseq, Lq, Lk;
  int64_t Tq, Tk;
  // ring steps (vx_attention_merge): 0 plain; 1 first block -> o_acc / lse; 2 merge into o_acc / lse;
  // 3 merge and write the final bf16 output
  int merge;
  float* o_acc;
  int64_t ld_acc;
  int q_blocks, kv_tiles, units;
  // Q tiles are numbered over (head, sequence, 128-row tile) in that order, tps per sequence; unit u
  // owns tiles [NT*u, NT*u + NT) of total_tiles. tps = q_blocks * NT (units never straddle two
  // sequences) except for packed frame attention, where tps = ceil(Lq / 128) and a unit may take its
  // last tiles from the next sequence (then it streams both sequences' K/V)
  int tps, total_tiles;
  float scale_log2;
  __nv_bfloat16* out;
  int64_t ldo;
  float* lse;
  // KV-split tail (plain and ring-merge modes): units >= split_from run as `parts` work items, each over
  // a contiguous range of KV tiles, writing normalised fp32 partial O + lse to part_o / part_lse
  // (item-major, ROWS rows each); fmha_split_merge combines them. work = total work items.
  int split_from, parts, work;
  float* part_o;
  float* part_lse;
  // dynamic work distribution: sched[0] = next work-item ticket past the first wave, sched[1] = CTAs
  // finished (the last one resets both, so the counters are zero again for the next launch on the
  // stream); nullptr = static round-robin (while a stream is being captured before the counters exist)
  unsigned* sched;
  // max-free launches (NOMAX kernel): a unit with a row whose result is not trustworthy (P or O out
  // of the fp32 range) is appended to fix_list (bad[0] = entries; more than fix_cap = recompute every
  // unit). The exact kernel then runs as a fixup (fixup = 1) over the listed units only: it exits at
  // once when the list is empty, and its last CTA clears bad[0] (bad[1] counts its CTAs). Plain
  // launches write every unit and the fixup overwrites the listed ones; ring-merge launches (in-place
  // O / lse accumulation) skip writing a flagged unit altogether, so the fixup merges it exactly once.
  unsigned* bad;
  unsigned* fix_list;
  int fix_cap;
  int fixup;
  int out32;  // out and ldo allow 32-byte row stores
};

// work-item queue depth (shared-memory ring from the TMA producer to the MMA and softmax warps)
constexpr int WQ = 4;

// work item w -> unit, first KV tile, KV tile count, part (-1: whole unit), tail index
struct WorkItem {
  int u, j0, cnt, part, t;
};
VX_DEVICE WorkItem work_item(const AttnArgs& a, int w) {
  if (w < a.split_from) return {w, 0, a.kv_tiles, -1, 0};
  const int x = w - a.split_from;
  const int t = x / a.parts, p = x - t * a.parts;
  const int j0 = p * a.kv_tiles / a.parts;  // host guarantees parts * kv_tiles < 2^31
  const int j1 = (p + 1) * a.kv_tiles / a.parts;
  return {a.split_from + t, j0, j1 - j0, p, t};
}

template <int D, int NT_ = (D == 128 ? 1 : 2), int BKV_ = 128, bool ALIAS_ = false, bool SUMV_ = false,
          bool PSM_ = false, bool PACK_ = false>
struct AttnCfg {
  // PACK: a unit's NT Q tiles may come from two consecutive sequences (frame attention, where
  // 1374 rows = 10.7 tiles would otherwise leave 1.3 of every 12 tile slots empty); every K/V stage
  // then has a slot per sequence
  static constexpr bool PACK = PACK_;
  static constexpr int KV_SLOTS = PACK ? 2 : 1;
  // PSM: P goes to shared memory (one 128 x 64-column SW128 tile per Q tile, K-major like Q) and the
  // PV MMA reads it from there (SS), so TMEM holds only S and O per tile and S_i(j+1) is issued as
  // soon as the softmax has loaded S_i(j), overlapping its exps (not aliased, 4 tiles still fit)
  static constexpr bool PSM = PSM_;
  static_assert(!(PSM_ && ALIAS_), "PSM and ALIAS are exclusive");
  // ALIAS: P is written over the first BKV/2 columns of S (4 tiles fit TMEM); S_i(j+1) is then
  // issued after PV_i(j) instead of running ahead
  static constexpr bool ALIAS = ALIAS_;
  // SUMV: the row sums come out of the PV MMA: V is extended by a panel of ones (N = D + 16), so
  // O_i[:, D] accumulates sum_k P_ik with the same lazy rescaling as O — no FADD row sums
  static constexpr bool SUMV = SUMV_;
  static constexpr int DO = D + (SUMV ? 8 : 0);            // O accumulator columns (N of the PV MMA)
  static constexpr int NT = NT_;                           // 128-row Q tiles per CTA (TMEM budget)
  static constexpr int BKV = BKV_;                         // KV rows per tile (score columns)
  // SUMV kernels (d = 64 product kernels): one shared ones panel instead of one per V stage, and two
  // Q buffers so a unit's Q loads while the previous unit still runs (the 64 KB reload was the
  // largest piece of the unit-boundary gap of 29-tile frame units); packed: 3 K/V stages to fit
  static constexpr int QBUF = SUMV_ ? 2 : 1;
  static constexpr int KST = D == 128 ? 2 : (BKV <= 64 ? (PACK && SUMV_ ? 3 : 4) : 3);
  static constexpr int PANEL_COLS = D == 32 ? 32 : 64;     // one swizzle atom wide (<= 128 B)
  static constexpr int PANELS = D / PANEL_COLS;            // D = 128: two 64-column panels
  static constexpr uint32_t ROW_BYTES = PANEL_COLS * 2;    // bytes per row inside a panel
  static constexpr uint32_t QPANEL_BYTES = 128 * ROW_BYTES;
  static constexpr uint32_t KVPANEL_BYTES = BKV * ROW_BYTES;
  static constexpr uint32_t Q_TILE_BYTES = PANELS * QPANEL_BYTES;
  static constexpr uint32_t KV_TILE_BYTES = PANELS * KVPANEL_BYTES;
  static constexpr uint32_t V_STAGE_BYTES = KV_TILE_BYTES;
  static constexpr uint32_t ONES_BYTES = SUMV ? KVPANEL_BYTES : 0;  // the ones panel (second MN atom of V)
  static constexpr int SWIZZLE = D == 32 ? 64 : 128;
  static constexpr uint32_t LAYOUT = D == 32 ? 4 : 2;      // SWIZZLE_64B / SWIZZLE_128B
  static constexpr uint32_t SBO = 8 * ROW_BYTES;           // 8-row core-matrix group
  static constexpr int THREADS = 128 + 128 * NT;
  static constexpr int ROWS = 128 * NT;                    // query rows per work unit
  static constexpr uint32_t BAR_BYTES = 512;
  static constexpr uint32_t P_TILE_BYTES = PSM ? 128 * 128 : 0;  // 128 rows x 128 B (BKV <= 64 bf16 used)
  static constexpr uint32_t K_STAGE_BYTES = KV_SLOTS * KV_TILE_BYTES;   // [K_A | K_B]
  static constexpr uint32_t VS_STAGE_BYTES = KV_SLOTS * V_STAGE_BYTES;  // [V_A | V_B]
  static constexpr uint32_t SMEM = QBUF * NT * Q_TILE_BYTES + NT * P_TILE_BYTES + KST * (K_STAGE_BYTES + VS_STAGE_BYTES) +
                                   ONES_BYTES + 1024 + BAR_BYTES;
  // TMEM columns: S_i [BKV fp32] ... | P_i [BKV/2] (neither ALIAS nor PSM) ... | O_i [DO fp32] ...
  static constexpr uint32_t O_BASE = ((NT * BKV + (ALIAS || PSM ? 0 : NT * BKV / 2)) + 31) / 32 * 32;
  static_assert(O_BASE + NT * DO <= 512, "TMEM budget");
  static_assert(!SUMV || ((ALIAS || PSM) && D == 64), "SUMV is implemented for the d=64 kernels");
  static_assert(!PSM || (D == 64 && BKV <= 64), "PSM: one 128-byte P row per query row");
  static_assert(!PACK || (ALIAS && !PSM), "PACK is implemented for the aliased kernel");
  static_assert(BKV % 16 == 0 && (BKV <= 64 || BKV % 64 == 0 || (BKV == 96 && ALIAS && D == 64)), "KV tile width");
  static __host__ __device__ constexpr uint32_t tS(int i) { return i * BKV; }
  static __host__ __device__ constexpr uint32_t tP(int i) { return ALIAS ? i * BKV : NT * BKV + i * (BKV / 2); }
  static __host__ __device__ constexpr uint32_t tO(int i) { return O_BASE + i * DO; }
};

// TMEM <-> register helpers for column counts that are multiples of 8
template <int N>
VX_DEVICE void tmem_ld_n(uint32_t taddr, uint32_t* r) {
  static_assert(N % 16 == 0, "ld width");
#pragma unroll
  for (int c = 0; c + 32 <= N; c += 32) tmem_ld32(taddr + c, r + c);
  if constexpr (N % 32 == 16) tmem_ld16(taddr + N - 16, r + N - 16);
}
template <int N>
VX_DEVICE void tmem_st_n(uint32_t taddr, const uint32_t* r) {
  static_assert(N % 8 == 0, "st width");
#pragma unroll
  for (int c = 0; c + 32 <= N; c += 32) tmem_st32(taddr + c, r + c);
  if constexpr (N % 32 >= 16) tmem_st16(taddr + N / 32 * 32, r + N / 32 * 32);
  if constexpr (N % 16 == 8) tmem_st8(taddr + N - 8, r + N - 8);
}

#ifdef VX_FMHA_TRACE
// diagnostic build only (tools/trace_fmha.py): clock64 stamps of CTA 0's first unit
__device__ unsigned long long* g_fmha_trace = nullptr;
#define VX_TRACE(slot)                                                                    \
  do {                                                                                    \
    if (g_fmha_trace && blockIdx.x == 0 && (slot) >= 0) g_fmha_trace[(slot)] = clock64(); \
  } while (0)
#else
#define VX_TRACE(slot) \
  do {                 \
  } while (0)
#endif
// trace slots (CTA 0's first two units, up to 32 KV tiles each: iteration jj = 32 * unit + j):
// softmax tile t (lane 0 of its first warp), point k < 8: (t * 64 + jj) * 8 + k (0 wait for S, 1 S
// ready, 2 max (exact kernel) / output stores begin (unit's last tile), 3 exps done, 4 P-ready
// arrive, 5 O final, 6 epilogue done, 7 O read); MMA thread: 4096 + (jj * 4 + i) * 2 + {0: p_full
// seen, 1: S(j+1) committed}, 6000 + 4 * unit + i: S(0) committed, 6100 + unit: q_full seen;
// producer: 6230 + unit q_empty seen, 6240 + 2 * unit + j: K stage j of the unit free
VX_DEVICE int trace_slot_sm(int unit_n, int wl, int lane, int tile, int j, int k) {
  return (unit_n < 2 && wl == 0 && lane == 0 && j < 32) ? (tile * 64 + unit_n * 32 + j) * 8 + k : -1;
}
VX_DEVICE int trace_slot_mma(int unit_n, int j, int i, int k) {
  return (unit_n < 2 && j < 32) ? 4096 + ((unit_n * 32 + j) * 4 + i) * 2 + k : -1;
}

template <bool B>
struct BoolTag {
  static constexpr bool value = B;
};

constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units


// EMU_PAIRS_OF_8: of every 8 exp pairs, this many use the FMA-pipe polynomial
template <int D, int EMU_PAIRS_OF_8, int NT_, int BKV_, bool ALIAS_, bool SUMV_, bool NOHINT = false,
          bool SPEC_ = false, bool LDSPLIT = false, bool PSM_ = false, bool PACK_ = false, bool NOMAX_ = false,
          bool QL2_ = false>
__global__ void __launch_bounds__(AttnCfg<D, NT_, BKV_, ALIAS_, SUMV_, PSM_, PACK_>::THREADS, 1)
    fmha_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  // fixup launch after a max-free one: nothing to do unless some unit was flagged; otherwise its work
  // items are the listed units (whole units, no KV split)
  int nwork = a.work;
  bool fix_all = false;
  if (a.fixup) {
    const unsigned nb = *reinterpret_cast<volatile unsigned*>(a.bad);
    if (nb == 0u) return;
    fix_all = nb > unsigned(a.fix_cap);
    nwork = fix_all ? a.units : int(nb);
  }
  auto item = [&](int w) -> WorkItem {
    if (a.fixup) return {fix_all ? w : int(a.fix_list[w]), 0, a.kv_tiles, -1, 0};
    return work_item(a, w);
  };
  using Cfg = AttnCfg<D, NT_, BKV_, ALIAS_, SUMV_, PSM_, PACK_>;
  constexpr bool ALIAS = ALIAS_;
  constexpr bool PACK = PACK_;
  // NOMAX: no running max at all — P = 2^(s * scale * log2e) with m = 0 (no row max, no vote, no
  // rescale; the first tile of a unit is no longer special). Exact whenever no P or O leaves the fp32
  // range, which the epilogue checks per row; units with a flagged row are recomputed by the exact
  // kernel (fixup launch over AttnArgs::fix_list).
  constexpr bool NOMAX = NOMAX_;
  constexpr bool QL2 = QL2_ && NOMAX_;  // (the exact kernel uses scale_log2 = 1 for pre-scaled q)
  static_assert(!NOMAX || (ALIAS_ && !PSM_ && ((SUMV_ && BKV_ == 48) || (!SUMV_ && BKV_ == 64))),
                "NOMAX is implemented for the aliased 4 x 48 ones-panel and 4 x 64 kernels");
  constexpr bool PSM = PSM_;
  // speculative exps (step_spec) need P writes that can be repeated before p_full: aliased or
  // shared-memory P only
  constexpr bool SPEC = SPEC_ && (ALIAS_ || PSM_);
  constexpr bool SUMV = SUMV_;
  constexpr int DO = Cfg::DO;
  constexpr int BKV = Cfg::BKV;
  constexpr int KST = Cfg::KST;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment by offsetting the __shared__ array itself (keeps the shared address space
  // visible to the compiler: LDS/STS instead of generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int NT = Cfg::NT;
  constexpr int QB = Cfg::QBUF;
  uint8_t* sQ = smem;                                 // QB x NT tiles
  [[maybe_unused]] uint8_t* sP = sQ + QB * NT * Cfg::Q_TILE_BYTES;  // PSM: NT P tiles (1024-aligned)
  uint8_t* sK = sP + NT * Cfg::P_TILE_BYTES;          // KST stages (K tile per slot)
  uint8_t* sV = sK + KST * Cfg::K_STAGE_BYTES;        // KST stages (V tile per slot)
  [[maybe_unused]] uint8_t* sOnes = sV + KST * Cfg::VS_STAGE_BYTES;  // SUMV: the ones panel (1024-aligned)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sOnes + Cfg::ONES_BYTES);
  uint64_t* q_full = bar;       // [QB]
  uint64_t* q_empty = bar + QB;  // [QB]
  uint64_t* k_full = bar + 2 * QB;
  uint64_t* k_empty = k_full + KST;
  uint64_t* v_full = k_empty + KST;
  uint64_t* v_empty = v_full + KST;
  uint64_t* s_full = v_empty + KST;  // [NT] MMA -> softmax: S_i(j) computed
  uint64_t* s_free = s_full + NT;    // [NT] softmax -> MMA: S_i(j) loaded, buffer reusable
  uint64_t* p_full = s_free + NT;    // [NT] softmax -> MMA: P_i(j) written (O rescaled)
  uint64_t* p_free = p_full + NT;    // [NT] MMA -> softmax: PV_i(j) done (P reusable, O stable)
  uint64_t* o_empty = p_free + NT;   // [NT] softmax -> MMA: O_i read by the epilogue
  uint64_t* wq_full = o_empty + NT;  // [WQ] producer -> consumers: work item published
  uint64_t* wq_empty = wq_full + WQ; // [WQ] MMA warp + softmax warps -> producer: slot read
  volatile int* wq = reinterpret_cast<volatile int*>(wq_empty + WQ);  // [WQ] work item indices
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wq_empty + WQ) + WQ;
  // NOMAX: [0] last unit this CTA appended to the fix list (plain launches: de-duplication);
  // [1 + (n & 1)] = n + 1 when a row of this CTA's n-th unit is flagged (ring-merge launches)
  [[maybe_unused]] volatile int* unit_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int b = 0; b < QB; ++b) {
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], 1);
    }
    for (int s = 0; s < KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < NT; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&p_free[i], 1);
      mbar_init(&o_empty[i], 4);
    }
    if constexpr (NOMAX_) {
      unit_flag[0] = -1;
      unit_flag[1] = 0;
      unit_flag[2] = 0;
    }
    for (int i = 0; i < WQ; ++i) {
      mbar_init(&wq_full[i], 1);
      mbar_init(&wq_empty[i], 1 + 4 * NT);  // the MMA warp and every softmax warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  if constexpr (SUMV) {  // the constant ones panel every V stage's descriptor points its second atom at
#if VX_FMHA_ONES_ALL
    const uint32_t ones = 0x3f803f80u;  // bf16x2 (1, 1)
    for (uint32_t o = threadIdx.x * 16; o < Cfg::ONES_BYTES; o += Cfg::THREADS * 16)
      *reinterpret_cast<uint4*>(sOnes + o) = make_uint4(ones, ones, ones, ones);
#else
    // one column of ones (MN index 0 -> O column D = the row sum), zeros in the other 7 columns the PV
    // MMA reads (N = D + 8): zero operands cost the tensor core less switching energy under the power
    // cap. SW128 MN-major rows of 128 B, one per key: logical 16-byte chunk 0 of row r sits at
    // physical chunk r % 8 (the panel is 1024-byte aligned).
    for (uint32_t o = threadIdx.x * 16; o < Cfg::ONES_BYTES; o += Cfg::THREADS * 16) {
      const uint32_t row = o >> 7, chunk = (o >> 4) & 7;
      const uint32_t w0 = (chunk ^ (row & 7)) == 0 ? 0x3f80u : 0u;  // bf16 1.0 in the chunk's first element
      *reinterpret_cast<uint4*>(sOnes + o) = make_uint4(w0, 0u, 0u, 0u);
    }
#endif
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // tile t of the (head, sequence, tile) numbering -> sequence g = head * nseq + seq, tile in sequence
  auto tile_seq = [&](int t, int& qt) -> int {
    const int g = t / a.tps;
    qt = t - g * a.tps;
    return g;
  };

  // the n-th work item of this CTA is published by the producer through wq[n % WQ]: the first is
  // blockIdx.x, later ones come from the launch's atomic ticket counter, so a CTA that started late
  // (its SM busy with a concurrent kernel, e.g. the NCCL ring transfer) simply takes fewer units
  auto wq_take = [&](uint32_t n) -> int {  // warp-collective consumer side
    const uint32_t slot = n % WQ;
    mbar_wait(&wq_full[slot], (n / WQ) & 1);
    const int w = wq[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&wq_empty[slot]);
    return w;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t pol_kv = policy_evict_last();
      const uint64_t pol_q = policy_evict_first();
      uint32_t c = 0;  // global K/V tile counter
      for (uint32_t n = 0;; ++n) {  // n: local unit counter
        const int w = n == 0 ? int(blockIdx.x)
                             : (a.sched ? int(gridDim.x + atomicAdd(a.sched, 1u)) : int(blockIdx.x + n * gridDim.x));
        {
          const uint32_t slot = n % WQ;
          mbar_wait(&wq_empty[slot], ((n / WQ) & 1) ^ 1);
          wq[slot] = w;
          mbar_arrive(&wq_full[slot]);
        }
        if (w >= nwork) break;
        const WorkItem wi = item(w);
        const int t0 = wi.u * NT;
        int qt0;
        const int gA = tile_seq(t0, qt0);
        const int last = (t0 + NT <= a.total_tiles ? t0 + NT : a.total_tiles) - 1;
        int qtl;
        const int nslot = PACK && tile_seq(last, qtl) != gA ? 2 : 1;  // K/V of one or two sequences
        int kv_row[2];
        for (int b = 0; b < nslot; ++b) {
          const int hb = (gA + b) / a.nseq;
          kv_row[b] = int(hb * a.Tk + (int64_t)(gA + b - hb * a.nseq) * a.Lk);
        }
        const uint32_t qb = QB == 2 ? (n & 1) : 0, qph = QB == 2 ? ((n >> 1) & 1) : (n & 1);
        mbar_wait(&q_empty[qb], qph ^ 1);
        VX_TRACE(n < 2 ? 6230 + int(n) : -1);
        mbar_expect_tx(&q_full[qb], NT * Cfg::Q_TILE_BYTES);
        for (int i = 0; i < NT; ++i) {
          int qt;
          const int g = tile_seq(t0 + i, qt);
          const int hq = g / a.nseq;
          // tiles past the last one (packed, final unit only) load any rows; their output is dropped
          const int q_row = t0 + i < a.total_tiles ? int(hq * a.Tq + (int64_t)(g - hq * a.nseq) * a.Lq + qt * 128) : 0;
          for (int pn = 0; pn < Cfg::PANELS; ++pn)
            tma_load_2d_hint(sQ + (qb * NT + i) * Cfg::Q_TILE_BYTES + pn * Cfg::QPANEL_BYTES, &tmQ, &q_full[qb],
                             pn * Cfg::PANEL_COLS, q_row, pol_q);
        }
        for (int j = wi.j0; j < wi.j0 + wi.cnt; ++j, ++c) {
          const uint32_t st = c % KST, ph = (c / KST) & 1;
          mbar_wait(&k_empty[st], ph ^ 1);
          VX_TRACE(n < 2 && j - wi.j0 < 2 ? 6240 + 2 * int(n) + (j - wi.j0) : -1);
          mbar_expect_tx(&k_full[st], nslot * Cfg::KV_TILE_BYTES);
          for (int b = 0; b < nslot; ++b)
            for (int pn = 0; pn < Cfg::PANELS; ++pn)
              tma_load_2d_hint(sK + st * Cfg::K_STAGE_BYTES + b * Cfg::KV_TILE_BYTES + pn * Cfg::KVPANEL_BYTES, &tmK,
                               &k_full[st], pn * Cfg::PANEL_COLS, kv_row[b] + BKV * j, pol_kv);
          mbar_wait(&v_empty[st], ph ^ 1);
          mbar_expect_tx(&v_full[st], nslot * Cfg::KV_TILE_BYTES);
          for (int b = 0; b < nslot; ++b)
            for (int pn = 0; pn < Cfg::PANELS; ++pn)
              tma_load_2d_hint(sV + st * Cfg::VS_STAGE_BYTES + b * Cfg::V_STAGE_BYTES + pn * Cfg::KVPANEL_BYTES, &tmV,
                               &v_full[st], pn * Cfg::PANEL_COLS, kv_row[b] + BKV * j, pol_kv);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // the whole warp runs the (warp-uniform) issue loop and waits; one elected lane issues the
    // tcgen05 ops, so descriptors and counters stay in uniform registers
    const bool lead = elect_one();
    {
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, BKV, 0, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16(128, DO, 0, 1);
      const uint32_t q0 = smem_u32(sQ);
      constexpr int KSTEPS_PER_PANEL = Cfg::PANEL_COLS / 16;
      // descriptors: one base per operand, offsets added in 16-byte units (smem addresses < 256 KB
      // keep the 14-bit start-address field from carrying into the next field)
      const uint64_t qdesc0 = make_sdesc(q0, 16, Cfg::SBO, Cfg::LAYOUT);
      uint32_t qsel = 0;  // byte offset of this unit's Q buffer
      auto issue_qk = [&](int i, uint32_t ks, bool issue = true) {
        const uint64_t kd = make_sdesc(ks, 16, Cfg::SBO, Cfg::LAYOUT);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t kstep = (k % KSTEPS_PER_PANEL) * 32;
          const uint32_t qoff = qsel + i * Cfg::Q_TILE_BYTES + (k / KSTEPS_PER_PANEL) * Cfg::QPANEL_BYTES + kstep;
          const uint32_t koff = (k / KSTEPS_PER_PANEL) * Cfg::KVPANEL_BYTES + kstep;
          mma_ss_if(lead && issue, tmem + Cfg::tS(i), qdesc0 + (qoff >> 4), kd + (koff >> 4), idesc_qk, k > 0);
        }
      };
      // V is the MN-major B operand: for D = 128 its two 64-column panels are the two MN atoms (LBO)
      [[maybe_unused]] const uint64_t pdesc0 = make_sdesc(smem_u32(sP), 16, 1024, 2);  // PSM: K-major SW128
      auto issue_pv = [&](int i, uint32_t vs, uint32_t acc) {
        // SUMV: the second MN atom (LBO away) is the shared ones panel
        const uint64_t vd = make_sdesc(vs, SUMV ? smem_u32(sOnes) - vs : Cfg::KVPANEL_BYTES, Cfg::SBO, Cfg::LAYOUT);
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          if constexpr (PSM)  // P_i from shared memory: 16 bf16 = 32 bytes per k-step within the 128-B row
            mma_ss_if(lead, tmem + Cfg::tO(i), pdesc0 + ((i * Cfg::P_TILE_BYTES + kk * 32) >> 4),
                      vd + ((kk * 16 * Cfg::ROW_BYTES) >> 4), idesc_pv, (acc | kk) != 0);
          else
            mma_ts_if(lead, tmem + Cfg::tO(i), tmem + Cfg::tP(i) + kk * 8, vd + ((kk * 16 * Cfg::ROW_BYTES) >> 4),
                      idesc_pv, (acc | kk) != 0);
        }
      };
      uint32_t c = 0;  // global K/V tile counter
      uint32_t n = 0;  // local unit counter
      uint32_t sfree_ph = 0, pfull_ph = 0;
      if constexpr (ALIAS) {
        for (;; ++n) {
          const int w = wq_take(n);
          if (w >= nwork) break;
          const WorkItem wi = item(w);
          const int nkv = wi.cnt;
          // PACK: bit i = Q tile i belongs to the unit's second sequence (K/V slot B of every stage)
          uint32_t bmask = 0;
          if constexpr (PACK) {
            int qt;
            const int gA = tile_seq(wi.u * NT, qt);
            for (int i = 1; i < NT; ++i)
              if (wi.u * NT + i < a.total_tiles && tile_seq(wi.u * NT + i, qt) != gA) bmask |= 1u << i;
          }
          auto koff = [&](int i) -> uint32_t { return PACK && ((bmask >> i) & 1) ? Cfg::KV_TILE_BYTES : 0; };
          auto voff = [&](int i) -> uint32_t { return PACK && ((bmask >> i) & 1) ? Cfg::V_STAGE_BYTES : 0; };
          const uint32_t qb = QB == 2 ? (n & 1) : 0, qph = QB == 2 ? ((n >> 1) & 1) : (n & 1);
          qsel = qb * NT * Cfg::Q_TILE_BYTES;
          mbar_wait(&q_full[qb], qph);
          VX_TRACE(n < 2 ? 6100 + int(n) : -1);
          tc_fence_after();
          {  // S(0): the previous unit's P / S columns were consumed by its last PVs (in order)
            const uint32_t st = c % KST, ph = (c / KST) & 1;
            mbar_wait(&k_full[st], ph);
            tc_fence_after();
            const uint32_t ks = smem_u32(sK + st * Cfg::K_STAGE_BYTES);
            for (int i = 0; i < NT; ++i) {
              issue_qk(i, ks + koff(i));
              mma_commit_if(lead, &s_full[i]);
              VX_TRACE(n < 2 ? 6000 + 4 * int(n) + i : -1);
            }
            mma_commit_if(lead, &k_empty[st]);
            mma_commit_if(lead && nkv == 1, &q_empty[qb]);
          }
          for (int j = 0; j < nkv; ++j, ++c) {
            const uint32_t st = c % KST, ph = (c / KST) & 1;
            const bool has_next = j + 1 < nkv;
            const uint32_t nst = (c + 1) % KST, nph = ((c + 1) / KST) & 1;
            const uint32_t vs = smem_u32(sV + st * Cfg::VS_STAGE_BYTES);
            const uint32_t nks = smem_u32(sK + nst * Cfg::K_STAGE_BYTES);
            mbar_wait(&v_full[st], ph);
            if (has_next) mbar_wait(&k_full[nst], nph);
            for (int i = 0; i < NT; ++i) {
              if (NOHINT) mbar_wait_nohint(&p_full[i], pfull_ph);
              else mbar_wait(&p_full[i], pfull_ph);
              // tile i's previous-unit epilogue has read O_i (per tile, so a unit boundary does not hold
              // every tile back to the slowest tile's epilogue; the softmax warps arrive o_empty before
              // this unit's first p_full, so the wait is already satisfied)
              if (j == 0) mbar_wait(&o_empty[i], (n & 1) ^ 1);
              VX_TRACE(trace_slot_mma(int(n), j, i, 0));
              tc_fence_after();
              issue_pv(i, vs + voff(i), j > 0);
              // S_i(j+1) overwrites P_i(j): executes after PV_i(j) (tcgen05 issue order). Predicated
              // rather than branched, so the issue path has no branch.
              issue_qk(i, nks + koff(i), has_next);
              mma_commit_if(lead && has_next, &s_full[i]);
              mma_commit_if(lead && !has_next, &p_free[i]);  // last PV of the unit
              VX_TRACE(trace_slot_mma(int(n), j, i, 1));
            }
            pfull_ph ^= 1;
            mma_commit_if(lead, &v_empty[st]);
            if (has_next) {
              mma_commit_if(lead, &k_empty[nst]);
              mma_commit_if(lead && j + 2 == nkv, &q_empty[qb]);
            }
          }
        }
      } else {
        for (;; ++n) {
          const int w = wq_take(n);
          if (w >= nwork) break;
          const int nkv = item(w).cnt;
          mbar_wait(q_full, n & 1);
          tc_fence_after();
          {  // S(0) of both tiles; the S buffers were released by the previous unit's last s_free
            const uint32_t st = c % KST, ph = (c / KST) & 1;
            mbar_wait(&k_full[st], ph);
            tc_fence_after();
            const uint32_t ks = smem_u32(sK + st * Cfg::K_STAGE_BYTES);
            for (int i = 0; i < NT; ++i) {
              if (n > 0) mbar_wait(&s_free[i], sfree_ph);
              tc_fence_after();
              issue_qk(i, ks);
              mma_commit_if(lead, &s_full[i]);
            }
            if (n > 0) sfree_ph ^= 1;
            mma_commit_if(lead, &k_empty[st]);
            mma_commit_if(lead && nkv == 1, q_empty);
          }
          for (int j = 0; j < nkv; ++j, ++c) {
            const uint32_t st = c % KST, ph = (c / KST) & 1;
            if (j + 1 < nkv) {  // run one KV tile ahead: S(j+1) as soon as S(j) has been loaded
              const uint32_t nst = (c + 1) % KST, nph = ((c + 1) / KST) & 1;
              mbar_wait(&k_full[nst], nph);
              const uint32_t nks = smem_u32(sK + nst * Cfg::K_STAGE_BYTES);
              for (int i = 0; i < NT; ++i) {
                mbar_wait(&s_free[i], sfree_ph);
                tc_fence_after();
                issue_qk(i, nks);
                mma_commit_if(lead, &s_full[i]);
              }
              sfree_ph ^= 1;
              mma_commit_if(lead, &k_empty[nst]);
              mma_commit_if(lead && j + 2 == nkv, q_empty);
            }
            const uint32_t vs = smem_u32(sV + st * Cfg::VS_STAGE_BYTES);
            mbar_wait(&v_full[st], ph);
            for (int i = 0; i < NT; ++i) {
              mbar_wait(&p_full[i], pfull_ph);
              if (j == 0) mbar_wait(&o_empty[i], (n & 1) ^ 1);  // the previous unit's epilogue has read O_i
              tc_fence_after();
              issue_pv(i, vs, j > 0);
              mma_commit_if(lead, &p_free[i]);
            }
            pfull_ph ^= 1;
            mma_commit_if(lead, &v_empty[st]);
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 4 + 4 * NT) {
    // ------------------------------------------------------------ softmax / epilogue, one WG per tile
    const int tile = (warp - 4) >> 2;
    const int wl = warp & 3;
    const int r = wl * 32 + lane;
    const uint32_t lane_off = uint32_t(wl * 32) << 16;
    const uint32_t S_addr = tmem + lane_off + Cfg::tS(tile);
    const uint32_t P_addr = tmem + lane_off + Cfg::tP(tile);
    const uint32_t O_addr = tmem + lane_off + Cfg::tO(tile);
    const float sl2 = a.scale_log2;
    const uint64_t SL2 = f2_pack(sl2, sl2);
    uint32_t sph = 0, pv_cnt = 0;
    [[maybe_unused]] int unit_n = 0;
    for (;; ++unit_n) {
      const int w = wq_take(uint32_t(unit_n));
      if (w >= nwork) break;
      const WorkItem wi = item(w);
      const int nkv = wi.cnt;
      const int t = wi.u * NT + tile;
      int qt;
      const int g = tile_seq(t, qt);
      const int h = g / a.nseq;
      const int s = g - h * a.nseq;
      const int q_local = qt * 128 + r;
      const bool row_valid = t < a.total_tiles && q_local < a.Lq;
      float m_run = NOMAX ? 0.f : -INFINITY;
      float l_run = 0.f;
      for (int j = 0; j < nkv; ++j) {
        VX_TRACE(trace_slot_sm(unit_n, wl, lane, tile, j, 0));
        if (NOHINT) mbar_wait_nohint(&s_full[tile], sph);
        else mbar_wait(&s_full[tile], sph);
        VX_TRACE(trace_slot_sm(unit_n, wl, lane, tile, j, 1));
        sph ^= 1;
        tc_fence_after();
        if constexpr (NOMAX && BKV == 64) {
          // 64-wide KV tiles (4 tiles: 4 x (64 S/P + 64 O) = 512 TMEM columns, row sums by FADD2): two
          // 32-column halves, P of half h to words [16h, 16h + 16) — over S columns the first half
          // has already loaded
          const int valid = a.Lk - BKV * (wi.j0 + j);
          uint64_t rs[2] = {0, 0};
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            uint32_t sr[32];
            uint32_t pk[16];
            tmem_ld32(S_addr + 32 * hf, sr);
            tmem_wait_ld();
            if (valid < BKV) {
#pragma unroll
              for (int c = 0; c < 32; ++c)
                if (32 * hf + c >= valid) sr[c] = 0xff800000u;
            }
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const uint64_t x = QL2 ? f2_pack(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1]))
                                     : f2_mul(f2_pack(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), SL2);
              float x0, x1, p0, p1;
              f2_unpack(x, x0, x1);
              if ((c & 7) >= 8 - EMU_PAIRS_OF_8) {
                ex2_poly2<2, true>(x0, x1, p0, p1);
              } else {
                p0 = ex2(x0);
                p1 = ex2(x1);
              }
              rs[c & 1] = f2_add(rs[c & 1], f2_pack(p0, p1));
              pk[c] = pack_bf16(p0, p1);
            }
            tmem_st16(P_addr + 16 * hf, pk);
          }
          float r0, r1;
          f2_unpack(f2_add(rs[0], rs[1]), r0, r1);
          l_run += r0 + r1;
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[tile]);
          continue;
        }
        if constexpr (BKV == 96) {
          // 96-wide KV tiles (3 Q tiles fit TMEM: 3 x (96 S/P + 72 O) = 504 columns), processed as two
          // 48-column halves A = S[0, 48), B = S[48, 96) so the registers stay those of one half. P (96
          // bf16 = 48 columns) goes over S[0, 48): P_A to columns 0-23 (once A is loaded), P_B to 24-47
          // (once A is consumed).
          const int valid = a.Lk - BKV * (wi.j0 + j);
          uint32_t sr[48];
          uint32_t pk[24];
          auto ld48 = [&](int half) {
            tmem_ld32(S_addr + 48 * half, sr);
            tmem_ld16(S_addr + 48 * half + 32, sr + 32);
            tmem_wait_ld();
          };
          auto mask48 = [&](int half) {
#pragma unroll
            for (int c = 0; c < 48; ++c)
              if (48 * half + c >= valid) sr[c] = 0xff800000u;
          };
          auto max48 = [&]() -> float {
            float mq[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) mq[q] = fmaxf(__uint_as_float(sr[q]), __uint_as_float(sr[q + 3]));
#pragma unroll
            for (int c = 6; c < 48; c += 6)
#pragma unroll
              for (int q = 0; q < 3; ++q) mq[q] = max3(mq[q], __uint_as_float(sr[c + q]), __uint_as_float(sr[c + 3 + q]));
            return fmaxf(fmaxf(mq[0], mq[1]), mq[2]) * sl2;
          };
          // 24 exp pairs of the half in sr -> pk; optionally stored as P words [pword, pword + 24)
          auto exps48 = [&](const float m, uint32_t pword, bool store) {
            const uint64_t NEGM = f2_pack(-m, -m);
#pragma unroll
            for (int c = 0; c < 24; ++c) {
              const uint64_t x = f2_fma(f2_pack(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), SL2, NEGM);
              float x0, x1, p0, p1;
              f2_unpack(x, x0, x1);
              if ((c & 7) >= 8 - EMU_PAIRS_OF_8) {
                ex2_poly2<2>(x0, x1, p0, p1);
              } else {
                p0 = ex2(x0);
                p1 = ex2(x1);
              }
              pk[c] = pack_bf16(p0, p1);
              if (store && c == 15) tmem_st16(P_addr + pword, pk);
            }
            if (store) tmem_st8(P_addr + pword + 16, pk + 16);
          };
          auto store_pk = [&](uint32_t pword) {
            tmem_st16(P_addr + pword, pk);
            tmem_st8(P_addr + pword + 16, pk + 16);
          };
          auto rescale_o96 = [&](const float alpha) {  // O_i (with the row-sum column) *= alpha
            uint32_t orr[32];
#pragma unroll
            for (int c0 = 0; c0 < DO; c0 += 32) {
              const int wd = DO - c0 >= 32 ? 32 : DO - c0;
              if (wd == 32) tmem_ld32(O_addr + c0, orr);
              else tmem_ld16(O_addr + c0, orr);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) orr[c] = __float_as_uint(__uint_as_float(orr[c]) * alpha);
              if (wd == 32) tmem_st32(O_addr + c0, orr);
              else if (wd == 16) tmem_st16(O_addr + c0, orr);
              else tmem_st8(O_addr + c0, orr);
            }
          };
          constexpr float GUARD = 120.0f;  // log2 units: P_A stays finite, so it can be rescaled in place
          bool done = false;
          if (SPEC && j > 0 && valid >= BKV) {
            // speculative: exps with the running max, tile max alongside
            ld48(0);
            exps48(m_run, 0, false);
            const float mxa = max48();
            if (!__any_sync(0xffffffff, mxa > m_run + GUARD)) {
              store_pk(0);
              ld48(1);
              exps48(m_run, 24, true);
              const float m_new = fmaxf(mxa, max48());
              const bool need = m_new > m_run + RESCALE_THRESHOLD;
              if (__any_sync(0xffffffff, need)) {  // rare: redo B, rescale P_A in place and O
                const float alpha = need ? ex2(m_run - m_new) : 1.0f;
                if (need) m_run = m_new;
                exps48(m_run, 24, true);
                uint32_t w[32];
                tmem_ld32(P_addr, w);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 24; ++c) {
                  const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[c]));
                  w[c] = pack_bf16(f.x * alpha, f.y * alpha);
                }
                tmem_st16(P_addr, w);
                tmem_st8(P_addr + 16, w + 16);
                rescale_o96(alpha);
              }
              done = true;
            }
          }
          if (!done) {  // exact: both halves' max first (first tile, masked tile, guard fallback)
            ld48(0);
            if (valid < BKV) mask48(0);
            const float mxa = max48();
            ld48(1);
            if (valid < BKV) mask48(1);
            const float m_new = fmaxf(mxa, max48());
            const bool need = m_new > m_run + RESCALE_THRESHOLD;
            const float alpha = need ? ex2(m_run - m_new) : 1.0f;
            if (need) m_run = m_new;
            exps48(m_run, 24, false);  // P_B, held until A has been reloaded (its S columns 24-47 are P_B's)
            ld48(0);
            if (valid < BKV) mask48(0);
            store_pk(24);
            exps48(m_run, 0, true);
            if (__any_sync(0xffffffff, need) && j > 0) rescale_o96(alpha);
          }
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[tile]);
          continue;
        }
        uint32_t sr[BKV];
        const int valid = a.Lk - BKV * (wi.j0 + j);
        // speculative tiles (48 wide) leave the last 16 S columns in flight: the first 16 exp pairs
        // only need columns 0-31, and the wait for the rest sits just before pair 16
        // (not with PSM: s_free is arrived right after the S load so S(j+1) can be issued into it)
        constexpr bool SPLIT_LD = SPEC && LDSPLIT && BKV == 48 && !PSM;
        const bool spec_now = (SPEC && j > 0 && valid >= BKV) || (NOMAX && valid >= BKV);
        if (SPLIT_LD && spec_now) {
          tmem_ld32(S_addr, sr);
          tmem_wait_ld();
          tmem_ld16(S_addr + 32, sr + 32);
        } else {
          tmem_ld_n<BKV>(S_addr, sr);
          tmem_wait_ld();
        }
        if constexpr (!ALIAS) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_free[tile]);
        }
        // row max of the tile (FMNMX3 chains), in log2 units
        auto tile_max = [&]() -> float {
          constexpr int CH = BKV / 16;  // independent FMNMX3 chains
          float mq[CH];
#pragma unroll
          for (int q = 0; q < CH; ++q) mq[q] = fmaxf(__uint_as_float(sr[q]), __uint_as_float(sr[q + CH]));
#pragma unroll
          for (int c = 2 * CH; c < BKV; c += 2 * CH)
#pragma unroll
            for (int q = 0; q < CH; ++q) mq[q] = max3(mq[q], __uint_as_float(sr[c + q]), __uint_as_float(sr[c + CH + q]));
          float mx = mq[0];
#pragma unroll
          for (int q = 1; q < CH; ++q) mx = fmaxf(mx, mq[q]);
          return mx * sl2;
        };
        // P = 2^(s * scale * log2e - m) for the whole tile, packed to bf16 and stored over S
        uint64_t acc[4];
        // PSM: this thread's row of its tile's P buffer (128-byte rows, 16-byte chunks XOR-swizzled by row
        // % 8 = the SW128 K-major layout the PV MMA reads); P_i(j-1) must have been consumed first
        [[maybe_unused]] uint8_t* prow = sP + tile * Cfg::P_TILE_BYTES + r * 128;
        [[maybe_unused]] bool pfree_waited = false;
        auto wait_pfree = [&]() {
          if (j > 0 && !pfree_waited) {  // PV_i(j-1) done: P buffer reusable, O stable
            mbar_wait(&p_free[tile], pv_cnt & 1);
            ++pv_cnt;
            tc_fence_after();
          }
          pfree_waited = true;
        };
        auto store_p_chunks = [&](const uint32_t* pk, int q0, int q1) {
#pragma unroll
          for (int q = q0; q < q1; ++q)
            *reinterpret_cast<uint4*>(prow + ((q ^ (r & 7)) * 16)) =
                make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        };
        auto exps = [&](const uint64_t NEGM, auto mid_wait) {
          acc[0] = acc[1] = acc[2] = acc[3] = 0;
          constexpr int NCHUNK = (BKV + 63) / 64;
#pragma unroll
          for (int hf = 0; hf < NCHUNK; ++hf) {
            constexpr int PAIRS = BKV >= 64 ? 32 : BKV / 2;  // column pairs in this chunk
            uint32_t pk[PAIRS];
#pragma unroll
            for (int c = 0; c < PAIRS; ++c) {
              if constexpr (decltype(mid_wait)::value && PAIRS == 24) {
                if (c == 16) tmem_wait_ld_dep16(sr + 32);
              }
              const int e = 64 * hf + 2 * c;
              // QL2 (max-free, q pre-scaled by log2(e)/sqrt(d)): the score already is the exponent
              const uint64_t x = QL2 ? f2_pack(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1]))
                                     : f2_fma(f2_pack(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])), SL2, NEGM);
              float x0, x1, p0, p1;
              f2_unpack(x, x0, x1);
              if ((c & 7) >= 8 - EMU_PAIRS_OF_8) {
                ex2_poly2<2, NOMAX>(x0, x1, p0, p1);
              } else {
                p0 = ex2(x0);
                p1 = ex2(x1);
              }
              if constexpr (!SUMV) acc[c & 3] = f2_add(acc[c & 3], f2_pack(p0, p1));
              pk[c] = pack_bf16(p0, p1);
              // 48-wide tiles: store the first 16 P columns while the last 8 pairs are computed
              if constexpr (PAIRS == 24) {
                if (c == 15) {
                  if constexpr (PSM) {
                    wait_pfree();
                    store_p_chunks(pk, 0, 4);
                  } else {
                    tmem_st16(P_addr + 32 * hf, pk);
                  }
                }
              }
            }
            VX_TRACE(trace_slot_sm(unit_n, wl, lane, tile, j, 3));
            if constexpr (PSM) {
              if constexpr (PAIRS == 24) {
                store_p_chunks(pk, 4, 6);
              } else {
                wait_pfree();
                store_p_chunks(pk, 0, PAIRS / 4);
              }
            } else {
              if (!ALIAS && hf == 0 && j > 0) {  // P_i(j-1) consumed and O stable (waited after the first exps)
                mbar_wait(&p_free[tile], pv_cnt & 1);
                ++pv_cnt;
                tc_fence_after();
              }
              if constexpr (PAIRS == 24) tmem_st8(P_addr + 32 * hf + 16, pk + 16);
              else tmem_st_n<PAIRS>(P_addr + 32 * hf, pk);
            }
          }
        };
        auto rescale_o = [&](const float alpha) {
          uint32_t orr[32];
#pragma unroll
          for (int c0 = 0; c0 < DO; c0 += 32) {
            const int w = DO - c0 >= 32 ? 32 : DO - c0;  // 32, 16 or 8 (never past this tile's O)
            if (w == 32) tmem_ld32(O_addr + c0, orr);
            else tmem_ld16(O_addr + c0, orr);  // an 8-wide tail reads 8 extra columns, unused
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) orr[c] = __float_as_uint(__uint_as_float(orr[c]) * alpha);
            if (w == 32) tmem_st32(O_addr + c0, orr);
            else if (w == 16) tmem_st16(O_addr + c0, orr);
            else tmem_st8(O_addr + c0, orr);
          }
        };
        auto row_sums = [&](const float alpha) {
          if constexpr (!SUMV) {
            float a0, a1, b0, b1;
            f2_unpack(f2_add(acc[0], acc[1]), a0, a1);
            f2_unpack(f2_add(acc[2], acc[3]), b0, b1);
            l_run = l_run * alpha + ((a0 + a1) + (b0 + b1));
          }
        };
        // exact: max first, then exps with the (possibly raised) running max
        auto step = [&](auto mask_tag) {
          if constexpr (decltype(mask_tag)::value) {
#pragma unroll
            for (int c = 0; c < BKV; ++c)
              if (c >= valid) sr[c] = 0xff800000u;
          }
          const float m_new = tile_max();
          const bool need = m_new > m_run + RESCALE_THRESHOLD;
          const float alpha = need ? ex2(m_run - m_new) : 1.0f;
          if (need) m_run = m_new;
          VX_TRACE(trace_slot_sm(unit_n, wl, lane, tile, j, 2));
          exps(f2_pack(-m_run, -m_run), BoolTag<false>{});
          row_sums(alpha);
          if (__any_sync(0xffffffff, need) && j > 0) rescale_o(alpha);
        };
        // speculative (unmasked tiles after the first): the running max almost never moves by more
        // than the threshold, so the exps start with it right away and the tile max is computed
        // alongside (off the critical path); a warp with a row that does need the new max redoes
        // the tile (rare)
        auto step_spec = [&]() {
          exps(f2_pack(-m_run, -m_run), BoolTag<SPLIT_LD>{});
          const float m_new = tile_max();
          const bool need = m_new > m_run + RESCALE_THRESHOLD;
          if (__any_sync(0xffffffff, need)) {
            const float alpha = need ? ex2(m_run - m_new) : 1.0f;
            if (need) m_run = m_new;
            exps(f2_pack(-m_run, -m_run), BoolTag<false>{});
            row_sums(alpha);
            rescale_o(alpha);
          } else {
            row_sums(1.0f);
          }
        };
        if constexpr (NOMAX) {
          if (valid < BKV) {
#pragma unroll
            for (int c = 0; c < BKV; ++c)
              if (c >= valid) sr[c] = 0xff800000u;
            exps(f2_pack(0.f, 0.f), BoolTag<false>{});
          } else {
            exps(f2_pack(0.f, 0.f), BoolTag<SPLIT_LD>{});
          }
        } else if (valid < BKV) {
          step(BoolTag<true>{});
        } else if (spec_now) {
          step_spec();
        } else {
          step(BoolTag<false>{});
        }
        tmem_wait_st();
        if constexpr (PSM) fence_proxy_async_smem();  // P stores visible to the tensor core's async proxy
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[tile]);
        VX_TRACE(trace_slot_sm(unit_n, wl, lane, tile, j, 4));
      }
      mbar_wait(&p_free[tile], pv_cnt & 1);
      ++pv_cnt;
      VX_TRACE(trace_slot_sm(unit_n, wl, lane, tile, nkv - 1, 5));
      tc_fence_after();
      constexpr int DL = (DO + 15) / 16 * 16;  // load width (a 72-column O reads 8 unused columns)
      uint32_t orr[DL];
      tmem_ld_n<DL>(O_addr, orr);
      tmem_wait_ld();
      if constexpr (SUMV) l_run = __uint_as_float(orr[D]);  // sum_k P_ik from the ones panel
      [[maybe_unused]] bool skip_unit = false;
      if constexpr (NOMAX) {
        // trustworthy iff 1e-30 < l < 1e30 and the O row is finite. The upper bound matters: every P is at
        // most l, so l < 1e30 (~2^100) proves every exponent was below 100, and the FMA-pipe exp2 (exponent
        // inserted into the float bits) is only valid below 2^128 — above that it wraps instead of giving
        // inf (measured: an upper bound of 3e38 lets large-logit rows through with 2e-2 errors). The
        // lower bound keeps the row's largest P far from the 2^-126 flush.
        uint64_t c4[4] = {0, 0, 0, 0};  // packed partial sums (NaN / inf propagate), a short dependency chain
#pragma unroll
        for (int c = 0; c < D / 2; ++c)
          c4[c & 3] = f2_add(c4[c & 3], f2_pack(__uint_as_float(orr[2 * c]), __uint_as_float(orr[2 * c + 1])));
        float c0, c1;
        f2_unpack(f2_add(f2_add(c4[0], c4[1]), f2_add(c4[2], c4[3])), c0, c1);
        const float chk = c0 + c1;
        const bool bad = row_valid && !(l_run > 1e-30f && l_run < 1e30f && fabsf(chk) < 3.0e38f);
        const bool wbad = __any_sync(0xffffffff, bad);
        auto append = [&]() {
          const unsigned idx = atomicAdd(a.bad, 1u);
          if (idx < unsigned(a.fix_cap)) a.fix_list[idx] = unsigned(wi.u);
        };
        if (a.merge == 0) {  // written anyway; the fixup overwrites the unit
          if (wbad && lane == 0 && atomicExch(const_cast<int*>(unit_flag), wi.u) != wi.u) append();
        } else {  // the whole unit is written only if none of its rows is flagged
          if (wbad && lane == 0) unit_flag[1 + (unit_n & 1)] = unit_n + 1;
          named_bar_sync(1, 128 * NT);
          skip_unit = unit_flag[1 + (unit_n & 1)] == unit_n + 1;
          if (skip_unit && tile == 0 && wl == 0 && lane == 0) append();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[tile]);
      VX_TRACE(trace_slot_sm(unit_n, wl, lane, tile, nkv - 1, 7));
      if (row_valid && !skip_unit) {
        const float inv = 1.0f / l_run;
        const int64_t orow = (int64_t)s * a.Lq + q_local;
        const float lse_new = (m_run + __log2f(l_run)) * 0.69314718055994531f;
        if (wi.part >= 0) {  // KV-split tail item: normalised fp32 partial + lse, merged by fmha_split_merge
          const int64_t item = (int64_t)wi.t * a.parts + wi.part;
          const int lr = tile * 128 + r;
          float4* dst = reinterpret_cast<float4*>(a.part_o + (item * Cfg::ROWS + lr) * D);
#pragma unroll
          for (int c = 0; c < D / 4; ++c)
            dst[c] = make_float4(__uint_as_float(orr[4 * c]) * inv, __uint_as_float(orr[4 * c + 1]) * inv,
                                 __uint_as_float(orr[4 * c + 2]) * inv, __uint_as_float(orr[4 * c + 3]) * inv);
          a.part_lse[item * Cfg::ROWS + lr] = lse_new;
        } else if (a.merge == 0) {
          VX_TRACE(trace_slot_sm(unit_n, wl, lane, tile, nkv - 1, 2));
          __nv_bfloat16* orow_p = a.out + orow * a.ldo + h * D;
#define VX_O(i) (__uint_as_float(orr[i]) * inv)
          if (a.out32) {  // 32-byte stores: each lane writes whole sectors, half the store transactions
#pragma unroll
            for (int c = 0; c < D / 16; ++c) {
              const int b = 16 * c;
              st_global_v8(orow_p + b, pack_bf16(VX_O(b), VX_O(b + 1)), pack_bf16(VX_O(b + 2), VX_O(b + 3)),
                           pack_bf16(VX_O(b + 4), VX_O(b + 5)), pack_bf16(VX_O(b + 6), VX_O(b + 7)),
                           pack_bf16(VX_O(b + 8), VX_O(b + 9)), pack_bf16(VX_O(b + 10), VX_O(b + 11)),
                           pack_bf16(VX_O(b + 12), VX_O(b + 13)), pack_bf16(VX_O(b + 14), VX_O(b + 15)));
            }
          } else {
            uint4* dst = reinterpret_cast<uint4*>(orow_p);
#pragma unroll
            for (int c = 0; c < D / 8; ++c) {
              const int b = 8 * c;
              dst[c] = make_uint4(pack_bf16(VX_O(b), VX_O(b + 1)), pack_bf16(VX_O(b + 2), VX_O(b + 3)),
                                  pack_bf16(VX_O(b + 4), VX_O(b + 5)), pack_bf16(VX_O(b + 6), VX_O(b + 7)));
            }
          }
#undef VX_O
          if (a.lse) a.lse[h * a.Tq + orow] = lse_new;
        } else {
          // ring step: log-sum-exp merge with the running (O, lse) of the blocks seen so far
          float* acc = a.o_acc + orow * a.ld_acc + h * D;
          float* lacc = a.lse + h * a.Tq + orow;
          float wa = 0.f, wb = inv, lse_out = lse_new;
          if (a.merge >= 2) {
            const float lp = *lacc;
            const float mx = fmaxf(lp, lse_new);
            const float ea = __expf(lp - mx), eb = __expf(lse_new - mx);
            const float rs = 1.0f / (ea + eb);
            wa = ea * rs;
            wb = eb * rs * inv;
            lse_out = mx + __logf(ea + eb);
          }
          if (a.merge == 3) {
            uint4* dst = reinterpret_cast<uint4*>(a.out + orow * a.ldo + h * D);
            const float4* a4 = reinterpret_cast<const float4*>(acc);
#pragma unroll
            for (int c = 0; c < D / 8; ++c) {
              const float4 p0 = a4[2 * c], p1 = a4[2 * c + 1];
#define VX_M(i, pv) (wa * (pv) + wb * __uint_as_float(orr[8 * c + i]))
              dst[c] = make_uint4(pack_bf16(VX_M(0, p0.x), VX_M(1, p0.y)), pack_bf16(VX_M(2, p0.z), VX_M(3, p0.w)),
                                  pack_bf16(VX_M(4, p1.x), VX_M(5, p1.y)), pack_bf16(VX_M(6, p1.z), VX_M(7, p1.w)));
#undef VX_M
            }
          } else {
            float4* a4 = reinterpret_cast<float4*>(acc);
#pragma unroll
            for (int c = 0; c < D / 4; ++c) {
              const float4 p = a.merge >= 2 ? a4[c] : make_float4(0.f, 0.f, 0.f, 0.f);
              a4[c] = make_float4(wa * p.x + wb * __uint_as_float(orr[4 * c + 0]),
                                  wa * p.y + wb * __uint_as_float(orr[4 * c + 1]),
                                  wa * p.z + wb * __uint_as_float(orr[4 * c + 2]),
                                  wa * p.w + wb * __uint_as_float(orr[4 * c + 3]));
            }
          }
          *lacc = lse_out;
        }
      }
      VX_TRACE(trace_slot_sm(unit_n, wl, lane, tile, nkv - 1, 6));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (a.fixup && threadIdx.x == 0) {  // a fixup that ran: the last CTA clears the list for the next launch
    __threadfence();
    if (atomicAdd(a.bad + 1, 1u) == gridDim.x - 1) {
      atomicExch(a.bad, 0u);
      atomicExch(a.bad + 1, 0u);
    }
  }
  if (a.sched && threadIdx.x == 0) {  // every ticket of this CTA is taken: the last CTA resets the counters
    __threadfence();
    if (atomicAdd(a.sched + 1, 1u) == gridDim.x - 1) {
      atomicExch(a.sched, 0u);
      atomicExch(a.sched + 1, 0u);
    }
  }
}

// Combines the KV-split tail items: one thread per (tail row, 4 output columns); the threads of a
// row are consecutive lanes of one warp (G4 divides 32). merge 0 writes out (+ lse); ring modes
// 1-3 fold the combined block into (o_acc, lse_acc) exactly like the FMHA epilogue does.
template <int D, int ROWS>
__global__ void __launch_bounds__(256) fmha_split_merge(const AttnArgs a) {
  constexpr int G4 = D / 4;
  static_assert(32 % G4 == 0, "row threads within one warp");
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)(a.units - a.split_from) * ROWS * G4;
  const int g = int(idx % G4);
  const int64_t rr = idx / G4;
  const int lr = int(rr % ROWS);
  const int t = int(rr / ROWS);
  const int u = a.split_from + t;
  const int per_head = a.nseq * a.q_blocks;
  const int h = u / per_head;
  const int rem = u - h * per_head;
  const int s = rem / a.q_blocks;
  const int qb = rem - s * a.q_blocks;
  const int q_local = qb * ROWS + lr;
  // no early return: every lane reaches the __syncwarp below
  const bool live = idx < total && q_local < a.Lq;
  const int64_t orow = (int64_t)s * a.Lq + q_local;
  float4 ob = make_float4(0.f, 0.f, 0.f, 0.f);
  float lse_b = 0.f, lp = -INFINITY;
  if (live) {
    const int64_t item0 = (int64_t)t * a.parts;
    float mx = -INFINITY;
    for (int p = 0; p < a.parts; ++p) mx = fmaxf(mx, a.part_lse[(item0 + p) * ROWS + lr]);
    float wsum = 0.f;
    for (int p = 0; p < a.parts; ++p) {
      const float wgt = __expf(a.part_lse[(item0 + p) * ROWS + lr] - mx);
      const float4 o = reinterpret_cast<const float4*>(a.part_o + ((item0 + p) * ROWS + lr) * D)[g];
      wsum += wgt;
      ob.x += wgt * o.x;
      ob.y += wgt * o.y;
      ob.z += wgt * o.z;
      ob.w += wgt * o.w;
    }
    const float inv = 1.0f / wsum;
    ob = make_float4(ob.x * inv, ob.y * inv, ob.z * inv, ob.w * inv);
    lse_b = mx + __logf(wsum);
    if (a.merge >= 2) lp = a.lse[h * a.Tq + orow];
  }
  __syncwarp();  // every lane of the row has read lse_acc before lane g == 0 overwrites it
  if (!live) return;
  if (a.merge == 0) {
    *reinterpret_cast<uint2*>(a.out + orow * a.ldo + h * D + 4 * g) =
        make_uint2(pack_bf16(ob.x, ob.y), pack_bf16(ob.z, ob.w));
    if (g == 0 && a.lse) a.lse[h * a.Tq + orow] = lse_b;
    return;
  }
  float wa = 0.f, wb = 1.f, lse_out = lse_b;
  if (a.merge >= 2) {
    const float mx = fmaxf(lp, lse_b);
    const float ea = __expf(lp - mx), eb = __expf(lse_b - mx);
    const float rs = 1.0f / (ea + eb);
    wa = ea * rs;
    wb = eb * rs;
    lse_out = mx + __logf(ea + eb);
  }
  float4* acc = reinterpret_cast<float4*>(a.o_acc + orow * a.ld_acc + h * D) + g;
  const float4 pa = a.merge >= 2 ? *acc : make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 m = make_float4(wa * pa.x + wb * ob.x, wa * pa.y + wb * ob.y, wa * pa.z + wb * ob.z,
                               wa * pa.w + wb * ob.w);
  if (a.merge == 3)
    *reinterpret_cast<uint2*>(a.out + orow * a.ldo + h * D + 4 * g) =
        make_uint2(pack_bf16(m.x, m.y), pack_bf16(m.z, m.w));
  else
    *acc = m;
  if (g == 0) a.lse[h * a.Tq + orow] = lse_out;
}

// The per-stream device buffers below are keyed by (current device, stream): the legacy default
// stream has the same handle on every device, and a buffer belongs to the device it was allocated on.
using StreamKey = std::pair<int, cudaStream_t>;
static StreamKey stream_key(cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  return {dev, st};
}

// Per-stream scratch for the KV-split tail (at most one wave of items: num_sms x ROWS x (D + 1)
// fp32). Allocated once per stream and kept; not allocated while the stream is being captured.
static float* split_scratch(cudaStream_t st, size_t floats) {
  static std::mutex mu;
  static std::map<StreamKey, std::pair<float*, size_t>> bufs;
  std::lock_guard<std::mutex> lock(mu);
  const StreamKey key = stream_key(st);
  auto it = bufs.find(key);
  if (it != bufs.end() && it->second.second >= floats) return it->second.first;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  float* p = nullptr;
  if (cudaMalloc(&p, floats * sizeof(float)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (it != bufs.end()) {  // grow: the old buffer may still be read by queued work on this stream
    cudaStreamSynchronize(st);
    cudaFree(it->second.first);
  }
  bufs[key] = {p, floats};
  return p;
}

// Per-stream unit list of the max-free launches' fixup (AttnArgs::fix_list), grown to the largest
// unit count seen; not allocated while the stream is being captured (the launch then runs the exact
// kernel only).
static unsigned* fix_buffer(cudaStream_t st, int64_t cap) {
  static std::mutex mu;
  static std::map<StreamKey, std::pair<unsigned*, int64_t>> bufs;
  std::lock_guard<std::mutex> lock(mu);
  const StreamKey key = stream_key(st);
  auto it = bufs.find(key);
  if (it != bufs.end() && it->second.second >= cap) return it->second.first;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  unsigned* p = nullptr;
  if (cudaMalloc(&p, cap * sizeof(unsigned)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (it != bufs.end()) {  // grow: queued work on this stream may still read the old list
    cudaStreamSynchronize(st);
    cudaFree(it->second.first);
  }
  bufs[key] = {p, cap};
  return p;
}

// Per-stream work-ticket counters of the FMHA and the max-free launches' fix-list count (4 x u32,
// zero between launches: each launch's last CTA resets them). Allocated and zeroed once per stream;
// not while the stream is being captured (the launch then falls back to static round-robin
// scheduling and the exact kernel).
static unsigned* sched_counters(cudaStream_t st) {
#ifdef VX_DIAG
  {  // diagnostic build only: VX_FMHA_STATIC=1 = static round-robin (read per launch for in-process A/B)
    const char* e = getenv("VX_FMHA_STATIC");
    if (e && atoi(e) == 1) return nullptr;
  }
#endif
  static std::mutex mu;
  static std::map<StreamKey, unsigned*> ctrs;
  std::lock_guard<std::mutex> lock(mu);
  const StreamKey key = stream_key(st);
  auto it = ctrs.find(key);
  if (it != ctrs.end()) return it->second;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  unsigned* p = nullptr;  // [ticket, CTAs done, bad flag, fixup CTAs done]
  if (cudaMalloc(&p, 4 * sizeof(unsigned)) != cudaSuccess || cudaMemset(p, 0, 4 * sizeof(unsigned)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  ctrs[key] = p;
  return p;
}

template <int D, int EMU, int NT = (D == 128 ? 1 : 2), int BKV = 128, bool ALIAS = false, bool SUMV = false,
          bool NOHINT = false, bool SPEC = false, bool LDSPLIT = false, bool PSM = false, bool PACK = false,
          bool NOMAX = false, bool QL2 = false>
static int launch_fmha(const void* q, const void* k, const void* v, AttnArgs args, cudaStream_t st) {
  using Cfg = AttnCfg<D, NT, BKV, ALIAS, SUMV, PSM, PACK>;
  CUtensorMap tq, tk, tv;
  constexpr int PC = Cfg::PANEL_COLS;
  if (!make_tmap_2d_bf16(&tq, q, (uint64_t)args.H * args.Tq, D, D, 128, PC, Cfg::SWIZZLE)) return VX_E_ARG;
  if (!make_tmap_2d_bf16(&tk, k, (uint64_t)args.H * args.Tk, D, D, BKV, PC, Cfg::SWIZZLE)) return VX_E_ARG;
  if (!make_tmap_2d_bf16(&tv, v, (uint64_t)args.H * args.Tk, D, D, BKV, PC, Cfg::SWIZZLE)) return VX_E_ARG;
  args.q_blocks = (args.Lq + Cfg::ROWS - 1) / Cfg::ROWS;
  args.kv_tiles = (args.Lk + BKV - 1) / BKV;
  args.tps = PACK ? (args.Lq + 127) / 128 : args.q_blocks * NT;
  if (PACK && (args.tps < NT || args.merge != 0)) return VX_E_ARG;  // a unit spans at most two sequences
  args.total_tiles = args.H * args.nseq * args.tps;
  args.units = (args.total_tiles + NT - 1) / NT;
  // KV-split tail: when the last wave of units would leave more than half the SMs idle, split each
  // of its units over `parts` CTAs (contiguous KV ranges) and merge the partials afterwards
  const int sms = num_sms();
  const int tail = args.units % sms;
  args.split_from = args.units;
  args.parts = 1;
#ifdef VX_DIAG
  static const bool split_on = [] {
    const char* e = getenv("VX_FMHA_SPLIT");  // diagnostic build only: 0 disables the KV-split tail
    return !(e && atoi(e) == 0);
  }();
#else
  constexpr bool split_on = true;
#endif
  // only for long units: each split costs a merge launch and fp32 partial round trips, which a
  // frame-attention unit (29 KV tiles) does not earn back (S=20 frame layer 0.215 -> 0.228 ms)
  // (not for a fixup, whose work items are listed units, nor for a max-free ring-merge step, whose
  // flagged units must not be merged by the split-merge kernel)
  if (split_on && !PACK && !args.fixup && !(NOMAX && args.merge != 0) && tail > 0 && 2 * tail <= sms &&
      args.kv_tiles >= 128) {
    int parts = sms / tail;
    if (parts > args.kv_tiles / 2) parts = args.kv_tiles / 2;  // >= 2 KV tiles per item
    if (parts >= 2 && (int64_t)parts * args.kv_tiles < (1ll << 31)) {
      float* scratch = split_scratch(st, (size_t)sms * Cfg::ROWS * (D + 1));
      if (scratch) {
        args.split_from = args.units - tail;
        args.parts = parts;
        args.part_o = scratch;
        args.part_lse = scratch + (size_t)sms * Cfg::ROWS * D;
      }
    }
  }
  args.work = args.split_from + (args.units - args.split_from) * args.parts;
  auto kern = fmha_kernel<D, EMU, NT, BKV, ALIAS, SUMV, NOHINT, SPEC, LDSPLIT, PSM, PACK, NOMAX, QL2>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return fail_cuda(e, "fmha: cudaFuncSetAttribute");
    attr_set = true;
  }
  const int grid = args.work < sms ? args.work : sms;
  args.sched = args.work > grid ? sched_counters(st) : nullptr;  // one wave: nothing to distribute
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(tq, tk, tv, args);
  VX_CHECK_LAUNCH("fmha launch");
  if (args.split_from < args.units) {
    const int64_t threads = (int64_t)(args.units - args.split_from) * Cfg::ROWS * (D / 4);
    fmha_split_merge<D, Cfg::ROWS><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(args);
    VX_CHECK_LAUNCH("fmha split merge");
  }
  return VX_OK;
}

static int attention_impl(const void* q, const void* k, const void* v, void* out, int64_t ldo, float* lse, int D,
                          int H, int nseq, int Lq, int Lk, int64_t Tq, int64_t Tk, int merge, float* o_acc,
                          int64_t ld_acc, int flags, void* stream) {
  VX_CHECK_ARG(q && k && v, "vx_attention: null pointer");
  VX_CHECK_ARG(merge == 1 || merge == 2 || out, "vx_attention: null out");
  VX_CHECK_ARG(D == 32 || D == 64 || D == 128, "vx_attention: head_dim %d unsupported (32, 64, 128)", D);
  VX_CHECK_ARG(H > 0 && nseq > 0 && Lq > 0 && Lk > 0, "vx_attention: empty problem");
  VX_CHECK_ARG((int64_t)nseq * Lq <= Tq && (int64_t)nseq * Lk <= Tk, "vx_attention: sequences exceed buffers");
  VX_CHECK_ARG((int64_t)H * Tq + 512 < (1ll << 31) && (int64_t)H * Tk + 512 < (1ll << 31),
               "vx_attention: too many rows for 32-bit TMA coordinates");
  VX_CHECK_ARG(!out || (ldo >= (int64_t)H * D && ldo % 8 == 0), "vx_attention: bad ldo");
  VX_CHECK_ARG(merge == 0 || (o_acc && lse && ld_acc >= (int64_t)H * D && ld_acc % 4 == 0),
               "vx_attention: merge needs o_acc [Tq, >= H*D] fp32 and lse");
  AttnArgs a{};
  a.H = H;
  a.nseq = nseq;
  a.Lq = Lq;
  a.Lk = Lk;
  a.Tq = Tq;
  a.Tk = Tk;
  a.merge = merge;
  a.o_acc = o_acc;
  a.ld_acc = ld_acc;
  // q_blocks / kv_tiles / units depend on the kernel configuration: set in launch_fmha
  const bool q_log2 = (flags & VX_ATTN_Q_LOG2) != 0;
  a.scale_log2 = q_log2 ? 1.0f : (1.0f / sqrtf(float(D))) * 1.4426950408889634f;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.ldo = ldo;
  a.out32 = out && (reinterpret_cast<uintptr_t>(out) % 32 == 0) && (ldo % 16 == 0) && (D % 16 == 0);
  a.lse = lse;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (D == 64) {
    // frame and global layers: 4 Q tiles x 48-wide KV tiles, P aliased onto S, row sums from a
    // ones panel appended to V, S-ready / P-ready waits without a suspend-time hint, exps started
    // with the running max (speculative; the tile max is checked afterwards) and 2 of 8 exp pairs on
    // the FMA pipe, the last 16 S columns loaded behind the first 16 exp pairs, and a branch-free
    // MMA issue path. Sustained S=200 global layer (tools/sustain_attn.sh): 954 TFLOP/s (EMU 1: 923,
    // 3: 922, 4: 887); isolated S=20: 1089.
#ifdef VX_DIAG
    // diagnostic build only (tools/, -DVX_DIAG): the measured alternatives of DESIGN.md §3.1
    static int emu = [] {
      const char* e = getenv("VX_FMHA_EMU");  // exp pairs (of 8) on the FMA pipe
      return e ? atoi(e) : 2;
    }();
    static int cfg = [] {
      const char* e = getenv("VX_FMHA_CFG");
      return e ? atoi(e) : 0;
    }();
    switch (cfg) {
      case 1: return launch_fmha<64, 2, 2, 128>(q, k, v, a, st);                       // 2 x 128 run-ahead
      case 3: return launch_fmha<64, 2, 3, 64>(q, k, v, a, st);                        // 3 x 64 run-ahead
      case 4: return launch_fmha<64, 2, 4, 64, true>(q, k, v, a, st);                  // 4 x 64 aliased
      case 13: return launch_fmha<64, 2, 4, 48, true, true, true>(q, k, v, a, st);     // exact max
      case 14: return launch_fmha<64, 2, 4, 48, true, true, false>(q, k, v, a, st);    // + suspend-hint waits
      case 15: return launch_fmha<64, 2, 4, 48, true, false, true>(q, k, v, a, st);    // FADD row sums
      case 16: return launch_fmha<64, 1, 4, 48, true, false, true>(q, k, v, a, st);
      case 20: return launch_fmha<64, 2, 4, 48, true, true, true, true, false>(q, k, v, a, st);  // one S load
      default: break;
    }
    switch (emu) {
      case 0: return launch_fmha<64, 0, 4, 48, true, true, true, true, true>(q, k, v, a, st);
      case 1: return launch_fmha<64, 1, 4, 48, true, true, true, true, true>(q, k, v, a, st);
      case 3: return launch_fmha<64, 3, 4, 48, true, true, true, true, true>(q, k, v, a, st);
      default: break;
    }
#endif
#if VX_FMHA_PSM
    return launch_fmha<64, 2, 4, 48, false, true, true, true, false, true>(q, k, v, a, st);
#elif VX_FMHA_W96
    return launch_fmha<64, 2, 3, 96, true, true, true, true, false>(q, k, v, a, st);
#else
    // frame attention (several sequences whose 128-row tile count is not a multiple of 4, e.g. 1374
    // rows = 11 tiles): units of 4 consecutive tiles across sequence boundaries
    const int tps = (Lq + 127) / 128;
#ifdef VX_DIAG
    static const bool pack_on = [] {
      const char* e = getenv("VX_FMHA_PACK");  // diagnostic build only: 0 = one sequence per unit
      return !(e && atoi(e) == 0);
    }();
#else
    constexpr bool pack_on = true;
#endif
    const bool pack = pack_on && merge == 0 && nseq > 1 && tps >= 4 && tps % 4 != 0;
    // run max-free first (NOMAX) and then the exact kernel as a fixup over the flagged units (it exits
    // at once when there are none); while the stream is being captured (no list storage) only the
    // exact kernel runs
    unsigned* flag = sched_counters(st);
    const int64_t cap = (int64_t)H * nseq * tps;  // >= units of any configuration
    unsigned* list = flag && cap < (1ll << 30) ? fix_buffer(st, cap) : nullptr;
    if (flag && list) {
      a.bad = flag + 2;
      a.fix_list = list;
      a.fix_cap = int(cap);
      constexpr int E = VX_FMHA_NOMAX_EMU;
      int e;
#if VX_FMHA_NOMAX_W64
      if (q_log2)
        e = pack ? launch_fmha<64, E, 4, 64, true, false, true, true, false, false, true, true, true>(q, k, v, a, st)
                 : launch_fmha<64, E, 4, 64, true, false, true, true, false, false, false, true, true>(q, k, v, a, st);
      else
        e = pack ? launch_fmha<64, E, 4, 64, true, false, true, true, false, false, true, true>(q, k, v, a, st)
                 : launch_fmha<64, E, 4, 64, true, false, true, true, false, false, false, true>(q, k, v, a, st);
#else
      if (q_log2)
        e = pack ? launch_fmha<64, E, 4, 48, true, true, true, true, true, false, true, true, true>(q, k, v, a, st)
                 : launch_fmha<64, E, 4, 48, true, true, true, true, true, false, false, true, true>(q, k, v, a, st);
      else
        e = pack ? launch_fmha<64, E, 4, 48, true, true, true, true, true, false, true, true>(q, k, v, a, st)
                 : launch_fmha<64, E, 4, 48, true, true, true, true, true, false, false, true>(q, k, v, a, st);
#endif
      if (e != VX_OK) return e;
      a.fixup = 1;
    }
    if (pack) return launch_fmha<64, 2, 4, 48, true, true, true, true, true, false, true>(q, k, v, a, st);
    return launch_fmha<64, 2, 4, 48, true, true, true, true, true>(q, k, v, a, st);
#endif
  }
  if (D == 128) return launch_fmha<128, 2>(q, k, v, a, st);
  return launch_fmha<32, 2>(q, k, v, a, st);
}

}  // namespace vx

extern "C" int vx_attention(const void* q, const void* k, const void* v, void* out, int64_t ldo, float* lse, int D,
                            int H, int nseq, int Lq, int Lk, int64_t Tq, int64_t Tk, void* stream) {
  return vx::attention_impl(q, k, v, out, ldo, lse, D, H, nseq, Lq, Lk, Tq, Tk, 0, nullptr, 0, 0, stream);
}

extern "C" int vx_attention_merge(const void* q, const void* k, const void* v, int mode, float* o_acc, int64_t ld_acc,
                                  float* lse_acc, void* out, int64_t ldo, int D, int H, int nseq, int Lq, int Lk,
                                  int64_t Tq, int64_t Tk, void* stream) {
  VX_CHECK_ARG(mode >= 1 && mode <= 3, "vx_attention_merge: mode must be 1 (first), 2 (merge) or 3 (final)");
  return vx::attention_impl(q, k, v, mode == 3 ? out : nullptr, ldo, lse_acc, D, H, nseq, Lq, Lk, Tq, Tk, mode, o_acc,
                            ld_acc, 0, stream);
}

extern "C" int vx_attention_ex(const void* q, const void* k, const void* v, int mode, float* o_acc, int64_t ld_acc,
                               float* lse_acc, void* out, int64_t ldo, int D, int H, int nseq, int Lq, int Lk,
                               int64_t Tq, int64_t Tk, int flags, void* stream) {
  VX_CHECK_ARG(mode >= 0 && mode <= 3, "vx_attention_ex: mode must be 0 (plain) or 1-3 (ring merge)");
  VX_CHECK_ARG((flags & ~VX_ATTN_Q_LOG2) == 0, "vx_attention_ex: unknown flags 0x%x", flags);
  return vx::attention_impl(q, k, v, mode == 1 || mode == 2 ? nullptr : out, ldo, lse_acc, D, H, nseq, Lq, Lk, Tq, Tk,
                            mode, o_acc, ld_acc, flags, stream);
}

#ifdef VX_FMHA_TRACE
extern "C" int vx_fmha_set_trace(void* buf) {
  cudaError_t e = cudaMemcpyToSymbol(vx::g_fmha_trace, &buf, sizeof(void*));
  return e == cudaSuccess ? 0 : -2;
}
#endif
