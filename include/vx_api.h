/*
 * vx_api.h — C ABI of the B200-native dense-view VGGT inference kernels.
 *
 * The reference (VGGT-X, arXiv 2509.25191) ships no operator/plugin/FFI
 * interface for this path: the hot path is described
 * only in PAPER.md:76-81 and the upstream `vggt` PyTorch modules.  Each entry
 * point below replaces one upstream PyTorch op of that path (SURVEY.md §8a
 * rows a1-a16, named in the comment); the Python host layer
 * (paper_2509_25191_b200/ops.py) binds them with ctypes, and INTEGRATION.md
 * shows the binding a `vggt` maintainer would add.
 *
 * Conventions
 *   - all tensors are device pointers owned by the caller (PyTorch caching
 *     allocator); the library never frees caller memory;
 *   - bf16 = __nv_bfloat16 storage, fp32 = float;
 *   - every call is asynchronous on `stream` (a cudaStream_t, may be NULL);
 *   - return 0 on success, a negative VX_E* code otherwise; the message of the
 *     last failure on the calling thread is available from vx_last_error().
 *     No C++ exception crosses this boundary.
 */
#ifndef VX_API_H
#define VX_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  VX_OK = 0,
  VX_E_ARG = -1,         /* invalid argument / unsupported shape */
  VX_E_CUDA = -2,        /* CUDA runtime / driver error */
  VX_E_UNSUPPORTED = -3  /* device is not sm_100 */
};

/* GEMM epilogues (D = A[M,K] . B[N,K]^T accumulated in fp32 TMEM). */
enum {
  VX_EPI_BF16 = 0,   /* out bf16 [M, ldo]   = D + bias                       (Linear)            */
  VX_EPI_GELU = 1,   /* out bf16 [M, ldo]   = gelu_erf(D + bias)             (Mlp.fc1 + GELU, a10) */
  VX_EPI_RESID = 2,  /* resid fp32 [M, ldr] += gamma * (D + bias); optional
                        kept bf16 [M, ldk] = new resid                       (proj/fc2 + LayerScale
                                                                              + residual, a9/a10/a11) */
  VX_EPI_QKV = 3,    /* qkv Linear + q/k LayerNorm(head_dim) + 2D RoPE, scattered
                        to q/k/v bf16 [H, T, head_dim]                       (Attention.qkv/q_norm/
                                                                              k_norm/rope, a4/a6);
                        without qk-norm and RoPE any head_dim % 32 == 0 (camera-head trunk, d = 128) */
  VX_EPI_PATCH = 4,  /* patch-embed: resid fp32 row (f*tpf + ps + p) = D + bias (PatchEmbed, a2)    */
  VX_EPI_F32 = 5     /* out fp32 [M, ldo]   = D + bias                                              */
};

typedef struct vx_epilogue {
  const float* bias;          /* [N] or NULL */
  void* out;                  /* VX_EPI_BF16/GELU/F32 output, row stride ldo elements */
  int64_t ldo;
  float* resid;               /* VX_EPI_RESID / VX_EPI_PATCH fp32 residual stream, stride ldr */
  int64_t ldr;
  const float* gamma;         /* VX_EPI_RESID LayerScale [N] */
  void* kept;                 /* VX_EPI_RESID optional bf16 copy of the new residual, stride ldk */
  int64_t ldk;
  void* q;                    /* VX_EPI_QKV outputs, each bf16 [H, T, head_dim] */
  void* k;
  void* v;
  const float* qn_w;          /* q_norm / k_norm affine [head_dim]; NULL disables qk-norm */
  const float* qn_b;
  const float* kn_w;
  const float* kn_b;
  const float* rope_cos;      /* [max_pos, head_dim/4] fp32; NULL disables RoPE */
  const float* rope_sin;
  int embed_dim;              /* C (=H*head_dim) */
  int head_dim;               /* 32 or 64 */
  int tokens_total;           /* T = rows of q/k/v per head */
  int tokens_per_frame;       /* tokens per view (RoPE positions, patch row remap) */
  int patch_start;            /* 1 + registers */
  int grid_w;                 /* patches per image row */
  float eps;                  /* q/k LayerNorm eps */
  float q_scale;              /* VX_EPI_QKV: q is multiplied by this before its bf16 store (0 = 1); the
                                 aggregator stores q * log2(e)/sqrt(head_dim) for VX_ATTN_Q_LOG2 */
  int col_offset;             /* VX_EPI_QKV: the B rows are rows col_offset .. col_offset+N-1 of the
                                 [3C, C] qkv weight (bias likewise sliced): output column c is q/k/v
                                 column col_offset + c. 0 = the whole weight (N = 3C); C with N = 2C
                                 writes K and V only, 0 with N = C q only (chunked-q global blocks) */
} vx_epilogue;

/* D[M,N] = A[M,K] (bf16, row stride lda) . B[N,K]^T (bf16, row stride ldb) with
 * epilogue `epi`.  K % 64 == 0, N % 32 == 0. tcgen05/TMEM/TMA persistent kernel. */
int vx_gemm(int epi, const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K,
            const vx_epilogue* ep, void* stream);

/* Flash attention (non-causal, no dropout) — replaces F.scaled_dot_product_attention in
 * Attention.forward for frame blocks (nseq = frames) and global blocks (nseq = 1) (a7/a8).
 *   q: bf16 [H, Tq, D]; k, v: bf16 [H, Tk, D]; sequence s of head h uses rows
 *   h*Tq + s*Lq .. +Lq (q) and h*Tk + s*Lk .. +Lk (k, v).
 *   out: bf16, row (s*Lq + i), columns h*D .. h*D+D-1, row stride ldo.
 *   lse: optional fp32 [H, Tq] natural-log log-sum-exp of the scaled scores.
 * D in {32, 64, 128} (128: camera-head trunk); scale = 1/sqrt(D).
 * When the last wave of 512-row work units would leave more than half the SMs idle, those units
 * are split over KV ranges and merged by a second kernel on the same stream; the fp32 partials
 * live in a per-stream scratch buffer (num_SMs x 512 x (D+1) floats, ~19 MB at D=64) allocated on
 * first use and kept. While the stream is being captured into a graph nothing is allocated and
 * the split is skipped unless the buffer already exists.
 * Work units past the first wave are claimed from a per-stream atomic ticket counter (4 x u32
 * allocated on the stream's first launch, reset by each launch's last CTA), so CTAs that start late
 * (SMs held by a concurrent kernel, e.g. an NCCL transfer) take fewer units; results do not depend
 * on the assignment (each unit's arithmetic is fixed).
 * D = 64 launches (plain and ring merge) run a max-free softmax (P = 2^score, no running max) and
 * then the exact kernel as a fixup over the work units with a row whose sum or output left the safe
 * fp32 range (a per-stream list; the fixup exits at once when it is empty): results are those of
 * the exact kernel either way, up to rounding. While the stream is being captured only the exact
 * kernel runs. */
int vx_attention(const void* q, const void* k, const void* v, void* out, int64_t ldo, float* lse,
                 int D, int H, int nseq, int Lq, int Lk, int64_t Tq, int64_t Tk, void* stream);
/* One K/V-ring step of frame-sharded global attention with the log-sum-exp merge
 * fused into the epilogue: mode 1 (first block) writes o_acc = O_blk (fp32 [Tq, ld_acc]) and
 * lse_acc = lse_blk ([H, Tq]); mode 2 merges: o_acc = w_a o_acc + w_b O_blk, lse_acc =
 * logaddexp(lse_acc, lse_blk); mode 3 merges and writes the final bf16 `out` (row stride ldo)
 * instead of o_acc.  Same shapes and head layout as vx_attention. */
int vx_attention_merge(const void* q, const void* k, const void* v, int mode, float* o_acc, int64_t ld_acc,
                       float* lse_acc, void* out, int64_t ldo, int D, int H, int nseq, int Lq, int Lk,
                       int64_t Tq, int64_t Tk, void* stream);
/* Both of the above with flags: mode 0 = vx_attention (out, optional lse in lse_acc), 1-3 =
 * vx_attention_merge.  VX_ATTN_Q_LOG2: q already holds q * log2(e)/sqrt(D) (the qkv epilogue's
 * q_scale), so the scores come out of the MMA in log2 units and the softmax skips one multiply per
 * score; results (out, natural-log lse) mean the same as without the flag. */
enum { VX_ATTN_Q_LOG2 = 1 };
int vx_attention_ex(const void* q, const void* k, const void* v, int mode, float* o_acc, int64_t ld_acc,
                    float* lse_acc, void* out, int64_t ldo, int D, int H, int nseq, int Lq, int Lk, int64_t Tq,
                    int64_t Tk, int flags, void* stream);

/* Camera head, fp32 parts ("bf16 except MLP in heads").
 * vx_linear_f32: out[M, N] = epi(X[M, K] . W[N, K]^T + bias), fp32 SIMT (X row stride ldx; ldx = 0
 * broadcasts one row, e.g. the (1, 1, 9) `empty_pose_tokens`).  Replaces CameraHead.embed_pose
 * (+ the SiLU of poseLN_modulation), pose_branch.fc1 + GELU and pose_branch.fc2 + the iterative
 * `pred_pose_enc + delta` update + activate_pose. */
enum {
  VX_LF_F32 = 0,        /* out fp32 = acc + bias                                   */
  VX_LF_GELU = 1,       /* out fp32 = gelu_erf(acc + bias)                         */
  VX_LF_SILU_BF16 = 2,  /* out bf16 = silu(acc + bias)                             */
  VX_LF_POSE = 3        /* N == 9: out fp32 pred = (prev ? prev : 0) + acc + bias;
                           act_out = activate_pose(pred) (T, quat linear; FoV relu) */
};
int vx_linear_f32(int epi, const float* X, int64_t ldx, const float* W, int64_t ldw, const float* bias, int M, int N,
                  int K, void* out, int64_t ldo, const float* prev, float* act_out, void* stream);
/* AdaLN modulation of the camera tokens (CameraHead.trunk_fn input): mod fp32 [S, 3D] = [shift | scale |
 * gate] (output of poseLN_modulation), out fp32 [S, D] = gate * (LN(tok) * (1 + scale) + shift) + tok
 * with the no-affine `adaln_norm` LayerNorm (eps).  D in {256, 512, 1024, 2048}. */
int vx_adaln_modulate(const float* tok, const float* mod, float* out, int S, int D, float eps, void* stream);

/* LayerNorm over the last dim (cols): y = (x - mean) * rstd * w + b.
 * x_dtype / y_dtype: 0 = fp32, 1 = bf16.  w/b may be NULL (no affine). (norm1/norm2, a5) */
int vx_layernorm(const void* x, int x_dtype, int64_t ldx, void* y, int y_dtype, int64_t ldy,
                 const float* w, const float* b, int rows, int cols, float eps, void* stream);
/* Same, reading output row r from input row (r / group_rows) * group_stride + group_offset +
 * r % group_rows — e.g. the DPT heads' patch tokens of each frame (group_rows = patches,
 * group_stride = tokens per frame, group_offset = patch_start) without a gather copy. */
int vx_layernorm_gather(const void* x, int x_dtype, int64_t ldx, void* y, int y_dtype, int64_t ldy,
                        const float* w, const float* b, int rows, int cols, float eps, int group_rows,
                        int group_stride, int group_offset, void* stream);

/* ResNet-normalise + im2col of (S,3,H,W) fp32 images into bf16 [S*P, Kpad] with
 * K order (c, ky, kx) and zero padding K..Kpad-1.  (Aggregator normalize + PatchEmbed, a1/a2) */
int vx_patchify(const float* images, void* out, int S, int H, int W, int patch, int Kpad,
                void* stream);

/* DINOv2 ViT-L/14-reg token assembly (a2', upstream DinoVisionTransformer.prepare_tokens_with_masks as
 * built by the VGGT aggregator) on the patch-embedded stream x fp32 [S * tpf, C] whose patch p of frame f
 * sits at row f*tpf + 1 + nreg + p: row f*tpf = cls + pos[0]; rows 1..nreg = reg (no position);
 * patch rows += pos[1 + p].  cls [C], reg [nreg, C], pos [1 + P, C] (already interpolated to the grid). */
int vx_dino_tokens(float* x, const float* cls, const float* reg, const float* pos, int S, int tpf, int nreg, int C,
                   void* stream);

/* Write camera (1) and register (R) tokens into the fp32 residual stream:
 * x[f*tpf + t] = (f == 0 ? tok[0] : tok[1])[t] for t < 1+R.  tokens: fp32 [2, 1+R, C]
 * (slice_expand_and_flatten + cat, a3) */
int vx_special_tokens(float* x, const float* tokens, int S, int tpf, int ntok, int C, void* stream);

/* Bilinear resize with align_corners=True of NHWC bf16 maps in [F, h, w, C] -> out [F, H, W, C]
 * (out_pad = 1: written into the interior of a zero-bordered [F, H+2, W+2, C] buffer), plus an
 * optional bf16 [H, W, C] map added after interpolation (DPT pos-embed).
 * (F.interpolate(mode="bilinear", align_corners=True) in DPTHead / FeatureFusionBlock, a14) */
int vx_upsample_bilinear(const void* in, int F, int h, int w, int C, void* out, int H, int W,
                         const void* add_hwc, int out_pad, void* stream);

/* Spatial GEMM for the DPT heads: rows are pixels of F frames.
 *   conv3x3 = 1: implicit-GEMM 3x3 / stride 1 / pad 1 convolution; A is a zero-padded NHWC
 *                bf16 buffer [F, H+2, W+2, Cin] (K = 9*Cin, weight K order (ky, kx, cin)); GEMM
 *                rows live on the padded grid and the border rows are discarded;
 *   conv3x3 = 0: 1x1 convolution / linear over dense NHWC rows [F*H*W, K].
 * Epilogue (per output element): v = acc + bias (+ pos[yo, xo, c]); relu?; + res1; + res2;
 *   out1 = v, out2 = relu(v) — bf16 NHWC, each tensor padded (1-pixel zero border) or dense.
 *   subsample2: stride-2 output (even y, x); shuffle = s: conv-transpose k = s, stride s with
 *   N = s*s*Cout ordered (i, j, c).
 * head_odim > 0 fuses the DPT output head (N == 32): relu(acc + bias) -> fp32 1x1 conv
 *   (head_w [odim, 32], head_b) -> activation (head_act 0: exp, 1: sign*expm1|x|) for the first
 *   odim-1 channels into head_pred [F, H, W, odim-1] and 1 + exp(x) into head_conf [F, H, W]. */
typedef struct vx_spatial {
  int conv3x3;
  int F, H, W;
  int subsample2;
  int shuffle;
  int relu;
  const void* pos;
  const void* res1;
  int res1_pad;
  const void* res2;
  int res2_pad;
  void* out1;
  int out1_pad;
  void* out2;
  int out2_pad;
  const float* head_w;
  const float* head_b;
  int head_odim;
  int head_act;
  float* head_pred;
  float* head_conf;
} vx_spatial;

int vx_gemm_spatial(const void* A, const void* B, int N, int K, const float* bias, const vx_spatial* sp,
                    void* stream);

/* Global-Alignment epipolar kernels, fp64, all image pairs in one launch.
 * Replace pkg/src/epialign/_kernels_cy.pyx pair_residuals (:26-54) / pair_accumulate (:57-116).
 *   F: [P, 3, 3] unit-Frobenius fundamental matrices; offsets: [P+1] prefix sums partitioning
 *   the correspondences xy_i, xy_j: [K, 2] (pixels) and weights w: [K].
 *   mode 0 = algebraic |x'^T F x|, 1 = geometric point-to-line distance (NaN / skipped when
 *   |(l0, l1)| < 1e-12); residuals < 1e-9 keep their loss but get a zero subgradient.
 * residuals: e [K], n_deg [P].  accumulate: out [P, 11] = (loss_sum, weight_sum, dL/dF row-major),
 * n_skipped [P]. */
int vx_epipolar_residuals(const double* F, const int64_t* offsets, const double* xy_i, const double* xy_j,
                          int num_pairs, int mode, double* e, int32_t* n_deg, void* stream);
int vx_epipolar_accumulate(const double* F, const int64_t* offsets, const double* xy_i, const double* xy_j,
                           const double* w, int num_pairs, int mode, double* out, int32_t* n_skipped,
                           void* stream);

/* Global-Alignment optimiser on the device ("plus the on-device chain rule and
 * Adam over 300 iterations").  Replaces the per-pair host loops of pkg/src/epialign/aligner.py:
 * _Problem._decode (:160-174), _pair_F (:176-185), residuals (:189-207), loss_and_gradient
 * (:209-278) and the adaptive-moment loop of align (:408-417).  All fp64, row-major 3x3 matrices.
 * Every pointer is device memory owned by the caller. */
typedef struct vx_ga_problem {
  int n_frames, n_pairs;
  int dim;          /* 9, or 10 with the log-focal parameter (optimize_focal) */
  int mode;         /* 0 algebraic, 1 geometric */
  int gauge;        /* gauge frame: its parameters never move */
  const int32_t* pair_ij;     /* [P, 2] frame indices (i, j) */
  const int64_t* offsets;     /* [P+1] correspondence prefix sums */
  const double* xy_i;         /* [K, 2] */
  const double* xy_j;         /* [K, 2] */
  const double* w;            /* [K] weights (residual calls ignore it) */
  const int32_t* frame_ptr;   /* [n+1] CSR over (pair, role) entries touching each frame */
  const int32_t* frame_ent;   /* [2P] entry = 2*pair + (frame is j), ascending pair order */
  const double* base_R;       /* [n, 9] canonical-gauge rotations */
  const double* base_t;       /* [n, 3] canonical-gauge translations */
  const double* base_Kinv;    /* [n, 9] inverse intrinsics */
  double* params;             /* [n, dim] pose residual blocks (6D rotation, translation, log focal) */
  double* adam_m;             /* [n, dim] first moments */
  double* adam_v;             /* [n, dim] second moments */
  double* Rs;                 /* [n, 9] decoded rotations (scratch, kept current by the calls) */
  double* ts;                 /* [n, 3] */
  double* Kinv;               /* [n, 9] */
  double* geom;               /* [P, 32] per-pair geometry: R_ij, t_ij, E, F/|F|, |F|, valid (scratch) */
  double* payload;            /* [P, 32] per-pair gradient contributions (scratch) */
  double* scalars;            /* [4 + 3*ceil(P/64)]: num, den, skipped (this evaluation), spare; then
                                 per-block partial sums (scratch) */
  int32_t* status;            /* [2]: [0] bit 0 degenerate 6D rotation, bit 1 zero total weight;
                                 [1] block counter, must be 0 on entry (left 0 on exit) */
} vx_ga_problem;

/* Rs/ts/Kinv <- decode(params). */
int vx_ga_decode(const vx_ga_problem* pb, void* stream);
/* Residuals at the decoded cameras: e [K] (NaN for degenerate lines and for every correspondence of
 * a pair whose fundamental matrix vanishes), deg_pair [P] (1 = pair degenerate), n_deg [P]. */
int vx_ga_residuals(const vx_ga_problem* pb, double* e, int32_t* deg_pair, int32_t* n_deg, void* stream);
/* One loss/gradient evaluation at the decoded cameras: grad [n, dim] (gauge block exactly 0),
 * scalars = (num, den, skipped). */
int vx_ga_loss_grad(const vx_ga_problem* pb, double* grad, void* stream);
/* `iters` full-batch adaptive-moment steps t = t0+1 .. t0+iters (1-based, as aligner.py:408):
 * loss trace -> trace[t-1]; bias corrections bc1[t-1] = 1 - beta1^t, bc2[t-1] = 1 - beta2^t;
 * skipped correspondences accumulated into *skipped_total.  Launched as one CUDA graph when
 * use_graph != 0.  Leaves params, moments and the decoded cameras current. */
int vx_ga_adam(const vx_ga_problem* pb, int t0, int iters, double lr, const double* bc1, const double* bc2,
               double* trace, double* skipped_total, int use_graph, void* stream);
/* Adaptive weights (pkg/src/epialign/weighting.py:56-109): histogram of the finite residuals clipped
 * to [edges[0], edges[n_bins]], density floor 1e-6, w = (f(e)/mean f)^alpha (0 for NaN residuals).
 * scratch: [n_bins] int64 counts; out_stats [2 + n_bins] = (avg density, finite count, densities). */
int vx_ga_adaptive_weights(const double* e, int64_t K, const double* edges, int n_bins, double alpha, double* w,
                           int64_t* counts, double* out_stats, void* stream);

/* Scene-level consumers of the predictions, csrc/scene.cu.
 *
 * vx_matched_points — pkg/src/epialign/pointcloud.py:91-130 select_matched_points with
 *   sample_depth (:66-88) and geometry.py:341-348 unproject.  Depth maps: `depth` holds every map
 *   (fp32 if depth_f32 else fp64) at element offsets map_offset[k], shape map_hw[2k] x map_hw[2k+1];
 *   frame f uses map slot[f].  Cameras R [n,9], t [n,3], Kinv [n,9] (fp64, world-to-camera).
 *   Per correspondence m: state[m] = 0 weight <= threshold, 1 emitted (points[m] = (p_i, p_j),
 *   gap[m] = |p_i - p_j|), 2 skipped (a depth sample <= 0), 3 non-finite depth sample. */
int vx_matched_points(const void* depth, int depth_f32, const int64_t* map_offset, const int32_t* map_hw,
                      const int32_t* slot, const double* R, const double* t, const double* Kinv,
                      const int32_t* pair_ij, const int64_t* offsets, int n_pairs, const double* xy_i,
                      const double* xy_j, const double* w, double threshold, double* points, double* gap,
                      int8_t* state, void* stream);
/* Dense world-point maps of VGGT depth: out[s, y, x] = R_s^T (depth[s,y,x] K_s^-1 (x, y, 1) - t_s),
 * fp32; extrinsic [S,3,4] world-to-camera, intrinsic [S,3,3]. */
int vx_unproject_depth(const float* depth, int S, int H, int W, const float* extrinsic, const float* intrinsic,
                       float* out, void* stream);
/* pairing.py:88-109: view angle (degrees) between the optical axes (third rows of R [n,9]) of every
 * pair i < j, in row-major upper-triangle order (n(n-1)/2 entries); flag = angle <= threshold. */
int vx_select_pairs(const double* R, int n, double threshold_deg, int8_t* flag, double* angle, void* stream);
/* metrics.py:89-118: RRE / RTE (degrees) of every pair i < j of the predicted rig against the ground
 * truth (gt_of[i] = ground-truth index of predicted frame i), upper-triangle order; with
 * order_invariant each pair writes (i, j) then (j, i).  zero_baseline = 1 where RTE was forced to 0. */
int vx_pairwise_errors(const double* Rp, const double* tp, const double* Rg, const double* tg,
                       const int32_t* gt_of, int n, int order_invariant, double* rre, double* rte,
                       uint8_t* zero_baseline, void* stream);

int vx_num_sms(void);
/* Kernels this library has launched in this process (a CUDA-graph replay counts its kernel nodes). */
uint64_t vx_launch_count(void);
const char* vx_last_error(void);
/* "vx <abi> sm_100a"; abi 0.2 added vx_epilogue.col_offset (a caller built against 0.1 passes a shorter
 * struct: rebuild against this header) */
const char* vx_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VX_API_H */
