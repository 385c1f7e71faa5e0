// Camera-head kernels outside the trunk GEMMs, all fp32 where VGGT-X keeps the
// head MLPs in full precision ("BFloat16 except MLP in heads"):
//
//   vx_linear_f32      tiled SIMT fp32 GEMM  out = epi(X W^T + b) for the pose embedding
//                      (`embed_pose`, Linear(9, 2C), fused SiLU -> bf16 operand of the AdaLN
//                      modulation GEMM) and the pose branch (`pose_branch` Mlp 2C -> C -> 9 with
//                      exact-erf GELU, the fc2 epilogue adding the refinement delta to the running
//                      pose encoding and applying activate_pose: T / quaternion linear, FoV relu)
//   vx_adaln_modulate  x = gate * (LN(tok) * (1 + scale) + shift) + tok with the no-affine LayerNorm
//                      (`adaln_norm`, eps 1e-6) and the [shift | scale | gate] split of the
//                      modulation output fused in one pass per camera token
//
// Both are tiny (S x 2C x 1-2K MACs per iteration) next to the trunk; they replace the eager
// torch / cuBLAS-SIMT calls of the round-1 host code so the whole camera head runs on libvx.
#include <math.h>

#include "../../include/vx_api.h"
#include "common.cuh"
#include "host_util.h"

namespace vx {

constexpr int LF_BM = 64, LF_BN = 64, LF_BK = 16, LF_THREADS = 256;

VX_DEVICE float gelu_erf_exact(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

// 64 x 64 output tile per CTA, 4 x 4 per thread; X [M, K] (row stride ldx, 0 = one broadcast row)
// and W [N, K] are both K-contiguous, staged K-major in shared memory.
__global__ void __launch_bounds__(LF_THREADS) linear_f32_kernel(int epi, const float* __restrict__ X, int64_t ldx,
                                                                const float* __restrict__ W, int64_t ldw,
                                                                const float* __restrict__ bias, int M, int N, int K,
                                                                void* out, int64_t ldo, const float* prev,
                                                                float* act_out) {
  __shared__ float sx[LF_BK][LF_BM + 4];
  __shared__ float sw[LF_BK][LF_BN + 4];
  const int m0 = blockIdx.y * LF_BM, n0 = blockIdx.x * LF_BN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += LF_BK) {
    // 64 rows x 16 k of each operand: 1024 elements, 4 per thread (k fastest: coalesced along K)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = threadIdx.x + i * LF_THREADS;
      const int r = e >> 4, kk = e & 15;
      const int gk = k0 + kk;
      const int gm = m0 + r, gn = n0 + r;
      sx[kk][r] = (gm < M && gk < K) ? X[(int64_t)gm * ldx + gk] : 0.f;
      sw[kk][r] = (gn < N && gk < K) ? W[(int64_t)gn * ldw + gk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < LF_BK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&sx[kk][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&sw[kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j] + (bias ? bias[n] : 0.f);
      switch (epi) {
        case VX_LF_GELU:
          v = gelu_erf_exact(v);
          [[fallthrough]];
        case VX_LF_F32:
          reinterpret_cast<float*>(out)[(int64_t)m * ldo + n] = v;
          break;
        case VX_LF_SILU_BF16:
          reinterpret_cast<__nv_bfloat16*>(out)[(int64_t)m * ldo + n] = __float2bfloat16_rn(v / (1.0f + __expf(-v)));
          break;
        case VX_LF_POSE: {  // pred = prev + delta; act_out = activate_pose(pred) (absT_quaR_FoV)
          const float p = (prev ? prev[(int64_t)m * ldo + n] : 0.f) + v;
          reinterpret_cast<float*>(out)[(int64_t)m * ldo + n] = p;
          act_out[(int64_t)m * ldo + n] = n >= 7 ? fmaxf(p, 0.f) : p;
          break;
        }
      }
    }
  }
}

// one warp per camera token; D = 128 * NV
template <int NV>
__global__ void __launch_bounds__(256) adaln_modulate_kernel(const float* __restrict__ tok, const float* __restrict__ mod,
                                                             float* __restrict__ out, int S, float eps) {
  constexpr int D = 128 * NV;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= S) return;
  const float* t = tok + (int64_t)row * D;
  float v[NV][4];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float4 x = *reinterpret_cast<const float4*>(t + (i * 32 + lane) * 4);
    v[i][0] = x.x; v[i][1] = x.y; v[i][2] = x.z; v[i][3] = x.w;
    s += (x.x + x.y) + (x.z + x.w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  const float mean = s * (1.0f / D);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u) q += (v[i][u] - mean) * (v[i][u] - mean);
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffff, q, o);
  const float rstd = rsqrtf(q * (1.0f / D) + eps);
  const float* md = mod + (int64_t)row * 3 * D;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * 4;
    const float4 sh = *reinterpret_cast<const float4*>(md + c);
    const float4 sc = *reinterpret_cast<const float4*>(md + D + c);
    const float4 g = *reinterpret_cast<const float4*>(md + 2 * D + c);
    const float shv[4] = {sh.x, sh.y, sh.z, sh.w}, scv[4] = {sc.x, sc.y, sc.z, sc.w}, gv[4] = {g.x, g.y, g.z, g.w};
    float o[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) o[u] = gv[u] * ((v[i][u] - mean) * rstd * (1.0f + scv[u]) + shv[u]) + v[i][u];
    *reinterpret_cast<float4*>(out + (int64_t)row * D + c) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace vx

extern "C" int vx_linear_f32(int epi, const float* X, int64_t ldx, const float* W, int64_t ldw, const float* bias,
                             int M, int N, int K, void* out, int64_t ldo, const float* prev, float* act_out,
                             void* stream) {
  using namespace vx;
  VX_CHECK_ARG(X && W && out, "vx_linear_f32: null pointer");
  VX_CHECK_ARG(M > 0 && N > 0 && K > 0, "vx_linear_f32: empty problem M=%d N=%d K=%d", M, N, K);
  VX_CHECK_ARG(epi >= VX_LF_F32 && epi <= VX_LF_POSE, "vx_linear_f32: unknown epilogue %d", epi);
  VX_CHECK_ARG(ldx >= 0 && ldw >= K && ldo >= N, "vx_linear_f32: bad strides");
  VX_CHECK_ARG(ldx == 0 || ldx >= K, "vx_linear_f32: ldx must be 0 (broadcast row) or >= K");
  VX_CHECK_ARG(epi != VX_LF_POSE || (act_out && N == 9), "vx_linear_f32: pose epilogue needs N == 9 and act_out");
  dim3 grid((N + LF_BN - 1) / LF_BN, (M + LF_BM - 1) / LF_BM);
  VX_CHECK_ARG(grid.y < 65536, "vx_linear_f32: M too large");
  linear_f32_kernel<<<grid, LF_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(epi, X, ldx, W, ldw, bias, M, N,
                                                                                   K, out, ldo, prev, act_out);
  VX_CHECK_LAUNCH("linear_f32 launch");
  return VX_OK;
}

extern "C" int vx_adaln_modulate(const float* tok, const float* mod, float* out, int S, int D, float eps,
                                 void* stream) {
  using namespace vx;
  VX_CHECK_ARG(tok && mod && out, "vx_adaln_modulate: null pointer");
  VX_CHECK_ARG(S > 0, "vx_adaln_modulate: no tokens");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int grid = (S + 7) / 8;
  switch (D) {
    case 256: adaln_modulate_kernel<2><<<grid, 256, 0, st>>>(tok, mod, out, S, eps); break;
    case 512: adaln_modulate_kernel<4><<<grid, 256, 0, st>>>(tok, mod, out, S, eps); break;
    case 1024: adaln_modulate_kernel<8><<<grid, 256, 0, st>>>(tok, mod, out, S, eps); break;
    case 2048: adaln_modulate_kernel<16><<<grid, 256, 0, st>>>(tok, mod, out, S, eps); break;
    default:
      set_error("vx_adaln_modulate: D=%d unsupported (256, 512, 1024, 2048)", D);
      return VX_E_ARG;
  }
  VX_CHECK_LAUNCH("adaln_modulate launch");
  return VX_OK;
}
