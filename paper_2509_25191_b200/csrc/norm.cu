// HBM-bound kernels of the aggregator: LayerNorm (fp32 residual -> bf16 GEMM
// operand), ResNet-normalise + im2col for the patch-embed GEMM, special-token
// writes.  SURVEY.md §8a rows a1, a3, a5.
#include "../../include/vx_api.h"
#include "common.cuh"
#include "host_util.h"

namespace vx {

template <typename T>
VX_DEVICE void load4(const T* p, float (&o)[4]);
template <>
VX_DEVICE void load4<float>(const float* p, float (&o)[4]) {
  float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <>
VX_DEVICE void load4<__nv_bfloat16>(const __nv_bfloat16* p, float (&o)[4]) {
  uint2 v = *reinterpret_cast<const uint2*>(p);
  __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&v.x);
  __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&v.y);
  float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
  o[0] = fa.x; o[1] = fa.y; o[2] = fb.x; o[3] = fb.y;
}
template <typename T>
VX_DEVICE void store4(T* p, const float (&o)[4]);
template <>
VX_DEVICE void store4<float>(float* p, const float (&o)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
}
template <>
VX_DEVICE void store4<__nv_bfloat16>(__nv_bfloat16* p, const float (&o)[4]) {
  *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]));
}

// one warp per row; NV = float4-groups per lane (cols = 128 * NV)
template <typename TI, typename TO, int NV>
__global__ void __launch_bounds__(256) layernorm_kernel(const TI* __restrict__ x, int64_t ldx, TO* __restrict__ y,
                                                        int64_t ldy, const float* __restrict__ w,
                                                        const float* __restrict__ b, int rows, float eps,
                                                        int g_rows, int g_stride, int g_off) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  constexpr int cols = 128 * NV;
  // input row gather: output row r reads row (r / g_rows) * g_stride + g_off + r % g_rows
  const int g = row / g_rows;
  const TI* xr = x + ((size_t)g * g_stride + g_off + (row - g * g_rows)) * ldx;
  float v[NV][4];
#pragma unroll
  for (int i = 0; i < NV; ++i) load4<TI>(xr + (i * 32 + lane) * 4, v[i]);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) s += (v[i][0] + v[i][1]) + (v[i][2] + v[i][3]);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  const float mean = s * (1.0f / cols);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float d = v[i][u] - mean;
      q += d * d;
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffff, q, o);
  const float rstd = rsqrtf(q * (1.0f / cols) + eps);
  TO* yr = y + (size_t)row * ldy;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * 4;
    float o[4];
    if (w) {
      float4 wv = __ldg(reinterpret_cast<const float4*>(w + c));
      float4 bv = b ? __ldg(reinterpret_cast<const float4*>(b + c)) : make_float4(0, 0, 0, 0);
      o[0] = (v[i][0] - mean) * rstd * wv.x + bv.x;
      o[1] = (v[i][1] - mean) * rstd * wv.y + bv.y;
      o[2] = (v[i][2] - mean) * rstd * wv.z + bv.z;
      o[3] = (v[i][3] - mean) * rstd * wv.w + bv.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) o[u] = (v[i][u] - mean) * rstd;
    }
    store4<TO>(yr + c, o);
  }
}

template <typename TI, typename TO>
static int ln_dispatch(const void* x, int64_t ldx, void* y, int64_t ldy, const float* w, const float* b, int rows,
                       int cols, float eps, cudaStream_t st, int g_rows, int g_stride, int g_off) {
  const int grid = (rows + 7) / 8;
  const TI* xi = reinterpret_cast<const TI*>(x);
  TO* yo = reinterpret_cast<TO*>(y);
  switch (cols / 128) {
#define VX_LN_CASE(nv) \
  case nv:                 \
    layernorm_kernel<TI, TO, nv><<<grid, 256, 0, st>>>(xi, ldx, yo, ldy, w, b, rows, eps, g_rows, g_stride, g_off); \
    break;
    VX_LN_CASE(1)
    VX_LN_CASE(2)
    VX_LN_CASE(4)
    VX_LN_CASE(8)
    VX_LN_CASE(16)
#undef VX_LN_CASE
    default:
      set_error("vx_layernorm: cols=%d unsupported (128*{1,2,4,8,16})", cols);
      return VX_E_ARG;
  }
  VX_CHECK_LAUNCH("layernorm launch");
  return VX_OK;
}

__global__ void patchify_kernel(const float* __restrict__ img, __nv_bfloat16* __restrict__ out, int S, int H, int W,
                                int ps, int Kpad) {
  const int gw = W / ps, gh = H / ps;
  const int P = gw * gh;
  const int K = 3 * ps * ps;
  const int64_t total = (int64_t)S * P * (Kpad / 2);
  const float mean[3] = {0.485f, 0.456f, 0.406f};
  const float stdv[3] = {0.229f, 0.224f, 0.225f};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int kp = int(i % (Kpad / 2));
    const int64_t rp = i / (Kpad / 2);
    const int p = int(rp % P);
    const int f = int(rp / P);
    const int py = p / gw, px = p - py * gw;
    float o[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = 2 * kp + u;
      if (k < K) {
        const int c = k / (ps * ps);
        const int r = k - c * ps * ps;
        const int ky = r / ps, kx = r - ky * ps;
        const float val = img[(((int64_t)f * 3 + c) * H + py * ps + ky) * W + px * ps + kx];
        o[u] = (val - mean[c]) / stdv[c];
      } else {
        o[u] = 0.f;
      }
    }
    reinterpret_cast<uint32_t*>(out)[i] = pack_bf16(o[0], o[1]);
  }
}

__global__ void special_tokens_kernel(float* __restrict__ x, const float* __restrict__ tok, int S, int tpf, int ntok,
                                      int C) {
  const int64_t total = (int64_t)S * ntok * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = int(i % C);
    const int t = int((i / C) % ntok);
    const int f = int(i / ((int64_t)C * ntok));
    const int which = f == 0 ? 0 : 1;
    x[((int64_t)f * tpf + t) * C + c] = tok[((int64_t)which * ntok + t) * C + c];
  }
}

// DINOv2 token assembly over the patch-embedded residual stream x [S * tpf, C] fp32 (patch p of frame
// f at row f*tpf + 1 + nreg + p): row f*tpf = cls + pos[0], rows 1..nreg = registers, patch rows += pos[1 + p].
// float4 per thread; C % 4 == 0.
__global__ void dino_tokens_kernel(float* __restrict__ x, const float* __restrict__ cls, const float* __restrict__ reg,
                                   const float* __restrict__ pos, int S, int tpf, int nreg, int C) {
  const int C4 = C / 4;
  const int64_t total = (int64_t)S * tpf * C4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c4 = int(i % C4);
    const int t = int((i / C4) % tpf);
    float4* xp = reinterpret_cast<float4*>(x) + i;
    if (t == 0) {
      const float4 a = reinterpret_cast<const float4*>(cls)[c4], b = reinterpret_cast<const float4*>(pos)[c4];
      *xp = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    } else if (t <= nreg) {
      *xp = reinterpret_cast<const float4*>(reg)[(int64_t)(t - 1) * C4 + c4];
    } else {
      const float4 b = reinterpret_cast<const float4*>(pos)[(int64_t)(t - nreg) * C4 + c4];
      float4 v = *xp;
      *xp = make_float4(v.x + b.x, v.y + b.y, v.z + b.z, v.w + b.w);
    }
  }
}

}  // namespace vx

extern "C" int vx_dino_tokens(float* x, const float* cls, const float* reg, const float* pos, int S, int tpf,
                              int nreg, int C, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(x && cls && pos && (nreg == 0 || reg) && S > 0 && tpf > 1 + nreg && C % 4 == 0,
               "vx_dino_tokens: bad args");
  const int64_t total = (int64_t)S * tpf * (C / 4);
  const int grid = int((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  dino_tokens_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, cls, reg, pos, S, tpf, nreg, C);
  VX_CHECK_LAUNCH("dino tokens launch");
  return VX_OK;
}

extern "C" int vx_layernorm_gather(const void* x, int x_dtype, int64_t ldx, void* y, int y_dtype, int64_t ldy,
                                   const float* w, const float* b, int rows, int cols, float eps, int group_rows,
                                   int group_stride, int group_offset, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(x && y, "vx_layernorm: null pointer");
  VX_CHECK_ARG(rows >= 0 && cols > 0 && cols % 128 == 0, "vx_layernorm: cols=%d must be a multiple of 128", cols);
  VX_CHECK_ARG(ldx % 8 == 0 && ldy % 8 == 0, "vx_layernorm: ld must be a multiple of 8");
  VX_CHECK_ARG(group_rows > 0 && group_offset >= 0 && group_stride >= group_rows + group_offset,
               "vx_layernorm: bad row gather (%d, %d, %d)", group_rows, group_stride, group_offset);
  if (rows == 0) return VX_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int gr = group_rows, gs = group_stride, go = group_offset;
  if (x_dtype == 0 && y_dtype == 1)
    return ln_dispatch<float, __nv_bfloat16>(x, ldx, y, ldy, w, b, rows, cols, eps, st, gr, gs, go);
  if (x_dtype == 1 && y_dtype == 1)
    return ln_dispatch<__nv_bfloat16, __nv_bfloat16>(x, ldx, y, ldy, w, b, rows, cols, eps, st, gr, gs, go);
  if (x_dtype == 0 && y_dtype == 0) return ln_dispatch<float, float>(x, ldx, y, ldy, w, b, rows, cols, eps, st, gr, gs, go);
  if (x_dtype == 1 && y_dtype == 0)
    return ln_dispatch<__nv_bfloat16, float>(x, ldx, y, ldy, w, b, rows, cols, eps, st, gr, gs, go);
  set_error("vx_layernorm: bad dtypes %d -> %d", x_dtype, y_dtype);
  return VX_E_ARG;
}

extern "C" int vx_layernorm(const void* x, int x_dtype, int64_t ldx, void* y, int y_dtype, int64_t ldy,
                            const float* w, const float* b, int rows, int cols, float eps, void* stream) {
  return vx_layernorm_gather(x, x_dtype, ldx, y, y_dtype, ldy, w, b, rows, cols, eps, rows > 0 ? rows : 1,
                             rows > 0 ? rows : 1, 0, stream);
}

extern "C" int vx_patchify(const float* images, void* out, int S, int H, int W, int patch, int Kpad, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(images && out, "vx_patchify: null pointer");
  VX_CHECK_ARG(S > 0 && H % patch == 0 && W % patch == 0, "vx_patchify: H, W must be multiples of the patch");
  VX_CHECK_ARG(Kpad % 2 == 0 && Kpad >= 3 * patch * patch, "vx_patchify: bad Kpad");
  const int64_t total = (int64_t)S * (H / patch) * (W / patch) * (Kpad / 2);
  const int grid = int((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  patchify_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      images, reinterpret_cast<__nv_bfloat16*>(out), S, H, W, patch, Kpad);
  VX_CHECK_LAUNCH("patchify launch");
  return VX_OK;
}

extern "C" int vx_special_tokens(float* x, const float* tokens, int S, int tpf, int ntok, int C, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(x && tokens && S > 0 && ntok <= tpf, "vx_special_tokens: bad args");
  const int64_t total = (int64_t)S * ntok * C;
  const int grid = int((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  special_tokens_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, tokens, S, tpf, ntok, C);
  VX_CHECK_LAUNCH("special tokens launch");
  return VX_OK;
}
