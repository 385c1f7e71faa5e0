// DPT-head HBM-bound kernels: bilinear (align_corners=True) resampling of NHWC bf16
// feature maps with an optional fused add (positional embedding / skip).
// Replaces F.interpolate(..., mode="bilinear", align_corners=True) + add in the upstream
// DPTHead / FeatureFusionBlock.
#include "../../include/vx_api.h"
#include "common.cuh"
#include "host_util.h"

namespace vx {

// grid: (ceil(W * C/(8*V) / 256), F, H); each thread V 16-byte channel chunks of one output pixel
// (V = 2 when C % 16 == 0: half the index / weight math per byte). Row weights are per block.
// Frames vary faster than rows, so one output row of the shared add table (the DPT pos-embed) is
// read from DRAM once and served from L2 to every frame (frame-major order re-read the whole
// 518^2 x 128 table per frame: 1.44 GB of DRAM reads per 16-frame resize for 0.43 GB of input).
template <int V>
__global__ void __launch_bounds__(256) upsample_bilinear_nhwc_kernel(
    const __nv_bfloat16* __restrict__ in, int h, int w, int C, __nv_bfloat16* __restrict__ out, int H, int W,
    const __nv_bfloat16* __restrict__ add_hwc, float sy, float sx, int out_pad) {
  const int cv = C / (8 * V);
  const int f = blockIdx.y, y = blockIdx.z;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= W * cv) return;
  const int x = t / cv, c8 = (t - x * cv) * V;
  // PyTorch area_pixel_compute_source_index with align_corners=True
  const float fy = sy * y, fx = sx * x;
  const int y0 = int(fy), x0 = int(fx);
  const int y1 = y0 + (y0 < h - 1 ? 1 : 0), x1 = x0 + (x0 < w - 1 ? 1 : 0);
  const float ly = fy - y0, lx = fx - x0;
  const float w00 = (1.f - ly) * (1.f - lx), w01 = (1.f - ly) * lx, w10 = ly * (1.f - lx), w11 = ly * lx;
  const __nv_bfloat16* base = in + (int64_t)f * h * w * C + c8 * 8;
  const uint4* pa = reinterpret_cast<const uint4*>(base + ((int64_t)y0 * w + x0) * C);
  const uint4* pb = reinterpret_cast<const uint4*>(base + ((int64_t)y0 * w + x1) * C);
  const uint4* pc = reinterpret_cast<const uint4*>(base + ((int64_t)y1 * w + x0) * C);
  const uint4* pd = reinterpret_cast<const uint4*>(base + ((int64_t)y1 * w + x1) * C);
  uint4 a[V], b[V], c[V], d[V], ad[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    a[v] = __ldg(pa + v);
    b[v] = __ldg(pb + v);
    c[v] = __ldg(pc + v);
    d[v] = __ldg(pd + v);
  }
  if (add_hwc) {
    const uint4* pe = reinterpret_cast<const uint4*>(add_hwc + ((int64_t)y * W + x) * C + c8 * 8);
#pragma unroll
    for (int v = 0; v < V; ++v) ad[v] = __ldg(pe + v);
  }
  const int64_t opix = out_pad ? ((int64_t)(f * (H + 2) + y + 1) * (W + 2) + x + 1) : (((int64_t)f * H + y) * W + x);
  uint4* po = reinterpret_cast<uint4*>(out + opix * C + c8 * 8);
  // packed fp32x2 arithmetic (FFMA2): a bf16x2 word widens with one shift / mask per half, the 4-tap
  // sum is one FMUL2 + three FFMA2 per channel pair, in the scalar expression's order
  const uint64_t W00 = f2_pack(w00, w00), W01 = f2_pack(w01, w01), W10 = f2_pack(w10, w10), W11 = f2_pack(w11, w11);
  auto widen = [](uint32_t x) { return f2_pack(__uint_as_float(x << 16), __uint_as_float(x & 0xffff0000u)); };
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const uint32_t* a2 = reinterpret_cast<const uint32_t*>(&a[v]);
    const uint32_t* b2 = reinterpret_cast<const uint32_t*>(&b[v]);
    const uint32_t* c2 = reinterpret_cast<const uint32_t*>(&c[v]);
    const uint32_t* d2 = reinterpret_cast<const uint32_t*>(&d[v]);
    const uint32_t* e2 = reinterpret_cast<const uint32_t*>(&ad[v]);
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint64_t t = f2_mul(widen(a2[k]), W00);
      t = f2_fma(widen(b2[k]), W01, t);
      t = f2_fma(widen(c2[k]), W10, t);
      t = f2_fma(widen(d2[k]), W11, t);
      float t0, t1;
      f2_unpack(t, t0, t1);
      const uint32_t r = pack_bf16(t0, t1);  // interpolated value rounded to bf16 like the library op
      if (add_hwc) {
        float u0, u1;
        f2_unpack(f2_add(widen(r), widen(e2[k])), u0, u1);
        o[k] = pack_bf16(u0, u1);
      } else {
        o[k] = r;
      }
    }
    po[v] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace vx

extern "C" int vx_upsample_bilinear(const void* in, int F, int h, int w, int C, void* out, int H, int W,
                                    const void* add_hwc, int out_pad, void* stream) {
  using namespace vx;
  VX_CHECK_ARG(in && out && F > 0 && h > 0 && w > 0 && H > 0 && W > 0, "vx_upsample_bilinear: bad args");
  VX_CHECK_ARG(C % 8 == 0, "vx_upsample_bilinear: C=%d must be a multiple of 8", C);
  const float sy = H > 1 ? float(h - 1) / float(H - 1) : 0.f;
  const float sx = W > 1 ? float(w - 1) / float(W - 1) : 0.f;
  VX_CHECK_ARG(H < 65536 && F < 65536, "vx_upsample_bilinear: grid too large");
  const auto* pin = reinterpret_cast<const __nv_bfloat16*>(in);
  auto* pout = reinterpret_cast<__nv_bfloat16*>(out);
  const auto* padd = reinterpret_cast<const __nv_bfloat16*>(add_hwc);
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (C % 16 == 0) {
    const dim3 grid((W * (C / 16) + 255) / 256, F, H);
    upsample_bilinear_nhwc_kernel<2><<<grid, 256, 0, st>>>(pin, h, w, C, pout, H, W, padd, sy, sx, out_pad);
  } else {
    const dim3 grid((W * (C / 8) + 255) / 256, F, H);
    upsample_bilinear_nhwc_kernel<1><<<grid, 256, 0, st>>>(pin, h, w, C, pout, H, W, padd, sy, sx, out_pad);
  }
  VX_CHECK_LAUNCH("upsample launch");
  return VX_OK;
}
