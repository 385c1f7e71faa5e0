// DPT-head HBM-bound kernels: bilinear (align_corners=True) resampling of NHWC bf16
// feature maps with an optional fused add (positional embedding / skip).
// Replaces F.interpolate(..., mode="bilinear", align_corners=True) + add in the upstream
// DPTHead / FeatureFusionBlock.
#include "../../include/vx_api.h"
#include "common.cuh"
#include "host_util.h"

namespace vx {

// grid: (ceil(W * C/8 / 256), H, F); each thread one 16-byte channel chunk of one output pixel.
// Row weights are per block, so the per-element index math is one div/mod by C/8.
__global__ void __launch_bounds__(256) upsample_bilinear_nhwc_kernel(
    const __nv_bfloat16* __restrict__ in, int h, int w, int C, __nv_bfloat16* __restrict__ out, int H, int W,
    const __nv_bfloat16* __restrict__ add_hwc, float sy, float sx, int out_pad) {
  const int cv = C >> 3;
  const int y = blockIdx.y, f = blockIdx.z;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= W * cv) return;
  const int x = t / cv, c8 = t - x * cv;
  // PyTorch area_pixel_compute_source_index with align_corners=True
  const float fy = sy * y, fx = sx * x;
  const int y0 = int(fy), x0 = int(fx);
  const int y1 = y0 + (y0 < h - 1 ? 1 : 0), x1 = x0 + (x0 < w - 1 ? 1 : 0);
  const float ly = fy - y0, lx = fx - x0;
  const float w00 = (1.f - ly) * (1.f - lx), w01 = (1.f - ly) * lx, w10 = ly * (1.f - lx), w11 = ly * lx;
  const __nv_bfloat16* base = in + (int64_t)f * h * w * C + c8 * 8;
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(base + ((int64_t)y0 * w + x0) * C));
  const uint4 b = __ldg(reinterpret_cast<const uint4*>(base + ((int64_t)y0 * w + x1) * C));
  const uint4 c = __ldg(reinterpret_cast<const uint4*>(base + ((int64_t)y1 * w + x0) * C));
  const uint4 d = __ldg(reinterpret_cast<const uint4*>(base + ((int64_t)y1 * w + x1) * C));
  const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
  const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c);
  const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&d);
  float2 e[4] = {};
  if (add_hwc) {
    const uint4 ad = __ldg(reinterpret_cast<const uint4*>(add_hwc + ((int64_t)y * W + x) * C + c8 * 8));
    const __nv_bfloat162* ad2 = reinterpret_cast<const __nv_bfloat162*>(&ad);
#pragma unroll
    for (int k = 0; k < 4; ++k) e[k] = __bfloat1622float2(ad2[k]);
  }
  uint32_t o[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 fa = __bfloat1622float2(a2[k]), fb = __bfloat1622float2(b2[k]);
    const float2 fc = __bfloat1622float2(c2[k]), fd = __bfloat1622float2(d2[k]);
    // interpolate (rounded to bf16 like the library op), then add
    const float v0 = __bfloat162float(__float2bfloat16_rn(w00 * fa.x + w01 * fb.x + w10 * fc.x + w11 * fd.x));
    const float v1 = __bfloat162float(__float2bfloat16_rn(w00 * fa.y + w01 * fb.y + w10 * fc.y + w11 * fd.y));
    o[k] = pack_bf16(v0 + e[k].x, v1 + e[k].y);
  }
  const int64_t opix = out_pad ? ((int64_t)(f * (H + 2) + y + 1) * (W + 2) + x + 1) : (((int64_t)f * H + y) * W + x);
  *reinterpret_cast<uint4*>(out + opix * C + c8 * 8) = make_uint4(o[0], o[1], o[2], o[3]);
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
  const dim3 grid((W * (C / 8) + 255) / 256, H, F);
  upsample_bilinear_nhwc_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(in), h, w, C, reinterpret_cast<__nv_bfloat16*>(out), H, W,
      reinterpret_cast<const __nv_bfloat16*>(add_hwc), sy, sx, out_pad);
  VX_CHECK_LAUNCH("upsample launch");
  return VX_OK;
}
