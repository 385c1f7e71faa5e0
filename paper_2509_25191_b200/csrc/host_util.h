// Host-side helpers: error reporting across the C ABI and TMA tensor-map encoding.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

namespace vx {

void set_error(const char* fmt, ...);
int fail_cuda(cudaError_t e, const char* where);
int num_sms();
// kernels launched by this library (vx_launch_count); graph replays count their kernel nodes
void count_launches(uint64_t n);

// 2D row-major bf16 tensor [rows, cols] with row stride `ld` elements, box [box_rows, box_cols].
// swizzle_bytes in {0, 32, 64, 128}.
bool make_tmap_2d_bf16(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld,
                       uint32_t box_rows, uint32_t box_cols, int swizzle_bytes);
// same for bf16 (f32 = false) or fp32 (f32 = true) elements
bool make_tmap_2d(CUtensorMap* m, const void* ptr, bool f32, uint64_t rows, uint64_t cols, uint64_t ld,
                  uint32_t box_rows, uint32_t box_cols, int swizzle_bytes);

}  // namespace vx

#define VX_CHECK_ARG(cond, ...)       \
  do {                                \
    if (!(cond)) {                    \
      vx::set_error(__VA_ARGS__);     \
      return VX_E_ARG;                \
    }                                 \
  } while (0)

// after every launch site: n = kernels launched since the previous check
#define VX_CHECK_LAUNCH_N(where, n)                         \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return vx::fail_cuda(_e, where); \
    vx::count_launches(n);                                  \
  } while (0)
#define VX_CHECK_LAUNCH(where) VX_CHECK_LAUNCH_N(where, 1)
