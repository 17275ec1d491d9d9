// tiles.cuh — the tile grid and S8's tile rectangle (src/preprocess.cpp:81-92),
// shared by binning.cu and the fused project+rect kernel in preprocess.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "bs_common.cuh"

namespace bs {

struct Grid {
  int W, H, pw, ph, cols, rows;
};

// static_cast<int>(float) with x86-64 cvttss2si semantics (out of range /
// NaN -> INT_MIN), the behaviour of the reference's casts on its platform.
__device__ __forceinline__ int x86_f2i(float f) {
  if (!(f > -2147483904.0f && f < 2147483648.0f)) return (int)0x80000000;
  return (int)f;
}

struct Rect {
  int tx0, tx1, ty0, ty1;
};

// x / p for the patch size p: a multiply by 1/p when p is a power of two
// (both round the same exact value x * 2^-k, so the bits are identical), an
// IEEE division otherwise.
__device__ __forceinline__ float div_patch(float x, int p) {
  if ((p & (p - 1)) == 0) return __fmul_rn(x, __uint_as_float((uint32_t)(127 - (31 - __clz(p))) << 23));
  return __fdiv_rn(x, (float)p);
}

// src/preprocess.cpp:81-92.  Returns false when rejected / empty.
__device__ __forceinline__ bool tile_rect(float x, float y, float radius, const Grid& g, Rect& r) {
  const float rr = ceilf(radius);
  const float x0 = __fsub_rn(x, rr), x1 = __fadd_rn(x, rr);
  const float y0 = __fsub_rn(y, rr), y1 = __fadd_rn(y, rr);
  if (x1 < 0.0f || y1 < 0.0f || x0 >= (float)g.W || y0 >= (float)g.H) return false;
  r.tx0 = max(0, x86_f2i(floorf(div_patch(x0, g.pw))));
  r.tx1 = min(g.cols - 1, x86_f2i(floorf(div_patch(x1, g.pw))));
  r.ty0 = max(0, x86_f2i(floorf(div_patch(y0, g.ph))));
  r.ty1 = min(g.rows - 1, x86_f2i(floorf(div_patch(y1, g.ph))));
  return r.tx0 <= r.tx1 && r.ty0 <= r.ty1;
}

// The project+rect kernel (preprocess.cu) for the frame pipeline: splat i
// stays at index i (no compaction; culled splats touch no tile), and the
// per-splat binning inputs of k_bin_rect are written in the same pass.
// counts[0] <- n (the item count the binning kernels read), counts[1] +=
// visible splats (caller zeroes it).
cudaError_t launch_project_bin(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam, const bs_camera* cam_dev,
                               const Grid& g, float4* xyab, float4* cop, float4* rgbr, uint32_t* touched,
                               uint2* rects, uint32_t* dkeys, uint32_t* dvals, int* diff, size_t diff_bytes,
                               bool smem_diff, int32_t* counts, cudaStream_t st, const Grid* g2 = nullptr,
                               int* diff2 = nullptr);

}  // namespace bs
