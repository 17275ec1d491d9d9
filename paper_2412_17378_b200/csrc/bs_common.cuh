// bs_common.cuh — shared device helpers for the B200 forward rasterizer.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#include "splatsim_b200.h"

#define BS_CUDA_TRY(expr)                              \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return BS_ERR_CUDA;         \
  } while (0)

#define TRY_BS(expr)                                   \
  do {                                                 \
    const int _s = (expr);                             \
    if (_s != BS_OK) return _s;                        \
  } while (0)

#define BS_LAUNCH_CHECK()                              \
  do {                                                 \
    bs::count_launches(1);                             \
    if (cudaPeekAtLastError() != cudaSuccess) {        \
      (void)cudaGetLastError();                        \
      return BS_ERR_CUDA;                              \
    }                                                  \
  } while (0)

namespace bs {

// Programmatic dependent launch (PDL): every kernel is launched with
// programmatic stream serialization and waits (griddepcontrol.wait) for its
// stream predecessor before touching memory, so a kernel's CTAs are
// scheduled — and run up to the wait — while the previous kernel drains (in
// streams and in the frame pipeline's CUDA graphs).  The wait is a no-op for
// kernels launched without the attribute.  BS_PDL=0 disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
inline bool pdl_enabled() {
  static const bool v = [] {
    const char* e = getenv("BS_PDL");
    return !(e && e[0] == '0');
  }();
  return v;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Library-wide kernel launch counter (bs_kernel_launches()).
void count_launches(unsigned long long n);

constexpr float kNearPlane = 0.01f;           // preprocess.hpp:47
constexpr float kAlphaClamp = 0.99f;          // blend.hpp:13
constexpr float kAlphaSkip = 1.0f / 255.0f;   // blend.hpp:14
constexpr float kStopThreshold = 1e-4f;       // blend.hpp:15

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over a caller workspace (all carve-outs 256-byte aligned).
struct WsCarver {
  char* base;
  size_t cap;
  size_t off = 0;
  bool ok = true;
  WsCarver(void* p, size_t c) : base(static_cast<char*>(p)), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += count * sizeof(T);
    if (off > cap) ok = false;
    return p;
  }
};

// Size-only variant of the carver (same layout rules; returns nullptr).
struct WsSizer {
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = align_up(off, 256);
    off += count * sizeof(T);
    return nullptr;
  }
};

// Per-frame variant predictor, shared by the host entry point
// bs_select_variant and the device-side selection of the sync-free pipeline.
// With L_t the list length of tile t, a static one-CTA-per-tile launch
// finishes no earlier than the heaviest tile (L_max) and no earlier than the
// balanced share sum(L)/(S*k) of S SMs with k resident tile-CTAs each; the
// fine-grained queue removes the first bound and (sub-tile culling) does less
// work per list entry, at a fixed queue/launch cost:
//   t_static ~ max(L_max, sum(L)/(S*k)),   t_fine ~ rho * sum(L)/(S*k) + c0
// FineGrainedCombined when t_static > t_fine, else SharedMemOpt (the
// selector's fallback, src/adaptive.cpp:27-28).  rho = 0.75 and c0 = 64 list
// entries are the B200 calibration from the C3 sweep (profiles/r1_c3_*.jsonl).
// Short lists: below kShortList entries per tile on average the fine-grained
// kernel's fixed per-task cost (queue claim, per-batch cull and compaction,
// 8 tasks per 16x16 tile) outweighs any balance it buys — the r2 selector
// sweep (profiles/r2_selector_sweep.jsonl) measured SharedMemOpt 10-40 %
// faster at every point with a mean list of <= 6 entries, FG faster from
// ~22 up (ties near 14).
constexpr double kShortList = 12.0;
__host__ __device__ inline int select_variant_formula(uint64_t total, uint32_t max_len, int32_t tiles, int pw, int ph,
                                                      int sm_count) {
  if (tiles > 0 && (double)total < kShortList * (double)tiles) return BS_SHARED_MEM_OPT;
  const double S = sm_count > 0 ? (double)sm_count : 148.0;
  const int pixels = pw * ph;
  const double k = pixels <= 128 ? 12.0 : (pixels <= 256 ? 6.0 : 3.0);  // resident tile CTAs per SM
  const double rho = 0.75, c0 = 64.0;
  const double balanced = (double)total / (S * k);
  const double t_static = fmax((double)max_len, balanced);
  const double t_fine = rho * balanced + c0;
  return t_static > t_fine ? BS_FINE_GRAINED_COMBINED : BS_SHARED_MEM_OPT;
}

// Sortable key of a float under operator< (ties -0 == +0 collapse).
__device__ __forceinline__ uint32_t float_sort_key(float f) {
  if (f == 0.0f) f = 0.0f;  // -0 -> +0
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace bs
