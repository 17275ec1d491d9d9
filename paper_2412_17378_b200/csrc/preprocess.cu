// preprocess.cu — P1-P4: EWA projection + order-preserving compaction.
//
// Compiled with --fmad=false: every float/double expression below rounds
// after each operation exactly like the reference built with
// -ffp-contract=off (/root/reference/proj/CMakeLists.txt:11-12).  The
// evaluation order is the oracle's documented Eigen 3.4 order
// (oracle/oracle.cpp covariance_of / project_covariance / project_gaussian):
// 3x3 float products reduce a0 + (a1 + a2); 2-row double products sum
// left to right.
//
// Layout: input AoS bs_gaussian3d (56 B, read once, 16 B-aligned rows are not
// guaranteed so it is read as 14 scalar floats: a warp touches 1792
// contiguous bytes, fully coalesced at sector granularity).  Output SoA of
// float4 (bs_splats).  HBM-bound: 56 B in + 48 B out per Gaussian.
#include <math.h>

#include "bs_common.cuh"
#include "scan.cuh"
#include "tiles.cuh"

namespace bs {

struct CamDev {
  float v[12];  // rows 0..2 of the row-major 4x4 view
  float fx, fy;
  int w, h;
};

struct Projected {
  float x, y, ca, cb, cc, depth, radius;
};

// src/scene.cpp:67-71 (see oracle covariance_of for the order).
__device__ __forceinline__ void covariance_of(const float* rot, const float* scale, float S[3][3]) {
  float qw = rot[0], qx = rot[1], qy = rot[2], qz = rot[3];
  const float n2 = (qx * qx + qz * qz) + (qy * qy + qw * qw);
  if (n2 > 0.0f) {
    const float n = __fsqrt_rn(n2);
    qx = __fdiv_rn(qx, n); qy = __fdiv_rn(qy, n); qz = __fdiv_rn(qz, n); qw = __fdiv_rn(qw, n);
  }
  const float tx = 2.0f * qx, ty = 2.0f * qy, tz = 2.0f * qz;
  const float twx = tx * qw, twy = ty * qw, twz = tz * qw;
  const float txx = tx * qx, txy = ty * qx, txz = tz * qx;
  const float tyy = ty * qy, tyz = tz * qy, tzz = tz * qz;
  float r[3][3];
  r[0][0] = 1.0f - (tyy + tzz); r[0][1] = txy - twz;          r[0][2] = txz + twy;
  r[1][0] = txy + twz;          r[1][1] = 1.0f - (txx + tzz); r[1][2] = tyz - twx;
  r[2][0] = txz - twy;          r[2][1] = tyz + twx;          r[2][2] = 1.0f - (txx + tyy);
  float m[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) m[i][j] = r[i][j] * scale[j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) S[i][j] = m[i][0] * m[j][0] + (m[i][1] * m[j][1] + m[i][2] * m[j][2]);
}

// src/preprocess.cpp:17-55.  Returns false when culled.
__device__ __forceinline__ bool project_one(const bs_gaussian3d& g, const CamDev& cam, Projected& o) {
  const float* V = cam.v;
  float p[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    p[i] = (V[i * 4 + 0] * g.mean[0] + (V[i * 4 + 1] * g.mean[1] + V[i * 4 + 2] * g.mean[2])) + V[i * 4 + 3];
  if (!(p[2] > kNearPlane)) return false;

  const double x = p[0], y = p[1], z = p[2];
  const double fx = cam.fx, fy = cam.fy;
  const double zz = z * z;
  const double jac[2][3] = {{fx / z, 0.0, -fx * x / zz}, {0.0, fy / z, -fy * y / zz}};
  float Sf[3][3];
  covariance_of(g.rot, g.scale, Sf);
  double t[2][3], u[2][3], c[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      t[i][j] = (jac[i][0] * (double)V[0 * 4 + j] + jac[i][1] * (double)V[1 * 4 + j]) + jac[i][2] * (double)V[2 * 4 + j];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      u[i][j] = (t[i][0] * (double)Sf[0][j] + t[i][1] * (double)Sf[1][j]) + t[i][2] * (double)Sf[2][j];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) c[i][j] = (u[i][0] * t[j][0] + u[i][1] * t[j][1]) + u[i][2] * t[j][2];

  const double det = c[0][0] * c[1][1] - c[0][1] * c[1][0];
  if (!(det > 0.0) || !isfinite(det)) return false;
  const double mid = 0.5 * (c[0][0] + c[1][1]);
  const double lambda_max = mid + sqrt(fmax(0.0, mid * mid - det));
  if (!(lambda_max > 0.0)) return false;

  o.x = (float)(fx * x / z) + 0.5f * (float)cam.w;
  o.y = (float)(fy * y / z) + 0.5f * (float)cam.h;
  o.ca = (float)(c[1][1] / det);
  o.cb = (float)(-c[0][1] / det);
  o.cc = (float)(c[0][0] / det);
  o.depth = (float)z;
  o.radius = (float)(3.0 * sqrt(lambda_max));
  if (!isfinite(o.ca) || !isfinite(o.cb) || !isfinite(o.cc) || !isfinite(o.radius)) return false;
  return true;
}

// power < cut  =>  opacity * expf(power) < 1/255 (1% margin in the exponent,
// far above every rounding error), so the exact exp can be skipped without
// changing a single decision.  opacity <= 0 -> everything skips.
// The cut is also clamped at glibc expf's underflow bound (x < -0x1.9fe368p6
// -> expf(x) = 0 -> alpha 0 -> skip), so the render path only ever evaluates
// the exact exp on [-103.97, 0] and needs no range guard.
__device__ __forceinline__ float power_cut_of(float opacity) {
  if (!(opacity > 0.0f)) return INFINITY;
  return fmaxf(logf(1.0f / (255.0f * opacity)) - 0.01f, -0x1.9fe368p6f);
}

__device__ __forceinline__ void load_g3d(const bs_gaussian3d* __restrict__ src, int64_t i, bs_gaussian3d& g) {
  const float* s = reinterpret_cast<const float*>(src + i);
  float* d = reinterpret_cast<float*>(&g);
#pragma unroll
  for (int k = 0; k < 14; ++k) d[k] = __ldg(s + k);
}

// camera from device memory (CUDA-graph replays of the frame pipeline read a
// per-frame camera the host copies in ahead of the launch)
__device__ __forceinline__ CamDev cam_of(const bs_camera* __restrict__ camd, const CamDev& cam) {
  if (!camd) return cam;
  CamDev c;
#pragma unroll
  for (int k = 0; k < 12; ++k) c.v[k] = __ldg(&camd->view[k]);
  c.fx = __ldg(&camd->focal[0]);
  c.fy = __ldg(&camd->focal[1]);
  c.w = __ldg(&camd->width);
  c.h = __ldg(&camd->height);
  return c;
}

__global__ void __launch_bounds__(256) k_project_flags(const bs_gaussian3d* __restrict__ g3d, int64_t n, CamDev cam_,
                                                       const bs_camera* __restrict__ camd,
                                                       uint32_t* __restrict__ block_counts) {
  bs::pdl_wait();
  const CamDev cam = cam_of(camd, cam_);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool vis = false;
  if (i < n) {
    bs_gaussian3d g;
    load_g3d(g3d, i, g);
    Projected o;
    vis = project_one(g, cam, o);
  }
  const int cnt = __syncthreads_count(vis);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = (uint32_t)cnt;
}

__global__ void __launch_bounds__(256) k_project_write(const bs_gaussian3d* __restrict__ g3d, int64_t n, CamDev cam_,
                                                       const bs_camera* __restrict__ camd,
                                                       const uint32_t* __restrict__ block_offsets, float4* __restrict__ xyab,
                                                       float4* __restrict__ cop, float4* __restrict__ rgbr) {
  bs::pdl_wait();
  const CamDev cam = cam_of(camd, cam_);
  __shared__ uint32_t warp_counts[8];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bs_gaussian3d g;
  Projected o;
  bool vis = false;
  if (i < n) {
    load_g3d(g3d, i, g);
    vis = project_one(g, cam, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ballot = __ballot_sync(0xffffffffu, vis);
  if (lane == 0) warp_counts[warp] = __popc(ballot);
  __syncthreads();
  uint32_t before = 0;
  for (int w = 0; w < warp; ++w) before += warp_counts[w];
  if (vis) {
    const uint32_t dst = block_offsets[blockIdx.x] + before + __popc(ballot & lanemask_lt());
    xyab[dst] = make_float4(o.x, o.y, o.ca, o.cb);
    cop[dst] = make_float4(o.cc, g.opacity, power_cut_of(g.opacity), o.depth);
    rgbr[dst] = make_float4(g.color[0], g.color[1], g.color[2], o.radius);
  }
}

// Frame-pipeline form of P1-P4 + the per-splat half of P5 in one pass:
// splat i is projected once, its float4 triple written at index i (culled
// splats write nothing and touch no tile), and k_bin_rect's outputs (tiles
// touched, packed rect, depth key, index, difference-grid corners) follow
// from the registers.  Tie order is unchanged: the compacted index of the
// reference is a monotone function of i.  SMEM_DIFF as in k_bin_rect.
// DIFF2: a second difference grid at grid g2 (the pw x ph tiles when the
// binning grid g is the 2pw x 2ph super-tile grid): its list lengths feed the
// tile statistics, the LPT order and the selector.  SMEM2: that grid too in
// shared memory (after the first), else global atomics.
// cp.async staging of the Gaussian chunks (k_project_bin)
constexpr int kStageBytes = 256 * (int)sizeof(bs_gaussian3d);  // 14,336
__host__ __device__ constexpr size_t kStageOff(int cells) { return ((size_t)cells * sizeof(int) + 15) & ~(size_t)15; }
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// (256, 2): 124 registers, no spills, 2 CTAs/SM — the 3-CTA budget (80
// registers) spilled 12-36 bytes and measured ~1 us slower per C2 frame
template <bool SMEM_DIFF, bool DIFF2, bool SMEM2>
__global__ void __launch_bounds__(256, 2) k_project_bin(const bs_gaussian3d* __restrict__ g3d, int64_t n, CamDev cam_,
                                                     const bs_camera* __restrict__ camd, Grid g,
                                                     float4* __restrict__ xyab, float4* __restrict__ cop,
                                                     float4* __restrict__ rgbr, uint32_t* __restrict__ touched,
                                                     uint2* __restrict__ rects, uint32_t* __restrict__ dkeys,
                                                     uint32_t* __restrict__ dvals, int* __restrict__ diff,
                                                     int32_t* __restrict__ counts, Grid g2, int* __restrict__ diff2,
                                                     bool staged) {
  bs::pdl_wait();
  extern __shared__ int s_diff[];
  const CamDev cam = cam_of(camd, cam_);
  const int stride = g.cols + 1;
  const int cells = stride * (g.rows + 1);
  const int stride2 = g2.cols + 1;
  const int cells2 = DIFF2 ? stride2 * (g2.rows + 1) : 0;
  int* dd = SMEM_DIFF ? s_diff : diff;
  int* dd2 = SMEM2 ? s_diff + cells : diff2;
  if (SMEM_DIFF) {
    for (int i = threadIdx.x; i < cells + (SMEM2 ? cells2 : 0); i += blockDim.x) s_diff[i] = 0;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[0] = (int32_t)n;
  int vis_n = 0;
  auto project = [&](int64_t i, const bs_gaussian3d& gs) {
      Projected o;
      uint32_t cnt = 0;
      uint2 pk = make_uint2(0u, 0u);
      if (project_one(gs, cam, o)) {
        ++vis_n;
        xyab[i] = make_float4(o.x, o.y, o.ca, o.cb);
        cop[i] = make_float4(o.cc, gs.opacity, power_cut_of(gs.opacity), o.depth);
        rgbr[i] = make_float4(gs.color[0], gs.color[1], gs.color[2], o.radius);
        Rect r;
        if (tile_rect(o.x, o.y, o.radius, g, r)) {
          const uint32_t w = (uint32_t)(r.tx1 - r.tx0 + 1), h = (uint32_t)(r.ty1 - r.ty0 + 1);
          cnt = w * h;
          pk = make_uint2((uint32_t)r.tx0 | ((uint32_t)r.ty0 << 16), w | (h << 16));
          atomicAdd(&dd[r.ty0 * stride + r.tx0], 1);
          atomicAdd(&dd[r.ty0 * stride + r.tx1 + 1], -1);
          atomicAdd(&dd[(r.ty1 + 1) * stride + r.tx0], -1);
          atomicAdd(&dd[(r.ty1 + 1) * stride + r.tx1 + 1], 1);
        }
        if (DIFF2) {
          Rect r2;
          if (tile_rect(o.x, o.y, o.radius, g2, r2)) {
            atomicAdd(&dd2[r2.ty0 * stride2 + r2.tx0], 1);
            atomicAdd(&dd2[r2.ty0 * stride2 + r2.tx1 + 1], -1);
            atomicAdd(&dd2[(r2.ty1 + 1) * stride2 + r2.tx0], -1);
            atomicAdd(&dd2[(r2.ty1 + 1) * stride2 + r2.tx1 + 1], 1);
          }
        }
      }
      touched[i] = cnt;
      rects[i] = pk;
      dkeys[i] = cnt ? float_sort_key(o.depth) : 0xffffffffu;
      dvals[i] = (uint32_t)i;
  };
  if (SMEM_DIFF && staged) {  // (staged: g3d 16-byte aligned, as cp.async needs)
    // grid-stride over 256-Gaussian chunks staged through shared memory:
    // the chunk's 14 KB arrive by coalesced 16-byte cp.async copies, double
    // buffered (the next chunk in flight while this one is projected), and
    // each thread reads its Gaussian from smem (stride 56 B: conflict-free
    // 8-byte loads) instead of 14 scattered 4-byte global loads
    char* const stage = reinterpret_cast<char*>(s_diff) + kStageOff(cells + (SMEM2 ? cells2 : 0));
    const int64_t chunks = (n + 255) / 256;
    auto issue = [&](int64_t ch, int buf) {
      const char* src = reinterpret_cast<const char*>(g3d + ch * 256);
      const int bytes = (int)(min((int64_t)256, n - ch * 256) * (int64_t)sizeof(bs_gaussian3d));
      char* dst = stage + buf * kStageBytes;
      for (int q = threadIdx.x; q * 16 < bytes; q += blockDim.x) {
        if (q * 16 + 16 <= bytes) cp_async16(dst + q * 16, src + q * 16);
        else cp_async8(dst + q * 16, src + q * 16);  // (bytes is a multiple of 8)
      }
      cp_async_commit();
    };
    int buf = 0;
    int64_t ch = blockIdx.x;
    if (ch < chunks) issue(ch, 0);
    for (; ch < chunks; ch += gridDim.x) {
      const int64_t nx = ch + gridDim.x;
      if (nx < chunks) {
        issue(nx, buf ^ 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const int64_t i = ch * 256 + threadIdx.x;
      if (i < n) {
        const float2* sp =
            reinterpret_cast<const float2*>(stage + buf * kStageBytes + threadIdx.x * sizeof(bs_gaussian3d));
        float2 v[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) v[k] = sp[k];
        bs_gaussian3d gs;
        memcpy(&gs, v, sizeof(gs));
        project(i, gs);
      }
      __syncthreads();  // the buffer is refilled two chunks later
      buf ^= 1;
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      bs_gaussian3d gs;
      load_g3d(g3d, i, gs);
      project(i, gs);
    }
  }
  const int tot = block_reduce_sum<int>(vis_n);
  if (threadIdx.x == 0 && tot) atomicAdd(&counts[1], tot);
  if (SMEM_DIFF) {
    __syncthreads();
    for (int i = threadIdx.x; i < cells; i += blockDim.x) {
      const int v = s_diff[i];
      if (v) atomicAdd(&diff[i], v);
    }
    if (SMEM2)
      for (int i = threadIdx.x; i < cells2; i += blockDim.x) {
        const int v = s_diff[cells + i];
        if (v) atomicAdd(&diff2[i], v);
      }
  }
}

cudaError_t launch_project_bin(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam, const bs_camera* cam_dev,
                               const Grid& g, float4* xyab, float4* cop, float4* rgbr, uint32_t* touched,
                               uint2* rects, uint32_t* dkeys, uint32_t* dvals, int* diff, size_t diff_bytes,
                               bool smem_diff, int32_t* counts, cudaStream_t st, const Grid* g2, int* diff2) {
  CamDev c{};
  if (cam) {
    for (int k = 0; k < 12; ++k) c.v[k] = cam->view[k];
    c.fx = cam->focal[0];
    c.fy = cam->focal[1];
    c.w = cam->width;
    c.h = cam->height;
  }
  const bs_camera* camd = cam ? nullptr : cam_dev;
  const int64_t nb = (n + 255) / 256;
  const Grid gg2 = g2 ? *g2 : g;
  const size_t diff2_bytes = g2 ? sizeof(int) * (size_t)(g2->cols + 1) * (g2->rows + 1) : 0;
  const bool smem2 = g2 && smem_diff && diff_bytes + diff2_bytes <= (size_t)64 * 1024;
  if (smem_diff) {
    const size_t sm = kStageOff((int)((diff_bytes + (smem2 ? diff2_bytes : 0)) / sizeof(int))) + 2 * (size_t)kStageBytes;
    // one kernel per combination; per-combination occupancy cached
    auto go = [&](auto kern) -> cudaError_t {
      static size_t attr_bytes[4] = {0, 0, 0, 0};
      static int per_sm[4] = {0, 0, 0, 0};
      const int slot = (g2 ? 1 : 0) + (smem2 ? 2 : 0);
      if (sm > attr_bytes[slot]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        attr_bytes[slot] = sm;
        per_sm[slot] = 0;
      }
      static int sms = 0;
      if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      }
      if (!per_sm[slot]) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[slot], kern, 256, sm);
        per_sm[slot] = per_sm[slot] < 1 ? 1 : (per_sm[slot] > 3 ? 3 : per_sm[slot]);  // each CTA flushes once
      }
      const int64_t grid = nb < (int64_t)sms * per_sm[slot] ? nb : (int64_t)sms * per_sm[slot];
      bs::launch_pdl(kern, (unsigned)(grid > 0 ? grid : 1), 256, sm, st, g3d, n, c, camd, g, xyab, cop, rgbr, touched, rects,
                                                             dkeys, dvals, diff, counts, gg2, diff2,
                                                             (reinterpret_cast<uintptr_t>(g3d) & 15) == 0);
      return cudaSuccess;
    };
    cudaError_t e;
    if (!g2) e = go(k_project_bin<true, false, false>);
    else if (smem2) e = go(k_project_bin<true, true, true>);
    else e = go(k_project_bin<true, true, false>);
    if (e != cudaSuccess) return e;
  } else if (g2) {
    bs::launch_pdl(k_project_bin<false, true, false>, (unsigned)(nb > 0 ? nb : 1), 256, 0, st, 
        g3d, n, c, camd, g, xyab, cop, rgbr, touched, rects, dkeys, dvals, diff, counts, gg2, diff2, false);
  } else {
    bs::launch_pdl(k_project_bin<false, false, false>, (unsigned)(nb > 0 ? nb : 1), 256, 0, st, 
        g3d, n, c, camd, g, xyab, cop, rgbr, touched, rects, dkeys, dvals, diff, counts, gg2, diff2, false);
  }
  count_launches(1);
  return cudaPeekAtLastError();
}

__global__ void k_splats_from_g2d(const bs_gaussian2d* __restrict__ g2d, int64_t n, float4* __restrict__ xyab,
                                  float4* __restrict__ cop, float4* __restrict__ rgbr) {
  bs::pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bs_gaussian2d g = g2d[i];
  xyab[i] = make_float4(g.x, g.y, g.conic_a, g.conic_b);
  cop[i] = make_float4(g.conic_c, g.opacity, power_cut_of(g.opacity), g.depth);
  rgbr[i] = make_float4(g.color[0], g.color[1], g.color[2], g.radius);
}

__global__ void k_splats_to_g2d(const float4* __restrict__ xyab, const float4* __restrict__ cop,
                                const float4* __restrict__ rgbr, int64_t n, bs_gaussian2d* __restrict__ g2d) {
  bs::pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 a = xyab[i], b = cop[i], c = rgbr[i];
  bs_gaussian2d g;
  g.x = a.x; g.y = a.y; g.conic_a = a.z; g.conic_b = a.w;
  g.conic_c = b.x; g.opacity = b.y; g.depth = b.w;
  g.color[0] = c.x; g.color[1] = c.y; g.color[2] = c.z; g.radius = c.w;
  g2d[i] = g;
}

}  // namespace bs

using namespace bs;

extern "C" size_t bs_preprocess_workspace_bytes(int64_t n) {
  const int64_t nb = (n + 255) / 256;
  WsSizer s;
  s.take<uint32_t>((size_t)nb);                   // block counts -> offsets
  s.take<uint32_t>((size_t)scan_num_blocks(nb));  // scan partials
  return s.off + 256;
}

static int preprocess_impl(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam, const bs_camera* cam_dev,
                           bs_splats out, int32_t* n_visible, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || (!cam && !cam_dev) || !n_visible || (n > 0 && (!g3d || !out.xyab || !out.cop || !out.rgbr)))
    return BS_ERR_INVALID_ARGUMENT;
  if (n >= (int64_t)0x7fffffff) return BS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) {
    BS_CUDA_TRY(cudaMemsetAsync(n_visible, 0, sizeof(int32_t), st));
    return BS_OK;
  }
  CamDev c{};
  if (cam) {
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 4; ++k) c.v[r * 4 + k] = cam->view[r * 4 + k];
    c.fx = cam->focal[0];
    c.fy = cam->focal[1];
    c.w = cam->width;
    c.h = cam->height;
  }
  const int64_t nb = (n + 255) / 256;
  WsCarver wc(ws, ws_bytes);
  uint32_t* counts = wc.take<uint32_t>((size_t)nb);
  uint32_t* partials = wc.take<uint32_t>((size_t)scan_num_blocks(nb));
  if (!wc.ok || !ws) return BS_ERR_WORKSPACE;
  bs::launch_pdl(k_project_flags, (unsigned)nb, 256, 0, st, g3d, n, c, cam ? nullptr : cam_dev, counts);
  BS_LAUNCH_CHECK();
  // exclusive scan of block counts in place; grand total -> n_visible (u32 == i32 bits for n < 2^31)
  BS_CUDA_TRY((exclusive_scan<uint32_t, uint32_t>(counts, counts, nb, nullptr, partials,
                                                 reinterpret_cast<uint32_t*>(n_visible), st)));
  bs::launch_pdl(k_project_write, (unsigned)nb, 256, 0, st, g3d, n, c, cam ? nullptr : cam_dev, counts,
                                                reinterpret_cast<float4*>(out.xyab), reinterpret_cast<float4*>(out.cop),
                                                reinterpret_cast<float4*>(out.rgbr));
  BS_LAUNCH_CHECK();
  return BS_OK;
}

extern "C" int bs_preprocess(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam, bs_splats out,
                             int32_t* n_visible, void* ws, size_t ws_bytes, void* stream) {
  if (!cam) return BS_ERR_INVALID_ARGUMENT;
  return preprocess_impl(g3d, n, cam, nullptr, out, n_visible, ws, ws_bytes, stream);
}

extern "C" int bs_preprocess_devcam(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam_dev, bs_splats out,
                                    int32_t* n_visible, void* ws, size_t ws_bytes, void* stream) {
  if (!cam_dev) return BS_ERR_INVALID_ARGUMENT;
  return preprocess_impl(g3d, n, nullptr, cam_dev, out, n_visible, ws, ws_bytes, stream);
}

extern "C" int bs_splats_from_g2d(const bs_gaussian2d* g2d, int64_t n, bs_splats out, void* stream) {
  if (n < 0 || (n > 0 && (!g2d || !out.xyab || !out.cop || !out.rgbr))) return BS_ERR_INVALID_ARGUMENT;
  if (n == 0) return BS_OK;
  bs::launch_pdl(k_splats_from_g2d, (unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream, 
      g2d, n, reinterpret_cast<float4*>(out.xyab), reinterpret_cast<float4*>(out.cop), reinterpret_cast<float4*>(out.rgbr));
  BS_LAUNCH_CHECK();
  return BS_OK;
}

extern "C" int bs_splats_to_g2d(bs_splats in, int64_t n, bs_gaussian2d* g2d, void* stream) {
  if (n < 0 || (n > 0 && (!g2d || !in.xyab || !in.cop || !in.rgbr))) return BS_ERR_INVALID_ARGUMENT;
  if (n == 0) return BS_OK;
  bs::launch_pdl(k_splats_to_g2d, (unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream, 
      reinterpret_cast<const float4*>(in.xyab), reinterpret_cast<const float4*>(in.cop),
      reinterpret_cast<const float4*>(in.rgbr), n, g2d);
  BS_LAUNCH_CHECK();
  return BS_OK;
}
