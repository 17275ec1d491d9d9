// capi.cu — library-level C-ABI entry points: version, status strings,
// variant names (include/splatsim/kernels.hpp:13-26, src/kernels.cpp:10-25),
// device query and the per-frame variant predictor.
#include <math.h>
#include <string.h>

#include "bs_common.cuh"

#include <atomic>

namespace bs {
static std::atomic<unsigned long long> g_launches{0};
void count_launches(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace bs

extern "C" uint64_t bs_kernel_launches(void) { return bs::g_launches.load(); }

extern "C" int bs_abi_version(void) { return BS_ABI_VERSION; }

extern "C" const char* bs_status_string(int status) {
  switch (status) {
    case BS_OK: return "ok";
    case BS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case BS_ERR_GRID_MISMATCH: return "binning grid does not match image dims";
    case BS_ERR_WORKSPACE: return "workspace too small";
    case BS_ERR_CAPACITY: return "capacity exceeded (u32 index space)";
    case BS_ERR_CUDA: return "CUDA error";
    case BS_ERR_UNSUPPORTED: return "unsupported configuration";
    case BS_ERR_LOGIC: return "selection already switched";
    case BS_ERR_NO_DEVICE: return "no CUDA device";
  }
  return "unknown status";
}

static const char* const kVariantNames[5] = {"Naive", "DynamicBlocks", "GaussianWise", "FineGrainedCombined",
                                             "SharedMemOpt"};

extern "C" const char* bs_variant_name(int variant) {
  if (variant < 0 || variant > 4) return "?";
  return kVariantNames[variant];
}

extern "C" int bs_variant_from_name(const char* name) {
  if (!name) return -1;
  for (int i = 0; i < 5; ++i)
    if (strcmp(name, kVariantNames[i]) == 0) return i;
  return -1;
}

extern "C" int bs_device_sm_count(int32_t* sm_count) {
  if (!sm_count) return BS_ERR_INVALID_ARGUMENT;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    (void)cudaGetLastError();
    return BS_ERR_NO_DEVICE;
  }
  int dev = 0, sms = 0;
  BS_CUDA_TRY(cudaGetDevice(&dev));
  BS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  *sm_count = sms;
  return BS_OK;
}

// Per-frame predictor (formula in bs_common.cuh).
extern "C" int bs_select_variant(const bs_tile_histogram* stats, int32_t width, int32_t height, int32_t pw, int32_t ph,
                                 int32_t sm_count) {
  if (!stats || width <= 0 || height <= 0 || pw <= 0 || ph <= 0) return BS_ERR_INVALID_ARGUMENT;
  return bs::select_variant_formula(stats->total, stats->max, stats->tiles, pw, ph, sm_count);
}

namespace bs {
__global__ void k_select_variant(const bs_tile_histogram* __restrict__ stats, int pw, int ph, int sm_count,
                                 int32_t* __restrict__ variant) {
  bs::pdl_wait();
  *variant = select_variant_formula(stats->total, stats->max, stats->tiles, pw, ph, sm_count);
}
}  // namespace bs

extern "C" int bs_select_variant_device(const bs_tile_histogram* stats, int32_t width, int32_t height, int32_t pw,
                                        int32_t ph, int32_t sm_count, int32_t* variant, void* stream) {
  if (!stats || !variant || width <= 0 || height <= 0 || pw <= 0 || ph <= 0) return BS_ERR_INVALID_ARGUMENT;
  bs::launch_pdl(bs::k_select_variant, 1, 1, 0, (cudaStream_t)stream, stats, pw, ph, sm_count, variant);
  BS_LAUNCH_CHECK();
  return BS_OK;
}

namespace bs {
__global__ void k_publish_i64(const int64_t* __restrict__ src, int64_t* dst) {
  bs::pdl_wait();
  *reinterpret_cast<volatile int64_t*>(dst) = *src;
  __threadfence_system();
}
}  // namespace bs

// 8 bytes from device memory to (mapped, pinned) host memory by a 1-thread
// kernel: no copy-engine transfer, so it never queues behind a large
// download running on another stream (a cudaMemcpyAsync D2H would).
extern "C" int bs_publish_i64(const int64_t* src_dev, int64_t* dst_host_mapped, void* stream) {
  if (!src_dev || !dst_host_mapped) return BS_ERR_INVALID_ARGUMENT;
  bs::launch_pdl(bs::k_publish_i64, 1, 1, 0, (cudaStream_t)stream, src_dev, dst_host_mapped);
  BS_LAUNCH_CHECK();
  return BS_OK;
}
