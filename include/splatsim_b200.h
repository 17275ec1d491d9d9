/*
 * splatsim_b200.h — C-ABI of the B200-native Balanced-3DGS forward rasterizer.
 *
 * Every entry point is extern "C", takes plain device pointers + sizes, is
 * stream-ordered on the `stream` argument (a cudaStream_t passed as void*,
 * NULL = legacy default stream), performs no hidden allocation (callers pass
 * workspace sized by the matching *_workspace_bytes query) and returns a
 * bs_status (0 = ok, < 0 = error; bs_status_string() names it).  There is no
 * CPU fallback: every call launches sm_100a kernels or fails.
 *
 * Reference interfaces replaced (/root/reference/proj/core, namespace splatsim):
 *   bs_preprocess        project_all / project_gaussian   include/splatsim/preprocess.hpp:57-59
 *                        (covariance_of scene.hpp:55, project_covariance preprocess.hpp:51-53)
 *   bs_bin_count+_sort   bin_tiles                         include/splatsim/preprocess.hpp:64-65
 *   bs_tile_stats        tile_load_histogram               include/splatsim/preprocess.hpp:67
 *   bs_render_forward    render_reference / run_kernel     include/splatsim/blend.hpp:100-102,
 *                                                          include/splatsim/kernels.hpp:104-106
 *   bs_frame_work        TileWork.consumed / trace inputs  src/kernels.cpp:283-298
 *   bs_select_variant    (per-frame form of) checkpoint    include/splatsim/adaptive.hpp:54-55
 *   bs_variant_name/_from_name  variant_name/_from_name    include/splatsim/kernels.hpp:25-26
 * Beyond the reference (it has no backward pass):
 *   bs_render_backward, bs_context_render_backward — per-splat gradients of
 *   render_reference's outputs (src/blend.cpp:8-42 differentiated).
 * The C++ host layer (splatsim_b200.hpp) restores the reference's value-typed
 * signatures and exceptions on top of this ABI.
 */
#ifndef SPLATSIM_B200_H
#define SPLATSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BS_ABI_VERSION 1

typedef enum bs_status {
  BS_OK = 0,
  BS_ERR_INVALID_ARGUMENT = -1, /* std::invalid_argument in the reference */
  BS_ERR_GRID_MISMATCH = -2,    /* "binning grid does not match image dims" */
  BS_ERR_WORKSPACE = -3,        /* workspace too small for this call */
  BS_ERR_CAPACITY = -4,         /* K exceeds the u32 point_list index space */
  BS_ERR_CUDA = -5,             /* a CUDA launch / runtime call failed */
  BS_ERR_UNSUPPORTED = -6,      /* patch larger than 1024 pixels, ... */
  BS_ERR_LOGIC = -7,            /* std::logic_error (selector already switched) */
  BS_ERR_NO_DEVICE = -8         /* no sm_100 device visible */
} bs_status;

/* Gaussian3D — include/splatsim/scene.hpp:16-22, by field (rot is w,x,y,z as
 * in the scene JSON, src/scene.cpp:124).  56 bytes, AoS. */
typedef struct bs_gaussian3d {
  float mean[3];
  float scale[3];
  float rot[4];
  float opacity;
  float color[3];
} bs_gaussian3d;

/* Camera — include/splatsim/scene.hpp:24-29.  view is row-major world->camera. */
typedef struct bs_camera {
  float view[16];
  float focal[2];
  int32_t width;
  int32_t height;
} bs_camera;

/* Gaussian2D — include/splatsim/preprocess.hpp:16-25, host interop layout (44 B). */
typedef struct bs_gaussian2d {
  float x, y;
  float conic_a, conic_b, conic_c;
  float opacity;
  float color[3];
  float depth;
  float radius;
} bs_gaussian2d;

/* Device-resident projected splats (SoA of float4, indexed by compacted id):
 *   xyab[i] = (x, y, conic_a, conic_b)
 *   cop[i]  = (conic_c, opacity, power_cut, depth)
 *   rgbr[i] = (r, g, b, radius)
 * power_cut is a conservative per-splat bound: power < power_cut implies
 * alpha < 1/255 (so the exact exp can be skipped without changing any
 * decision).  Each array holds n_cap float4 (16-byte aligned). */
typedef struct bs_splats {
  float* xyab;
  float* cop;
  float* rgbr;
} bs_splats;

/* KernelVariant — include/splatsim/kernels.hpp:13-19 (same order / names). */
typedef enum bs_variant {
  BS_NAIVE = 0,
  BS_DYNAMIC_BLOCKS = 1,
  BS_GAUSSIAN_WISE = 2,
  BS_FINE_GRAINED_COMBINED = 3,
  BS_SHARED_MEM_OPT = 4,
  BS_VARIANT_AUTO = -1 /* bs_render_forward: not accepted; use bs_select_variant */
} bs_variant;

/* Alpha arithmetic.
 *   BS_ALPHA_EXACT: alpha = min(0.99, opacity * expf(power)) with expf
 *     bit-identical to glibc 2.39 libm (the reference's std::exp(float)),
 *     serial float transmittance for every skip/stop decision, double
 *     colour/depth accumulators — the reference semantics bit for bit.
 *   BS_ALPHA_FAST: ex2.approx alpha, float accumulators and (Gaussian-wise
 *     variants) prefix-product stop decisions as in the paper's Alg. 6.
 *     Within 1e-4 of the reference; stop/skip flips at the termination
 *     boundary are possible and are counted by the parity tests. */
typedef enum bs_alpha_mode { BS_ALPHA_EXACT = 0, BS_ALPHA_FAST = 1 } bs_alpha_mode;

/* RenderOutput — include/splatsim/blend.hpp:86-97 (device pointers, P = W*H). */
typedef struct bs_frame_out {
  float* color;     /* f32[3P], rgb interleaved */
  float* alpha;     /* f32[P] */
  float* depth;     /* f32[P] */
  float* final_t;   /* f32[P] */
  int32_t* contrib; /* i32[P] committed steps */
  int32_t* term;    /* i32[P] 1-based termination index, 0 = none */
} bs_frame_out;

/* Backward render inputs: dL/d(outputs) of one frame (device pointers). */
typedef struct bs_frame_grad_in {
  const float* dl_dcolor; /* f32[3P] */
  const float* dl_dalpha; /* f32[P] or NULL (zero) */
  const float* dl_ddepth; /* f32[P] or NULL (zero) */
} bs_frame_grad_in;

/* Per-splat gradients, the bs_splats layout (f32x4 per splat), accumulated:
 *   xyab: d/dx, d/dy, d/dconic_a, d/dconic_b
 *   cop:  d/dconic_c, d/dopacity, 0, d/ddepth
 *   rgbr: d/dr, d/dg, d/db, 0 */
typedef struct bs_splat_grads {
  float* xyab;
  float* cop;
  float* rgbr;
} bs_splat_grads;

/* TileHistogram summary — include/splatsim/preprocess.hpp:38-45. */
typedef struct bs_tile_histogram {
  uint32_t min;
  uint32_t max;
  uint32_t p50; /* nearest-rank, as src/preprocess.cpp:130-134 */
  uint32_t p99;
  double mean;
  uint64_t total;    /* K */
  int32_t tiles;     /* T */
  int32_t nonempty;  /* tiles with count > 0 */
} bs_tile_histogram;

/* ---- library ---- */
int bs_abi_version(void);
const char* bs_status_string(int status);
/* Number of SMs of the current device (148 on B200); fails without a GPU. */
int bs_device_sm_count(int32_t* sm_count);
const char* bs_variant_name(int variant);
int bs_variant_from_name(const char* name); /* -1 when unknown */

/* ---- P1-P4: EWA projection + order-preserving compaction ----
 * Projects n Gaussians (device AoS) through cam (host struct), writes the
 * survivors in input order to out[0..n_visible) and *n_visible (device i32).
 * Semantics: src/preprocess.cpp:17-64 (near cull, det/eigen culls, no +0.3
 * dilation).  out arrays must hold n entries. */
size_t bs_preprocess_workspace_bytes(int64_t n);
int bs_preprocess(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam, bs_splats out, int32_t* n_visible,
                  void* ws, size_t ws_bytes, void* stream);

/* Same, with the camera read from DEVICE memory at run time (what a CUDA
 * graph of the frame replays with a per-frame camera). */
int bs_preprocess_devcam(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam_dev, bs_splats out,
                         int32_t* n_visible, void* ws, size_t ws_bytes, void* stream);

/* Interop: device AoS Gaussian2D <-> splats (fills power_cut). */
int bs_splats_from_g2d(const bs_gaussian2d* g2d, int64_t n, bs_splats out, void* stream);
int bs_splats_to_g2d(bs_splats in, int64_t n, bs_gaussian2d* g2d, void* stream);

/* ---- P5: binning (bit-exact with src/preprocess.cpp:66-115) ----
 * Two calls so the host can size point_list without a hidden sync:
 *   bs_bin_count: per-splat tile rects, stable depth sort of the visible
 *     splats, exclusive scan of tiles-touched.  Writes K to *k_total (an i64
 *     in device memory or in mapped pinned host memory, stored by a kernel).
 *     Reads the splat count from *n_visible (device) — n_cap bounds it.
 *   bs_bin_sort: duplicates (tile, id) pairs in depth order, stable radix sort
 *     by tile id, tile ranges.  k is K read back by the host.  Must be given
 *     the same workspace the matching bs_bin_count call used.
 * Workspace: bs_bin_workspace_bytes(n_cap, W, H, pw, ph, k_cap) with
 * k_cap >= k; bs_bin_sort returns BS_ERR_WORKSPACE if k > k_cap.
 * tile_ranges holds 2*T u32 ([start, end) per tile, row-major tiles). */
size_t bs_bin_workspace_bytes(int64_t n_cap, int32_t width, int32_t height, int32_t pw, int32_t ph, int64_t k_cap);
int bs_bin_count(bs_splats g, int64_t n_cap, const int32_t* n_visible, int32_t width, int32_t height, int32_t pw,
                 int32_t ph, int64_t* k_total, void* ws, size_t ws_bytes, void* stream);
/* Frame-pipeline fusion of bs_preprocess + bs_bin_count (no reference
 * counterpart of its own: project_all + the counting half of bin_tiles,
 * src/preprocess.cpp:57-64, 66-92).  Splats are NOT compacted: splat i stays
 * at index i of out, culled splats touch no tile.  counts (2 x i32, device):
 * counts[0] <- n, the item count to pass as n_visible to bs_bin_sort*;
 * counts[1] <- the visible count.  Tile lists then index the uncompacted
 * arrays, in the reference's order (compaction is monotone).  Exactly one of
 * cam (host) / cam_dev (device) is used (cam wins).  Workspace: the bin one. */
int bs_preprocess_bin_count(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam, const bs_camera* cam_dev,
                            bs_splats out, int32_t* counts, int32_t width, int32_t height, int32_t pw, int32_t ph,
                            int64_t* k_total, void* ws, size_t ws_bytes, void* stream);
/* Super-tile form for the frame pipeline (power-of-two pw, ph; replaces
 * project_all + bin_tiles' counting, src/preprocess.cpp:57-92, inside a
 * frame — the reference's own lists stay available via bs_bin_sort): the lists
 * are binned at 2pw x 2ph (bs_bin_sort* follow with 2pw, 2ph) and
 * tile_ranges (2 x T, T = pw x ph tiles; may be NULL) receives the pw x ph
 * list lengths (for bs_tile_stats / bs_frame_work) — or later, from the same
 * aux, bs_super_tile_lengths.  aux: bs_super_aux_bytes(width, height, pw, ph)
 * bytes. */
size_t bs_super_aux_bytes(int32_t width, int32_t height, int32_t pw, int32_t ph);
int bs_preprocess_bin_count_super(const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam,
                                  const bs_camera* cam_dev, bs_splats out, int32_t* counts, int32_t width,
                                  int32_t height, int32_t pw, int32_t ph, int64_t* k_total, void* ws,
                                  size_t ws_bytes, uint32_t* tile_ranges, void* aux, size_t aux_bytes,
                                  void* stream);
int bs_super_tile_lengths(void* aux, size_t aux_bytes, int32_t width, int32_t height, int32_t pw, int32_t ph,
                          uint32_t* tile_ranges, void* stream);
int bs_bin_sort(bs_splats g, int64_t n_cap, const int32_t* n_visible, int32_t width, int32_t height, int32_t pw,
                int32_t ph, int64_t k, uint32_t* point_list, uint32_t* tile_ranges, void* ws, size_t ws_bytes,
                void* stream);

/* Sync-free form of bs_bin_sort (chunked path; bs_bin_async_supported says
 * whether the grid qualifies): K stays on the device and point_list holds
 * k_cap entries.  If K > k_cap nothing is written to point_list and every
 * tile range is written empty; the caller reads K (the k_total of the
 * matching bs_bin_count) later, grows point_list and runs again. */
int bs_bin_sort_async(bs_splats g, int64_t n_cap, const int32_t* n_visible, int32_t width, int32_t height, int32_t pw,
                      int32_t ph, int64_t k_cap, uint32_t* point_list, uint32_t* tile_ranges, void* ws,
                      size_t ws_bytes, void* stream);
int bs_bin_async_supported(int32_t width, int32_t height, int32_t pw, int32_t ph);

/* ---- P6: tile statistics + LPT task order ----
 * counts[t] = end - start; stats as tile_load_histogram (written to device
 * memory at *stats); task_order = tiles by list length descending, ties by
 * tile id ascending (the fine-grained queue order).  counts/task_order may be
 * NULL. */
size_t bs_tile_stats_workspace_bytes(int32_t tiles);
int bs_tile_stats(const uint32_t* tile_ranges, int32_t tiles, bs_tile_histogram* stats, uint32_t* counts,
                  uint32_t* task_order, void* ws, size_t ws_bytes, void* stream);

/* Frame-pipeline form of the above (one launch, T <= 32768): sum / max /
 * mean / nonempty in *stats (device; min, p50, p99 left 0) and task_order =
 * tiles by eighth-octave length bucket descending, tile id ascending within a
 * bucket (lengths inside a bucket differ by < 9 %: an LPT order for the
 * fine-grained queue without a full sort). */
int bs_tile_order(const uint32_t* tile_ranges, int32_t tiles, bs_tile_histogram* stats, uint32_t* task_order,
                  void* stream);
/* bs_tile_order + bs_select_variant_device in one launch: *variant (device)
 * <- the selector's choice (select_variant_formula) on the same statistics
 * (tile_load_histogram, src/preprocess.cpp:117-136, feeding the per-frame
 * predictor of the balanced/baseline choice, src/adaptive.cpp:16-32). */
int bs_tile_order_select(const uint32_t* tile_ranges, int32_t tiles, bs_tile_histogram* stats,
                         uint32_t* task_order, int32_t width, int32_t height, int32_t pw, int32_t ph,
                         int32_t sm_count, int32_t* variant, void* stream);

/* ---- R1-R8: forward render ----
 * variant: bs_variant (not AUTO).  task_order: LPT tile order from
 * bs_tile_stats (required for BS_FINE_GRAINED_COMBINED, ignored otherwise;
 * NULL = index order).  bg: host rgb.  Writes every pixel of out.
 * Output equals render_reference (pixel-wise variants) or
 * render_gaussianwise (GaussianWise / FineGrainedCombined).
 * Workspace holds the dynamic-queue counter (reset by the call). */
/* queue counters (256 B) + the FineGrainedCombined tail hand-off slots
 * (64 B/pixel) + parked-task records (8 B per 4 pixels): ~66 B/pixel, e.g.
 * 137 MB at 1080p, 548 MB at 4K. */
size_t bs_render_workspace_bytes(int32_t width, int32_t height);
int bs_render_forward(int variant, int alpha_mode, bs_splats g, const uint32_t* point_list,
                      const uint32_t* tile_ranges, const uint32_t* task_order, int32_t width, int32_t height,
                      int32_t pw, int32_t ph, const float bg[3], bs_frame_out out, void* ws, size_t ws_bytes,
                      void* stream);

/* Sync-free auto mode: variant_dev points to the device int32 written by
 * bs_select_variant_device.  Launches the selector's candidates
 * (FineGrainedCombined, SharedMemOpt); all but the selected one exit at
 * entry, so the host never waits for the selection. */
int bs_render_forward_auto(const int32_t* variant_dev, int alpha_mode, bs_splats g, const uint32_t* point_list,
                           const uint32_t* tile_ranges, const uint32_t* task_order, int32_t width, int32_t height,
                           int32_t pw, int32_t ph, const float bg[3], bs_frame_out out, void* ws, size_t ws_bytes,
                           void* stream);

/* Resident FineGrainedCombined CTAs per SM for the following launches (0 =
 * as many as fit, the default).  With several frame contexts streaming
 * views concurrently, 3 leaves room for the other context's preprocess and
 * binning kernels to overlap the render (process-wide setting). */
int bs_render_set_fine_occupancy(int32_t ctas_per_sm);

/* The frame context's render entry: bs_render_forward (super_lists = 0) /
 * bs_render_forward_super (super_lists = 1), variant -1 = the device-selected
 * one (variant_dev), with a per-call FineGrainedCombined occupancy cap
 * (fine_ctas_per_sm > 0; 0 = the process default above) — each context keeps
 * its own (bs_context_set_fine_occupancy). */
int bs_render_forward_ctx(int variant, const int32_t* variant_dev, int alpha_mode, bs_splats g,
                          const uint32_t* point_list, const uint32_t* tile_ranges, const uint32_t* task_order,
                          int32_t width, int32_t height, int32_t pw, int32_t ph, const float bg[3], bs_frame_out out,
                          int32_t super_lists, int32_t fine_ctas_per_sm, void* ws, size_t ws_bytes, void* stream);

/* Work counters of a rendered frame (src/kernels.cpp:283-298):
 *   evaluated = sum_p consumed(p), consumed = term > 0 ? term : list_len(tile(p))
 *   committed = sum_p contrib(p)
 * written to device u64[2] = {evaluated, committed}. */
int bs_frame_work(const int32_t* term, const int32_t* contrib, const uint32_t* tile_ranges, int32_t width,
                  int32_t height, int32_t pw, int32_t ph, uint64_t* evaluated_committed, void* stream);

/* ---- S-1: per-frame variant predictor (host call, host struct) ----
 * Returns the bs_variant the B200 cost model predicts fastest for a frame
 * with these tile statistics.  Host-only logic. */
int bs_select_variant(const bs_tile_histogram* stats, int32_t width, int32_t height, int32_t pw, int32_t ph,
                      int32_t sm_count);

/* Device form of bs_select_variant: reads the histogram bs_tile_stats wrote
 * (device pointer) and writes the chosen bs_variant to *variant (device
 * int32), stream-ordered — same formula, same decision. */
int bs_select_variant_device(const bs_tile_histogram* stats, int32_t width, int32_t height, int32_t pw, int32_t ph,
                             int32_t sm_count, int32_t* variant, void* stream);

/* ---- diagnostics ----
 * y[i] = the device exp the render kernels use in alpha_mode (EXACT: the
 * glibc-identical expf, through the same in-range function and shared-memory
 * table the render's eval_step calls on [-0x1.9fe368p6, 0], the general one
 * elsewhere; FAST: ex2.approx).  Used by the parity tests to pin the exact
 * path against the host libm.  _range: x = the float with bit pattern
 * first_bits + i (exhaustive sweeps without an input array). */
int bs_test_expf(const float* x, float* y, int64_t n, int alpha_mode, void* stream);
int bs_test_expf_range(uint32_t first_bits, int64_t n, float* y, int alpha_mode, void* stream);

/* ---- host-side helpers (implemented in the C++ host layer) ----
 * gen_clustered_scene (src/workload.cpp:198-246, include/splatsim/workload.hpp:68-76):
 * writes n Gaussians to the HOST array out. */
int bs_host_gen_clustered_scene(int32_t n, int32_t n_clusters, uint64_t seed, double cluster_sigma,
                                double background_fraction, const bs_camera* cam, bs_gaussian3d* out);

/* Measured training run (the B200 form of the reference's run_training_sim,
 * src/adaptive.cpp:34-129; C++: splatsim::run_training): a clustered scene
 * moves linearly from the *_start to the *_end parameters over total_iters
 * iterations (regenerated at `keyframes` points), FineGrainedCombined and
 * SharedMemOpt are timed on the device per keyframe, the selector
 * checkpoints every check_interval iterations until the first loss.  Writes
 * report_csv (NUL-terminated, truncated to csv_cap) and its full length. */
typedef struct bs_training_params {
  int32_t total_iters, keyframes, width, height, patch_width, patch_height;
  float focal;
  int32_t n_gaussians;
  uint64_t seed;
  double background_fraction_start, background_fraction_end;
  double cluster_sigma_start, cluster_sigma_end;
  double opacity_scale_start, opacity_scale_end;
} bs_training_params;
int bs_host_run_training(const bs_training_params* params, int32_t check_interval, char* csv, size_t csv_cap,
                         size_t* csv_len);

/* ---- host-buffer frame API (the drop-in for project_all -> bin_tiles ->
 * run_kernel on HOST data) ----
 * A context owns a CUDA stream and device buffers that grow on demand.
 * bs_render_frame_host copies the Gaussians host->device, runs the whole
 * forward on the device, and copies the RenderOutput planes device->host
 * (each output pointer may be NULL to skip that plane).  variant = -1 picks
 * the variant per frame with bs_select_variant. */
typedef struct bs_context bs_context;

typedef struct bs_frame_info {
  int32_t variant;          /* variant actually rendered */
  int32_t n_visible;
  int64_t k;                /* tile instances */
  bs_tile_histogram stats;  /* tile_load_histogram of the frame */
  uint64_t evaluated;       /* sum consumed (pairs blended under serial semantics) */
  uint64_t committed;       /* sum contrib */
} bs_frame_info;

int bs_context_create(bs_context** out, int alpha_mode);
int bs_context_destroy(bs_context* ctx);
/* cudaStream_t of the context (as void*) */
void* bs_context_stream(bs_context* ctx);
int bs_render_frame_host(bs_context* ctx, const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam, int32_t pw,
                         int32_t ph, int32_t variant, const float bg[3], float* color, float* alpha, float* depth,
                         float* final_t, int32_t* contrib, int32_t* term, bs_frame_info* info);

/* Pipelined form (async mode contexts): enqueues the upload, the frame and
 * the download of the requested planes on three streams and returns; three
 * frames are in flight, so frame i+1's upload and frame i-1's download overlap
 * frame i's kernels.  Host buffers (pinned for overlap) must stay valid and
 * untouched until bs_context_sync, after which every output is final (frames
 * whose K outgrew point_list are re-rendered and re-downloaded there).  Falls
 * back to bs_render_frame_host when the context is not in async mode. */
int bs_render_frame_host_async(bs_context* ctx, const bs_gaussian3d* g3d, int64_t n, const bs_camera* cam, int32_t pw,
                               int32_t ph, int32_t variant, const float bg[3], float* color, float* alpha,
                               float* depth, float* final_t, int32_t* contrib, int32_t* term);

/* Same pipeline on DEVICE Gaussians (g3d_dev), stream-ordered on the context
 * stream (bs_context_set_stream; NULL = the context's own stream).  out: the
 * caller's device planes, or all-NULL for context-owned planes.  The only
 * host wait is the 8-byte K readback that sizes point_list; with variant = -1
 * the variant is selected on the device.  info != NULL additionally waits for
 * the frame and fills it (otherwise bs_context_last_info does that later). */
int bs_render_frame_device(bs_context* ctx, const bs_gaussian3d* g3d_dev, int64_t n, const bs_camera* cam, int32_t pw,
                           int32_t ph, int32_t variant, const float bg[3], bs_frame_out out, bs_frame_info* info);
/* Stream for the following frames: NULL = the legacy default stream; the
 * context's own stream is the value bs_context_stream() returned before. */
int bs_context_set_stream(bs_context* ctx, void* stream);
/* A batch of views over several contexts from one native loop (the
 * reference renders one view per run_kernel call, src/kernels.cpp:268-301): view i
 * renders cams[view_ids[i]] with ctxs[i % nctx] (into that context's own
 * planes); flush_bufs (nctx device buffers, may be NULL) are zeroed, flush_bytes
 * each, on the view's stream before it (an L2 flush when larger than L2). */
int bs_render_views(bs_context* const* ctxs, int32_t nctx, const bs_gaussian3d* g3d_dev, int64_t n,
                    const bs_camera* cams, const int32_t* view_ids, int32_t count, int32_t pw, int32_t ph,
                    int32_t variant, const float bg[3], void* const* flush_bufs, size_t flush_bytes);
/* A batch of views of ONE scene from HOST memory (the host-buffer form of
 * bs_render_views): the scene is uploaded once per call (ctxs[0]'s upload
 * stream), view i = cams[view_ids[i]] renders on ctxs[i % nctx] (async
 * frame body; every context must be in async mode) and its six planes are
 * downloaded into host_out[6i .. 6i+5] = color, alpha, depth, final_t,
 * contrib, term (pinned host memory for full speed; NULL skips a plane).
 * Outputs are final after bs_context_sync on every context; the host
 * buffers of one call must stay untouched until then. */
int bs_render_views_host(bs_context* const* ctxs, int32_t nctx, const bs_gaussian3d* g3d_host, int64_t n,
                         const bs_camera* cams, const int32_t* view_ids, int32_t count, int32_t pw, int32_t ph,
                         int32_t variant, const float bg[3], void* const* host_out);
/* The context-owned planes frames with an empty bs_frame_out render into
 * (device pointers, valid until the next such frame or the context's destroy). */
int bs_context_frame(bs_context* ctx, bs_frame_out* out);
/* Render from super-tile lists (binned at 2pw x 2ph; same outputs as
 * run_kernel / render_reference on the pw x ph lists, src/kernels.cpp:268-301,
 * src/blend.cpp:55-107): tile_ranges holds, per
 * pw x ph tile, its super-tile's range (bs_super_tile_ranges); the render
 * keeps the entries whose pw x ph rectangle contains the tile — exactly the
 * tile's list, term counted over it.  variant: FineGrainedCombined,
 * SharedMemOpt, or -1 (device-selected from variant_dev, as
 * bs_render_forward_auto).  Power-of-two pw, ph. */
int bs_render_forward_super(int variant, const int32_t* variant_dev, int alpha_mode, bs_splats g,
                            const uint32_t* point_list, const uint32_t* tile_ranges, const uint32_t* task_order,
                            int32_t width, int32_t height, int32_t pw, int32_t ph, const float bg[3],
                            bs_frame_out out, void* ws, size_t ws_bytes, void* stream);
int bs_super_tile_ranges(const uint32_t* super_ranges, int32_t width, int32_t height, int32_t pw, int32_t ph,
                         uint32_t* tile_ranges, void* stream);
/* Backward render (the reference has no backward pass): the
 * per-splat gradients of a frame's colour / alpha / depth under
 * render_reference semantics (src/blend.cpp:8-42), the forward's skip /
 * stop decisions held fixed; no gradient through a clamped alpha (0.99).
 * fwd: the forward's outputs for the same inputs (colour, depth, final_t
 * read).  gout accumulates (caller zeroes).  super_lists = 1: the frame
 * pipeline's super-tile lists (as bs_render_forward_super).  ws: a render
 * workspace (>= 256 bytes; its queue counters).  Checked against the CPU
 * oracle's analytic gradient, which finite differences of the reference
 * forward pin (tests/test_backward_oracle.py). */
int bs_render_backward(int alpha_mode, bs_splats g, const uint32_t* point_list, const uint32_t* tile_ranges,
                       const uint32_t* task_order, int32_t width, int32_t height, int32_t pw, int32_t ph,
                       const float bg[3], bs_frame_out fwd, bs_frame_grad_in gin, bs_splat_grads gout,
                       int super_lists, void* ws, size_t ws_bytes, void* stream);
/* Backward render of a frame context's last frame (bs_render_frame_device,
 * bs_render_views...; the frame pipeline's training step): per-Gaussian
 * gradients at the INPUT index i of that frame's g3d array (culled Gaussians
 * receive none), accumulated into caller-zeroed gout holding >= n entries
 * per array.  Verifies pending async frames first.  BS_ERR_UNSUPPORTED when
 * the frame ran the compacting projection (BS_NO_FUSED_PRE=1). */
int bs_context_render_backward(bs_context* ctx, bs_frame_grad_in gin, bs_splat_grads gout);
/* 1 if the context's last frame was binned into super-tile lists (frames
 * >= 1 Mpixel with power-of-two patches and a FineGrainedCombined /
 * SharedMemOpt / device-selected variant; BS_NO_SUPER=1 disables), else 0. */
int bs_context_list_mode(bs_context* ctx, int32_t* super_lists);
/* 8 bytes device -> mapped pinned host memory (cudaMallocHost) by a 1-thread
 * kernel on stream: unlike a D2H memcpy it does not queue behind other
 * streams' downloads on the copy engine. */
int bs_publish_i64(const int64_t* src_dev, int64_t* dst_host_mapped, void* stream);
/* Async mode for bs_render_frame_device: no host wait inside a frame.
 * point_list is sized from a capacity (3 x the first K, regrown to 3 x K
 * whenever a K passes 2/3 of it);
 * a frame's K is checked at the NEXT call on the context (or at
 * bs_context_sync / bs_context_last_info), and a frame whose K exceeded the
 * capacity is rendered again then, before anything else, with the same
 * inputs — so inputs and outputs must stay valid until that next call.
 * Outputs are final once bs_context_sync returns (reruns = frames re-rendered
 * so far). */
int bs_context_set_async(bs_context* ctx, int32_t on);
int bs_context_sync(bs_context* ctx, int64_t* reruns);
/* CUDA-graph mode for async frames: the first frame of a configuration
 * (inputs, outputs, dims, variant, bg, buffers) runs normally, later ones
 * replay a captured graph of the same kernels with the new camera (copied in
 * ahead of the launch) — one launch instead of ~45.  Off by default.
 * bs_context_graph_launches counts the replays. */
int bs_context_set_graphs(bs_context* ctx, int32_t on);
/* This context's FineGrainedCombined resident CTAs per SM (0 = the process
 * default, bs_render_set_fine_occupancy).  With several contexts streaming
 * views concurrently, 3 leaves SM room for the other contexts' preprocess and
 * binning kernels to overlap the render. */
int bs_context_set_fine_occupancy(bs_context* ctx, int32_t ctas_per_sm);
int bs_context_graph_launches(bs_context* ctx, int64_t* launches);
/* Drops pending K checks without waiting (after capturing a frame into a
 * CUDA graph: the captured call's check never ran).  The caller then owns
 * capacity safety for replays. */
int bs_context_drop_pending(bs_context* ctx);
/* point_list capacity (entries) and how many times it has grown (diagnostics). */
int bs_context_capacity(bs_context* ctx, int64_t* point_list_cap, int64_t* grows);
int bs_context_last_info(bs_context* ctx, bs_frame_info* info);
/* Per-stage CUDA-event timing of the following frames (6 stages: preprocess,
 * bin_count, k_readback, bin_sort, stats_select, render); bs_context_stage_ms
 * waits for the last frame and writes n >= 6 floats (ms). */
int bs_context_enable_timing(bs_context* ctx, int32_t on);
int bs_context_stage_ms(bs_context* ctx, float* ms, int32_t n);

/* Number of kernel launches issued by this library since load (evidence
 * counter for bench.py's gpu_launches). */
uint64_t bs_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* SPLATSIM_B200_H */
