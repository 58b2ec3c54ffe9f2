/* gsf_cuda.h — C-ABI of the B200-native CG-SLAM rasterizer / track-step / map-step.
 *
 * This is the drop-in boundary for the reference's hot path (arxiv 2403.16095 "gsfield",
 * /root/reference/proj).  Every entry point below replaces one reference C++ function;
 * the citation next to it names the interface it stands in for.  Plain C types only:
 * pointers, sizes, PODs.  No torch types, no C++ types.
 *
 * Conventions
 *   - Images are row-major (x fastest), index y*W + x, like gsf::Image (core/image.hpp:10-48).
 *     RGB images interleave channels: rgb[3*(y*W+x) + c].
 *   - Per-primitive host arrays are AoS per primitive, like GaussianPrimitive
 *     (geometry/primitive.hpp:16-59): mean[3*i+a], log_scale[3*i+a], quat[4*i+k] (w,x,y,z),
 *     opacity_logit[i], sh[3*K*i + 3*b + c] (K coefficients per channel, 1/4/9/16).
 *   - The device keeps the map as SoA fp32 ([field][P]); poses, loss scalars and the
 *     camera rotation are fp64.  Pixel maps are returned as fp32.
 *   - Every function returns a gsf_status.  GSF_OK = 0.  On failure gsf_last_error(ctx)
 *     holds the message the reference would have put in its exception, and
 *     gsf_last_error_index(ctx) the offending primitive index (or -1).
 *   - A context owns one CUDA device + stream.  It is not thread-safe; use one per thread.
 *   - There is no CPU fallback: if the device or the kernels are unavailable every call
 *     fails with GSF_ECUDA.
 */
#ifndef GSF_CUDA_H
#define GSF_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSF_ABI_VERSION 1

typedef enum {
  GSF_OK = 0,
  GSF_EINVAL = 1,        /* std::invalid_argument in the reference */
  GSF_ENONFINITE = 2,    /* invalid_argument("render: primitive i has non-finite parameters") */
  GSF_EDIVERGED = 3,     /* std::runtime_error("... diverged ...") */
  GSF_ECUDA = 4,         /* device / launch failure (no fallback exists) */
  GSF_EUNSUPPORTED = 5,  /* a runtime value the device path does not implement (e.g. tile_size != 16) */
  GSF_ENOMEM = 6,
  GSF_ERUNTIME = 7       /* any other std::runtime_error of the reference (e.g. an empty first frame) */
} gsf_status;

typedef struct gsf_ctx_s* gsf_ctx;

/* CameraIntrinsics (geometry/camera.hpp:9-36). */
typedef struct {
  double fx, fy, cx, cy;
  int32_t width, height;
  double depth_scale, near_plane, far_plane;
} gsf_intrinsics;

/* RasterConfig (raster/config.hpp:5-16).  tile_size must be 16 on the device path;
 * threads is accepted and ignored (the device has its own parallelism). */
typedef struct {
  double alpha_clamp, alpha_skip, termination_threshold, footprint_sigma, dilation;
  int32_t tile_size;
  int32_t uncertainty_full_gradient;
  int32_t threads;
} gsf_raster_cfg;

/* CameraPose (geometry/pose.hpp:13-49): p_cam = exp(rotation_tangent) p_world + translation. */
typedef struct {
  double rotation_tangent[3];
  double translation[3];
} gsf_pose;

/* LossWeights (loss/losses.hpp:13-31). */
typedef struct {
  double w_color, w_ssim, w_geo, w_align, w_iso, w_var;
  double t_color, t_geo;
  double iso_epsilon, opacity_floor;
  int32_t normalize_by_valid;
} gsf_loss_weights;

/* TrackerConfig (track/tracker.hpp:11-22). */
typedef struct {
  double lr_rotation, lr_translation;
  int32_t iterations, ba_window, ba_iterations, keyframe_interval, recent_keyframes;
  int32_t freeze_oldest_pose;
  double degraded_loss_ratio;
} gsf_tracker_cfg;

/* The MapperConfig fields used by map_step / sliding_ba (map/mapper.hpp:21-41). */
typedef struct {
  int32_t sh_coeffs;
  double scene_extent, lr_mean, lr_sh, lr_opacity, lr_scale, lr_rotation;
  int32_t densify_interval;   /* DensifyConfig::interval; densify runs on the host layer */
  double densify_grad_threshold, densify_split_factor, densify_size_fraction, densify_cull_opacity;
  double uncertainty_tau, uncertainty_reduced_opacity;   /* UncertaintyConfig */
  uint64_t seed;
  gsf_raster_cfg raster;
  gsf_loss_weights weights;
  int32_t init_stride, spawn_stride;          /* pixel sampling strides of initialize / spawn */
  double spawn_opacity_threshold, init_opacity;
} gsf_mapper_cfg;

/* Host view of a primitive list (std::vector<GaussianPrimitive>). */
typedef struct {
  int64_t count;
  int32_t sh_coeffs;
  double* mean;           /* 3*count */
  double* log_scale;      /* 3*count */
  double* quat;           /* 4*count */
  double* opacity_logit;  /* count */
  double* sh;             /* 3*sh_coeffs*count */
  double* uncertainty;    /* count, may be NULL */
  uint8_t* observed;      /* count, may be NULL */
} gsf_map_host;

/* RenderOutput (raster/output.hpp:15-28) + the per-pixel parts of BlendRecord
 * (dominant, median_prim, visible; output.hpp:32-45).  Any pointer may be NULL. */
typedef struct {
  float* color;               /* 3*W*H */
  float* alpha_depth;         /* W*H */
  float* median_depth;
  uint8_t* median_valid;
  float* opacity;
  float* uncertainty;
  float* final_transmittance;
  int32_t* per_pixel_count;
  int32_t* dominant;          /* -1 where no contributor */
  int32_t* median_prim;       /* -1 where T never crossed 0.5 */
  float* dominant_weight;     /* alpha*T of the dominant contributor (0 if none) */
  uint8_t* visible;           /* count (per primitive) */
  int32_t has_uncertainty;    /* out */
  int64_t num_visible;        /* out: primitives surviving culling */
  int64_t num_pairs;          /* out: (tile, primitive) list entries */
} gsf_render_out;

/* UpstreamGradients (raster/output.hpp:54-60).  NULL = that map carries no gradient. */
typedef struct {
  const float* d_color;        /* 3*W*H */
  const float* d_alpha_depth;
  const float* d_median_depth;
  const float* d_opacity;
  const float* d_uncertainty;
} gsf_upstream;

/* GradientBundle (raster/output.hpp:64-77).  Any array pointer may be NULL. */
typedef struct {
  float* d_mean;            /* 3*count */
  float* d_log_scale;       /* 3*count */
  float* d_quat;            /* 4*count */
  float* d_opacity_logit;   /* count */
  float* d_sh;              /* 3*K*count */
  float* d_mean2d;          /* 2*count */
  double d_pose[6];         /* out: (rot, trans) in the CameraPose::perturbed tangent */
} gsf_grads_out;

/* TrackResult (track/tracker.hpp:28-33). */
typedef struct {
  gsf_pose pose;
  double final_loss;
  int32_t degraded;
  int32_t iterations_run;
  double initial_loss;
} gsf_track_result;

/* Loss scalars of evaluate_tracking_loss / evaluate_mapping_loss (losses.hpp:65-87). */
typedef struct {
  double color, ssim, geo, align, iso, var, total;
  int32_t valid_color, valid_geo, any_empty_mask;
} gsf_loss_terms;

/* ---- context ------------------------------------------------------------------------ */
int gsf_abi_version(void);
int gsf_ctx_create(int device, gsf_ctx* out);
int gsf_ctx_destroy(gsf_ctx ctx);
const char* gsf_last_error(gsf_ctx ctx);
int64_t gsf_last_error_index(gsf_ctx ctx);
/* Device-side kernel launches issued by this context since creation (evidence counter). */
int64_t gsf_kernel_launches(gsf_ctx ctx);
/* Binning capacities: (tile, primitive) pairs and per-tile bucket entries.  Renders grow both on
 * overflow (retry with the loop's maxima; GSF_EUNSUPPORTED if still exceeded), so reserve only
 * pre-sizes them to skip that retry (a value <= 0 leaves a capacity unchanged; smaller values are
 * honoured too, which the overflow tests use). */
int gsf_reserve(gsf_ctx ctx, int64_t pair_cap, int64_t bucket_cap);
int gsf_capacity(gsf_ctx ctx, int64_t* pair_cap, int64_t* bucket_cap);
/* Trust-region candidates of the last tracked frame (the primitives its iterations project;
 * measurement evidence for the preprocess's algorithmic bytes), -1 on error. */
int64_t gsf_track_candidates(gsf_ctx ctx);
int gsf_synchronize(gsf_ctx ctx);

/* ---- timing hooks (benchmark evidence; no effect on results) -------------------------------
 * CUDA events on the context's stream (profiling runs the loops eagerly, not as graphs).  Kernel
 * classes for gsf_profile_read: 0 preprocess, 1 tile sort + list build (binning), 2 blend (forward),
 * 3 backward (per-pixel reverse sweep), 4 chain (per-primitive fp64 chain + pose reduction),
 * 5 SSIM, 6 Adam, 7 (unused), 8 pose Jacobians (k_posejac, timed on the side stream it overlaps
 * the binning on). */
int gsf_profile_enable(gsf_ctx ctx, int32_t on);
int gsf_profile_read(gsf_ctx ctx, int32_t kernel_class, double* total_ms, int64_t* launches);
int gsf_event_record(gsf_ctx ctx, int32_t slot);                       /* slot 0..7 */
int gsf_event_elapsed(gsf_ctx ctx, int32_t a, int32_t b, double* ms);  /* waits for b */

/* ---- map residency ------------------------------------------------------------------
 * Replaces the implicit per-call read of const std::vector<GaussianPrimitive>& in every
 * reference entry point: the map is uploaded once and stays resident.  Validation of
 * non-finite parameters (rasterizer.cpp:34-44) happens at upload and again on device. */
int gsf_map_upload(gsf_ctx ctx, const gsf_map_host* map);
int gsf_map_download(gsf_ctx ctx, gsf_map_host* map);   /* map->count must match */
int64_t gsf_map_count(gsf_ctx ctx);
/* SH coefficients per colour channel of the context's map (K of GaussianPrimitive::sh). */
int32_t gsf_map_sh_coeffs(gsf_ctx ctx);
/* Reset the Adam moments/step counts of the primitive optimizer (PrimitiveOptimizer,
 * map/mapper.hpp:92-105) — a fresh MapState. */
int gsf_optimizer_reset(gsf_ctx ctx);

/* ---- forward / backward (raster/rasterizer.hpp:19-35) --------------------------------- */
/* render(): observed_depth may be NULL (then has_uncertainty = 0). */
int gsf_render(gsf_ctx ctx, const gsf_pose* pose, const gsf_intrinsics* K,
               const float* observed_depth, const gsf_raster_cfg* cfg, gsf_render_out* out);
/* render_backward() over the record of the most recent gsf_render on this context.
 * observed_depth must be the same buffer contents as for that render (or NULL). */
int gsf_render_backward(gsf_ctx ctx, const gsf_upstream* up, const float* observed_depth,
                        gsf_grads_out* out);
/* The CSR BlendRecord of the most recent render (output.hpp:32-45, rasterizer.cpp:240-259).
 * Call with prim == NULL to get *total; then again with buffers of that size. */
int gsf_render_record(gsf_ctx ctx, uint32_t* row_start, int32_t* prim, float* alpha,
                      float* transmittance, int64_t* total);

/* Tile binning of the most recent render, for bit-exact checks of the binning:
 * tile_range[2*tiles] ([start, end) into the pair list; [0, 0) for an empty tile) and
 * pair_prim[M] (every tile list as primitive ids in (depth, id) order: the tile_lists of
 * rasterizer.cpp:193-212 built from sorted_visible, :69-79).
 * Any pointer may be NULL; capacities are checked against the counts of gsf_render_out. */
int gsf_render_tiles(gsf_ctx ctx, int32_t* tile_range, int64_t tiles_cap, int32_t* pair_prim,
                     int64_t pair_cap);

/* ---- losses (loss/losses.hpp:77-94) over the most recent render ----------------------- */
int gsf_tracking_loss(gsf_ctx ctx, const float* target_rgb, const float* observed_depth,
                      const gsf_loss_weights* w, gsf_loss_terms* out, float* d_color,
                      float* d_alpha_depth);
int gsf_mapping_loss(gsf_ctx ctx, const float* target_rgb, const float* observed_depth,
                     const gsf_loss_weights* w, gsf_loss_terms* out, float* d_color,
                     float* d_alpha_depth, float* d_median_depth, float* d_uncertainty,
                     float* d_log_scale_direct);
/* ssim / ssim_with_gradient (loss/ssim.hpp:11-14); d_x may be NULL. */
int gsf_ssim(gsf_ctx ctx, const float* x, const float* y, int32_t w, int32_t h, double* value,
             float* d_x);

/* ---- frames resident on the device --------------------------------------------------- */
/* Upload one RGB-D observation into slot `slot` (rgb 3*W*H, depth W*H, meters). */
int gsf_frame_upload(gsf_ctx ctx, int32_t slot, const float* rgb, const float* depth,
                     int32_t width, int32_t height);

/* ---- track / map / bundle adjustment --------------------------------------------------- */
/* track_frame (track/tracker.hpp:38-42, tracker.cpp:30-84) against frame slot `slot`. */
int gsf_track_frame(gsf_ctx ctx, int32_t slot, const gsf_pose* initial, const gsf_intrinsics* K,
                    const gsf_tracker_cfg* tcfg, const gsf_loss_weights* w,
                    const gsf_raster_cfg* rcfg, gsf_track_result* out);
/* One tracking iteration's objective and pose gradient at `pose` against frame slot `slot`:
 * render -> evaluate_tracking_loss -> render_backward (pose part) of tracker.cpp:42-63, on the
 * fused device path track_frame uses (per-primitive SE(3) Jacobians, no chain pass). */
int gsf_tracking_gradient(gsf_ctx ctx, int32_t slot, const gsf_pose* pose, const gsf_intrinsics* K,
                          const gsf_loss_weights* w, const gsf_raster_cfg* rcfg, gsf_loss_terms* terms,
                          double d_pose[6]);
/* Same call with host frame buffers: uploads rgb/depth into slot 0 first (e2e path). */
int gsf_track_frame_host(gsf_ctx ctx, const float* rgb, const float* depth,
                         const gsf_pose* initial, const gsf_intrinsics* K,
                         const gsf_tracker_cfg* tcfg, const gsf_loss_weights* w,
                         const gsf_raster_cfg* rcfg, gsf_track_result* out);
/* map_step (map/mapper.hpp:101-103): window = frame slots + their poses; trace gets
 * `iterations` loss values. */
int gsf_map_step(gsf_ctx ctx, const int32_t* slots, const gsf_pose* poses, int32_t n,
                 const gsf_intrinsics* K, const gsf_mapper_cfg* mcfg, int32_t iterations,
                 double* trace);
/* sliding_ba (track/tracker.hpp:55-57).  poses is updated in place; frame_ids pick the anchor.
 * With a communicator set (gsf_comm_init), each rank passes the full window and renders
 * only the keyframes it owns (k mod nranks == rank).  Per iteration one exchange: the loss, a
 * divergence flag and the window pose gradients in one fp64 all-reduce, the Gaussian gradients in
 * one fp32 all-reduce bucketed by parameter group (each group's Adam waits only for its bucket);
 * every rank returns the same map and all window poses. */
int gsf_sliding_ba(gsf_ctx ctx, const int32_t* slots, gsf_pose* poses, const int32_t* frame_ids,
                   int32_t n, const gsf_intrinsics* K, const gsf_tracker_cfg* tcfg,
                   const gsf_mapper_cfg* mcfg, int32_t iterations, double* trace);

/* initialize_map (map/mapper.hpp:84-87, mapper.cpp:125-148): replaces the context's map with
 * one backprojected primitive per init_stride-sampled valid-depth pixel of frame `slot` seen from
 * `pose` (row-major pixel order) and resets the optimizer state (a fresh MapState).  An empty
 * frame fails with GSF_ERUNTIME ("cannot initialize a map: first frame has no usable depth"). */
int gsf_initialize_map(gsf_ctx ctx, int32_t slot, const gsf_pose* pose, const gsf_intrinsics* K,
                       const gsf_mapper_cfg* mcfg, int64_t* count);

/* spawn_gaussians (map/mapper.hpp:89-93, mapper.cpp:150-170): appends one primitive per
 * spawn_stride-sampled pixel of frame `slot` with valid depth where the most recent render on
 * this context (the reference's `rendered` argument; same intrinsics) has accumulated opacity
 * below spawn_opacity_threshold.  Adam moments and densify statistics of the new primitives
 * start at zero. */
int gsf_spawn_gaussians(gsf_ctx ctx, int32_t slot, const gsf_pose* pose, const gsf_intrinsics* K,
                        const gsf_mapper_cfg* mcfg, int32_t* spawned);

/* render_reference (raster/rasterizer.hpp:24-28, rasterizer.cpp:263-296): the brute-force oracle
 * render — every pixel blends its whole depth-ordered list without early termination. */
int gsf_render_reference(gsf_ctx ctx, const gsf_pose* pose, const gsf_intrinsics* K, const float* observed_depth,
                         const gsf_raster_cfg* cfg, gsf_render_out* out);

/* save_checkpoint / load_checkpoint (io/checkpoint.hpp:16-20): the GSFMAP01 file of the context's
 * map with intrinsics K.  Loading replaces the map (a fresh MapState) and returns its intrinsics. */
int gsf_checkpoint_save(gsf_ctx ctx, const char* path, const gsf_intrinsics* K);
int gsf_checkpoint_load(gsf_ctx ctx, const char* path, gsf_intrinsics* K);

/* StructuralChange (map/mapper.hpp:66-70). */
typedef struct {
  int32_t split, cloned, removed;
} gsf_structural_change;

/* densify_and_cull (map/mapper.hpp:96-98, mapper.cpp:172-230) on the context's map and its
 * densification statistics: decisions on the device, the split offsets drawn on the host from the
 * map state's std::mt19937_64 (seeded with mcfg->seed the first time after the map state was
 * created: gsf_map_upload, gsf_initialize_map or gsf_optimizer_reset), one std::normal_distribution
 * per split parent, exactly as the reference.  gsf_map_step runs it every densify_interval
 * mapping iterations. */
int gsf_densify_and_cull(gsf_ctx ctx, const gsf_mapper_cfg* mcfg, gsf_structural_change* out);

/* MapState::grad_accum / grad_count (map/mapper.hpp:76-77): the densification statistics of the
 * context's map (count entries each). */
int gsf_map_stats_upload(gsf_ctx ctx, const double* grad_accum, const int32_t* grad_count);
int gsf_map_stats_download(gsf_ctx ctx, double* grad_accum, int32_t* grad_count);

/* accumulate_uncertainty / prune_unreliable (map/uncertainty.hpp:33-39).  Each view is
 * rendered on the device from (slot depth, pose). */
int gsf_accumulate_uncertainty(gsf_ctx ctx, const int32_t* slots, const gsf_pose* poses,
                               int32_t n, const gsf_intrinsics* K, const gsf_raster_cfg* rcfg,
                               int32_t* observed_count);
int gsf_prune_unreliable(gsf_ctx ctx, double tau, double reduced_opacity, int32_t* reduced);

/* ---- SLAM pipeline (slam/system.hpp, system.cpp:31-154) on the context's map ------------ */
typedef struct gsf_slam_s* gsf_slam;

/* RunConfig fields the pipeline reads (io/config.hpp:16-35). */
typedef struct {
  gsf_intrinsics intrinsics;
  gsf_tracker_cfg tracker;
  gsf_mapper_cfg mapper;      /* mapper.seed is replaced by `seed` (system.cpp:20-24) */
  int32_t map_iterations;     /* MapperConfig::iterations per keyframe window (60) */
  int32_t init_iterations;    /* MapperConfig::init_iterations of the bootstrap (120) */
  uint64_t seed;
} gsf_slam_cfg;

/* FrameLog (slam/system.hpp:17-34) plus the frame's trajectory pose.  The *_ms fields are
 * wall-clock milliseconds of each stage (device work included). */
typedef struct {
  int32_t frame;
  double timestamp;
  double track_loss;
  int32_t track_iterations, track_degraded, keyframe;
  int64_t primitives;
  double track_ms, map_ms, ba_ms, uncertainty_ms, spawn_ms;
  double kf_psnr_db, kf_depth_l1_cm;
  gsf_pose pose;
} gsf_frame_log;

/* SlamSystem over the context: the first processed frame bootstraps the map (initialize_map +
 * map_step(init_iterations)); every later frame is tracked from the constant-velocity prediction,
 * and every keyframe_interval-th frame runs map_step over the selected window, sliding_ba,
 * accumulate_uncertainty + prune_unreliable and spawn_gaussians.  Frames use device slot 0 and
 * keyframe k slot 1 + k of the context.  Host rgb (3*W*H) / depth (W*H) in stream order. */
int gsf_slam_create(gsf_ctx ctx, const gsf_slam_cfg* cfg, gsf_slam* out);
int gsf_slam_destroy(gsf_slam slam);
int gsf_slam_process(gsf_slam slam, int32_t index, double timestamp, const float* rgb, const float* depth,
                     gsf_frame_log* log);
int32_t gsf_slam_keyframes(gsf_slam slam);
int32_t gsf_slam_degraded_frames(gsf_slam slam);

/* ---- multi-GPU (keyframe-sharded sliding_ba) ----------------------------------------- */
/* Which window keyframes rank `rank` of `nranks` renders: out[i] = 1 if owned.  Pure host
 * logic, usable without a device (ctx may be NULL). */
int gsf_ba_partition(int32_t n, int32_t nranks, int32_t rank, uint8_t* owned);
int gsf_comm_unique_id(uint8_t id[128]);
/* NCCL communicator of a keyframe-sharded job (one context per GPU/rank); id from rank 0's
 * gsf_comm_unique_id, distributed by the caller. */
int gsf_comm_init(gsf_ctx ctx, int32_t nranks, int32_t rank, const uint8_t id[128]);
/* Host-staged communicator: the same sharded paths, with every sum-all-reduce staged through pinned
 * host memory and handed to the caller's callback (e.g. an MPI / gloo process group).  The callback
 * sums `count` elements of `dtype` in place across ranks and returns 0 on success. */
enum { GSF_DT_U32 = 3, GSF_DT_F32 = 7, GSF_DT_F64 = 8 };   /* ncclUint32 / ncclFloat32 / ncclFloat64 */
typedef int (*gsf_host_allreduce_fn)(void* buf, size_t count, int32_t dtype, void* user);
int gsf_comm_init_host(gsf_ctx ctx, int32_t nranks, int32_t rank, gsf_host_allreduce_fn fn, void* user);

#ifdef __cplusplus
}
#endif
#endif /* GSF_CUDA_H */
