// kernels.h — host-side launch wrappers of the sm_100a kernels and the device workspace.
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace gsfk {

// A window keyframe's pose, its Adam moments and its summed pose gradient (sliding_ba / map_step).
struct KfPose {
  double rot[3], trans[3];
  double m[6], v[6];
  double t;
  double grad[6];
};

// Keyframe bookkeeping folded into the chain's pose sum (mapping views): copy the view's pose
// gradient and loss out, and stage the next view's camera, without launches of their own.
struct PoseSumPost {
  KfPose* kf = nullptr;
  int grab = -1;              // keyframe whose grad receives d_pose (-1: none)
  double* loss_acc = nullptr; // += the view's total loss
  double* trace = nullptr;    // [trace_index] = the view's total loss (if trace_index >= 0)
  int trace_index = -1;
  int next = -1;              // keyframe whose camera becomes ds->cam (-1: none)
};

// Optional CUDA-event brackets around named kernels (bench / roofline evidence only).
struct Profiler {
  struct Mark { int name; cudaEvent_t a, b; };
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<Mark> pending;
  double total_ms[16] = {0};
  int64_t count[16] = {0};
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void begin(int name, cudaStream_t st) {
    if (!on) return;
    Mark m{name, get(), get()};
    cudaEventRecord(m.a, st);
    pending.push_back(m);
  }
  void end(cudaStream_t st) {
    if (!on || pending.empty()) return;
    cudaEventRecord(pending.back().b, st);
  }
  void resolve() {   // after a stream sync
    for (Mark& m : pending) {
      float ms = 0.0f;
      if (cudaEventElapsedTime(&ms, m.a, m.b) == cudaSuccess) {
        total_ms[m.name] += ms;
        count[m.name] += 1;
      }
      pool.push_back(m.a);
      pool.push_back(m.b);
    }
    pending.clear();
  }
};
enum ProfName { PROF_PREPROCESS = 0, PROF_SORT = 1, PROF_BLEND = 2, PROF_BACKWARD = 3, PROF_CHAIN = 4, PROF_SSIM = 5,
                PROF_ADAM = 6, PROF_BINNING = 7, PROF_POSEJAC = 8, PROF_NUM = 9 };

// Device workspace of one context.  Capacities grow on demand (never shrink).
struct Workspace {
  int64_t P_cap = 0, pair_cap = 0, npix_cap = 0, tiles_cap = 0;
  // tracking: k_posejac runs on a side branch beside the binning (fork after k_preprocess, join
  // before the blend); created with the context
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // tracking: longest-first CTA order of the tile kernels (k_lpt, from the previous iteration's
  // per-quadrant step counts) on a second side branch: fork after the backward, join before the
  // next blend.  Two buffers of [1 + 5 tiles_cap]: [0] = the tile count the orders were built for
  // (0 = none: identity order), then the blend's tile order, then the backward's quadrant order.
  cudaStream_t side2 = nullptr;
  cudaEvent_t ev_lfork = nullptr, ev_ljoin = nullptr;
  uint32_t* order = nullptr;    // 2 * (1 + 5 tiles_cap)
  int2* qstat = nullptr;        // 4 tiles_cap: per (tile, quadrant) forward (warp, entry) steps, list length
  // per primitive, id-indexed (written by k_preprocess for the visible ones)
  BlendG* bg_id = nullptr;
  GuardG* gg_id = nullptr;
  BlendG* bg_slot = nullptr;   // tracking: the same records indexed by visible slot (compact)
  GuardG* gg_slot = nullptr;
  uint32_t* sslot = nullptr;   // tracking: tile lists as visible slots (beside sid)
  // tracking: per (tile, quadrant) work list of the pose backward, written by k_blend_track's walk:
  // the visible slots of the entries whose footprint can reach the quadrant's 8x8 block, in list
  // order, at 4 start + q (end - start) (4 pair_cap); lastc = each pixel's last contributor as an
  // index into its quadrant's list (+1)
  uint32_t* qlist = nullptr;
  int32_t* lastc = nullptr;
  uint32_t* cand = nullptr;    // tracking: trust-region candidate ids (k_candidates)
  double* depth_id = nullptr;
  int4* rect_id = nullptr;
  uint8_t* visible = nullptr;
  float* pj_id = nullptr;       // P * kPjFloats: pose matrices of the visible primitives at their list slot
  uint32_t* pj_slot = nullptr;  // P: id -> slot of its pose Jacobian
  WorldG* world = nullptr;      // P: view-independent part, cached per tracked frame (k_world)
  double* support = nullptr;    // P: footprint support of the same cache (NaN = invalid primitive)
  // per tile: bins[t * kBinStride] = fill cursor of the tile's bucket (+ its list-start scan word at
  // +2), then the counters; one memset
  uint32_t* bins = nullptr;
  uint32_t* tile_fill = nullptr;
  uint32_t* bin_counters = nullptr;   // BinCounter slots
  uint32_t* big_ids = nullptr;        // P: primitives with more than kBigPairs tiles
  uint32_t* vis_list = nullptr;       // P: visible ids (any order): pose Jacobians, chain
  uint32_t* pair_base = nullptr;      // P: first primitive-major pair slot of a visible primitive
  int2* ranges = nullptr;
  double* loss_part = nullptr;  // rows * LS_NUM (+ group rows of the single-warp tracking blend)
  int loss_rows = 0;            // rows the last loss-partial producer wrote (tiles, or 4 tiles)
  // per (tile, primitive) pair: scattered keys/ids, then each tile's list sorted by (depth, id)
  unsigned long long* bucket = nullptr; // tiles * bucket_cap keys (fp32 depth bits << 32 | id), scatter order
  int64_t bucket_cap = 0;
  unsigned long long* skey = nullptr;   // the same keys, each tile's list in (depth, id) order
  uint32_t* sid = nullptr;
  float* partials = nullptr;   // pair_cap * 10, primitive-major: pair_base[id] + rectangle index
  // per pixel (render outputs + backward inputs)
  float* color = nullptr;      // 3*npix, interleaved
  float* alpha_depth = nullptr;
  float* median_depth = nullptr;
  uint8_t* median_valid = nullptr;
  float* opacity = nullptr;
  float* uncertainty = nullptr;
  float* final_T = nullptr;
  int32_t* count = nullptr;
  int32_t* dominant = nullptr;
  int32_t* median_prim = nullptr;
  float* dominant_w = nullptr;
  int32_t* last = nullptr;
  uint8_t* pxcode = nullptr;     // tracking: per pixel, the signs of the loss seeds (pixel_seed_code)
  uint32_t* fix_list = nullptr;  // render API: pixels flagged for the exact-decision fix-up (k_pixel_fixup)
  float* obs = nullptr;         // observed depth of the API render (npix)
  float* upstream = nullptr;    // explicit upstream maps for gsf_render_backward (7*npix)
  float* dssim = nullptr;       // 3*npix: d(w_ssim * ssim loss)/d colour (mapping)
  float* ssim_tmp = nullptr;    // SSIM scratch maps (see loss.cu)
  // temporaries
  float* qpart = nullptr;       // [pair][4 quadrants][10] partials of k_backward_q (k_pair_combine folds them)
  uint32_t* qflag = nullptr;    // per pair: 4 bytes, quadrant q's slot written (k_backward_q -> k_pair_combine)
  double* pose_part = nullptr;  // chain blocks * 6 (or 4 tiles * 6 + group rows for the tracking backward)
  uint32_t* wtickets = nullptr; // zeroed group tickets of the single-warp grid reductions (self-resetting)
  int64_t wtickets_half = 0;    // entries per region: [0, half) blend, [half, 2 half) backward
  double* red_part = nullptr;   // generic per-block fp64 partials (ssim, then iso)
  int64_t red_iso_offset = 0;
  int ssim_blocks = 0, iso_blocks = 0;
  Profiler* prof = nullptr;
};

// binning.cu
void run_binning(Workspace& ws, DevState* ds, int64_t P, int tiles_x, int ntiles, cudaStream_t st, int64_t* launches,
                 bool want_slots = false, bool any_order = false);

// raster_fwd.cu
struct FwdArgs {
  const float* params;   // [D][P]
  int64_t P;
  int32_t K;
  RasterParams rp;
  BlendConsts kc;
  int32_t W, H;
  double near_plane, far_plane;
  const float* obs;          // observed depth for the U map (nullable)
  const float* loss_rgb;     // target colour for the fused loss epilogue (nullable)
  const float* loss_depth;   // sensor depth for the loss masks (nullable)
  LossParams lp;
  int iteration;             // loop iteration (for device-side checks), -1 outside loops
  bool want_posejac = false; // tracking: emit the per-primitive pose Jacobians (ws.pj_id)
  bool keep_maps = true;     // tracking loop: colour / alpha depth / opacity maps are not read back
  // k_blend_track's outputs for the two-pixel pose backward: 0 = last contributor as a list index
  // (ws.last) only, 1 = the per-quadrant work lists (ws.qlist) + ws.lastc only (inside the tracking
  // loop), 2 = both (gsf_tracking_gradient, whose render stays the context's latest)
  int qmode = 0;
  bool bins_clean = false;   // tracking loop: the previous iteration's blend re-zeroed the bins (no memset)
  bool clean_bins = false;   // tracking loop: the blend re-zeroes the bins once the binning is consumed
  bool fuse_loss_final = false;  // tracking: the blend's last CTA runs the loss finalize
  bool use_world = false;        // preprocess from ws.world / ws.support (run_world ran for this map)
  const uint32_t* cand = nullptr;  // tracking: candidate ids (run_candidates), used while ds->cand_ok
  bool want_pair_base = true;    // primitive-major pair slots for a parameter-gradient backward
  const uint32_t* order = nullptr;  // tracking: CTA order buffer (Workspace::order half) of the blend
  bool join_order = false;          // wait for the k_lpt branch (ws.ev_ljoin) before the blend
};
void run_forward(Workspace& ws, DevState* ds, const FwdArgs& a, cudaStream_t st, int64_t* launches);
// per-primitive validation + view-independent cache (ws.world, ws.support)
void run_world(Workspace& ws, DevState* ds, const float* params, int64_t P, const RasterParams& rp, cudaStream_t st,
               int64_t* launches);
// trust-region candidate list of the tracking loop (once per frame, after run_world, at its first camera)
void run_candidates(Workspace& ws, DevState* ds, const float* params, int64_t P, const RasterParams& rp,
                    double theta_max, double dist_max, cudaStream_t st, int64_t* launches);
// tracking: longest-first CTA orders for the next iteration (ws.qstat -> out, a Workspace::order half)
void run_lpt(Workspace& ws, int ntiles, uint32_t* out, cudaStream_t st, int64_t* launches);
void run_loss_tiles(Workspace& ws, int mode, const float* rgb, const float* depth, bool has_unc, int W, int H,
                    double near_plane, double far_plane, float floor, cudaStream_t st, int64_t* launches);

// raster_bwd.cu
enum SeedMode { SEED_EXPLICIT = 0, SEED_TRACK = 1, SEED_MAP = 2 };
struct BwdArgs {
  const float* params;
  int64_t P;
  int32_t K;
  RasterParams rp;
  BlendConsts kc;
  int32_t W, H;
  double near_plane, far_plane;
  const float* obs;          // sensor depth (U map gradient / loss masks), nullable
  const float* target_rgb;   // loss target (tracking/mapping seeds)
  const float* up_color;     // explicit seeds (SEED_EXPLICIT), nullable each
  const float* up_adepth;
  const float* up_mdepth;
  const float* up_opacity;
  const float* up_uncert;
  LossParams lp;
  int seed_mode;
  bool pose_only;            // tracking: skip per-primitive parameter gradients
  bool fused_pose = false;   // pose_only + ws.pj_id valid: pose through per-primitive Jacobians
  int update_iter = -1;      // >= 0: the tracking backward's last CTA also takes this iteration's pose step
  const uint32_t* order = nullptr;  // tracking: CTA order buffer (Workspace::order half) of the pose backward
  float* grads;              // [D][P] parameter gradients (full mode)
  double iso_w = 0.0;        // > 0: k_chain also adds the iso term's direct log-scale gradient (losses.cpp:272-280)
  PoseSumPost post;          // mapping views: k_pose_sum's keyframe bookkeeping
  double iso_eps = 0.0;
  float* d_mean2d;           // [2][P] (full mode, nullable)
};
// true when the backward also ran the pose step of a.update_iter (k_track_update is then skipped)
bool run_backward(Workspace& ws, DevState* ds, const BwdArgs& a, cudaStream_t st, int64_t* launches);
// seed maps (3 colour planes interleaved, then ad, md, u planes) of the last render's loss
void run_seeds_out(Workspace& ws, DevState* ds, int mode, const float* target, const float* depth, const LossParams& lp,
                   int W, int H, double near_plane, double far_plane, float* out, cudaStream_t st, int64_t* launches);

// loss.cu
void run_loss_finalize(Workspace& ws, DevState* ds, const LossParams& lp, int tiles, int64_t npix, int iteration,
                       cudaStream_t st, int64_t* launches);
void run_ssim(Workspace& ws, DevState* ds, const float* x, const float* y, int W, int H, float weight_grad,
              float* d_out, cudaStream_t st, int64_t* launches);
void run_iso(Workspace& ws, DevState* ds, const float* params, int64_t P, double w_iso, double eps, float* grads,
             cudaStream_t st, int64_t* launches);

// optim.cu
struct AdamGroups {
  double lr[5];   // mean, log_scale, quat, opacity, sh
};
void run_adam(float* params, const float* grads, float* m, float* v, int64_t P, int D, const AdamGroups& g, double step,
              cudaStream_t st, int64_t* launches);
// Adam over the fields [f0, f1) of the SoA map only (the per-group buckets of a sharded sliding_ba)
void run_adam_fields(float* params, const float* grads, float* m, float* v, int64_t P, int f0, int f1,
                     const AdamGroups& g, double step, cudaStream_t st, int64_t* launches);
void run_track_update(DevState* ds, int iteration, cudaStream_t st, int64_t* launches);

// densify.cu (mapper.cpp:172-230, 261-269)
void run_densify_stats(const uint8_t* visible, const float* d_mean2d, double* accum, int32_t* cnt, int64_t P, int W, int H,
                       cudaStream_t st, int64_t* launches);
void run_densify_codes(const float* params, int64_t P, const double* accum, const int32_t* cnt, double cull_opacity,
                       double grad_threshold, double size_boundary, uint8_t* code, cudaStream_t st, int64_t* launches);
void run_densify_build(const float* params, const float* m, const float* v, const double* nu, const uint8_t* observed,
                       int64_t P_old, int D, const int32_t* src, const uint8_t* kind, const int32_t* zidx, const double* z,
                       double log_split, int64_t P_new, float* params_n, float* m_n, float* v_n, double* nu_n,
                       uint8_t* observed_n, cudaStream_t st, int64_t* launches);

// spawn.cu: initialize_map / spawn_gaussians candidates (one per stride-sampled pixel)
struct BackprojectArgs {
  const float* depth;     // sensor depth of the frame (W*H)
  const float* rgb;       // frame colour, interleaved (3*W*H)
  const float* opacity;   // current render's accumulated opacity (spawn) or nullptr (initialize)
  double threshold;       // spawn_opacity_threshold
  double fx, fy, cx, cy, near_plane, far_plane;
  double Rinv[9], tinv[3];   // pose.inverse(): exp(-rot), -(R^T t)
  double logit0;          // logit(init_opacity)
  int W, H, stride, K;
  int cells_x;
  int64_t cells;
};
int64_t run_backproject_count(const BackprojectArgs& a, uint32_t* blk_cnt, uint32_t* blk_off, uint32_t* total,
                              cudaStream_t st, int64_t* launches);
void run_backproject_write(const BackprojectArgs& a, const uint32_t* blk_off, int64_t P_old, int64_t P_new, float* params,
                           double* nu, uint8_t* observed, cudaStream_t st, int64_t* launches);

// uncert.cu
void run_uncertainty_view(const Workspace& ws, const float* params, int64_t P, const float* obs, int W, int H,
                          double near_plane, double far_plane, const DevState* ds, double* sum, uint32_t* cnt,
                          cudaStream_t st, int64_t* launches);
void run_uncertainty_finalize(const double* sum, const uint32_t* cnt, double* nu, uint8_t* observed, int64_t P,
                              uint32_t* observed_count, cudaStream_t st, int64_t* launches);
void run_prune(const double* nu, float* opacity_logit, int64_t P, double tau, float target, uint32_t* reduced,
               cudaStream_t st, int64_t* launches);

}  // namespace gsfk
