/* gsf_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU fp64 restatement of the reference hot path (/root/reference/proj, "gsfield"), used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.  It is
 * never linked into, loaded by or called from the product (paper_2403_16095_b200/).
 *
 * Every function cites the reference file:line it restates.  Parity of this restatement
 * is pinned by the reference's own known-answer tests (tests/golden/, tests/test_oracle_*.py)
 * and by finite-difference gradient checks (verify/gradcheck.cpp:47-128 restated).
 */
#ifndef GSF_ORACLE_H
#define GSF_ORACLE_H

#include "../include/gsf_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_result orc_result;      /* RenderResult (raster/output.hpp:47-50) */
typedef struct orc_mapstate orc_mapstate;  /* MapState (map/mapper.hpp:113-123) */

typedef struct {
  double* color; double* alpha_depth; double* median_depth; uint8_t* median_valid;
  double* opacity; double* uncertainty; double* final_transmittance; int32_t* per_pixel_count;
  int32_t* dominant; int32_t* median_prim; double* dominant_weight; uint8_t* visible;
  int32_t has_uncertainty;
} orc_maps;

typedef struct {
  const double* d_color; const double* d_alpha_depth; const double* d_median_depth;
  const double* d_opacity; const double* d_uncertainty;
} orc_upstream;

typedef struct {
  double* d_mean; double* d_log_scale; double* d_quat; double* d_opacity_logit; double* d_sh;
  double* d_mean2d; double d_pose[6];
} orc_grads;

const char* orc_last_error(void);
int orc_threads(void);   /* OpenMP threads used by the parallel loops (the reference's parallel_for) */

/* render / render_reference (rasterizer.cpp:168-296).  brute_force selects render_reference. */
int orc_render(const gsf_map_host* map, const gsf_pose* pose, const gsf_intrinsics* K,
               const double* observed_depth, const gsf_raster_cfg* cfg, int brute_force,
               orc_result** out);
void orc_result_free(orc_result* r);
int orc_result_maps(const orc_result* r, orc_maps* out);
int64_t orc_result_record_total(const orc_result* r);
int orc_result_record(const orc_result* r, uint32_t* row_start, int32_t* prim, double* alpha,
                      double* transmittance);

/* render_backward (rasterizer.cpp:339-572) over r's record. */
int orc_render_backward(const gsf_map_host* map, const gsf_pose* pose, const gsf_intrinsics* K,
                        const orc_result* r, const orc_upstream* up, const double* observed_depth,
                        const gsf_raster_cfg* cfg, orc_grads* out);

/* evaluate_tracking_loss (losses.cpp:284-339) / evaluate_mapping_loss (losses.cpp:156-282).
 * Seed outputs may be NULL.  d_log_scale_direct is 3*P (zeros when the iso term is off). */
int orc_tracking_loss(const orc_result* r, const double* target_rgb, const double* observed_depth,
                      const gsf_intrinsics* K, const gsf_loss_weights* w, gsf_loss_terms* out,
                      double* d_color, double* d_alpha_depth);
int orc_mapping_loss(const gsf_map_host* map, const orc_result* r, const double* target_rgb,
                     const double* observed_depth, const gsf_intrinsics* K,
                     const gsf_loss_weights* w, gsf_loss_terms* out, double* d_color,
                     double* d_alpha_depth, double* d_median_depth, double* d_uncertainty,
                     double* d_log_scale_direct);
/* ssim / ssim_with_gradient (ssim.cpp:110-195).  d_x may be NULL. */
int orc_ssim(const double* x, const double* y, int w, int h, double* value, double* d_x);

/* AdamState::step (adam.cpp:40-53) on a flat array; m, v, t are caller state. */
void orc_adam_step(double* params, const double* grads, double* m, double* v, int64_t n,
                   uint64_t* t, double lr, double beta1, double beta2, double eps);

/* track_frame (tracker.cpp:30-84).  rgb 3*W*H, depth W*H. */
int orc_track_frame(const gsf_map_host* map, const double* rgb, const double* depth,
                    const gsf_pose* initial, const gsf_intrinsics* K, const gsf_tracker_cfg* tcfg,
                    const gsf_loss_weights* w, const gsf_raster_cfg* rcfg, gsf_track_result* out);

/* MapState + map_step (mapper.cpp:232-281) + sliding_ba (tracker.cpp:119-183). */
int orc_mapstate_create(const gsf_map_host* map, const gsf_mapper_cfg* mcfg, orc_mapstate** out);
void orc_mapstate_free(orc_mapstate* s);
int64_t orc_mapstate_count(const orc_mapstate* s);
int orc_mapstate_get(const orc_mapstate* s, gsf_map_host* out);
int orc_map_step(orc_mapstate* s, int n, const double* const* rgbs, const double* const* depths,
                 const gsf_pose* poses, const gsf_intrinsics* K, const gsf_mapper_cfg* mcfg,
                 int iterations, double* trace);
int orc_sliding_ba(orc_mapstate* s, int n, const double* const* rgbs, const double* const* depths,
                   gsf_pose* poses, const int32_t* frame_ids, const gsf_intrinsics* K,
                   const gsf_tracker_cfg* tcfg, const gsf_mapper_cfg* mcfg, int iterations,
                   double* trace);

/* accumulate_uncertainty / prune_unreliable (uncertainty.cpp:17-100).  The map's
 * uncertainty/observed arrays are updated in place. */
int orc_mapstate_put(orc_mapstate* st, const gsf_map_host* map);
int orc_mapstate_append(orc_mapstate* st, const gsf_map_host* map);
int orc_mapstate_set_stats(orc_mapstate* st, const double* accum, const int32_t* count);
int orc_mapstate_densify(orc_mapstate* st, const gsf_mapper_cfg* cfg, int32_t* change);
int orc_backproject(const double* rgb, const double* depth, const double* opacity, const gsf_pose* pose,
                    const gsf_intrinsics* K, const gsf_mapper_cfg* cfg, int stride, gsf_map_host* out, int64_t* count);
int orc_uncertainty_partials(const gsf_map_host* map, int n, const orc_result* const* records,
                             const double* const* depths, const gsf_pose* poses, const gsf_intrinsics* K,
                             double* sum_out, int32_t* count_out);
int orc_accumulate_uncertainty(gsf_map_host* map, int n, const orc_result* const* records,
                               const double* const* depths, const gsf_pose* poses,
                               const gsf_intrinsics* K, int32_t* observed_count);
int orc_prune_unreliable(gsf_map_host* map, double tau, double reduced_opacity, int32_t* reduced);

/* Gradient check with a linear probe objective (gradcheck.cpp:47-128 + test_gradients.cpp:17-61).
 * probe maps: color 3HW, depth/opacity/uncert/median HW (uncert may be NULL). */
typedef struct { int32_t total, checked, skipped; double max_rel_err, worst_analytic, worst_fd; int32_t worst_index; } orc_gradcheck_report;
int orc_gradcheck_linear(const gsf_map_host* map, const gsf_pose* pose, const gsf_intrinsics* K,
                         const gsf_raster_cfg* cfg, const double* observed_depth,
                         const double* a_color, const double* a_depth, const double* a_opacity,
                         const double* a_uncert, const double* a_median, double step,
                         double denom_floor, orc_gradcheck_report* rep);

/* Test fixtures (tests/test_utils.hpp:13-65): random_scene with std::mt19937(seed). */
int orc_random_scene(uint32_t seed, int count, int sh_coeffs, double max_opacity, double min_scale,
                     double max_scale, gsf_map_host* out);
void orc_wavy_depth(int w, int h, double base, int hole_every, double* out);

/* Config defaults of the reference structs. */
void orc_default_raster(gsf_raster_cfg* c);
void orc_default_weights(gsf_loss_weights* w, int handheld_real);
void orc_default_tracker(gsf_tracker_cfg* c);
void orc_default_mapper(gsf_mapper_cfg* c);

/* fp32 mirror of the device decision path (mirror.cpp): bit-exact reference for tile keys,
 * sort order, tile ranges, per-pixel counts and ids of the CUDA kernels, which share its
 * arithmetic through paper_2403_16095_b200/csrc/gsf_shared.cuh. */
typedef struct {
  uint8_t* visible;        /* P */
  int32_t* rank_to_id;     /* V (depth order) */
  int32_t* tile_range;     /* 2*num_tiles: [start, end) into the sorted pair list */
  int32_t* pair_rank;      /* sorted pair list entries (rank), capacity given below */
  int64_t pair_capacity;
  float* color; float* alpha_depth; float* median_depth; uint8_t* median_valid; float* opacity;
  float* uncertainty; float* final_transmittance; int32_t* per_pixel_count; int32_t* dominant;
  int32_t* median_prim; float* dominant_weight; int32_t* last_index;
  int64_t num_visible, num_pairs;
  int64_t num_flagged;     /* pixels re-blended by the exact-decision fix-up */
} mir_out;
int mir_render(const gsf_map_host* map, const gsf_pose* pose, const gsf_intrinsics* K,
               const float* observed_depth, const gsf_raster_cfg* cfg, mir_out* out);

#ifdef __cplusplus
}
#endif
#endif
