// finalize.cuh — block-level tails shared by the stand-alone finalize kernels and the
// "last CTA done" epilogues of k_blend / k_backward_pose (tracking loop).
//
//   block_reduce_rows   fixed-order sum of a [rows][NV] fp64 partial array by one 256-thread CTA
//   loss_scalars        losses.cpp:284-339 / :156-282 scalar tails + the loop checks of
//                       track_frame (tracker.cpp:45-60) and map_step (mapper.cpp:247-254)
//   track_update        tracker.cpp:62-70: pose Adam, CameraPose::perturbed, next camera
//   last_cta            grid-wide ticket: true in exactly one CTA, after every CTA's writes
#pragma once

#include "common.cuh"

namespace gsfk {

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// out[0..NV) (shared) = column sums of part[rows][NV]; thread t owns rows t, t+NT, ... so the
// summation order is fixed.  Requires blockDim.x == NT; ends with a __syncthreads().
template <int NV, int NT = 256>
__device__ __forceinline__ void block_reduce_rows(const double* part, int rows, double* out, double (*s_red)[NV]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
#pragma unroll 4
  for (int r = tid; r < rows; r += NT) {
    const double* row = part + static_cast<int64_t>(r) * NV;
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] += __ldcg(row + q);
  }
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double t = warp_sum_f64(acc[q]);
    if (lane == 0) s_red[warp][q] = t;
  }
  __syncthreads();
  if (tid < NV) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) t += s_red[w][tid];
    out[tid] = t;
  }
  __syncthreads();
}

// One CTA of the grid returns true, after all CTAs have called this; the global writes of the
// threads that pass wrote=true are visible to it (only they pay for the fence, so the CTA's other
// output stores do not stall its exit).  `counter` must be zero before the launch; the last CTA
// re-zeroes it.
__device__ __forceinline__ bool last_cta(uint32_t* counter, int* s_flag, bool wrote) {
  if (wrote) __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const bool last = atomicAdd(counter, 1u) == gridDim.x - 1;
    if (last) *counter = 0u;   // no other CTA touches it any more: ready for the next launch
    *s_flag = last ? 1 : 0;
  }
  __syncthreads();
  if (*s_flag) __threadfence();
  return *s_flag != 0;
}

// Two-level fixed-order reduction for grids of single-warp CTAs (blockDim.x == 32): CTA r wrote
// row part[r][NV] (r = row, default blockIdx.x).  The last CTA of each group of 32 consecutive rows sums the group (lane l takes
// row l, then a fixed shuffle tree) into gpart[g]; the last group sums gpart the same way.  Returns
// true in exactly one CTA, whose lane 0 then holds the totals in out[NV].  gt[] (one ticket per
// group) and *top must be zero before the launch; they are re-zeroed here.
template <int NV>
__device__ __forceinline__ bool warp_grid_reduce(const double* part, double* gpart, int rows, uint32_t* gt, uint32_t* top,
                                                 double* out, bool wrote, int row = -1) {
  const int lane = threadIdx.x & 31;
  const int r = row >= 0 ? row : static_cast<int>(blockIdx.x), g = r >> 5, g0 = g << 5, gn = min(32, rows - g0);
  const int ngroups = (rows + 31) >> 5;
#ifdef GSF_RELEASE_TICKET
  // the row's writer publishes it with a release RMW on the group ticket (no full SC fence)
  __syncwarp();
  unsigned last = 0;
  if (lane == 0) {
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&gt[g]) : "memory");
    last = prev == static_cast<unsigned>(gn - 1);
    if (last) gt[g] = 0u;
  }
  (void)wrote;
#else
  if (wrote) __threadfence();
  __syncwarp();
  unsigned last = 0;
  if (lane == 0) {
    last = atomicAdd(&gt[g], 1u) == static_cast<unsigned>(gn - 1);
    if (last) gt[g] = 0u;
  }
#endif
  if (!__shfl_sync(0xffffffffu, last, 0)) return false;
  __threadfence();
  double v[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = lane < gn ? __ldcg(part + static_cast<int64_t>(g0 + lane) * NV + q) : 0.0;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum_f64(v[q]);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) gpart[static_cast<int64_t>(g) * NV + q] = v[q];
    __threadfence();
    last = atomicAdd(top, 1u) == static_cast<unsigned>(ngroups - 1);
    if (last) *top = 0u;
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return false;
  __threadfence();
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = 0.0;
  for (int i = lane; i < ngroups; i += 32)
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] += __ldcg(gpart + static_cast<int64_t>(i) * NV + q);
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    v[q] = warp_sum_f64(v[q]);
    if (lane == 0) out[q] = v[q];
  }
  return true;
}

// Scalar tails of the tracking (mode 1) and mapping (mode 2) losses; thread 0 only.
static __device__ __noinline__ void loss_scalars(DevState* ds, const LossParams& lp, const double* tot, double ssim_sum, double iso_sum,
                                    int64_t npix, int iteration) {
  if (ds->halt) return;
  for (int q = 0; q < LS_NUM; ++q) ds->loss[q] = tot[q];
  const double hw = static_cast<double>(npix);
  const bool nbv = lp.normalize_by_valid != 0;
  const double cc = tot[LS_COLOR_CNT], cg = tot[LS_GEO_CNT], ca = tot[LS_ALIGN_CNT], cv = tot[LS_VAR_CNT];
  if (lp.mode == 1) {
    const double color = cc > 0.0 ? tot[LS_COLOR_SUM] / (3.0 * (nbv ? cc : hw)) : 0.0;
    const double geo = cg > 0.0 ? tot[LS_GEO_SUM] / (nbv ? cg : hw) : 0.0;
    const double total = lp.t_color * color + lp.t_geo * geo;
    const double m_color = nbv ? cc : hw, m_geo = nbv ? cg : hw;
    ds->term_color = color;
    ds->term_geo = geo;
    ds->term_align = ds->term_var = ds->term_ssim = ds->term_iso = 0.0;
    ds->loss_total = total;
    ds->seed_color = (lp.t_color > 0.0 && m_color > 0.0) ? lp.t_color / (3.0 * m_color) : 0.0;
    ds->seed_geo = (lp.t_geo > 0.0 && m_geo > 0.0) ? lp.t_geo / m_geo : 0.0;
    ds->any_empty = (cc == 0.0 || cg == 0.0) ? 1 : 0;
    if (iteration == 0) {
      ds->initial_loss = total;
      if (cc == 0.0 && cg == 0.0) {   // tracker.cpp:46-53
        ds->halt = 1;
        ds->halt_iter = 0;
        ds->final_loss = total;
        ds->degraded = 1;
        return;
      }
    }
    if (iteration >= 0 && !isfinite(total)) {   // tracker.cpp:55-60
      ds->halt = 2;
      ds->halt_iter = iteration;
    }
  } else if (lp.mode == 2) {
    bool warn = false;
    const double color = hw > 0.0 ? tot[LS_COLOR_SUM] / (3.0 * hw) : 0.0;
    auto masked = [&](double sum, double c) {
      if (c == 0.0) { warn = true; return 0.0; }
      return sum / (nbv ? c : hw);
    };
    const double geo = masked(tot[LS_GEO_SUM], cg);
    const double align = masked(tot[LS_ALIGN_SUM], ca);
    double var = 0.0;
    if (ds->has_obs) var = masked(tot[LS_VAR_SUM], cv);
    else warn = true;
    const double ssim = lp.w_ssim > 0.0 ? 1.0 - ssim_sum / (3.0 * hw) : 0.0;
    const double iso = ds->V > 0 ? iso_sum / static_cast<double>(ds->V) : 0.0;
    const double total = lp.w_color * color + lp.w_ssim * ssim + lp.w_geo * geo + lp.w_align * align + lp.w_iso * iso +
                         lp.w_var * var;
    const double m_geo = nbv ? cg : hw, m_align = nbv ? ca : hw, m_var = nbv ? cv : hw;
    ds->term_color = color;
    ds->term_geo = geo;
    ds->term_align = align;
    ds->term_var = var;
    ds->term_ssim = ssim;
    ds->term_iso = iso;
    ds->loss_total = total;
    ds->any_empty = warn ? 1 : 0;
    ds->seed_color = lp.w_color > 0.0 ? lp.w_color / (3.0 * hw) : 0.0;
    ds->seed_geo = (lp.w_geo > 0.0 && m_geo > 0.0) ? lp.w_geo / m_geo : 0.0;
    ds->seed_align = (lp.w_align > 0.0 && m_align > 0.0) ? lp.w_align / m_align : 0.0;
    ds->seed_var = (lp.w_var > 0.0 && ds->has_obs && m_var > 0.0) ? lp.w_var / m_var : 0.0;
    if (iteration >= 0 && !isfinite(total)) {
      ds->halt = 2;
      ds->halt_iter = iteration;
    }
  }
}

// log_map (lie.cpp:30-52)
__device__ inline void log_map_dev(const double* R, double* out) {
  const double trace = R[0] + R[4] + R[8];
  double ct = (trace - 1.0) * 0.5;
  ct = ct < -1.0 ? -1.0 : (ct > 1.0 ? 1.0 : ct);
  const double theta = acos(ct);
  const double vee[3] = {R[7] - R[5], R[2] - R[6], R[3] - R[1]};
  if (theta < 1e-8) {
    const double f = 0.5 * (1.0 + theta * theta / 6.0);
    for (int i = 0; i < 3; ++i) out[i] = f * vee[i];
    return;
  }
  if (theta > 3.14159265358979323846 - 1e-3) {
    double outer[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) outer[3 * i + j] = (0.5 * (R[3 * i + j] + R[3 * j + i]) - ct * (i == j ? 1.0 : 0.0)) / (1.0 - ct);
    int a = 0;
    for (int i = 1; i < 3; ++i)
      if (outer[4 * i] > outer[4 * a]) a = i;
    const double sq = sqrt(outer[4 * a]);
    double ax[3] = {outer[0 * 3 + a] / sq, outer[1 * 3 + a] / sq, outer[2 * 3 + a] / sq};
    if (ax[0] * vee[0] + ax[1] * vee[1] + ax[2] * vee[2] < 0.0)
      for (int i = 0; i < 3; ++i) ax[i] = -ax[i];
    for (int i = 0; i < 3; ++i) out[i] = theta * ax[i];
    return;
  }
  const double f = theta / (2.0 * sin(theta));
  for (int i = 0; i < 3; ++i) out[i] = f * vee[i];
}

// tracker.cpp:62-70 on the device; thread 0 only.  bc1/bc2 = 1 - beta^t come from the host
// (std::pow, as adam.cpp computes them); the current rotation is the camera's W = exp(rot).
// Every DevState read is issued before any write so the chain is not serialised on memory.
static __device__ __noinline__ void track_update(DevState* ds, int iteration, double bc1, double bc2) {
  if (ds->halt) return;
  double g[6], m[6], v[6], trans[3], Rc[9];
  for (int a = 0; a < 6; ++a) { g[a] = ds->d_pose[a]; m[a] = ds->adam_m[a]; v[a] = ds->adam_v[a]; }
  for (int a = 0; a < 3; ++a) trans[a] = ds->pose_trans[a];
  for (int a = 0; a < 9; ++a) Rc[a] = ds->cam.W[a];
  const double lr_rot = ds->lr_rot, lr_trans = ds->lr_trans;
  const double fx = ds->cam.fx, fy = ds->cam.fy, cx = ds->cam.cx, cy = ds->cam.cy;
  const double nearp = ds->cam.near_plane, farp = ds->cam.far_plane;
  const int width = ds->cam.width, height = ds->cam.height;
  const double t = ds->adam_t + 1.0;
  double delta[6];
  for (int a = 0; a < 6; ++a) {
    m[a] = 0.9 * m[a] + (1.0 - 0.9) * g[a];
    v[a] = 0.999 * v[a] + (1.0 - 0.999) * g[a] * g[a];
    const double lr = a < 3 ? lr_rot : lr_trans;
    delta[a] = 0.0 - lr * (m[a] / bc1) / (sqrt(v[a] / bc2) + 1e-8);
  }
  // perturbed(): R <- exp(d_rot) R, t <- exp(d_rot) t + d_trans
  double dR[9], Rn[9];
  exp_map_d(delta, dR);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Rn[3 * i + j] = dR[3 * i + 0] * Rc[0 * 3 + j] + dR[3 * i + 1] * Rc[1 * 3 + j] + dR[3 * i + 2] * Rc[2 * 3 + j];
  double tn[3];
  for (int i = 0; i < 3; ++i) tn[i] = dR[3 * i + 0] * trans[0] + dR[3 * i + 1] * trans[1] + dR[3 * i + 2] * trans[2] + delta[3 + i];
  double rn[3];
  log_map_dev(Rn, rn);
  const Cam nc = make_cam(rn, tn, fx, fy, cx, cy, width, height, nearp, farp);
  ds->adam_t = t;
  for (int a = 0; a < 6; ++a) { ds->adam_m[a] = m[a]; ds->adam_v[a] = v[a]; }
  for (int i = 0; i < 3; ++i) {
    ds->pose_rot[i] = rn[i];
    ds->pose_trans[i] = tn[i];
  }
  ds->iterations_run = iteration + 1;
  ds->cam = nc;
  if (ds->cand_ok) {   // leave the trust region -> later iterations preprocess every primitive
    // p' = Q p + (t' - Q t0) with Q = W' W0^T: |p' - p| <= angle(Q) |p| + |t' - Q t0|
    double tr = 0.0, u[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < 9; ++a) tr += nc.W[a] * ds->cand_W0[a];
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) u[j] += ds->cand_W0[3 * i + j] * ds->cand_t0[i];
    double d2 = 0.0;
    for (int i = 0; i < 3; ++i) {
      const double e = nc.t[i] - (nc.W[3 * i] * u[0] + nc.W[3 * i + 1] * u[1] + nc.W[3 * i + 2] * u[2]);
      d2 += e * e;
    }
    if (!(0.5 * (tr - 1.0) >= ds->cand_cos_min) || !(sqrt(d2) <= ds->cand_dist_max)) ds->cand_ok = 0;
  }
}

}  // namespace gsfk
