// optim.cu — fused Adam over the SoA map, the fp64 pose update of track_frame, densify stats.
//
//   k_adam          AdamState::step (adam.cpp:40-53) for all five parameter groups of
//                   PrimitiveOptimizer::step (mapper.cpp:72-117) in one pass over [D][P]; fp32
//                   storage, fp64 arithmetic, dense over every entry like the reference.
//   k_track_update  tracker.cpp:62-70: the two pose AdamStates on zero-initialised deltas, then
//                   CameraPose::perturbed (pose.hpp:44-48) and the next iteration's camera, all
//                   on the device so a whole track_frame can be one CUDA graph.
//   k_densify_stats mapper.cpp:261-269 (screen-space gradient norms in NDC units).
#include "kernels.h"

namespace gsfk {

namespace {

__global__ void __launch_bounds__(256) k_adam(float* __restrict__ params, const float* __restrict__ grads,
                                              float* __restrict__ m, float* __restrict__ v, int64_t P, int D, AdamGroups g,
                                              double bc1, double bc2) {
  const int64_t n = static_cast<int64_t>(D) * P;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int f = static_cast<int>(i / P);
    const int grp = f < 3 ? 0 : (f < 6 ? 1 : (f < 10 ? 2 : (f < 11 ? 3 : 4)));
    const double gr = grads[i];
    const double mm = 0.9 * static_cast<double>(m[i]) + (1.0 - 0.9) * gr;
    const double vv = 0.999 * static_cast<double>(v[i]) + (1.0 - 0.999) * gr * gr;
    m[i] = static_cast<float>(mm);
    v[i] = static_cast<float>(vv);
    const double upd = g.lr[grp] * (mm / bc1) / (sqrt(vv / bc2) + 1e-8);
    params[i] = static_cast<float>(static_cast<double>(params[i]) - upd);
  }
}

// log_map (lie.cpp:30-52)
__device__ void log_map_dev(const double* R, double* out) {
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
  if (theta > M_PI - 1e-3) {
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

__global__ void k_track_update(DevState* ds, int iteration) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (ds->halt) return;
  ds->adam_t += 1.0;
  const double bc1 = 1.0 - pow(0.9, ds->adam_t);
  const double bc2 = 1.0 - pow(0.999, ds->adam_t);
  double delta[6];
  for (int a = 0; a < 6; ++a) {
    const double g = ds->d_pose[a];
    ds->adam_m[a] = 0.9 * ds->adam_m[a] + (1.0 - 0.9) * g;
    ds->adam_v[a] = 0.999 * ds->adam_v[a] + (1.0 - 0.999) * g * g;
    const double lr = a < 3 ? ds->lr_rot : ds->lr_trans;
    delta[a] = 0.0 - lr * (ds->adam_m[a] / bc1) / (sqrt(ds->adam_v[a] / bc2) + 1e-8);
  }
  // perturbed(): R <- exp(d_rot) R, t <- exp(d_rot) t + d_trans
  double dR[9], Rc[9], Rn[9];
  exp_map_d(delta, dR);
  exp_map_d(ds->pose_rot, Rc);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Rn[3 * i + j] = dR[3 * i + 0] * Rc[0 * 3 + j] + dR[3 * i + 1] * Rc[1 * 3 + j] + dR[3 * i + 2] * Rc[2 * 3 + j];
  double tn[3];
  for (int i = 0; i < 3; ++i)
    tn[i] = dR[3 * i + 0] * ds->pose_trans[0] + dR[3 * i + 1] * ds->pose_trans[1] + dR[3 * i + 2] * ds->pose_trans[2] + delta[3 + i];
  double rn[3];
  log_map_dev(Rn, rn);
  for (int i = 0; i < 3; ++i) {
    ds->pose_rot[i] = rn[i];
    ds->pose_trans[i] = tn[i];
  }
  ds->iterations_run = iteration + 1;
  const Cam old = ds->cam;
  ds->cam = make_cam(ds->pose_rot, ds->pose_trans, old.fx, old.fy, old.cx, old.cy, old.width, old.height, old.near_plane,
                     old.far_plane);
}

__global__ void k_densify_stats(const uint8_t* __restrict__ visible, const float* __restrict__ d_mean2d,
                                float* __restrict__ accum, int32_t* __restrict__ cnt, int64_t P, double hw, double hh) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P || !visible[i]) return;
  const double nx = d_mean2d[i] * hw, ny = d_mean2d[P + i] * hh;
  accum[i] = static_cast<float>(static_cast<double>(accum[i]) + sqrt(nx * nx + ny * ny));
  cnt[i] += 1;
}

}  // namespace

void run_adam(float* params, const float* grads, float* m, float* v, int64_t P, int D, const AdamGroups& g, double step,
              cudaStream_t st, int64_t* L) {
  const int64_t n = static_cast<int64_t>(D) * P;
  if (n == 0) return;
  const double bc1 = 1.0 - std::pow(0.9, step);
  const double bc2 = 1.0 - std::pow(0.999, step);
  const int blocks = static_cast<int>(std::min<int64_t>(div_up(n, 256), 148 * 16));
  k_adam<<<blocks, 256, 0, st>>>(params, grads, m, v, P, D, g, bc1, bc2);
  ++*L;
}

void run_track_update(DevState* ds, int iteration, cudaStream_t st, int64_t* L) {
  k_track_update<<<1, 32, 0, st>>>(ds, iteration);
  ++*L;
}

void run_densify_stats(const uint8_t* visible, const float* d_mean2d, float* accum, int32_t* cnt, int64_t P, int W, int H,
                       cudaStream_t st, int64_t* L) {
  if (P <= 0) return;
  k_densify_stats<<<div_up(P, 256), 256, 0, st>>>(visible, d_mean2d, accum, cnt, P, 0.5 * W, 0.5 * H);
  ++*L;
}

}  // namespace gsfk
