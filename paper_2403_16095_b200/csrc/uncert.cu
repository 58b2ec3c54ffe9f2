// uncert.cu — per-primitive depth uncertainty (Eq. 13) and unreliable-primitive pruning.
//
//   k_uncert_view      accumulate_uncertainty (uncertainty.cpp:35-64) for one view: every
//                      valid-depth pixel adds alpha*T*(D - z_owner)^2 to its dominant primitive
//                      (the dominant weight is kept per pixel by the blend, so no CSR walk).
//   k_uncert_finalize  uncertainty.cpp:75-85: nu = sum / count, observed flags.
//   k_prune            prune_unreliable (uncertainty.cpp:89-100).
#include "kernels.h"

namespace gsfk {

namespace {

__global__ void k_uncert_view(const int32_t* __restrict__ dominant, const float* __restrict__ dom_w,
                              const float* __restrict__ obs, int64_t npix, double near_plane, double far_plane,
                              const float* __restrict__ params, int64_t P, const DevState* ds, double* __restrict__ sum,
                              uint32_t* __restrict__ cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= npix) return;
  const int32_t owner = dominant[i];
  if (owner < 0) return;
  const double d = obs[i];
  if (!isfinite(d) || d <= near_plane || d >= far_plane) return;
  const double* W = ds->cam.W;
  const double z = W[6] * params[owner] + W[7] * params[P + owner] + W[8] * params[2 * P + owner] + ds->cam.t[2];
  const double r = d - z;
  atomicAdd(&sum[owner], static_cast<double>(dom_w[i]) * r * r);
  atomicAdd(&cnt[owner], 1u);
}

__global__ void k_uncert_finalize(const double* __restrict__ sum, const uint32_t* __restrict__ cnt, double* __restrict__ nu,
                                  uint8_t* __restrict__ observed, int64_t P, uint32_t* observed_count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  if (cnt[i] > 0) {
    nu[i] = sum[i] / cnt[i];
    observed[i] = 1;
    atomicAdd(observed_count, 1u);
  } else {
    observed[i] = 0;
  }
}

__global__ void k_prune(const double* __restrict__ nu, float* __restrict__ opacity_logit, int64_t P, double tau, float target,
                        uint32_t* reduced) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  if (nu[i] > tau && opacity_logit[i] != target) {
    opacity_logit[i] = target;
    atomicAdd(reduced, 1u);
  }
}

}  // namespace

void run_uncertainty_view(const Workspace& ws, const float* params, int64_t P, const float* obs, int W, int H,
                          double near_plane, double far_plane, const DevState* ds, double* sum, uint32_t* cnt,
                          cudaStream_t st, int64_t* L) {
  const int64_t npix = static_cast<int64_t>(W) * H;
  k_uncert_view<<<div_up(npix, 256), 256, 0, st>>>(ws.dominant, ws.dominant_w, obs, npix, near_plane, far_plane, params, P,
                                                   ds, sum, cnt);
  ++*L;
}

void run_uncertainty_finalize(const double* sum, const uint32_t* cnt, double* nu, uint8_t* observed, int64_t P,
                              uint32_t* observed_count, cudaStream_t st, int64_t* L) {
  if (P <= 0) return;
  k_uncert_finalize<<<div_up(P, 256), 256, 0, st>>>(sum, cnt, nu, observed, P, observed_count);
  ++*L;
}

void run_prune(const double* nu, float* opacity_logit, int64_t P, double tau, float target, uint32_t* reduced, cudaStream_t st,
               int64_t* L) {
  if (P <= 0) return;
  k_prune<<<div_up(P, 256), 256, 0, st>>>(nu, opacity_logit, P, tau, target, reduced);
  ++*L;
}

}  // namespace gsfk
