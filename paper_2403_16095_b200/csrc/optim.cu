// optim.cu — fused Adam over the SoA map and the fp64 pose update of track_frame.
//
//   k_adam          AdamState::step (adam.cpp:40-53) for all five parameter groups of
//                   PrimitiveOptimizer::step (mapper.cpp:72-117) in one pass over [D][P]; fp32
//                   storage, fp64 arithmetic, dense over every entry like the reference.
//   k_track_update  tracker.cpp:62-70: the two pose AdamStates on zero-initialised deltas, then
//                   CameraPose::perturbed (pose.hpp:44-48) and the next iteration's camera, all
//                   on the device so a whole track_frame can be one CUDA graph.
#include "kernels.h"
#include "finalize.cuh"

namespace gsfk {

namespace {

// One field per blockIdx.y, so the group and learning rate are uniform per CTA (no per-element
// 64-bit division to find the field); each thread streams kAdamPer elements of that field.
constexpr int kAdamPer = 4;
__global__ void __launch_bounds__(256) k_adam(float* __restrict__ params, const float* __restrict__ grads,
                                              float* __restrict__ m, float* __restrict__ v, int64_t P, AdamGroups g,
                                              double ibc1, double ibc2, int f0) {
  const int f = f0 + static_cast<int>(blockIdx.y);
  const int grp = f < 3 ? 0 : (f < 6 ? 1 : (f < 10 ? 2 : (f < 11 ? 3 : 4)));
  const double lr = g.lr[grp];
  const int64_t base = static_cast<int64_t>(f) * P;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x * kAdamPer + threadIdx.x;
#pragma unroll
  for (int u = 0; u < kAdamPer; ++u) {
    const int64_t i = i0 + static_cast<int64_t>(u) * blockDim.x;
    if (i >= P) break;
    const int64_t e = base + i;
    const double gr = grads[e];
    const double mm = 0.9 * static_cast<double>(m[e]) + (1.0 - 0.9) * gr;
    const double vv = 0.999 * static_cast<double>(v[e]) + (1.0 - 0.999) * gr * gr;
    m[e] = static_cast<float>(mm);
    v[e] = static_cast<float>(vv);
    // the bias corrections as host reciprocals (ibc = 1 / bc): two fp64 divisions fewer per entry
    // (the kernel is FP64-bound, not HBM-bound: 145 -> 107 us at 994k x 14); one fp64 ulp apart
    // from m / bc before the fp32 store
    const double upd = lr * (mm * ibc1) / (sqrt(vv * ibc2) + 1e-8);
    params[e] = static_cast<float>(static_cast<double>(params[e]) - upd);
  }
}

__global__ void k_track_update(DevState* ds, int iteration, double bc1, double bc2) {
  if (threadIdx.x == 0 && blockIdx.x == 0) track_update(ds, iteration, bc1, bc2);
}

}  // namespace

void run_adam_fields(float* params, const float* grads, float* m, float* v, int64_t P, int f0, int f1,
                     const AdamGroups& g, double step, cudaStream_t st, int64_t* L) {
  if (P == 0 || f1 <= f0) return;
  const double bc1 = 1.0 - std::pow(0.9, step);
  const double bc2 = 1.0 - std::pow(0.999, step);
  const dim3 grid(static_cast<unsigned>(div_up(P, 256 * kAdamPer)), static_cast<unsigned>(f1 - f0));
  k_adam<<<grid, 256, 0, st>>>(params, grads, m, v, P, g, 1.0 / bc1, 1.0 / bc2, f0);
  ++*L;
}

void run_adam(float* params, const float* grads, float* m, float* v, int64_t P, int D, const AdamGroups& g, double step,
              cudaStream_t st, int64_t* L) {
  run_adam_fields(params, grads, m, v, P, 0, D, g, step, st, L);
}

void run_track_update(DevState* ds, int iteration, cudaStream_t st, int64_t* L) {
  // AdamState bias corrections at step t = iteration + 1 (adam.cpp:40-53), host std::pow
  const double t = static_cast<double>(iteration + 1);
  k_track_update<<<1, 32, 0, st>>>(ds, iteration, 1.0 - std::pow(0.9, t), 1.0 - std::pow(0.999, t));
  ++*L;
}

}  // namespace gsfk
