// densify.cu — densify_and_cull (map/mapper.cpp:172-230) and its statistics (:261-269).
//
//   k_densify_stats  grad_accum += |d_mean2d| in NDC units, grad_count += 1 for visible primitives
//                    (fp64 accumulators like the reference's std::vector<double>)
//   k_densify_codes  per primitive: 0 culled (opacity below cull_opacity), 1 kept, 2 split (the
//                    parent is replaced by two children), 3 cloned (kept + one copy appended)
//   k_densify_build  the new SoA map: kept primitives in order, then the appended ones in parent
//                    order (two children per split, one copy per clone); Adam moments follow the
//                    kept entries (AdamState::filter) and start at zero for appended ones (append)
//
// The children's offsets z ~ N(0, I) come from the map state's std::mt19937_64 on the host, one
// fresh std::normal_distribution per split parent as in the reference, so they are the reference's
// draws; the host also orders the output (one pass over the codes).
#include "kernels.h"

namespace gsfk {

namespace {

__global__ void k_densify_stats(const uint8_t* __restrict__ visible, const float* __restrict__ d_mean2d,
                                double* __restrict__ accum, int32_t* __restrict__ cnt, int64_t P, double hw, double hh) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P || !visible[i]) return;
  const double nx = static_cast<double>(d_mean2d[i]) * hw, ny = static_cast<double>(d_mean2d[P + i]) * hh;
  accum[i] += sqrt(nx * nx + ny * ny);
  cnt[i] += 1;
}

__global__ void k_densify_codes(const float* __restrict__ params, int64_t P, const double* __restrict__ accum,
                                const int32_t* __restrict__ cnt, double cull_opacity, double grad_threshold,
                                double size_boundary, uint8_t* __restrict__ code) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const double op = 1.0 / (1.0 + exp(-static_cast<double>(params[10 * P + i])));   // primitive.hpp:11,33
  uint8_t c = 1;
  if (op < cull_opacity) {
    c = 0;
  } else if (cnt[i] != 0 && accum[i] / cnt[i] > grad_threshold) {
    double smax = exp(static_cast<double>(params[3 * P + i]));
    smax = fmax(smax, exp(static_cast<double>(params[4 * P + i])));
    smax = fmax(smax, exp(static_cast<double>(params[5 * P + i])));
    c = smax > size_boundary ? 2 : 3;
  }
  code[i] = c;
}

// kind: 0 kept (moments carried), 1 clone (moments zero), 2 child (offset mean, shrunken scale)
__global__ void k_densify_build(const float* __restrict__ params, const float* __restrict__ m, const float* __restrict__ v,
                                const double* __restrict__ nu, const uint8_t* __restrict__ observed, int64_t P_old, int D,
                                const int32_t* __restrict__ src, const uint8_t* __restrict__ kind,
                                const int32_t* __restrict__ zidx, const double* __restrict__ z, double log_split,
                                int64_t P_new, float* __restrict__ params_n, float* __restrict__ m_n,
                                float* __restrict__ v_n, double* __restrict__ nu_n, uint8_t* __restrict__ observed_n) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= P_new) return;
  const int64_t s = src[j];
  const int kd = kind[j];
  for (int f = 0; f < D; ++f) {
    params_n[f * P_new + j] = params[f * P_old + s];
    m_n[f * P_new + j] = kd == 0 ? m[f * P_old + s] : 0.0f;
    v_n[f * P_new + j] = kd == 0 ? v[f * P_old + s] : 0.0f;
  }
  nu_n[j] = nu[s];
  observed_n[j] = observed[s];
  if (kd != 2) return;
  // child: mean = p.mean + (R diag(s)) z, log_scale = p.log_scale - log(split_factor)  (mapper.cpp:195-203)
  const double qw0 = params[6 * P_old + s], qx0 = params[7 * P_old + s], qy0 = params[8 * P_old + s],
               qz0 = params[9 * P_old + s];
  const double qn = sqrt(qw0 * qw0 + qx0 * qx0 + qy0 * qy0 + qz0 * qz0);
  const double w = qw0 / qn, x = qx0 / qn, y = qy0 / qn, zq = qz0 / qn;
  const double R[3][3] = {{1 - 2 * (y * y + zq * zq), 2 * (x * y - w * zq), 2 * (x * zq + w * y)},
                          {2 * (x * y + w * zq), 1 - 2 * (x * x + zq * zq), 2 * (y * zq - w * x)},
                          {2 * (x * zq - w * y), 2 * (y * zq + w * x), 1 - 2 * (x * x + y * y)}};
  double sc[3], ls[3];
  for (int a = 0; a < 3; ++a) {
    ls[a] = params[(3 + a) * P_old + s];
    sc[a] = exp(ls[a]);
  }
  const double* zz = z + 3 * static_cast<int64_t>(zidx[j]);
  for (int a = 0; a < 3; ++a) {
    const double off = R[a][0] * sc[0] * zz[0] + R[a][1] * sc[1] * zz[1] + R[a][2] * sc[2] * zz[2];
    params_n[a * P_new + j] = static_cast<float>(static_cast<double>(params[a * P_old + s]) + off);
    params_n[(3 + a) * P_new + j] = static_cast<float>(ls[a] - log_split);
  }
}

}  // namespace

void run_densify_stats(const uint8_t* visible, const float* d_mean2d, double* accum, int32_t* cnt, int64_t P, int W, int H,
                       cudaStream_t st, int64_t* L) {
  if (P <= 0) return;
  k_densify_stats<<<div_up(P, 256), 256, 0, st>>>(visible, d_mean2d, accum, cnt, P, 0.5 * W, 0.5 * H);
  ++*L;
}

void run_densify_codes(const float* params, int64_t P, const double* accum, const int32_t* cnt, double cull_opacity,
                       double grad_threshold, double size_boundary, uint8_t* code, cudaStream_t st, int64_t* L) {
  if (P <= 0) return;
  k_densify_codes<<<div_up(P, 256), 256, 0, st>>>(params, P, accum, cnt, cull_opacity, grad_threshold, size_boundary, code);
  ++*L;
}

void run_densify_build(const float* params, const float* m, const float* v, const double* nu, const uint8_t* observed,
                       int64_t P_old, int D, const int32_t* src, const uint8_t* kind, const int32_t* zidx, const double* z,
                       double log_split, int64_t P_new, float* params_n, float* m_n, float* v_n, double* nu_n,
                       uint8_t* observed_n, cudaStream_t st, int64_t* L) {
  if (P_new <= 0) return;
  k_densify_build<<<div_up(P_new, 256), 256, 0, st>>>(params, m, v, nu, observed, P_old, D, src, kind, zidx, z, log_split,
                                                      P_new, params_n, m_n, v_n, nu_n, observed_n);
  ++*L;
}

}  // namespace gsfk
