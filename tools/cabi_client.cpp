// cabi_client.cpp — a plain C++ caller of the drop-in boundary (include/gsf_cuda.h only, no torch,
// no Python): the sequence the reference's SlamSystem runs per frame, through the C-ABI.
//
//   synthetic room (io/synthetic.cpp) -> gsf_map_upload -> render the ground-truth frame ->
//   gsf_frame_upload -> gsf_track_frame from a perturbed pose -> gsf_map_step -> gsf_render_record
//
// Prints one JSON line; exits non-zero on any failure.  Built by __graft_entry__.build() next to
// the library (tools/cabi_client), run by tests/test_gpu_parity.py::test_cabi_client_from_cpp.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gsf_cuda.h"
#include "../tools/synth/gsf_synth.h"   // scene generator (tools, not the product)

#define CHECK(call)                                                                          \
  do {                                                                                       \
    const int rc_ = (call);                                                                  \
    if (rc_ != GSF_OK) {                                                                     \
      std::fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, ctx ? gsf_last_error(ctx) : ""); \
      return 1;                                                                              \
    }                                                                                        \
  } while (0)

int main() {
  gsf_ctx ctx = nullptr;
  CHECK(gsf_ctx_create(0, &ctx));
  // map: the reference room generator, 50k primitives
  gsf_map_host m{};
  CHECK(gsf_synth_room(50000, 4.0, 3, 0, &m));
  const int64_t P = m.count;
  std::vector<double> mean(3 * P), ls(3 * P), quat(4 * P), op(P), sh(3 * P);
  m.mean = mean.data(); m.log_scale = ls.data(); m.quat = quat.data(); m.opacity_logit = op.data(); m.sh = sh.data();
  CHECK(gsf_synth_room(50000, 4.0, 3, 0, &m));
  CHECK(gsf_map_upload(ctx, &m));
  std::vector<gsf_pose> orbit(50);
  CHECK(gsf_synth_orbit(50, 1.0, 0.0, orbit.data()));
  const gsf_intrinsics K{300.0, 300.0, 159.5, 119.5, 320, 240, 1.0, 0.1, 10.0};
  gsf_raster_cfg rc{0.99, 1.0 / 255.0, 1e-8, 3.0, 0.3, 16, 1, 0};
  // ground-truth frame at orbit pose 2
  const size_t npix = static_cast<size_t>(K.width) * K.height;
  std::vector<float> rgb(3 * npix), depth(npix);
  gsf_render_out out{};
  out.color = rgb.data();
  out.alpha_depth = depth.data();
  CHECK(gsf_render(ctx, &orbit[2], &K, nullptr, &rc, &out));
  CHECK(gsf_frame_upload(ctx, 0, rgb.data(), depth.data(), K.width, K.height));
  // track from a perturbed start (TrackerConfig / LossWeights::indoor_synthetic defaults)
  gsf_pose start = orbit[2];
  start.rotation_tangent[0] += 0.004;
  start.translation[1] -= 0.006;
  gsf_tracker_cfg tc{0.0015, 0.00215, 40, 4, 10, 30, 2, 1, 2.0};
  gsf_loss_weights w{0.7, 0.1, 0.25, 0.25, 0.1, 0.15, 0.2, 1.0, 1.0, 0.1, 1};
  gsf_track_result tr{};
  CHECK(gsf_track_frame(ctx, 0, &start, &K, &tc, &w, &rc, &tr));
  double err0 = 0.0, err1 = 0.0;
  for (int a = 0; a < 3; ++a) {
    err0 += std::pow(start.translation[a] - orbit[2].translation[a], 2);
    err1 += std::pow(tr.pose.translation[a] - orbit[2].translation[a], 2);
  }
  // one mapping step on the tracked keyframe, then the CSR record of a render
  gsf_mapper_cfg mc{};
  mc.sh_coeffs = 1; mc.scene_extent = 4.0; mc.lr_mean = 1.6e-4; mc.lr_sh = 2.5e-3; mc.lr_opacity = 5e-2;
  mc.lr_scale = 5e-3; mc.lr_rotation = 1e-3; mc.densify_interval = 0; mc.densify_grad_threshold = 2e-4;
  mc.densify_split_factor = 1.6; mc.densify_size_fraction = 0.01; mc.densify_cull_opacity = 0.005;
  mc.uncertainty_tau = 0.025; mc.uncertainty_reduced_opacity = 0.005; mc.seed = 0; mc.raster = rc; mc.weights = w;
  mc.init_stride = 2; mc.spawn_stride = 2; mc.spawn_opacity_threshold = 0.5; mc.init_opacity = 0.5;
  const int32_t slot = 0;
  double trace[3];
  CHECK(gsf_map_step(ctx, &slot, &tr.pose, 1, &K, &mc, 3, trace));
  CHECK(gsf_render(ctx, &tr.pose, &K, nullptr, &rc, &out));
  int64_t total = 0;
  CHECK(gsf_render_record(ctx, nullptr, nullptr, nullptr, nullptr, &total));
  std::printf("{\"primitives\": %lld, \"visible\": %lld, \"iterations\": %d, \"initial_loss\": %.6g, \"final_loss\": %.6g, "
              "\"trans_err_before\": %.6g, \"trans_err_after\": %.6g, \"map_trace\": [%.6g, %.6g, %.6g], "
              "\"record_entries\": %lld, \"kernel_launches\": %lld}\n",
              static_cast<long long>(P), static_cast<long long>(out.num_visible), tr.iterations_run, tr.initial_loss,
              tr.final_loss, std::sqrt(err0), std::sqrt(err1), trace[0], trace[1], trace[2],
              static_cast<long long>(total), static_cast<long long>(gsf_kernel_launches(ctx)));
  const bool ok = tr.iterations_run == 40 && tr.final_loss < tr.initial_loss && std::isfinite(trace[2]) && total > 0;
  CHECK(gsf_ctx_destroy(ctx));
  return ok ? 0 : 2;
}
