// synth.cpp — synthetic scene / trajectory generators for the benchmark and tests (tools/, not the
// product: built into tools/synth/libgsf_synth.so, never into libgsf_cuda.so).
//
// Restates io/synthetic.cpp:39-186 (room scene, orbit trajectory) so the benchmark builds the
// same Replica-shaped inputs the reference's own generator would, draw for draw from
// std::mt19937_64 with libstdc++'s distributions.  Frames are rendered on the device by the
// caller (the reference's brute-force render_reference is O(pixels x primitives)).
#include <algorithm>
#include <cmath>
#include <random>
#include <vector>

#include "gsf_synth.h"

namespace {

constexpr double kC0 = 0.28209479177387814;

struct V3 {
  double x, y, z;
  V3(double a = 0, double b = 0, double c = 0) : x(a), y(b), z(c) {}
};
V3 operator+(const V3& a, const V3& b) { return V3(a.x + b.x, a.y + b.y, a.z + b.z); }
V3 operator*(double s, const V3& a) { return V3(s * a.x, s * a.y, s * a.z); }

struct Prim {
  V3 mean;
  double ls;
  double logit;
  V3 sh0;
};

double logit(double p) { return std::log(p / (1.0 - p)); }

V3 textured_color(double u, double v, const V3& phase, std::mt19937_64& rng) {   // synthetic.cpp:30-38
  std::uniform_real_distribution<double> jitter(-0.08, 0.08);
  const double ph[3] = {phase.x, phase.y, phase.z};
  double c[3];
  for (int ch = 0; ch < 3; ++ch)
    c[ch] = 0.5 + 0.33 * std::sin(3.1 * u + ph[ch]) * std::cos(2.3 * v + 1.7 * ph[ch]) + jitter(rng);
  for (double& x : c) x = std::min(std::max(x, 0.02), 0.98);
  return V3(c[0], c[1], c[2]);
}

Prim surface(const V3& pos, double scale, double opacity, const V3& rgb) {   // synthetic.cpp:40-49
  return Prim{pos, std::log(scale), logit(opacity), V3((rgb.x - 0.5) / kC0, (rgb.y - 0.5) / kC0, (rgb.z - 0.5) / kC0)};
}

void wall_grid(std::vector<Prim>& prims, const V3& origin, const V3& u_axis, const V3& v_axis, double side, int n, int layers,
               double opacity, const V3& phase, std::mt19937_64& rng) {   // synthetic.cpp:51-66
  const double spacing = side / n;
  const double scale = 0.55 * spacing;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double u = (i + 0.5) * spacing - 0.5 * side;
      const double v = (j + 0.5) * spacing - 0.5 * side;
      const V3 pos = origin + u * u_axis + v * v_axis;
      const V3 rgb = textured_color(u, v, phase, rng);
      for (int l = 0; l < layers; ++l) prims.push_back(surface(pos, scale, opacity, rgb));
    }
}

std::vector<Prim> build_room(int count, double extent, int wall_layers, std::mt19937_64& rng) {   // :68-116
  std::vector<Prim> prims;
  const double h = 0.5 * extent;
  const int layers = std::max(1, wall_layers);
  const int object_budget = std::min(count / 10, 450);
  const int wall_budget = count - object_budget;
  const int n = std::max(2, static_cast<int>(std::sqrt(wall_budget / (6.0 * layers))));
  std::uniform_real_distribution<double> uphase(0.0, 6.28);
  const V3 x(1, 0, 0), y(0, 1, 0), z(0, 0, 1);
  struct Face { V3 origin, u, v; };
  const Face faces[6] = {{h * z, x, y}, {(-h) * z, x, y}, {h * x, z, y}, {(-h) * x, z, y}, {h * y, x, z}, {(-h) * y, x, z}};
  for (const Face& f : faces) {
    const V3 phase(uphase(rng), uphase(rng), uphase(rng));
    wall_grid(prims, f.origin, f.u, f.v, extent, n, layers, 0.98, phase, rng);
  }
  const V3 centers[3] = {V3(-0.3 * h, 0.62 * h, 0.25 * h), V3(0.35 * h, 0.66 * h, -0.2 * h), V3(0.05 * h, 0.7 * h, 0.45 * h)};
  const V3 tints[3] = {V3(0.85, 0.3, 0.25), V3(0.25, 0.7, 0.85), V3(0.8, 0.75, 0.2)};
  const double radius = 0.12 * extent;
  const int per_object = std::max(object_budget / 3 - 1, 1);
  std::normal_distribution<double> dir(0.0, 1.0);
  std::uniform_real_distribution<double> shade(-0.1, 0.1);
  const double shell_area = 4.0 * M_PI * radius * radius;
  const double obj_scale = 0.7 * std::sqrt(shell_area / per_object);
  for (int o = 0; o < 3; ++o) {
    prims.push_back(surface(centers[o], 0.45 * radius, 0.995, tints[o]));
    for (int i = 0; i < per_object; ++i) {
      V3 d(dir(rng), dir(rng), dir(rng));
      double len = std::sqrt(d.x * d.x + d.y * d.y + d.z * d.z);
      if (len < 1e-6) {
        d = V3(1, 0, 0);
        len = 1.0;
      }
      d = V3(d.x / len, d.y / len, d.z / len);   // Eigen's normalize(): *this /= norm()
      const double s = shade(rng);
      V3 rgb(tints[o].x + s, tints[o].y + s, tints[o].z + s);
      rgb.x = std::min(std::max(rgb.x, 0.02), 0.98);
      rgb.y = std::min(std::max(rgb.y, 0.02), 0.98);
      rgb.z = std::min(std::max(rgb.z, 0.02), 0.98);
      prims.push_back(surface(centers[o] + radius * d, obj_scale, 0.98, rgb));
    }
  }
  return prims;
}

// look_at + from_matrix (synthetic.cpp:139-150): returns rotation tangent and translation
void look_at(const V3& p, const V3& target, gsf_pose* out) {
  V3 f(target.x - p.x, target.y - p.y, target.z - p.z);
  double fl = std::sqrt(f.x * f.x + f.y * f.y + f.z * f.z);
  f = V3(f.x / fl, f.y / fl, f.z / fl);   // Eigen's normalized(): / norm()
  V3 r(f.y * 0.0 - f.z * 1.0, f.z * 0.0 - f.x * 0.0, f.x * 1.0 - f.y * 0.0);   // forward x UnitY
  double rl = std::sqrt(r.x * r.x + r.y * r.y + r.z * r.z);
  if (rl < 1e-9) { r = V3(1, 0, 0); rl = 1.0; }
  r = V3(r.x / rl, r.y / rl, r.z / rl);
  const V3 d(f.y * r.z - f.z * r.y, f.z * r.x - f.x * r.z, f.x * r.y - f.y * r.x);   // forward x right
  const double R[3][3] = {{r.x, r.y, r.z}, {d.x, d.y, d.z}, {f.x, f.y, f.z}};
  // log_map (lie.cpp:30-52)
  const double trace = R[0][0] + R[1][1] + R[2][2];
  const double ct = std::clamp((trace - 1.0) * 0.5, -1.0, 1.0);
  const double th = std::acos(ct);
  const double vee[3] = {R[2][1] - R[1][2], R[0][2] - R[2][0], R[1][0] - R[0][1]};
  double w[3];
  if (th < 1e-8) {
    for (int i = 0; i < 3; ++i) w[i] = 0.5 * (1.0 + th * th / 6.0) * vee[i];
  } else if (th > M_PI - 1e-3) {
    double o[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) o[i][j] = (0.5 * (R[i][j] + R[j][i]) - ct * (i == j)) / (1.0 - ct);
    int a = 0;
    for (int i = 1; i < 3; ++i)
      if (o[i][i] > o[a][a]) a = i;
    const double sq = std::sqrt(o[a][a]);
    double ax[3] = {o[0][a] / sq, o[1][a] / sq, o[2][a] / sq};
    if (ax[0] * vee[0] + ax[1] * vee[1] + ax[2] * vee[2] < 0.0)
      for (double& v : ax) v = -v;
    for (int i = 0; i < 3; ++i) w[i] = th * ax[i];
  } else {
    for (int i = 0; i < 3; ++i) w[i] = th / (2.0 * std::sin(th)) * vee[i];
  }
  for (int i = 0; i < 3; ++i) out->rotation_tangent[i] = w[i];
  const double P[3] = {p.x, p.y, p.z};
  for (int i = 0; i < 3; ++i) out->translation[i] = -(R[i][0] * P[0] + R[i][1] * P[1] + R[i][2] * P[2]);
}

}  // namespace

extern "C" {

int gsf_synth_room(int32_t primitive_count, double extent, int32_t wall_layers, uint64_t seed, gsf_map_host* map) {
  if (!map || primitive_count < 1) return GSF_EINVAL;
  std::mt19937_64 rng(seed);
  const std::vector<Prim> prims = build_room(primitive_count, extent, wall_layers, rng);
  const int64_t P = static_cast<int64_t>(prims.size());
  if (!map->mean) {
    map->count = P;
    map->sh_coeffs = 1;
    return GSF_OK;
  }
  if (map->count != P || map->sh_coeffs != 1) return GSF_EINVAL;
  for (int64_t i = 0; i < P; ++i) {
    const Prim& q = prims[i];
    map->mean[3 * i] = q.mean.x; map->mean[3 * i + 1] = q.mean.y; map->mean[3 * i + 2] = q.mean.z;
    for (int a = 0; a < 3; ++a) map->log_scale[3 * i + a] = q.ls;
    map->quat[4 * i] = 1.0; map->quat[4 * i + 1] = 0.0; map->quat[4 * i + 2] = 0.0; map->quat[4 * i + 3] = 0.0;
    map->opacity_logit[i] = q.logit;
    map->sh[3 * i] = q.sh0.x; map->sh[3 * i + 1] = q.sh0.y; map->sh[3 * i + 2] = q.sh0.z;
    if (map->uncertainty) map->uncertainty[i] = 0.0;
    if (map->observed) map->observed[i] = 0;
  }
  return GSF_OK;
}

int gsf_synth_orbit(int32_t frames, double radius, double height, gsf_pose* poses) {   // synthetic.cpp:152-186
  if (frames < 1 || !(radius > 0.0) || !poses) return GSF_EINVAL;
  const double sweep = 6.283185307179586;
  std::vector<double> s(frames, 0.0);
  if (frames >= 2) {
    for (int i = 1; i < frames; ++i) s[i] = s[i - 1] + 1.0 / (frames - 1);
    s[frames - 1] = 1.0;
  }
  for (int i = 0; i < frames; ++i) {
    const double th = sweep * s[i];
    look_at(V3(radius * std::cos(th), height, radius * std::sin(th)), V3(0.0, height, 0.0), &poses[i]);
  }
  return GSF_OK;
}

}  // extern "C"
