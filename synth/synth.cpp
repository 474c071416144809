// synth.cpp — synthetic depth streams (host only).
//
// Restates the reference's analytic scenes (proj/core/src/synth.cpp:20-373:
// ray-cast primitives, smoothstep motion, mm quantisation with Gaussian noise
// from mt19937(seed + t * 2654435761)) and adds the BASELINE.json scenes the
// reference never shipped:
//   deforming_sphere  (config 1: ~30k surfels at 320x240)
//   articulated_body  (config 2: ~200k surfels, ~1.5k nodes at 640x480)
// These frames are the shared input of the CUDA path and the CPU oracle.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "../include/dynsurf_synth.h"

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr double kPi = 3.14159265358979323846;

struct P3 {
  double x = 0, y = 0, z = 0;
};
inline P3 p3(double a, double b, double c) { return P3{a, b, c}; }
inline P3 operator+(P3 a, P3 b) { return p3(a.x + b.x, a.y + b.y, a.z + b.z); }
inline P3 operator-(P3 a, P3 b) { return p3(a.x - b.x, a.y - b.y, a.z - b.z); }
inline P3 operator*(double s, P3 a) { return p3(s * a.x, s * a.y, s * a.z); }
inline double dot(P3 a, P3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline double len(P3 a) { return std::sqrt(dot(a, a)); }

struct R3 {  // row-major rotation
  double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  P3 operator*(P3 v) const {
    return p3((m[0] * v.x + m[1] * v.y) + m[2] * v.z, (m[3] * v.x + m[4] * v.y) + m[5] * v.z,
              (m[6] * v.x + m[7] * v.y) + m[8] * v.z);
  }
  R3 operator*(const R3& b) const {
    R3 o;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        o.m[i * 3 + j] = (m[i * 3] * b.m[j] + m[i * 3 + 1] * b.m[3 + j]) + m[i * 3 + 2] * b.m[6 + j];
    return o;
  }
  R3 t() const {
    R3 o;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) o.m[i * 3 + j] = m[j * 3 + i];
    return o;
  }
};
// Eigen::AngleAxisd(angle, unit axis).toRotationMatrix() (synth.cpp:27-28)
R3 axis_angle(P3 axis, double angle) {
  const double s = std::sin(angle), c = std::cos(angle);
  const P3 sa = s * axis, ca = (1.0 - c) * axis;
  R3 r;
  double t = ca.x * axis.y;
  r.m[1] = t - sa.z;
  r.m[3] = t + sa.z;
  t = ca.x * axis.z;
  r.m[2] = t + sa.y;
  r.m[6] = t - sa.y;
  t = ca.y * axis.z;
  r.m[5] = t - sa.x;
  r.m[7] = t + sa.x;
  r.m[0] = ca.x * axis.x + c;
  r.m[4] = ca.y * axis.y + c;
  r.m[8] = ca.z * axis.z + c;
  return r;
}
R3 rot_x(double a) { return axis_angle(p3(1, 0, 0), a); }
R3 rot_y(double a) { return axis_angle(p3(0, 1, 0), a); }
R3 rot_z(double a) { return axis_angle(p3(0, 0, 1), a); }

double smoothstep(double u) {
  u = std::clamp(u, 0.0, 1.0);
  return u * u * (3.0 - 2.0 * u);
}

// ---- primitives (synth.cpp:40-73 + capsules / ellipsoids for the new scenes)
struct RectZ {
  double z0, x0, x1, y0, y1;
};
struct Sphere {
  P3 c;
  double r;
};
struct Sheet {
  double half_width, radius, z_front, half_angle;
};
struct Ellipsoid {  // x = c + R * diag(a) * unit-sphere
  P3 c;
  R3 R;
  P3 a;
};
struct Capsule {
  P3 a, b;
  double r;
};
struct Scene {
  std::vector<RectZ> rects;
  std::vector<Sphere> spheres;
  std::vector<Sheet> sheets;
  std::vector<Ellipsoid> ellipsoids;
  std::vector<Capsule> capsules;
  std::vector<struct SineSheet> sines;
};

double ray_rect(P3 o, P3 d, const RectZ& r) {  // synth.cpp:75-84
  if (std::abs(d.z) < 1e-12) return kInf;
  const double s = (r.z0 - o.z) / d.z;
  if (s <= 1e-9) return kInf;
  const double x = o.x + s * d.x, y = o.y + s * d.y;
  if (x < r.x0 || x > r.x1 || y < r.y0 || y > r.y1) return kInf;
  return s;
}
double ray_sphere(P3 o, P3 d, const Sphere& sp) {  // synth.cpp:86-99
  const P3 oc = o - sp.c;
  const double a = dot(d, d), b = 2.0 * dot(oc, d), c = dot(oc, oc) - sp.r * sp.r;
  const double disc = b * b - 4.0 * a * c;
  if (disc < 0) return kInf;
  const double sq = std::sqrt(disc);
  const double s1 = (-b - sq) / (2.0 * a);
  if (s1 > 1e-9) return s1;
  const double s2 = (-b + sq) / (2.0 * a);
  if (s2 > 1e-9) return s2;
  return kInf;
}
double ray_sheet(P3 o, P3 d, const Sheet& sh) {  // synth.cpp:101-122
  const double cz = sh.z_front + sh.radius;
  const double vy = o.y, vz = o.z - cz;
  const double a = d.y * d.y + d.z * d.z;
  if (a < 1e-18) return kInf;
  const double b = 2.0 * (vy * d.y + vz * d.z);
  const double c = vy * vy + vz * vz - sh.radius * sh.radius;
  const double disc = b * b - 4.0 * a * c;
  if (disc < 0) return kInf;
  const double sq = std::sqrt(disc);
  for (const double s : {(-b - sq) / (2.0 * a), (-b + sq) / (2.0 * a)}) {
    if (s <= 1e-9) continue;
    const P3 hit = o + s * d;
    const double phi = std::atan2(hit.y, cz - hit.z);
    if (std::abs(phi) > sh.half_angle) continue;
    if (std::abs(hit.x) > sh.half_width) continue;
    return s;
  }
  return kInf;
}
double ray_ellipsoid(P3 o, P3 d, const Ellipsoid& e) {
  const R3 rt = e.R.t();
  P3 ol = rt * (o - e.c), dl = rt * d;
  ol = p3(ol.x / e.a.x, ol.y / e.a.y, ol.z / e.a.z);
  dl = p3(dl.x / e.a.x, dl.y / e.a.y, dl.z / e.a.z);
  return ray_sphere(ol, dl, Sphere{p3(0, 0, 0), 1.0});
}
double ray_capsule(P3 o, P3 d, const Capsule& cp) {
  double best = std::min(ray_sphere(o, d, Sphere{cp.a, cp.r}), ray_sphere(o, d, Sphere{cp.b, cp.r}));
  const P3 ax = cp.b - cp.a;
  const double L = len(ax);
  if (L < 1e-12) return best;
  const P3 u = (1.0 / L) * ax;
  const P3 w = o - cp.a;
  const P3 dp = d - dot(d, u) * u, wp = w - dot(w, u) * u;
  const double a = dot(dp, dp), b = 2.0 * dot(dp, wp), c = dot(wp, wp) - cp.r * cp.r;
  if (a > 1e-18) {
    const double disc = b * b - 4.0 * a * c;
    if (disc >= 0) {
      const double sq = std::sqrt(disc);
      for (const double s : {(-b - sq) / (2.0 * a), (-b + sq) / (2.0 * a)}) {
        if (s <= 1e-9) continue;
        const double h = dot(w + s * d, u);
        if (h < 0 || h > L) continue;
        best = std::min(best, s);
        break;
      }
    }
  }
  return best;
}
double dist_rect(P3 p, const RectZ& r) {
  const double dx = p.x - std::clamp(p.x, r.x0, r.x1);
  const double dy = p.y - std::clamp(p.y, r.y0, r.y1);
  const double dz = p.z - r.z0;
  return std::sqrt(dx * dx + dy * dy + dz * dz);
}
double dist_sphere(P3 p, const Sphere& s) { return std::abs(len(p - s.c) - s.r); }
double dist_sheet(P3 p, const Sheet& sh) {
  const double cz = sh.z_front + sh.radius;
  const double phi = std::atan2(p.y, cz - p.z);
  const double dx = std::max(0.0, std::abs(p.x) - sh.half_width);
  if (std::abs(phi) <= sh.half_angle) {
    const double rho = std::hypot(p.y, p.z - cz);
    return std::hypot(dx, rho - sh.radius);
  }
  const double edge = std::copysign(sh.half_angle, phi);
  const double ey = sh.radius * std::sin(edge), ez = cz - sh.radius * std::cos(edge);
  return std::hypot(dx, std::hypot(p.y - ey, p.z - ez));
}
double dist_capsule(P3 p, const Capsule& cp) {
  const P3 ax = cp.b - cp.a;
  const double L2 = dot(ax, ax);
  const double h = L2 > 0 ? std::clamp(dot(p - cp.a, ax) / L2, 0.0, 1.0) : 0.0;
  return std::abs(len(p - (cp.a + h * ax)) - cp.r);
}
double dist_ellipsoid(P3 p, const Ellipsoid& e) {
  // First-order distance |f|/|grad f| of f = |x/a|^2 - 1 (adequate as an oracle
  // for mm-scale residual checks near the surface).
  const P3 l = e.R.t() * (p - e.c);
  const P3 q = p3(l.x / e.a.x, l.y / e.a.y, l.z / e.a.z);
  const double f = dot(q, q) - 1.0;
  const P3 g = p3(2 * q.x / e.a.x, 2 * q.y / e.a.y, 2 * q.z / e.a.z);
  const double gl = len(g);
  return gl > 0 ? std::abs(f) / gl : len(l);
}

// Config 4 (solver micro-bench) surface: a height field z = z0 + a sin(kx x + phase)
// sin(ky y) filling the whole field of view, so the node count scales with the
// image size (~130 surfels per node at f/z ~ 465).
struct SineSheet {
  double z0, a, kx, ky, phase;
};
double ray_sine(P3 o, P3 d, const SineSheet& h) {
  if (d.z <= 1e-9) return kInf;
  double s = (h.z0 - o.z) / d.z;
  for (int it = 0; it < 40; ++it) {
    const P3 q = o + s * d;
    const double z = h.z0 + h.a * std::sin(h.kx * q.x + h.phase) * std::sin(h.ky * q.y);
    const double ns = (z - o.z) / d.z;
    if (std::abs(ns - s) < 1e-12) {
      s = ns;
      break;
    }
    s = ns;
  }
  return s > 1e-9 ? s : kInf;
}
double dist_sine(P3 p, const SineSheet& h) {
  return std::abs(p.z - (h.z0 + h.a * std::sin(h.kx * p.x + h.phase) * std::sin(h.ky * p.y)));
}

double scene_raycast(P3 o, P3 d, const Scene& s) {
  double best = kInf;
  for (const auto& r : s.sines) best = std::min(best, ray_sine(o, d, r));
  for (const auto& r : s.rects) best = std::min(best, ray_rect(o, d, r));
  for (const auto& r : s.spheres) best = std::min(best, ray_sphere(o, d, r));
  for (const auto& r : s.sheets) best = std::min(best, ray_sheet(o, d, r));
  for (const auto& r : s.ellipsoids) best = std::min(best, ray_ellipsoid(o, d, r));
  for (const auto& r : s.capsules) best = std::min(best, ray_capsule(o, d, r));
  return best;
}
double scene_distance(P3 p, const Scene& s) {
  double best = kInf;
  for (const auto& r : s.sines) best = std::min(best, dist_sine(p, r));
  for (const auto& r : s.rects) best = std::min(best, dist_rect(p, r));
  for (const auto& r : s.spheres) best = std::min(best, dist_sphere(p, r));
  for (const auto& r : s.sheets) best = std::min(best, dist_sheet(p, r));
  for (const auto& r : s.ellipsoids) best = std::min(best, dist_ellipsoid(p, r));
  for (const auto& r : s.capsules) best = std::min(best, dist_capsule(p, r));
  return best;
}

enum Kind {
  kStaticPlane = 0,
  kRigidOrbit,
  kBendingSheet,
  kArticulatedTwoPart,
  kOpenToClose,
  kTangentialSlide,
  kTurntable,
  kDeformingSphere,
  kArticulatedBody,
  kSineSheet,
  kLargeScene,
  kNumKinds
};
const char* kNames[kNumKinds] = {"static_plane",     "rigid_orbit",    "bending_sheet",
                                 "articulated_two_part", "open_to_close", "tangential_slide",
                                 "turntable",        "deforming_sphere", "articulated_body",
                                 "sine_sheet",       "large_scene"};
int default_frames(int kind) {  // synth.cpp:213-224 (+ new scenes)
  switch (kind) {
    case kStaticPlane: return 10;
    case kRigidOrbit: return 50;
    case kBendingSheet: return 100;
    case kArticulatedTwoPart: return 60;
    case kOpenToClose: return 96;
    case kTangentialSlide: return 72;
    case kTurntable: return 360;
    case kDeformingSphere: return 10;
    case kArticulatedBody: return 100;
    case kSineSheet: return 10;
    case kLargeScene: return 60;
  }
  return 60;
}

// synth.cpp:156-211 constants
constexpr double kOrbitStepRad = 0.4 * kPi / 180.0;
constexpr double kSheetHalfWidth = 0.18, kSheetHalfArc = 0.135, kSheetZ = 0.95;
constexpr double kSheetMaxAngle = 55.0 * kPi / 180.0;
constexpr double kCloseSphereRadius = 0.055;
constexpr double kSlideEdgeStart = -0.35, kSlideEdgeTravel = 0.852, kSlideLowZ = 1.0,
                 kSlideHighZ = 0.96, kSlideHalfHeight = 0.20, kSlideHalfWidth = 1.2;

double open_close_gap(double u) {
  if (u <= 0.57) return 0.18 + (0.008 - 0.18) * smoothstep(u / 0.57);
  if (u <= 0.78) return 0.008 + (0.05 - 0.008) * smoothstep((u - 0.57) / 0.21);
  return 0.05 + (0.008 - 0.05) * smoothstep((u - 0.78) / 0.22);
}
double bending_angle(double u) {
  constexpr double lead = 0.1;
  if (u <= lead) return 0.0;
  return kSheetMaxAngle * smoothstep((u - lead) / (1.0 - lead));
}
// smooth 0 -> 1 -> 0 cycle used by the articulated body
double swing(double u, double phase) { return 0.5 - 0.5 * std::cos(2.0 * kPi * (u + phase)); }

// Config 2 body: torso + head + two-link arms + legs, joint rotations in the
// image plane and a breathing torso; ~0.9 m^2 visible at ~1.2 m.
void articulated_body(Scene& s, double u, P3 o = P3()) {
  const double breathe = 1.0 + 0.015 * std::sin(2.0 * kPi * u);
  const P3 torso_c = o + p3(0.0, 0.12, 1.22);
  s.ellipsoids.push_back({torso_c, rot_z(0.04 * std::sin(2.0 * kPi * u)),
                          p3(0.35 * breathe, 0.46, 0.17 * breathe)});
  const P3 neck = o + p3(0.0, -0.29, 1.22);
  const R3 nod = rot_x(0.12 * std::sin(2.0 * kPi * u));
  s.spheres.push_back({neck + nod * p3(0.0, -0.16, 0.0), 0.15});
  for (int side = -1; side <= 1; side += 2) {
    const P3 shoulder = o + p3(0.36 * side, -0.18, 1.22);
    const double raise = (22.0 + 40.0 * swing(u, side > 0 ? 0.0 : 0.25)) * kPi / 180.0;
    const R3 r_up = rot_z(-side * raise);
    const P3 elbow = shoulder + r_up * p3(0.0, 0.40, 0.0);
    const double bend = (15.0 + 45.0 * swing(u, side > 0 ? 0.1 : 0.35)) * kPi / 180.0;
    const R3 r_lo = r_up * rot_z(side * bend);
    const P3 wrist = elbow + r_lo * p3(0.0, 0.36, 0.0);
    s.capsules.push_back({shoulder, elbow, 0.10});
    s.capsules.push_back({elbow, wrist, 0.085});
    const P3 hip = o + p3(0.15 * side, 0.46, 1.22);
    const R3 r_leg = rot_z(side * (6.0 + 10.0 * swing(u, side > 0 ? 0.5 : 0.0)) * kPi / 180.0);
    s.capsules.push_back({hip, hip + r_leg * p3(0.0, 0.55, 0.0), 0.12});
  }
}

Scene scene_at(int kind, double u) {  // synth.cpp:275-334 (+ new scenes)
  Scene s;
  switch (kind) {
    case kStaticPlane:
      s.rects.push_back({1.0, -0.4, 0.4, -0.3, 0.3});
      break;
    case kRigidOrbit:
      s.spheres.push_back({p3(-0.11, -0.03, 1.15), 0.10});
      s.spheres.push_back({p3(0.10, 0.05, 1.05), 0.08});
      s.spheres.push_back({p3(0.0, -0.09, 0.93), 0.065});
      break;
    case kBendingSheet: {
      const double alpha = bending_angle(u);
      if (alpha < 1e-6)
        s.rects.push_back({kSheetZ, -kSheetHalfWidth, kSheetHalfWidth, -kSheetHalfArc, kSheetHalfArc});
      else
        s.sheets.push_back({kSheetHalfWidth, kSheetHalfArc / alpha, kSheetZ, alpha});
      break;
    }
    case kArticulatedTwoPart: {
      s.spheres.push_back({p3(-0.085, 0.0, 1.0), 0.06});
      const double beta = (60.0 * kPi / 180.0) * smoothstep(u);
      const P3 hinge = p3(0.03, 0.0, 1.0);
      s.spheres.push_back({hinge + rot_z(beta) * p3(0.10, 0.0, 0.0), 0.05});
      break;
    }
    case kOpenToClose: {
      const double xc = kCloseSphereRadius + 0.5 * open_close_gap(u);
      s.spheres.push_back({p3(-xc, 0.0, 1.0), kCloseSphereRadius});
      s.spheres.push_back({p3(xc, 0.0, 1.0), kCloseSphereRadius});
      break;
    }
    case kTangentialSlide: {
      const double edge = kSlideEdgeStart + kSlideEdgeTravel * u;
      s.rects.push_back({kSlideLowZ, -kSlideHalfWidth, kSlideHalfWidth, -kSlideHalfHeight, kSlideHalfHeight});
      s.rects.push_back({kSlideHighZ, edge, kSlideHalfWidth, -kSlideHalfHeight, kSlideHalfHeight});
      break;
    }
    case kTurntable: {
      const double theta = 4.0 * kPi * u;
      const R3 spin = rot_y(theta);
      const P3 axis_point = p3(0.0, 0.0, 1.1);
      s.spheres.push_back({axis_point + spin * p3(0.07, 0.01, 0.0), 0.05});
      s.spheres.push_back({axis_point + spin * (rot_y(140.0 * kPi / 180.0) * p3(0.09, -0.025, 0.0)), 0.04});
      break;
    }
    case kDeformingSphere: {
      // Config 1: r = 0.2 m ellipsoid centred 0.6 m ahead; semi-axes breathe
      // anisotropically (non-rigid) and the body turns slowly.
      const double a = 0.04 * std::sin(2.0 * kPi * u);
      s.ellipsoids.push_back({p3(0.0, 0.0, 0.72), rot_y(0.15 * u) * rot_z(0.1 * u),
                              p3(0.24 * (1.0 + a), 0.24 * (1.0 - 0.5 * a), 0.24 * (1.0 + 0.5 * a))});
      break;
    }
    case kArticulatedBody:
      articulated_body(s, u);
      break;
    case kSineSheet:  // 2 cm waves travelling ~1.3 mm per frame over 10 frames
      s.sines.push_back({1.2, 0.02, 2.0 * kPi / 0.4, 2.0 * kPi / 0.3, 0.2 * kPi * u});
      break;
    case kLargeScene: {
      // Config 3: a wide back wall band (revealed by the panning camera every
      // frame), an articulated body at ~2.3 m and two spheres closing into
      // contact (open-to-close topology change): ~5 m^2 visible at 1280x960.
      s.rects.push_back({3.3, -2.4, 2.4, -0.55, 0.55});
      articulated_body(s, u, p3(-0.45, 0.0, 1.1));
      const double xc = 0.16 + 0.5 * open_close_gap(u) * 2.0;
      s.spheres.push_back({p3(0.75 - xc, 0.05, 2.0), 0.16});
      s.spheres.push_back({p3(0.75 + xc, 0.05, 2.0), 0.16});
      break;
    }
  }
  return s;
}

double normalized_time(int t, int frames) { return frames > 1 ? double(t) / double(frames - 1) : 0.0; }

void camera_pose(int kind, int t, R3& R, P3& tr) {  // synth.cpp:336-344
  R = R3();
  tr = P3();
  if (kind == kLargeScene) {  // slow pan about the vertical axis: new wall every frame
    R = rot_y(0.25 * kPi / 180.0 * t);
    return;
  }
  if (kind != kRigidOrbit) return;
  const P3 pivot = p3(0.0, 0.0, 1.1);
  R = rot_y(kOrbitStepRad * t);
  tr = pivot - R * pivot;
}

}  // namespace

extern "C" {

int32_t ds_synth_scenario(const char* name) {
  if (!name) return -1;
  for (int i = 0; i < kNumKinds; ++i)
    if (std::strcmp(name, kNames[i]) == 0) return i;
  return -1;
}
const char* ds_synth_scenario_name(int32_t k) { return (k >= 0 && k < kNumKinds) ? kNames[k] : "unknown"; }
int32_t ds_synth_default_frames(int32_t k) { return (k >= 0 && k < kNumKinds) ? default_frames(k) : -1; }

// SyntheticSequence::render_depth (synth.cpp:346-373)
ds_status ds_synth_render_depth(int32_t kind, int32_t frames, const ds_config* cfg, double noise,
                                uint32_t seed, int32_t t, uint16_t* out) {
  if (kind < 0 || kind >= kNumKinds) return DS_ERR_UNKNOWN_SCENARIO;
  if (!cfg || !out) return DS_ERR_INVALID_ARGUMENT;
  if (frames <= 0) frames = default_frames(kind);
  const Scene scene = scene_at(kind, normalized_time(t, frames));
  R3 R;
  P3 origin;
  camera_pose(kind, t, R, origin);
  std::mt19937 rng(seed + uint32_t(t) * 2654435761u);
  std::normal_distribution<double> gauss(0.0, noise);
  const int W = cfg->width, H = cfg->height;
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      out[size_t(y) * W + x] = 0;
      const P3 dir = R * p3((x - cfg->cx) / cfg->fx, (y - cfg->cy) / cfg->fy, 1.0);
      const double s = scene_raycast(origin, dir, scene);
      if (!std::isfinite(s)) continue;
      double mm = s * 1000.0;
      if (noise > 0) mm += gauss(rng);
      const long v = std::lround(mm);
      if (v < 100 || v > 5000) continue;
      out[size_t(y) * W + x] = uint16_t(v);
    }
  return DS_OK;
}
ds_status ds_synth_camera_pose(int32_t kind, int32_t frames, int32_t t, double* pose) {
  if (kind < 0 || kind >= kNumKinds) return DS_ERR_UNKNOWN_SCENARIO;
  (void)frames;
  R3 R;
  P3 tr;
  camera_pose(kind, t, R, tr);
  for (int i = 0; i < 9; ++i) pose[i] = R.m[i];
  pose[9] = tr.x;
  pose[10] = tr.y;
  pose[11] = tr.z;
  return DS_OK;
}
double ds_synth_surface_distance(int32_t kind, int32_t frames, const double* p, int32_t t) {
  if (kind < 0 || kind >= kNumKinds) return kInf;
  if (frames <= 0) frames = default_frames(kind);
  return scene_distance(p3(p[0], p[1], p[2]), scene_at(kind, normalized_time(t, frames)));
}

}  // extern "C"
