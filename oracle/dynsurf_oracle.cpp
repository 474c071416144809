// dynsurf_oracle.cpp — CPU fp64 restatement of the SurfelWarp reference hot path.
//
// TEST INFRASTRUCTURE ONLY (see dynsurf_oracle.h). Every stage below cites the
// reference function it restates (paths relative to /root/reference/proj/core).
// Arithmetic is double precision throughout, like the reference
// (include/dynsurf/geometry.hpp:3-4). Small-vector sums are evaluated strictly
// left to right ((a0*b0 + a1*b1) + a2*b2 ...); the CUDA product follows the same
// order for every quantity that feeds a discrete decision, so discrete outputs
// (node sets, KNN indices, z-buffer winners, correspondence pairs, JtJ pattern,
// fusion winners, removal masks) can be compared bit-exactly on shared inputs.
// Build: oracle/Makefile (-O2 -ffp-contract=off, no -mfma, like the reference's
// x86-64 baseline Release build, proj/CMakeLists.txt:8-10).

#include "dynsurf_oracle.h"

#include <algorithm>
#include <array>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstring>
#include <deque>
#include <limits>
#include <optional>
#include <string>
#include <unordered_map>
#include <vector>

namespace ora {

// ---------------------------------------------------------------- small math
struct V3 {
  double c[3] = {0, 0, 0};
  double& operator[](int i) { return c[i]; }
  double operator[](int i) const { return c[i]; }
};
struct Q4 {
  double c[4] = {0, 0, 0, 0};  // (w, x, y, z)
  double& operator[](int i) { return c[i]; }
  double operator[](int i) const { return c[i]; }
};
struct M3 {
  double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};  // row-major
  double& operator()(int r, int k) { return m[r * 3 + k]; }
  double operator()(int r, int k) const { return m[r * 3 + k]; }
};
struct M4 {
  double m[16] = {0};
  double& operator()(int r, int k) { return m[r * 4 + k]; }
  double operator()(int r, int k) const { return m[r * 4 + k]; }
};

static inline V3 mk(double a, double b, double d) { V3 v; v[0] = a; v[1] = b; v[2] = d; return v; }
static inline Q4 mq(double w, double x, double y, double z) {
  Q4 q; q[0] = w; q[1] = x; q[2] = y; q[3] = z; return q;
}
static inline V3 operator+(const V3& a, const V3& b) { return mk(a[0] + b[0], a[1] + b[1], a[2] + b[2]); }
static inline V3 operator-(const V3& a, const V3& b) { return mk(a[0] - b[0], a[1] - b[1], a[2] - b[2]); }
static inline V3 operator-(const V3& a) { return mk(-a[0], -a[1], -a[2]); }
static inline V3 operator*(double s, const V3& a) { return mk(s * a[0], s * a[1], s * a[2]); }
static inline V3 operator/(const V3& a, double s) { return mk(a[0] / s, a[1] / s, a[2] / s); }
static inline double dot(const V3& a, const V3& b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
static inline double sqn(const V3& a) { return dot(a, a); }
static inline double nrm(const V3& a) { return std::sqrt(sqn(a)); }
static inline V3 cross(const V3& a, const V3& b) {
  return mk(a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]);
}
static inline Q4 operator+(const Q4& a, const Q4& b) {
  return mq(a[0] + b[0], a[1] + b[1], a[2] + b[2], a[3] + b[3]);
}
static inline Q4 operator-(const Q4& a, const Q4& b) {
  return mq(a[0] - b[0], a[1] - b[1], a[2] - b[2], a[3] - b[3]);
}
static inline Q4 operator*(double s, const Q4& a) { return mq(s * a[0], s * a[1], s * a[2], s * a[3]); }
static inline Q4 operator/(const Q4& a, double s) { return mq(a[0] / s, a[1] / s, a[2] / s, a[3] / s); }
static inline Q4 operator-(const Q4& a) { return mq(-a[0], -a[1], -a[2], -a[3]); }
static inline double dot(const Q4& a, const Q4& b) {
  return ((a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]) + a[3] * b[3];
}
static inline double nrm(const Q4& a) { return std::sqrt(dot(a, a)); }
static inline V3 mul(const M3& r, const V3& p) {
  return mk((r(0, 0) * p[0] + r(0, 1) * p[1]) + r(0, 2) * p[2],
            (r(1, 0) * p[0] + r(1, 1) * p[1]) + r(1, 2) * p[2],
            (r(2, 0) * p[0] + r(2, 1) * p[1]) + r(2, 2) * p[2]);
}
static inline M3 mul(const M3& a, const M3& b) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o(i, j) = (a(i, 0) * b(0, j) + a(i, 1) * b(1, j)) + a(i, 2) * b(2, j);
  return o;
}
static inline M3 transpose(const M3& a) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o(i, j) = a(j, i);
  return o;
}

// geometry.cpp:7-12
static Q4 qmul(const Q4& a, const Q4& b) {
  return mq(a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
            a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
            a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
            a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]);
}
static inline Q4 qconj(const Q4& q) { return mq(q[0], -q[1], -q[2], -q[3]); }
// geometry.cpp:14-21  quat_multiply(q, p) == L(q) p
static M4 qleft(const Q4& q) {
  M4 m;
  const double v[16] = {q[0], -q[1], -q[2], -q[3], q[1], q[0], -q[3], q[2],
                        q[2], q[3],  q[0], -q[1], q[3], -q[2], q[1], q[0]};
  std::memcpy(m.m, v, sizeof v);
  return m;
}
// geometry.cpp:23-30  quat_multiply(p, q) == R(q) p
static M4 qright(const Q4& q) {
  M4 m;
  const double v[16] = {q[0], -q[1], -q[2], -q[3], q[1], q[0],  q[3], -q[2],
                        q[2], -q[3], q[0], q[1],  q[3], q[2], -q[1], q[0]};
  std::memcpy(m.m, v, sizeof v);
  return m;
}
// geometry.cpp:32-42
static Q4 quat_from_rotvec(const V3& om) {
  const double angle = nrm(om);
  if (angle < 1e-12) {
    Q4 q = mq(1.0, 0.5 * om[0], 0.5 * om[1], 0.5 * om[2]);
    return q / nrm(q);
  }
  const double half = 0.5 * angle;
  const V3 axis = om / angle;
  const double s = std::sin(half);
  return mq(std::cos(half), s * axis[0], s * axis[1], s * axis[2]);
}
// geometry.cpp:44-50 — Eigen::Quaterniond(Matrix3d) (Shoemake branch order),
// normalize, then canonical w >= 0.
static Q4 quat_from_matrix(const M3& m) {
  Q4 q;  // (w, x, y, z)
  double t = (m(0, 0) + m(1, 1)) + m(2, 2);
  if (t > 0.0) {
    t = std::sqrt(t + 1.0);
    q[0] = 0.5 * t;
    t = 0.5 / t;
    q[1] = (m(2, 1) - m(1, 2)) * t;
    q[2] = (m(0, 2) - m(2, 0)) * t;
    q[3] = (m(1, 0) - m(0, 1)) * t;
  } else {
    int i = 0;
    if (m(1, 1) > m(0, 0)) i = 1;
    if (m(2, 2) > m(i, i)) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    t = std::sqrt(m(i, i) - m(j, j) - m(k, k) + 1.0);
    q[1 + i] = 0.5 * t;
    t = 0.5 / t;
    q[0] = (m(k, j) - m(j, k)) * t;
    q[1 + j] = (m(j, i) + m(i, j)) * t;
    q[1 + k] = (m(k, i) + m(i, k)) * t;
  }
  q = q / nrm(q);
  if (q[0] < 0) q = -q;
  return q;
}
// geometry.cpp:52-56 — normalize then Quaterniond::toRotationMatrix
static M3 matrix_from_quat(const Q4& qin) {
  const Q4 q = qin / nrm(qin);
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  M3 r;
  r(0, 0) = 1.0 - (tyy + tzz);
  r(0, 1) = txy - twz;
  r(0, 2) = txz + twy;
  r(1, 0) = txy + twz;
  r(1, 1) = 1.0 - (txx + tzz);
  r(1, 2) = tyz - twx;
  r(2, 0) = txz - twy;
  r(2, 1) = tyz + twx;
  r(2, 2) = 1.0 - (txx + tyy);
  return r;
}

// geometry.hpp:36-69 (Se3)
struct Rig {
  M3 R;
  V3 t;
  V3 apply(const V3& p) const { return mul(R, p) + t; }
  V3 rotate(const V3& d) const { return mul(R, d); }
  Rig inverse() const {
    Rig o;
    o.R = transpose(R);
    o.t = -mul(o.R, t);
    return o;
  }
  Rig operator*(const Rig& b) const {
    Rig o;
    o.R = mul(R, b.R);
    o.t = mul(R, b.t) + t;
    return o;
  }
};
static Rig rig_from12(const double* p) {
  Rig r;
  for (int i = 0; i < 9; ++i) r.R.m[i] = p[i];
  r.t = mk(p[9], p[10], p[11]);
  return r;
}
static void rig_to12(const Rig& r, double* p) {
  for (int i = 0; i < 9; ++i) p[i] = r.R.m[i];
  p[9] = r.t[0]; p[10] = r.t[1]; p[11] = r.t[2];
}
// geometry.cpp:65-76
static Rig se3_increment(const V3& om, const V3& dt, const Rig& t) {
  Rig inc;
  inc.R = matrix_from_quat(quat_from_rotvec(om));
  inc.t = dt;
  Rig out = inc * t;
  out.R = matrix_from_quat(quat_from_matrix(out.R));  // renormalize_rotation
  return out;
}

// geometry.hpp:71-85, geometry.cpp:78-125
struct DQ {
  Q4 r = mq(1, 0, 0, 0);
  Q4 d = mq(0, 0, 0, 0);
};
static DQ dq_from_rig(const Rig& t) {
  DQ dq;
  dq.r = quat_from_matrix(t.R);
  dq.d = 0.5 * qmul(mq(0.0, t.t[0], t.t[1], t.t[2]), dq.r);
  return dq;
}
static DQ dq_normalized(const DQ& q) {  // geometry.cpp:102-109
  const double a = nrm(q.r);
  const double b = dot(q.r, q.d) / a;
  DQ o;
  o.r = q.r / a;
  o.d = q.d / a - (b / (a * a)) * q.r;
  return o;
}
static Rig dq_to_rig(const DQ& q) {  // geometry.cpp:86-93
  const DQ n = dq_normalized(q);
  Rig t;
  t.R = matrix_from_quat(n.r);
  const Q4 tq = qmul(n.d, qconj(n.r));
  t.t = mk(2.0 * tq[1], 2.0 * tq[2], 2.0 * tq[3]);
  return t;
}
static DQ dq_mul(const DQ& a, const DQ& b) {  // geometry.cpp:95-100
  DQ o;
  o.r = qmul(a.r, b.r);
  o.d = qmul(a.r, b.d) + qmul(a.d, b.r);
  return o;
}
static DQ dq_increment(const V3& om, const V3& dt) {  // geometry.cpp:120-125
  Rig inc;
  inc.R = matrix_from_quat(quat_from_rotvec(om));
  inc.t = dt;
  return dq_from_rig(inc);
}
static constexpr double kDegenerate = 1e-8;  // geometry.hpp:89
// geometry.cpp:127-147
static std::optional<DQ> blend(int n, const DQ* dqs, const double* w) {
  if (n <= 0) return std::nullopt;
  Q4 rs = mq(0, 0, 0, 0), ds = mq(0, 0, 0, 0);
  const Q4 pivot = dqs[0].r;
  for (int i = 0; i < n; ++i) {
    const double sign = (dot(pivot, dqs[i].r) < 0.0) ? -1.0 : 1.0;
    const double ww = sign * w[i];
    rs = rs + ww * dqs[i].r;
    ds = ds + ww * dqs[i].d;
  }
  if (nrm(rs) < kDegenerate) return std::nullopt;
  DQ sum;
  sum.r = rs;
  sum.d = ds;
  return dq_normalized(sum);
}
// geometry.cpp:156-159
static inline double skin_weight(const V3& x, const V3& p, double sigma) {
  const double d2 = sqn(x - p);
  return std::exp(-d2 / (2.0 * sigma * sigma));
}

// ------------------------------------------------------------------ types
struct Cfg : or_config {};
struct Surf {
  V3 p;
  V3 n = mk(0, 0, 1);
  double r = 0, c = 0;
  int32_t ti = 0, to = 0;
};
constexpr int kMaxSkin = 8;  // types.hpp:50
struct Skin {
  int32_t idx[kMaxSkin] = {0};
  double w[kMaxSkin] = {0};
  int count = 0;
  double wsum() const {
    double s = 0;
    for (int i = 0; i < count; ++i) s += w[i];
    return s;
  }
};
struct Node {
  V3 p;
  double sigma = 0.025;
  DQ T;
  std::vector<int32_t> nbr;
  V3 live() const { return dq_to_rig(T).apply(p); }  // warp_field.hpp:21
};
struct Model {
  std::vector<Surf> ref, live;
  std::vector<Skin> skin;
  size_t size() const { return ref.size(); }
};
struct Frame {
  int w = 0, h = 0, index = 0, valid_count = 0;
  std::vector<V3> vert, nrm;
  std::vector<double> conf, rad;
  std::vector<uint8_t> vvalid, valid;
};
struct Err {
  int code;
  std::string msg;
};
[[noreturn]] static void fail(int code, const std::string& m) { throw Err{code, m}; }

// types.hpp:11-39 (CameraIntrinsics)
struct Cam {
  double fx, fy, cx, cy;
  int w, h;
  explicit Cam(const Cfg& c) : fx(c.fx), fy(c.fy), cx(c.cx), cy(c.cy), w(c.width), h(c.height) {}
  void project(const V3& p, double& u, double& v) const {
    u = fx * p[0] / p[2] + cx;
    v = fy * p[1] / p[2] + cy;
  }
  V3 backproject(double px, double py, double d) const {
    return mk(d * (px - cx) / fx, d * (py - cy) / fy, d);
  }
  double mean_focal() const { return 0.5 * (fx + fy); }
  double max_radial() const {
    double best = 0;
    for (int corner = 0; corner < 4; ++corner) {
      const double x = (corner & 1) ? double(w - 1) : 0.0;
      const double y = (corner & 2) ? double(h - 1) : 0.0;
      best = std::max(best, std::hypot(x - cx, y - cy));
    }
    return best;
  }
};

// ------------------------------------------------------------ voxel hash
// spatial_grid.hpp:16-136: uniform hash, exact kNN by rings ordered (d2, idx),
// strict-< existence query.
struct NB {
  double d2;
  int32_t i;
  bool operator<(const NB& o) const { return d2 != o.d2 ? d2 < o.d2 : i < o.i; }
};
class Voxels {
 public:
  explicit Voxels(double cell) : cell_(cell), inv_(1.0 / cell) {}
  int32_t add(const V3& p) {
    const int32_t id = int32_t(pts_.size());
    pts_.push_back(p);
    int32_t c[3];
    coord(p, c);
    cells_[key(c[0], c[1], c[2])].push_back(id);
    for (int a = 0; a < 3; ++a) {
      lo_[a] = std::min(lo_[a], c[a]);
      hi_[a] = std::max(hi_[a], c[a]);
    }
    return id;
  }
  bool any_within(const V3& q, double radius) const {
    if (pts_.empty()) return false;
    int32_t c[3];
    coord(q, c);
    const int reach = int(std::ceil(radius * inv_));
    const double r2 = radius * radius;
    for (int dz = -reach; dz <= reach; ++dz)
      for (int dy = -reach; dy <= reach; ++dy)
        for (int dx = -reach; dx <= reach; ++dx) {
          auto it = cells_.find(key(c[0] + dx, c[1] + dy, c[2] + dz));
          if (it == cells_.end()) continue;
          for (int32_t id : it->second)
            if (sqn(pts_[id] - q) < r2) return true;
        }
    return false;
  }
  std::vector<NB> knn(const V3& q, int k) const {
    std::vector<NB> best;
    if (pts_.empty() || k <= 0) return best;
    int32_t c[3];
    coord(q, c);
    int max_ring = 0;
    for (int a = 0; a < 3; ++a) {
      max_ring = std::max(max_ring, std::abs(c[a] - lo_[a]));
      max_ring = std::max(max_ring, std::abs(c[a] - hi_[a]));
    }
    ++max_ring;
    auto consider = [&](const std::vector<int32_t>& ids) {
      for (int32_t id : ids) {
        const NB cand{sqn(pts_[id] - q), id};
        if (int(best.size()) == k && !(cand < best.back())) continue;
        best.insert(std::lower_bound(best.begin(), best.end(), cand), cand);
        if (int(best.size()) > k) best.pop_back();
      }
    };
    for (int ring = 0; ring <= max_ring; ++ring) {
      if (int(best.size()) == k) {
        const double bound = double(ring - 1) * cell_;
        if (bound > 0 && bound * bound > best.back().d2) break;
      }
      for (int dz = -ring; dz <= ring; ++dz)
        for (int dy = -ring; dy <= ring; ++dy)
          for (int dx = -ring; dx <= ring; ++dx) {
            if (std::max({std::abs(dx), std::abs(dy), std::abs(dz)}) != ring) continue;
            auto it = cells_.find(key(c[0] + dx, c[1] + dy, c[2] + dz));
            if (it != cells_.end()) consider(it->second);
          }
    }
    return best;
  }

 private:
  void coord(const V3& p, int32_t* c) const {
    for (int a = 0; a < 3; ++a) c[a] = int32_t(std::floor(p[a] * inv_));
  }
  static int64_t key(int32_t x, int32_t y, int32_t z) {
    const int64_t b = int64_t(1) << 20;
    return ((int64_t(x) + b) << 42) | ((int64_t(y) + b) << 21) | (int64_t(z) + b);
  }
  double cell_, inv_;
  std::vector<V3> pts_;
  std::unordered_map<int64_t, std::vector<int32_t>> cells_;
  int32_t lo_[3] = {0, 0, 0}, hi_[3] = {0, 0, 0};
};

// ------------------------------------------------------- dense LDLT (Eigen)
// Restates Eigen::LDLT (solver.cpp:225, 386): diagonal pivoting on the
// largest remaining |diagonal|, zero pivots kept, pseudo-inverse of D with
// tolerance DBL_MIN at solve time. In-place on a row-major n x n copy.
static std::vector<double> ldlt_solve(int n, std::vector<double> a, const std::vector<double>& b) {
  std::vector<int> perm(n);
  std::vector<double> temp(n);
  auto A = [&](int r, int c) -> double& { return a[size_t(r) * n + c]; };
  bool zero_all = false;
  for (int k = 0; k < n; ++k) {
    int big = k;
    double bv = std::abs(A(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A(i, i)) > bv) { bv = std::abs(A(i, i)); big = i; }
    perm[k] = big;
    if (big != k) {
      // symmetric swap of rows/cols k and big (only the lower triangle is used)
      for (int c = 0; c < k; ++c) std::swap(A(k, c), A(big, c));
      for (int r = big + 1; r < n; ++r) std::swap(A(r, k), A(r, big));
      std::swap(A(k, k), A(big, big));
      for (int i = k + 1; i < big; ++i) {
        const double tmp = A(i, k);
        A(i, k) = A(big, i);
        A(big, i) = tmp;
      }
    }
    if (k > 0) {
      for (int c = 0; c < k; ++c) temp[c] = A(c, c) * A(k, c);
      double s = 0;
      for (int c = 0; c < k; ++c) s += A(k, c) * temp[c];
      A(k, k) -= s;
      for (int r = k + 1; r < n; ++r) {
        double acc = 0;
        const double* row = &a[size_t(r) * n];
        for (int c = 0; c < k; ++c) acc += row[c] * temp[c];
        A(r, k) -= acc;
      }
    }
    const double akk = A(k, k);
    const bool valid = std::abs(akk) > 0.0;
    if (k == 0 && !valid) {
      zero_all = true;
      break;
    }
    if (valid)
      for (int r = k + 1; r < n; ++r) A(r, k) /= akk;
  }
  std::vector<double> x(b);
  if (zero_all) {
    std::fill(x.begin(), x.end(), 0.0);
    return x;
  }
  for (int k = 0; k < n; ++k) std::swap(x[k], x[perm[k]]);
  for (int r = 0; r < n; ++r) {  // L y = Pb (unit lower)
    double s = x[r];
    for (int c = 0; c < r; ++c) s -= A(r, c) * x[c];
    x[r] = s;
  }
  for (int i = 0; i < n; ++i) {
    if (std::abs(A(i, i)) > DBL_MIN) x[i] /= A(i, i);
    else x[i] = 0.0;
  }
  for (int r = n - 1; r >= 0; --r) {  // L^T z = y
    double s = x[r];
    for (int c = r + 1; c < n; ++c) s -= A(c, r) * x[c];
    x[r] = s;
  }
  for (int k = n - 1; k >= 0; --k) std::swap(x[k], x[perm[k]]);
  return x;
}

// symmetric Jacobi eigenvalues (restates Eigen::SelfAdjointEigenSolver /
// JacobiSVD results; solver.cpp:163, fusion.cpp:175)
static std::vector<double> sym_eigenvalues(int n, std::vector<double> a) {
  auto A = [&](int r, int c) -> double& { return a[size_t(r) * n + c]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += A(p, q) * A(p, q);
    if (off < 1e-300) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (A(p, q) == 0.0) continue;
        const double theta = (A(q, q) - A(p, p)) / (2.0 * A(p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) /
                         (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * akq;
          A(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * aqk;
          A(q, k) = s * apk + c * aqk;
        }
      }
  }
  std::vector<double> ev(n);
  for (int i = 0; i < n; ++i) ev[i] = A(i, i);
  return ev;
}
static double sigma_max3(const M3& s) {
  std::vector<double> ata(9, 0.0);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = 0;
      for (int k = 0; k < 3; ++k) acc += s(k, i) * s(k, j);
      ata[i * 3 + j] = acc;
    }
  const auto ev = sym_eigenvalues(3, ata);
  const double m = std::max({ev[0], ev[1], ev[2], 0.0});
  return std::sqrt(m);
}

// ---------------------------------------------------------- fp32 mirroring
static inline double f32(double v) { return double(float(v)); }
static void round_surf(Surf& s) {
  for (int a = 0; a < 3; ++a) {
    s.p[a] = f32(s.p[a]);
    s.n[a] = f32(s.n[a]);
  }
  s.r = f32(s.r);
  s.c = f32(s.c);
}
static void round_model(Model& m) {
  for (auto& s : m.ref) round_surf(s);
  for (auto& s : m.live) round_surf(s);
  for (auto& e : m.skin)
    for (int i = 0; i < e.count; ++i) e.w[i] = f32(e.w[i]);
}

// ------------------------------------------------------ depth processing
static const double kMinAbsNz = std::cos(75.0 * M_PI / 180.0);
// depth_processing.cpp:14-32
static void backproject(const uint16_t* depth, int w, int h, const Cfg& cfg, std::vector<V3>& vert,
                        std::vector<uint8_t>& vvalid) {
  if (w != cfg.width || h != cfg.height)
    fail(1, "depth image size does not match intrinsics");
  const Cam k(cfg);
  vert.assign(size_t(w) * h, V3());
  vvalid.assign(size_t(w) * h, 0);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const uint16_t raw = depth[size_t(y) * w + x];
      if (raw == 0) continue;
      const double d = raw * 1e-3;
      if (d < cfg.depth_min || d > cfg.depth_max) continue;
      vert[size_t(y) * w + x] = k.backproject(x, y, d);
      vvalid[size_t(y) * w + x] = 1;
    }
}
// depth_processing.cpp:34-57
static void estimate_normals(const std::vector<V3>& v, const std::vector<uint8_t>& vv, int w,
                             int h, std::vector<V3>& n, std::vector<uint8_t>& nv) {
  n.assign(size_t(w) * h, V3());
  nv.assign(size_t(w) * h, 0);
  auto at = [&](int x, int y) { return size_t(y) * w + x; };
  for (int y = 1; y + 1 < h; ++y)
    for (int x = 1; x + 1 < w; ++x) {
      if (!vv[at(x, y)] || !vv[at(x - 1, y)] || !vv[at(x + 1, y)] || !vv[at(x, y - 1)] ||
          !vv[at(x, y + 1)])
        continue;
      const V3 tu = v[at(x + 1, y)] - v[at(x - 1, y)];
      const V3 tv = v[at(x, y + 1)] - v[at(x, y - 1)];
      V3 c = cross(tu, tv);
      const double len = nrm(c);
      if (len < 1e-12) continue;
      c = c / len;
      if (dot(c, v[at(x, y)]) > 0) c = -c;
      n[at(x, y)] = c;
      nv[at(x, y)] = 1;
    }
}
// depth_processing.cpp:59-69
static double confidence(double px, double py, const Cfg& cfg) {
  const Cam k(cfg);
  const double mr = k.max_radial();
  const double g = mr > 0 ? std::hypot(px - k.cx, py - k.cy) / mr : 0.0;
  return std::exp(-(g * g) / (2.0 * 0.6 * 0.6));
}
static double radius_of(double d, double f, double nz) {
  const double a = std::max(std::abs(nz), kMinAbsNz);
  return std::sqrt(2.0) * d / (f * a);
}
// depth_processing.cpp:71-101
static void bilateral(const uint16_t* in, int w, int h, double ss, double sd, uint16_t* out) {
  const double i2s = 1.0 / (2.0 * ss * ss), i2d = 1.0 / (2.0 * sd * sd);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const uint16_t c = in[size_t(y) * w + x];
      out[size_t(y) * w + x] = 0;
      if (c == 0) continue;
      double ws = 0, vs = 0;
      for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx) {
          const int nx = x + dx, ny = y + dy;
          if (nx < 0 || nx >= w || ny < 0 || ny >= h) continue;
          const uint16_t s = in[size_t(ny) * w + nx];
          if (s == 0) continue;
          const double dd = double(s) - double(c);
          const double wb = std::exp(-(dx * dx + dy * dy) * i2s - dd * dd * i2d);
          ws += wb;
          vs += wb * s;
        }
      out[size_t(y) * w + x] = uint16_t(std::lround(vs / ws));
    }
}
// depth_processing.cpp:103-138
static Frame build_frame(const uint16_t* depth_in, int w, int h, int index, const Cfg& cfg) {
  Frame f;
  f.w = w;
  f.h = h;
  f.index = index;
  std::vector<uint16_t> filtered;
  const uint16_t* depth = depth_in;
  if (cfg.bilateral_filter) {
    filtered.resize(size_t(w) * h);
    bilateral(depth_in, w, h, cfg.bilateral_sigma_space, cfg.bilateral_sigma_depth,
              filtered.data());
    depth = filtered.data();
  }
  backproject(depth, w, h, cfg, f.vert, f.vvalid);
  std::vector<uint8_t> nv;
  estimate_normals(f.vert, f.vvalid, w, h, f.nrm, nv);
  f.conf.assign(size_t(w) * h, 0.0);
  f.rad.assign(size_t(w) * h, 0.0);
  f.valid.assign(size_t(w) * h, 0);
  const Cam k(cfg);
  const double focal = k.mean_focal();
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t i = size_t(y) * w + x;
      if (!f.vvalid[i] || !nv[i]) continue;
      f.valid[i] = 1;
      ++f.valid_count;
      f.conf[i] = confidence(x, y, cfg);
      f.rad[i] = radius_of(f.vert[i][2], focal, f.nrm[i][2]);
    }
  return f;
}

// ------------------------------------------------------------ warp field
// warp_field.cpp:11-22
static std::optional<DQ> blend_entry(const Skin& e, const std::vector<Node>& nodes) {
  if (e.count == 0) return std::nullopt;
  DQ dqs[kMaxSkin];
  for (int i = 0; i < e.count; ++i) dqs[i] = nodes[e.idx[i]].T;
  return blend(e.count, dqs, e.w);
}
// warp_field.cpp:42-56
static void node_edges(std::vector<Node>& nodes, int k_nb) {
  const int n = int(nodes.size());
  for (int j = 0; j < n; ++j) {
    std::vector<NB> cands;
    cands.reserve(n);
    for (int i = 0; i < n; ++i) {
      if (i == j) continue;
      cands.push_back({sqn(nodes[i].p - nodes[j].p), i});
    }
    const int k = std::min<int>(k_nb, int(cands.size()));
    std::partial_sort(cands.begin(), cands.begin() + k, cands.end());
    nodes[j].nbr.clear();
    for (int i = 0; i < k; ++i) nodes[j].nbr.push_back(cands[i].i);
  }
}
// warp_field.cpp:60-79
static std::vector<Skin> skin_bulk(const std::vector<Surf>& s, const std::vector<Node>& nodes,
                                   const Cfg& cfg) {
  Voxels grid(cfg.node_sigma);
  for (const auto& nd : nodes) grid.add(nd.p);
  std::vector<Skin> table(s.size());
  for (size_t i = 0; i < s.size(); ++i) {
    const auto nbs = grid.knn(s[i].p, cfg.knn_k);
    Skin& e = table[i];
    for (const auto& nb : nbs) {
      e.idx[e.count] = nb.i;
      e.w[e.count] = skin_weight(s[i].p, nodes[nb.i].p, nodes[nb.i].sigma);
      ++e.count;
    }
  }
  return table;
}
// warp_field.cpp:83-102
static void init_warp_field(Model& m, std::vector<Node>& nodes_out, const Cfg& cfg) {
  if (m.ref.empty()) fail(2, "init_warp_field: no reference surfels");
  std::vector<Node> nodes;
  Voxels acc(cfg.node_sigma);
  for (const auto& s : m.ref) {
    if (acc.any_within(s.p, cfg.node_sigma)) continue;
    acc.add(s.p);
    Node nd;
    nd.p = s.p;
    nd.sigma = cfg.node_sigma;
    nodes.push_back(nd);
  }
  node_edges(nodes, cfg.node_neighbor_k);
  m.skin = skin_bulk(m.ref, nodes, cfg);
  nodes_out = std::move(nodes);
}
// warp_field.cpp:104-126
static std::optional<Surf> fwd_warp_surfel(const Surf& ref, const Skin& e,
                                           const std::vector<Node>& nodes) {
  const auto b = blend_entry(e, nodes);
  if (!b) return std::nullopt;
  const Rig w = dq_to_rig(*b);
  Surf live = ref;
  live.p = w.apply(ref.p);
  live.n = w.rotate(ref.n);
  return live;
}
static std::optional<Surf> inv_warp_surfel(const Surf& live, const Skin& e,
                                           const std::vector<Node>& nodes) {
  const auto b = blend_entry(e, nodes);
  if (!b) return std::nullopt;
  const Rig inv = dq_to_rig(*b).inverse();
  Surf ref = live;
  ref.p = inv.apply(live.p);
  ref.n = inv.rotate(live.n);
  return ref;
}
// warp_field.cpp:128-140
static int forward_warp(Model& m, const std::vector<Node>& nodes) {
  int degenerate = 0;
  for (size_t i = 0; i < m.size(); ++i) {
    const auto w = fwd_warp_surfel(m.ref[i], m.skin[i], nodes);
    if (w) m.live[i] = *w;
    else {
      m.live[i] = m.ref[i];
      ++degenerate;
    }
  }
  return degenerate;
}
// warp_field.cpp:142-184
static int extend_warp_field(const std::vector<Surf>& app, std::vector<Node>& nodes,
                             const Cfg& cfg) {
  if (app.empty()) return 0;
  const int existing = int(nodes.size());
  Voxels occ(cfg.node_sigma);
  for (const auto& nd : nodes) occ.add(nd.p);
  Voxels existing_only = occ;
  int appended = 0;
  for (const auto& s : app) {
    if (occ.any_within(s.p, cfg.node_sigma)) continue;
    occ.add(s.p);
    Node nd;
    nd.p = s.p;
    nd.sigma = cfg.node_sigma;
    if (existing > 0) {
      const auto nbs = existing_only.knn(s.p, cfg.knn_k);
      DQ dqs[kMaxSkin];
      double ws[kMaxSkin];
      int c = 0;
      for (const auto& nb : nbs) {
        dqs[c] = nodes[nb.i].T;
        ws[c] = skin_weight(s.p, nodes[nb.i].p, nodes[nb.i].sigma);
        ++c;
      }
      const auto b = blend(c, dqs, ws);
      if (b) nd.T = *b;
    }
    nodes.push_back(nd);
    ++appended;
  }
  if (appended > 0) node_edges(nodes, cfg.node_neighbor_k);
  return appended;
}
// warp_field.cpp:186-236
static void update_skinning_incremental(std::vector<Skin>& table, const std::vector<Surf>& ref,
                                        const std::vector<Node>& nodes, int first_new,
                                        const Cfg& cfg) {
  const int total = int(nodes.size());
  if (first_new >= total) return;
  struct Slot {
    double d2;
    int32_t i;
    double w;
    bool operator<(const Slot& o) const { return d2 != o.d2 ? d2 < o.d2 : i < o.i; }
  };
  for (size_t s = 0; s < table.size(); ++s) {
    Skin& e = table[s];
    const V3& pos = ref[s].p;
    Slot slots[kMaxSkin];
    int count = e.count;
    for (int m = 0; m < count; ++m) {
      const int32_t id = e.idx[m];
      slots[m] = Slot{sqn(nodes[id].p - pos), id, e.w[m]};
    }
    std::sort(slots, slots + count);
    bool changed = false;
    for (int32_t j = first_new; j < total; ++j) {
      const Slot cand{sqn(nodes[j].p - pos), j, skin_weight(pos, nodes[j].p, nodes[j].sigma)};
      if (count < cfg.knn_k) {
        slots[count++] = cand;
        std::sort(slots, slots + count);
        changed = true;
      } else if (cand < slots[count - 1]) {
        slots[count - 1] = cand;
        std::sort(slots, slots + count);
        changed = true;
      }
    }
    if (!changed) continue;
    e.count = count;
    for (int m = 0; m < count; ++m) {
      e.idx[m] = slots[m].i;
      e.w[m] = slots[m].w;
    }
  }
}

// ------------------------------------------------------------------ raster
static inline int ss_coord(double u, int factor) { return int(std::floor(factor * (u + 0.5))); }
struct IndexMap {
  int w = 0, h = 0, factor = 1;
  std::vector<int32_t> idx;
  std::vector<double> depth;
};
// raster.cpp:8-30
static IndexMap render_index_map(const std::vector<Surf>& live, const Rig& pose, const Cfg& cfg,
                                 int factor) {
  IndexMap map;
  map.factor = factor;
  map.w = cfg.width * factor;
  map.h = cfg.height * factor;
  map.idx.assign(size_t(map.w) * map.h, -1);
  map.depth.assign(size_t(map.w) * map.h, std::numeric_limits<double>::infinity());
  const Rig w2c = pose.inverse();
  const Cam k(cfg);
  for (size_t i = 0; i < live.size(); ++i) {
    const V3 pc = w2c.apply(live[i].p);
    if (pc[2] <= 0) continue;
    double u, v;
    k.project(pc, u, v);
    const int sx = ss_coord(u, factor), sy = ss_coord(v, factor);
    if (sx < 0 || sx >= map.w || sy < 0 || sy >= map.h) continue;
    const size_t c = size_t(sy) * map.w + sx;
    if (pc[2] < map.depth[c]) {
      map.depth[c] = pc[2];
      map.idx[c] = int32_t(i);
    }
  }
  return map;
}
struct ModelMaps {
  int w = 0, h = 0;
  std::vector<V3> vert, nrm;
  std::vector<int32_t> idx;
  std::vector<double> depth;
  std::vector<uint8_t> valid;
};
// raster.cpp:32-121
static ModelMaps render_model_maps(const std::vector<Surf>& live, const Rig& pose, const Cfg& cfg,
                                   int t_now, int t_last) {
  const int W = cfg.width, H = cfg.height;
  const double kInf = std::numeric_limits<double>::infinity();
  ModelMaps mm;
  mm.w = W;
  mm.h = H;
  mm.vert.assign(size_t(W) * H, V3());
  mm.nrm.assign(size_t(W) * H, V3());
  mm.idx.assign(size_t(W) * H, -1);
  mm.depth.assign(size_t(W) * H, kInf);
  mm.valid.assign(size_t(W) * H, 0);
  bool any_stable = false;
  for (const auto& s : live)
    if (s.c > cfg.delta_stable) {
      any_stable = true;
      break;
    }
  const bool bootstrap = (t_now - t_last <= cfg.delta_recent) || !any_stable;
  std::vector<double> sd(size_t(W) * H, kInf), pd(size_t(W) * H, kInf);
  std::vector<int32_t> si(size_t(W) * H, -1), pi(size_t(W) * H, -1);
  const Rig w2c = pose.inverse();
  const Cam k(cfg);
  const double focal = k.mean_focal();
  auto inb = [&](int x, int y) { return x >= 0 && x < W && y >= 0 && y < H; };
  for (size_t i = 0; i < live.size(); ++i) {
    const Surf& s = live[i];
    const bool stable = s.c > cfg.delta_stable;
    const bool recent = (t_now - s.to) <= cfg.delta_recent;
    if (!stable && !(bootstrap && recent)) continue;
    const V3 pc = w2c.apply(s.p);
    if (pc[2] <= 0) continue;
    const V3 nc = w2c.rotate(s.n);
    if (dot(nc, pc) >= 0) continue;
    double u, v;
    k.project(pc, u, v);
    const int cx = int(std::lround(u)), cy = int(std::lround(v));
    if (inb(cx, cy) && pc[2] < pd[size_t(cy) * W + cx]) {
      pd[size_t(cy) * W + cx] = pc[2];
      pi[size_t(cy) * W + cx] = int32_t(i);
    }
    const double rpx = s.r * focal / pc[2];
    const double r2 = rpx * rpx;
    auto splat = [&](int x, int y) {
      if (!inb(x, y)) return;
      const size_t c = size_t(y) * W + x;
      if (pc[2] < sd[c]) {
        sd[c] = pc[2];
        si[c] = int32_t(i);
      }
    };
    for (int y = int(std::ceil(v - rpx)); y <= int(std::floor(v + rpx)); ++y)
      for (int x = int(std::ceil(u - rpx)); x <= int(std::floor(u + rpx)); ++x) {
        const double dx = x - u, dy = y - v;
        if (dx * dx + dy * dy <= r2) splat(x, y);
      }
    splat(cx, cy);
  }
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const size_t c = size_t(y) * W + x;
      int32_t win = pi[c];
      double dep = pd[c];
      if (win < 0) {
        win = si[c];
        dep = sd[c];
      }
      if (win < 0) continue;
      mm.idx[c] = win;
      mm.vert[c] = live[win].p;
      mm.nrm[c] = live[win].n;
      mm.depth[c] = dep;
      mm.valid[c] = 1;
    }
  return mm;
}

// ------------------------------------------------------------------ solver
constexpr double kGateDist = 0.03;   // solver.hpp:14
constexpr double kGateNormal = 0.7;  // solver.hpp:15
constexpr int kRigidMinPairs = 100;  // solver.hpp:19
struct Pair {
  int32_t s = -1;
  int px = 0, py = 0;
  V3 vm, vd, nd;
};
// solver.cpp:244-271
static std::vector<Pair> find_correspondences(const Frame& f, const ModelMaps& mm, const Rig& pose) {
  std::vector<Pair> pairs;
  if (f.w != mm.w || f.h != mm.h) fail(1, "find_correspondences: map resolutions differ");
  for (int y = 0; y < f.h; ++y)
    for (int x = 0; x < f.w; ++x) {
      const size_t c = size_t(y) * f.w + x;
      if (!f.valid[c] || !mm.valid[c]) continue;
      const V3 vd = pose.apply(f.vert[c]);
      const V3 nd = pose.rotate(f.nrm[c]);
      const V3& vm = mm.vert[c];
      if (nrm(vm - vd) >= kGateDist) continue;
      if (dot(mm.nrm[c], nd) <= kGateNormal) continue;
      Pair p;
      p.s = mm.idx[c];
      p.px = x;
      p.py = y;
      p.vm = vm;
      p.vd = vd;
      p.nd = nd;
      pairs.push_back(p);
    }
  return pairs;
}

// solver.cpp:29-49 (solver_detail::BlendState)
struct BlendState {
  Q4 rs, ds;
  double sw[kMaxSkin] = {0};
  int count = 0;
  bool degenerate = true;
};
static BlendState blend_state(const Skin& e, const std::vector<Node>& nodes) {
  BlendState st;
  st.count = e.count;
  if (e.count == 0) return st;
  const Q4 pivot = nodes[e.idx[0]].T.r;
  for (int m = 0; m < e.count; ++m) {
    const DQ& dq = nodes[e.idx[m]].T;
    const double sign = (dot(pivot, dq.r) < 0.0) ? -1.0 : 1.0;
    const double w = sign * e.w[m];
    st.sw[m] = w;
    st.rs = st.rs + w * dq.r;
    st.ds = st.ds + w * dq.d;
  }
  st.degenerate = nrm(st.rs) < kDegenerate;
  return st;
}
// solver.cpp:51-56
static V3 warp_point(const BlendState& st, const V3& p) {
  DQ raw;
  raw.r = st.rs;
  raw.d = st.ds;
  return dq_to_rig(dq_normalized(raw)).apply(p);
}
// 4x4 helpers for the blend Jacobian
static M4 m4_mul(const M4& a, const M4& b) {
  M4 o;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double s = 0;
      for (int k = 0; k < 4; ++k) s += a(i, k) * b(k, j);
      o(i, j) = s;
    }
  return o;
}
static M4 m4_add(const M4& a, const M4& b) {
  M4 o;
  for (int i = 0; i < 16; ++i) o.m[i] = a.m[i] + b.m[i];
  return o;
}
static M4 m4_scale(double s, const M4& a) {
  M4 o;
  for (int i = 0; i < 16; ++i) o.m[i] = s * a.m[i];
  return o;
}
static M4 m4_outer(const Q4& a, const Q4& b) {
  M4 o;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) o(i, j) = a[i] * b[j];
  return o;
}
static M4 m4_eye() {
  M4 o;
  for (int i = 0; i < 4; ++i) o(i, i) = 1.0;
  return o;
}
static const M4 kConj = [] {
  M4 c;
  c(0, 0) = 1; c(1, 1) = -1; c(2, 2) = -1; c(3, 3) = -1;
  return c;
}();
// solver.cpp:58-92 — dy/db, 3x8 row-major
static void blend_jacobian(const BlendState& st, const V3& p, double* out24) {
  const Q4& br = st.rs;
  const Q4& bd = st.ds;
  const double a = nrm(br);
  const Q4 rh = br / a;
  const double rd = dot(br, bd);
  const Q4 nr = br / a;
  const Q4 nd = bd / a - (rd / (a * a * a)) * br;
  const M4 dnr_dbr = m4_scale(1.0 / a, m4_add(m4_eye(), m4_scale(-1.0, m4_outer(rh, rh))));
  const double a3 = a * a * a, a5 = a3 * a * a;
  M4 t1 = m4_add(m4_add(m4_outer(bd, br), m4_outer(br, bd)), m4_scale(rd, m4_eye()));
  const M4 dnd_dbr = m4_add(m4_scale(-1.0 / a3, t1), m4_scale(3.0 * rd / a5, m4_outer(br, br)));
  const M4 dnd_dbd = m4_add(m4_scale(1.0 / a, m4_eye()), m4_scale(-1.0 / a3, m4_outer(br, br)));
  const Q4 pq = mq(0, p[0], p[1], p[2]);
  const M4 dy_dnr = m4_add(m4_add(qright(qmul(pq, qconj(nr))), m4_mul(qleft(qmul(nr, pq)), kConj)),
                           m4_scale(2.0, m4_mul(qleft(nd), kConj)));
  const M4 dy_dnd = m4_scale(2.0, qright(qconj(nr)));
  const M4 A = m4_add(m4_mul(dy_dnr, dnr_dbr), m4_mul(dy_dnd, dnd_dbr));
  const M4 B = m4_mul(dy_dnd, dnd_dbd);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 4; ++c) {
      out24[r * 8 + c] = A(r + 1, c);
      out24[r * 8 + 4 + c] = B(r + 1, c);
    }
}
// solver.cpp:94-112 — dy/dxi_slot, 3x6 row-major
static void node_jacobian(const double* dy_db, const BlendState& st, const Skin& e,
                          const std::vector<Node>& nodes, int slot, double* out18) {
  const DQ& dq = nodes[e.idx[slot]].T;
  const double w = st.sw[slot];
  const M4 rr = qright(dq.r), rdm = qright(dq.d);
  double db[8][6] = {{0}};
  for (int row = 0; row < 4; ++row)
    for (int c = 0; c < 3; ++c) {
      db[row][c] = 0.5 * w * rr(row, c + 1);      // d real / d omega
      db[4 + row][c] = 0.5 * w * rdm(row, c + 1);  // d dual / d omega
      db[4 + row][3 + c] = 0.5 * w * rr(row, c + 1);  // d dual / d t
    }
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 6; ++c) {
      double s = 0;
      for (int k = 0; k < 8; ++k) s += dy_db[r * 8 + k] * db[k][c];
      out18[r * 6 + c] = s;
    }
}
static M3 skew(const V3& v) {
  M3 m;
  m(0, 0) = 0; m(0, 1) = -v[2]; m(0, 2) = v[1];
  m(1, 0) = v[2]; m(1, 1) = 0; m(1, 2) = -v[0];
  m(2, 0) = -v[1]; m(2, 1) = v[0]; m(2, 2) = 0;
  return m;
}
// solver.cpp:114-130
static void reg_terms(const Rig& tj, const Rig& ti, const V3& pj, V3& r, double* jj, double* ji) {
  const V3 a = tj.apply(pj), b = ti.apply(pj);
  r = a - b;
  const M3 sa = skew(a), sb = skew(b);
  for (int i = 0; i < 3; ++i)
    for (int c = 0; c < 3; ++c) {
      jj[i * 6 + c] = -sa(i, c);
      jj[i * 6 + 3 + c] = (i == c) ? 1.0 : 0.0;
      ji[i * 6 + c] = sb(i, c);
      ji[i * 6 + 3 + c] = (i == c) ? -1.0 : 0.0;
    }
}
// solver.cpp:132-155
static double data_energy(const std::vector<Pair>& pairs, const Model& m,
                          const std::vector<Node>& nodes) {
  double e = 0;
  for (const auto& pr : pairs) {
    const BlendState st = blend_state(m.skin[pr.s], nodes);
    if (st.degenerate) continue;
    const V3 vm = warp_point(st, m.ref[pr.s].p);
    const double r = dot(pr.nd, vm - pr.vd);
    e += r * r;
  }
  return e;
}
static double reg_energy(const std::vector<Node>& nodes) {
  std::vector<Rig> T(nodes.size());
  for (size_t j = 0; j < nodes.size(); ++j) T[j] = dq_to_rig(nodes[j].T);
  double e = 0;
  for (size_t j = 0; j < nodes.size(); ++j)
    for (int32_t i : nodes[j].nbr) e += sqn(T[j].apply(nodes[j].p) - T[i].apply(nodes[j].p));
  return e;
}
static double total_energy(const std::vector<Pair>& pairs, const Model& m,
                           const std::vector<Node>& nodes, double lambda) {
  return data_energy(pairs, m, nodes) + lambda * reg_energy(nodes);
}
// solver.cpp:157-167
static void assert_normal_equations(int dim, const std::vector<double>& h) {
  double mx = 0;
  for (double v : h) mx = std::max(mx, std::abs(v));
  const double scale = std::max(1.0, mx);
  double asym = 0;
  for (int i = 0; i < dim; ++i)
    for (int j = 0; j < dim; ++j)
      asym = std::max(asym, std::abs(h[size_t(i) * dim + j] - h[size_t(j) * dim + i]));
  if (asym > 1e-9 * scale) fail(3, "normal equations lost symmetry");
  for (int b = 0; b + 6 <= dim; b += 6) {
    std::vector<double> blk(36);
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) blk[r * 6 + c] = h[size_t(b + r) * dim + b + c];
    const auto ev = sym_eigenvalues(6, blk);
    if (*std::min_element(ev.begin(), ev.end()) < -1e-8 * scale)
      fail(3, "normal equations diagonal block not PSD");
  }
}

// Normal equations of one GN iteration (solver.cpp:327-369). Returns pairs
// of this iteration's association through `pairs_out`.
struct NormalEq {
  int dim = 0;
  std::vector<double> h, g;
  std::vector<uint8_t> touched;  // N x N block pattern (d5)
};
static void assemble(const std::vector<Pair>& pairs, const Model& m, const std::vector<Node>& nodes,
                     double lambda, NormalEq& ne) {
  const int n = int(nodes.size());
  ne.dim = 6 * n;
  ne.h.assign(size_t(ne.dim) * ne.dim, 0.0);
  ne.g.assign(ne.dim, 0.0);
  ne.touched.assign(size_t(n) * n, 0);
  auto H = [&](int r, int c) -> double& { return ne.h[size_t(r) * ne.dim + c]; };
  for (const auto& pr : pairs) {
    const Skin& e = m.skin[pr.s];
    const BlendState st = blend_state(e, nodes);
    if (st.degenerate) continue;
    const V3& pref = m.ref[pr.s].p;
    const V3 vm = warp_point(st, pref);
    const double r = dot(pr.nd, vm - pr.vd);
    double dy_db[24];
    blend_jacobian(st, pref, dy_db);
    double rows[kMaxSkin][6];
    for (int s = 0; s < e.count; ++s) {
      double J[18];
      node_jacobian(dy_db, st, e, nodes, s, J);
      for (int c = 0; c < 6; ++c)
        rows[s][c] = (pr.nd[0] * J[c] + pr.nd[1] * J[6 + c]) + pr.nd[2] * J[12 + c];
    }
    for (int m1 = 0; m1 < e.count; ++m1) {
      const int j1 = e.idx[m1];
      for (int c = 0; c < 6; ++c) ne.g[6 * j1 + c] += rows[m1][c] * r;
      for (int m2 = 0; m2 < e.count; ++m2) {
        const int j2 = e.idx[m2];
        ne.touched[size_t(j1) * n + j2] = 1;
        for (int a = 0; a < 6; ++a)
          for (int b = 0; b < 6; ++b) H(6 * j1 + a, 6 * j2 + b) += rows[m1][a] * rows[m2][b];
      }
    }
  }
  std::vector<Rig> T(n);
  for (int j = 0; j < n; ++j) T[j] = dq_to_rig(nodes[j].T);
  for (int j = 0; j < n; ++j) {
    const V3& pj = nodes[j].p;
    for (int32_t i : nodes[j].nbr) {
      V3 r;
      double jj[18], ji[18];
      reg_terms(T[j], T[i], pj, r, jj, ji);
      auto add_block = [&](int bj, int bi, const double* A, const double* B) {
        ne.touched[size_t(bj) * n + bi] = 1;
        for (int a = 0; a < 6; ++a)
          for (int b = 0; b < 6; ++b) {
            const double v = (A[a] * B[b] + A[6 + a] * B[6 + b]) + A[12 + a] * B[12 + b];
            H(6 * bj + a, 6 * bi + b) += lambda * v;
          }
      };
      add_block(j, j, jj, jj);
      add_block(i, i, ji, ji);
      add_block(j, i, jj, ji);
      add_block(i, j, ji, jj);
      for (int a = 0; a < 6; ++a) {
        ne.g[6 * j + a] += lambda * ((jj[a] * r[0] + jj[6 + a] * r[1]) + jj[12 + a] * r[2]);
        ne.g[6 * i + a] += lambda * ((ji[a] * r[0] + ji[6 + a] * r[1]) + ji[12 + a] * r[2]);
      }
    }
  }
}

// solver.cpp:277-286
static std::vector<Node> apply_increments(const std::vector<Node>& nodes,
                                          const std::vector<double>& delta) {
  std::vector<Node> out = nodes;
  for (size_t j = 0; j < out.size(); ++j) {
    const V3 om = mk(delta[6 * j], delta[6 * j + 1], delta[6 * j + 2]);
    const V3 t = mk(delta[6 * j + 3], delta[6 * j + 4], delta[6 * j + 5]);
    out[j].T = dq_normalized(dq_mul(dq_increment(om, t), out[j].T));
  }
  return out;
}

// Optional replacement of the LM step's dense LDLT (solver.cpp:386). Only the
// bench's CPU reference arm installs one (LAPACK Cholesky on all host
// threads), so that a 9k x 9k config-2 system solves in seconds instead of
// minutes; every other use of the oracle runs the restated Eigen LDLT.
static or_dense_solver_fn g_dense_solver = nullptr;
static int64_t g_dense_solves = 0;

struct SolveReport {
  int iterations = 0, correspondences = 0;
  double e0 = 0, e1 = 0, mean_r = 0;
};
// solver.cpp:296-422
static SolveReport solve_nonrigid(std::vector<Node>& nodes, const Model& model, const Frame& f,
                                  const Rig& pose, int t_now, int t_last, const Cfg& cfg,
                                  bool mirror) {
  SolveReport rep;
  const int n = int(nodes.size());
  if (n == 0 || model.size() == 0) return rep;
  const int dim = 6 * n;
  Model work;
  work.ref = model.ref;
  work.skin = model.skin;
  work.live.resize(model.size());
  std::vector<Pair> pairs;
  double mu = 0;
  NormalEq ne;
  for (int iter = 0; iter < cfg.max_gn_iters; ++iter) {
    forward_warp(work, nodes);
    if (mirror)
      for (auto& s : work.live) round_surf(s);
    const ModelMaps mm = render_model_maps(work.live, pose, cfg, t_now, t_last);
    pairs = find_correspondences(f, mm, pose);
    const double e_pre = total_energy(pairs, model, nodes, cfg.lambda);
    if (iter == 0) {
      rep.e0 = e_pre;
      rep.e1 = e_pre;
    }
    assemble(pairs, model, nodes, cfg.lambda, ne);
    double ginf = 0;
    for (double v : ne.g) ginf = std::max(ginf, std::abs(v));
    if (ginf < 1e-14) break;
    assert_normal_equations(dim, ne.h);
    double tr = 0;
    for (int i = 0; i < dim; ++i) tr += ne.h[size_t(i) * dim + i];
    const double mu_floor = 1e-6 * tr / dim;
    mu = std::max(mu, mu_floor);
    bool accepted = false;
    double e_post = e_pre;
    std::vector<Node> cand;
    double gnorm = 0;
    for (double v : ne.g) gnorm += v * v;
    gnorm = std::sqrt(gnorm);
    std::vector<double> neg_g(dim);
    for (int i = 0; i < dim; ++i) neg_g[i] = -ne.g[i];
    for (int attempt = 0; attempt < 8 && !accepted; ++attempt) {
      std::vector<double> damped = ne.h;
      for (int i = 0; i < dim; ++i) damped[size_t(i) * dim + i] += mu;
      std::vector<double> delta;
      ++g_dense_solves;
      if (g_dense_solver) {  // bench reference arm: the same step by multithreaded LAPACK
        delta.assign(dim, 0.0);
        if (g_dense_solver(dim, damped.data(), neg_g.data(), delta.data()) != 0)
          delta.assign(dim, std::numeric_limits<double>::quiet_NaN());
      } else {
        delta = ldlt_solve(dim, damped, neg_g);
      }
      bool finite = true;
      for (double v : delta) finite = finite && std::isfinite(v);
      double res = 0;
      if (finite) {
        for (int i = 0; i < dim; ++i) {
          double acc = 0;
          const double* row = &damped[size_t(i) * dim];
          for (int j = 0; j < dim; ++j) acc += row[j] * delta[j];
          acc += ne.g[i];
          res += acc * acc;
        }
        res = std::sqrt(res);
      }
      if (!finite || res > 1e-6 * (gnorm + 1.0)) {
        mu = std::max(mu_floor, mu * 10.0);
        continue;
      }
      cand = apply_increments(nodes, delta);
      e_post = total_energy(pairs, model, cand, cfg.lambda);
      if (e_post <= e_pre) accepted = true;
      else mu = std::max(mu_floor, mu * 10.0);
    }
    if (!accepted) break;
    mu = std::max(mu_floor, mu * 0.1);
    nodes = cand;
    ++rep.iterations;
    rep.e1 = e_post;
    if (e_pre - e_post < 1e-4 * std::max(e_pre, 1e-300)) break;
  }
  rep.correspondences = int(pairs.size());
  double abs_sum = 0;
  int counted = 0;
  for (const auto& pr : pairs) {
    const BlendState st = blend_state(model.skin[pr.s], nodes);
    if (st.degenerate) continue;
    const V3 vm = warp_point(st, model.ref[pr.s].p);
    abs_sum += std::abs(dot(pr.nd, vm - pr.vd));
    ++counted;
  }
  rep.mean_r = counted > 0 ? abs_sum / counted : 0.0;
  return rep;
}

struct RigidResult {
  Rig pose;
  int pairs = 0;
  double mean_r = 0;
  bool low = false;
};
// solver.cpp:171-242
static RigidResult rigid_align(const Frame& f, const ModelMaps& mm, const Rig& init, const Cfg& cfg) {
  static constexpr int kIters[3] = {4, 3, 3};
  const Cam k(cfg);
  const Rig rinv = init.inverse();
  Rig cur = init;
  int final_pairs = 0;
  double final_abs = 0;
  for (int level = 2; level >= 0; --level) {
    const int stride = 1 << level;
    for (int it = 0; it < kIters[level]; ++it) {
      std::vector<double> h(36, 0.0), g(6, 0.0);
      int pairs = 0;
      double abs_r = 0;
      for (int y = 0; y < f.h; y += stride)
        for (int x = 0; x < f.w; x += stride) {
          const size_t c = size_t(y) * f.w + x;
          if (!f.valid[c]) continue;
          const V3 vw = cur.apply(f.vert[c]);
          const V3 pr = rinv.apply(vw);
          if (pr[2] <= 0) continue;
          double u, v;
          k.project(pr, u, v);
          const int ui = int(std::lround(u)), vi = int(std::lround(v));
          if (ui < 0 || ui >= mm.w || vi < 0 || vi >= mm.h) continue;
          const size_t mc = size_t(vi) * mm.w + ui;
          if (!mm.valid[mc]) continue;
          const V3& vm = mm.vert[mc];
          const V3& nm = mm.nrm[mc];
          if (nrm(vw - vm) >= kGateDist) continue;
          if (dot(cur.rotate(f.nrm[c]), nm) <= kGateNormal) continue;
          const double r = dot(nm, vw - vm);
          const V3 cr = cross(vw, nm);
          const double J[6] = {cr[0], cr[1], cr[2], nm[0], nm[1], nm[2]};
          for (int a = 0; a < 6; ++a) {
            for (int b = 0; b < 6; ++b) h[a * 6 + b] += J[a] * J[b];
            g[a] += J[a] * r;
          }
          ++pairs;
          abs_r += std::abs(r);
        }
      if (level == 0) {
        final_pairs = pairs;
        final_abs = abs_r;
      }
      if (pairs < 6) continue;
      std::vector<double> ng(6);
      for (int a = 0; a < 6; ++a) ng[a] = -g[a];
      const auto xi = ldlt_solve(6, h, ng);
      bool finite = true;
      for (double v : xi) finite = finite && std::isfinite(v);
      if (!finite) continue;
      cur = se3_increment(mk(xi[0], xi[1], xi[2]), mk(xi[3], xi[4], xi[5]), cur);
    }
  }
  RigidResult res;
  res.pairs = final_pairs;
  if (final_pairs < kRigidMinPairs) {
    res.pose = init;
    res.low = true;
    res.mean_r = final_pairs > 0 ? final_abs / final_pairs : 0.0;
    return res;
  }
  res.pose = cur;
  res.mean_r = final_abs / final_pairs;
  return res;
}

// ------------------------------------------------------------------ fusion
struct Cand {
  Surf s;
  int px = 0, py = 0;
};
// fusion.cpp:9-75
static int fuse_depth(const Frame& f, Model& m, const IndexMap& im, const Rig& pose, int t_now,
                      const Cfg& cfg, std::vector<Cand>& cands) {
  int fused = 0;
  const int fac = im.factor;
  std::vector<uint8_t> once(m.size(), 0);
  for (int y = 0; y < f.h; ++y)
    for (int x = 0; x < f.w; ++x) {
      const size_t c = size_t(y) * f.w + x;
      if (!f.valid[c]) continue;
      const V3 vd = pose.apply(f.vert[c]);
      const V3 nd = pose.rotate(f.nrm[c]);
      int32_t best = -1;
      double bc = 0, bd2 = 0;
      for (int sy = fac * y; sy < fac * (y + 1); ++sy)
        for (int sx = fac * x; sx < fac * (x + 1); ++sx) {
          const int32_t id = im.idx[size_t(sy) * im.w + sx];
          if (id < 0) continue;
          const Surf& s = m.live[id];
          const double d2 = sqn(s.p - vd);
          if (d2 >= cfg.delta_distance * cfg.delta_distance) continue;
          if (dot(nd, s.n) < cfg.delta_normal) continue;
          const bool better = best < 0 || s.c > bc ||
                              (s.c == bc && (d2 < bd2 || (d2 == bd2 && id < best)));
          if (better) {
            best = id;
            bc = s.c;
            bd2 = d2;
          }
        }
      if (best < 0) {
        Cand cd;
        cd.s.p = vd;
        cd.s.n = nd;
        cd.s.r = f.rad[c];
        cd.s.c = f.conf[c];
        cd.s.ti = t_now;
        cd.s.to = t_now;
        cd.px = x;
        cd.py = y;
        cands.push_back(cd);
        continue;
      }
      if (once[best]) continue;
      once[best] = 1;
      Surf& s = m.live[best];
      const double c_old = s.c, c_d = f.conf[c], c_new = c_old + c_d;
      s.p = (c_old * s.p + c_d * vd) / c_new;
      V3 nn = (c_old * s.n + c_d * nd) / c_new;
      s.n = nn / nrm(nn);
      s.r = (c_old * s.r + c_d * f.rad[c]) / c_new;
      s.c = c_new;
      s.to = t_now;
      ++fused;
    }
  return fused;
}
// fusion.cpp:77-122
static std::optional<Skin> skin_appended(const V3& x, const std::vector<V3>& nl,
                                         const std::vector<Node>& nodes, const Cfg& cfg) {
  const int n = int(nodes.size());
  if (n == 0) return std::nullopt;
  std::vector<NB> cands;
  cands.reserve(n);
  for (int32_t j = 0; j < n; ++j) cands.push_back({sqn(nl[j] - x), j});
  const int k = std::min(int(cfg.knn_k), n);
  std::partial_sort(cands.begin(), cands.begin() + k, cands.end());
  const int32_t n0 = cands[0].i;
  Skin e;
  e.idx[e.count] = n0;
  e.w[e.count] = skin_weight(x, nl[n0], nodes[n0].sigma);
  ++e.count;
  for (int m = 1; m < k; ++m) {
    const int32_t j = cands[m].i;
    const double lp = nrm(nl[j] - nl[n0]);
    const double rp = nrm(nodes[j].p - nodes[n0].p);
    if (rp <= 0) continue;
    const double ratio = lp / rp;
    if (ratio <= 1.0 - cfg.epsilon || ratio >= 1.0 + cfg.epsilon) continue;
    e.idx[e.count] = j;
    e.w[e.count] = skin_weight(x, nl[j], nodes[j].sigma);
    ++e.count;
  }
  if (e.wsum() < cfg.delta_nn) return std::nullopt;
  return e;
}
// fusion.cpp:128-146
static std::optional<V3> inv_warp_reweighted(const V3& x, const Skin& e,
                                             const std::vector<Node>& nodes,
                                             const std::vector<V3>& nl) {
  DQ dqs[kMaxSkin];
  double ws[kMaxSkin];
  for (int m = 0; m < e.count; ++m) {
    const int32_t j = e.idx[m];
    dqs[m] = nodes[j].T;
    ws[m] = skin_weight(x, nl[j], nodes[j].sigma);
  }
  const auto b = blend(e.count, dqs, ws);
  if (!b) return std::nullopt;
  return dq_to_rig(*b).inverse().apply(x);
}
// fusion.cpp:148-166
static std::optional<M3> inverse_warp_strain(const V3& x, const Skin& e,
                                             const std::vector<Node>& nodes,
                                             const std::vector<V3>& nl) {
  if (e.count == 0) return std::nullopt;
  constexpr double kStep = 1e-3;
  const auto c0 = inv_warp_reweighted(x, e, nodes, nl);
  if (!c0) return std::nullopt;
  M3 st;
  for (int a = 0; a < 3; ++a) {
    V3 pr = x;
    pr[a] += kStep;
    const auto sh = inv_warp_reweighted(pr, e, nodes, nl);
    if (!sh) return std::nullopt;
    const V3 col = (*sh - *c0) / kStep;
    for (int r = 0; r < 3; ++r) st(r, a) = col[r];
  }
  return st;
}
// fusion.cpp:168-177
static bool check_compressive(const V3& x, const Skin& e, const std::vector<Node>& nodes,
                              const std::vector<V3>& nl, const Cfg& cfg) {
  const auto st = inverse_warp_strain(x, e, nodes, nl);
  if (!st) return false;
  return sigma_max3(*st) <= 1.0 + cfg.epsilon;
}
// fusion.cpp:179-218
static std::vector<uint8_t> remove_surfels(const Model& m, const IndexMap& im, const Rig& pose,
                                           int t_now, const Cfg& cfg) {
  std::vector<uint8_t> rm(m.size(), 0);
  const Rig w2c = pose.inverse();
  const Cam k(cfg);
  const int fac = im.factor;
  for (size_t i = 0; i < m.size(); ++i) {
    const Surf& s = m.live[i];
    if (t_now - s.ti > cfg.t_low_confid && s.c < cfg.delta_stable) {
      rm[i] = 1;
      continue;
    }
    const V3 pc = w2c.apply(s.p);
    if (pc[2] <= 0) continue;
    double u, v;
    k.project(pc, u, v);
    const int sx = ss_coord(u, fac), sy = ss_coord(v, fac);
    for (int dy = -1; dy <= 1 && !rm[i]; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int nx = sx + dx, ny = sy + dy;
        if (nx < 0 || nx >= im.w || ny < 0 || ny >= im.h) continue;
        const int32_t j = im.idx[size_t(ny) * im.w + nx];
        if (j < 0 || size_t(j) == i) continue;
        const Surf& o = m.live[j];
        if (o.c <= cfg.delta_stable) continue;
        if (o.c <= s.c) continue;
        if (nrm(o.p - s.p) >= cfg.delta_distance) continue;
        if (dot(o.n, s.n) < cfg.delta_normal) continue;
        rm[i] = 1;
        break;
      }
  }
  return rm;
}
struct Outcome {
  int fused = 0, appended = 0, removed = 0, comp = 0, low = 0, new_nodes = 0, degen = 0;
};
// fusion.cpp:220-307
static Outcome apply_fusion(Model& m, const Frame& f, std::vector<Node>& nodes, const Rig& pose,
                            int t_now, const Cfg& cfg, bool mirror) {
  Outcome out;
  const IndexMap im = render_index_map(m.live, pose, cfg, cfg.supersample_factor);
  std::vector<Cand> cands;
  out.fused = fuse_depth(f, m, im, pose, t_now, cfg, cands);
  if (mirror) {
    for (auto& s : m.live) round_surf(s);
    for (auto& c : cands) round_surf(c.s);
  }
  std::vector<V3> nl(nodes.size());
  for (size_t j = 0; j < nodes.size(); ++j) nl[j] = nodes[j].live();
  std::vector<std::pair<Surf, Skin>> acc;
  for (const auto& cd : cands) {
    const auto e = skin_appended(cd.s.p, nl, nodes, cfg);
    if (!e) {
      ++out.low;
      continue;
    }
    if (cfg.compressive_check && !check_compressive(cd.s.p, *e, nodes, nl, cfg)) {
      ++out.comp;
      continue;
    }
    acc.emplace_back(cd.s, *e);
  }
  const size_t old = m.size();
  for (auto& [s, e] : acc) {
    m.live.push_back(s);
    m.ref.push_back(s);
    m.skin.push_back(e);
  }
  if (mirror) round_model(m);
  out.appended = int(acc.size());
  const auto rm = remove_surfels(m, im, pose, t_now, cfg);
  size_t wr = 0;
  std::vector<uint8_t> app_flag(m.size(), 0), comp_app;
  for (size_t i = old; i < m.size(); ++i) app_flag[i] = 1;
  comp_app.reserve(m.size());
  for (size_t i = 0; i < m.size(); ++i) {
    if (rm[i]) {
      ++out.removed;
      continue;
    }
    if (wr != i) {
      m.live[wr] = m.live[i];
      m.ref[wr] = m.ref[i];
      m.skin[wr] = m.skin[i];
    }
    comp_app.push_back(app_flag[i]);
    ++wr;
  }
  m.live.resize(wr);
  m.ref.resize(wr);
  m.skin.resize(wr);
  for (size_t i = 0; i < m.size(); ++i) {
    const auto b = inv_warp_surfel(m.live[i], m.skin[i], nodes);
    if (b) m.ref[i] = *b;
    else {
      m.ref[i] = m.live[i];
      ++out.degen;
    }
  }
  if (mirror) round_model(m);
  std::vector<Surf> app_ref;
  for (size_t i = 0; i < m.size(); ++i)
    if (comp_app[i]) app_ref.push_back(m.ref[i]);
  const int first_new = int(nodes.size());
  out.new_nodes = extend_warp_field(app_ref, nodes, cfg);
  if (out.new_nodes > 0) update_skinning_incremental(m.skin, m.ref, nodes, first_new, cfg);
  if (mirror) round_model(m);
  return out;
}

// ------------------------------------------------------------------ reinit
// reinit.cpp:9-26
static bool should_reinit(int n, const double* mr, const int32_t* app, int t_now, int t_last,
                          const Cfg& cfg) {
  if (cfg.periodic_reinit_interval > 0 && t_now - t_last >= cfg.periodic_reinit_interval)
    return true;
  if (n < cfg.reinit_window) return false;
  for (int i = 0; i < cfg.reinit_window; ++i) {
    if (mr[n - 1 - i] <= cfg.reinit_energy_threshold) return false;
    if (app[n - 1 - i] <= cfg.reinit_append_threshold) return false;
  }
  return true;
}
// reinit.cpp:28-89
static int clean_and_reset(Model& m, std::vector<Node>& nodes, const Frame& f, const Rig& pose,
                           const Cfg& cfg, int* survivors_out) {
  const Cam k(cfg);
  const Rig w2c = pose.inverse();
  const double gate = cfg.delta_distance_reinit;
  std::vector<Surf> surv;
  int removed = 0;
  auto inb = [&](int x, int y) { return x >= 0 && x < f.w && y >= 0 && y < f.h; };
  for (size_t i = 0; i < m.size(); ++i) {
    const Surf& s = m.live[i];
    const V3 pc = w2c.apply(s.p);
    bool keep = true;
    if (pc[2] > 0 && dot(w2c.rotate(s.n), pc) < 0) {
      double u, v;
      k.project(pc, u, v);
      const int ui = int(std::lround(u)), vi = int(std::lround(v));
      if (ui >= 0 && ui < k.w && vi >= 0 && vi < k.h) {
        bool corr = false, occl = false, anym = false;
        for (int dy = -1; dy <= 2 && !corr; ++dy)
          for (int dx = -1; dx <= 2; ++dx) {
            const int x = ui + dx, y = vi + dy;
            if (!inb(x, y) || !f.vvalid[size_t(y) * f.w + x]) continue;
            const size_t c = size_t(y) * f.w + x;
            anym = true;
            if (f.vert[c][2] < pc[2] - gate) occl = true;
            if (!f.valid[c]) continue;
            const V3 vd = pose.apply(f.vert[c]);
            if (nrm(vd - s.p) >= gate) continue;
            if (dot(pose.rotate(f.nrm[c]), s.n) < cfg.delta_normal) continue;
            corr = true;
            break;
          }
        keep = corr || occl || !anym;
      }
    }
    if (keep) surv.push_back(s);
    else ++removed;
  }
  if (surv.empty()) fail(2, "clean_and_reset: no surfel survived");
  m.live = surv;
  m.ref = surv;
  if (survivors_out) *survivors_out = int(surv.size());
  init_warp_field(m, nodes, cfg);
  return removed;
}

// ---------------------------------------------------------------- state/pipeline
struct State {
  Cfg cfg;
  bool mirror = false;
  Model m;
  std::vector<Node> nodes;
  Frame f;
};
struct Pipe {
  Cfg cfg;
  bool mirror = false;
  State st;
  Rig pose;
  bool initialized = false;
  int t_last = 0;
  std::deque<double> mr_win;
  std::deque<int32_t> app_win;
};
static double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
// pipeline.cpp:42-72
static void initialize_from_frame(Pipe& p) {
  const Frame& f = p.st.f;
  std::vector<Surf> surf;
  for (int y = 0; y < f.h; ++y)
    for (int x = 0; x < f.w; ++x) {
      const size_t c = size_t(y) * f.w + x;
      if (!f.valid[c]) continue;
      Surf s;
      s.p = p.pose.apply(f.vert[c]);
      s.n = p.pose.rotate(f.nrm[c]);
      s.r = f.rad[c];
      s.c = f.conf[c];
      s.ti = f.index;
      s.to = f.index;
      surf.push_back(s);
    }
  if (surf.empty()) fail(2, "initialization frame has no valid depth pixels");
  p.st.m = Model{};
  p.st.m.ref = surf;
  p.st.m.live = surf;
  if (p.mirror) round_model(p.st.m);
  init_warp_field(p.st.m, p.st.nodes, p.cfg);
  if (p.mirror) round_model(p.st.m);
  p.t_last = f.index;
  p.mr_win.clear();
  p.app_win.clear();
  p.initialized = true;
}
static void fill_rigid(const RigidResult& r, or_rigid_result* o) {
  rig_to12(r.pose, o->pose);
  o->correspondences = r.pairs;
  o->low_confidence = r.low ? 1 : 0;
  o->mean_residual = r.mean_r;
}
// pipeline.cpp:74-142
static void process_frame(Pipe& p, const uint16_t* depth, int w, int h, int index,
                          or_frame_stats* st) {
  std::memset(st, 0, sizeof *st);
  st->frame = index;
  const double t0 = now_ms();
  double ph = now_ms();
  p.st.f = build_frame(depth, w, h, index, p.cfg);
  st->depth_ms = now_ms() - ph;
  st->valid_pixels = p.st.f.valid_count;
  Model& m = p.st.m;
  std::vector<Node>& nodes = p.st.nodes;
  if (!p.initialized) {
    p.pose = Rig();
    initialize_from_frame(p);
    st->surfel_count = int(m.size());
    st->node_count = int(nodes.size());
    rig_to12(p.pose, st->pose);
    st->total_ms = now_ms() - t0;
    return;
  }
  const int t_now = index;
  ph = now_ms();
  const ModelMaps mm = render_model_maps(m.live, p.pose, p.cfg, t_now, p.t_last);
  const RigidResult rr = rigid_align(p.st.f, mm, p.pose, p.cfg);
  fill_rigid(rr, &st->rigid);
  p.pose = rr.pose;
  st->rigid_ms = now_ms() - ph;
  ph = now_ms();
  const SolveReport sr = solve_nonrigid(nodes, m, p.st.f, p.pose, t_now, p.t_last, p.cfg, p.mirror);
  st->solver.iterations = sr.iterations;
  st->solver.correspondences = sr.correspondences;
  st->solver.initial_energy = sr.e0;
  st->solver.final_energy = sr.e1;
  st->solver.mean_residual = sr.mean_r;
  st->solve_ms = now_ms() - ph;
  ph = now_ms();
  forward_warp(m, nodes);
  if (p.mirror) round_model(m);
  const Outcome oc = apply_fusion(m, p.st.f, nodes, p.pose, t_now, p.cfg, p.mirror);
  st->fusion.fused = oc.fused;
  st->fusion.appended = oc.appended;
  st->fusion.removed = oc.removed;
  st->fusion.compressive_rejected = oc.comp;
  st->fusion.low_support_rejected = oc.low;
  st->fusion.new_nodes = oc.new_nodes;
  st->fusion.degenerate_warps = oc.degen;
  st->fusion_ms = now_ms() - ph;
  p.mr_win.push_back(sr.mean_r);
  p.app_win.push_back(oc.appended);
  while (int(p.mr_win.size()) > p.cfg.reinit_window) p.mr_win.pop_front();
  while (int(p.app_win.size()) > p.cfg.reinit_window) p.app_win.pop_front();
  ph = now_ms();
  const std::vector<double> mr(p.mr_win.begin(), p.mr_win.end());
  const std::vector<int32_t> ap(p.app_win.begin(), p.app_win.end());
  if (should_reinit(int(mr.size()), mr.data(), ap.data(), t_now, p.t_last, p.cfg)) {
    st->reinit = 1;
    try {
      st->reinit_removed = clean_and_reset(m, nodes, p.st.f, p.pose, p.cfg, nullptr);
      if (p.mirror) round_model(m);
    } catch (const Err& e) {
      if (e.code != 2) throw;
      st->reinit_removed = int(m.size());
      initialize_from_frame(p);
    }
    p.t_last = t_now;
    p.mr_win.clear();
    p.app_win.clear();
  }
  st->reinit_ms = now_ms() - ph;
  st->surfel_count = int(m.size());
  st->node_count = int(nodes.size());
  rig_to12(p.pose, st->pose);
  st->total_ms = now_ms() - t0;
}

static ModelMaps maps_from(const int32_t* idx, const double* vert, const double* nrmv,
                           const uint8_t* valid, int w, int h) {
  ModelMaps mm;
  mm.w = w;
  mm.h = h;
  const size_t n = size_t(w) * h;
  mm.idx.assign(idx, idx + n);
  mm.valid.assign(valid, valid + n);
  mm.vert.resize(n);
  mm.nrm.resize(n);
  mm.depth.assign(n, 0.0);
  for (size_t i = 0; i < n; ++i) {
    mm.vert[i] = mk(vert[3 * i], vert[3 * i + 1], vert[3 * i + 2]);
    mm.nrm[i] = mk(nrmv[3 * i], nrmv[3 * i + 1], nrmv[3 * i + 2]);
  }
  return mm;
}
static Skin skin_from(const int32_t* idx, const double* w, int count) {
  Skin e;
  e.count = count;
  for (int i = 0; i < count; ++i) {
    e.idx[i] = idx[i];
    e.w[i] = w[i];
  }
  return e;
}
static std::vector<V3> v3s(const double* p, int n) {
  std::vector<V3> o(n);
  for (int i = 0; i < n; ++i) o[i] = mk(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
  return o;
}
static DQ dq_from8(const double* p) {
  DQ d;
  for (int i = 0; i < 4; ++i) {
    d.r[i] = p[i];
    d.d[i] = p[4 + i];
  }
  return d;
}
static void dq_to8(const DQ& d, double* p) {
  for (int i = 0; i < 4; ++i) {
    p[i] = d.r[i];
    p[4 + i] = d.d[i];
  }
}

thread_local std::string g_err;

}  // namespace ora

using namespace ora;

struct or_state : ora::State {};
struct or_pipeline : ora::Pipe {};

#define OR_TRY(expr)                  \
  try {                               \
    expr;                             \
  } catch (const ora::Err& e) {       \
    ora::g_err = e.msg;               \
    return e.code;                    \
  }

extern "C" {

void or_default_config(or_config* c) {
  std::memset(c, 0, sizeof *c);
  c->node_sigma = 0.025;
  c->knn_k = 4;
  c->node_neighbor_k = 8;
  c->lambda = 5.0;
  c->max_gn_iters = 10;
  c->delta_distance = 0.001;
  c->delta_normal = 0.85;
  c->epsilon = 0.2;
  c->delta_stable = 10.0;
  c->t_low_confid = 30;
  c->delta_recent = 2;
  c->delta_nn = 0.03;
  c->supersample_factor = 4;
  c->compressive_check = 1;
  c->depth_min = 0.1;
  c->depth_max = 5.0;
  c->bilateral_filter = 0;
  c->bilateral_sigma_space = 4.5;
  c->bilateral_sigma_depth = 30.0;
  c->reinit_energy_threshold = 0.005;
  c->reinit_append_threshold = 3000;
  c->reinit_window = 3;
  c->periodic_reinit_interval = 0;
  c->delta_distance_reinit = 0.010;
}
const char* or_last_error(void) { return ora::g_err.c_str(); }

or_state* or_state_new(const or_config* cfg) {
  auto* s = new or_state();
  std::memcpy(static_cast<or_config*>(&s->cfg), cfg, sizeof(or_config));
  return s;
}
void or_state_free(or_state* s) { delete s; }
void or_state_set_mirror(or_state* s, int32_t mirror) { s->mirror = mirror != 0; }
void or_state_set_config(or_state* s, const or_config* cfg) {
  std::memcpy(static_cast<or_config*>(&s->cfg), cfg, sizeof(or_config));
}

void or_set_model(or_state* s, int32_t n, const double* rp, const double* rn, const double* rr,
                  const double* rc, const int32_t* rti, const int32_t* rto, const double* lp,
                  const double* ln, const double* lr, const double* lc, const int32_t* lti,
                  const int32_t* lto, const int32_t* si, const double* sw, const int32_t* sc) {
  Model& m = s->m;
  m.ref.assign(n, Surf());
  m.live.assign(n, Surf());
  m.skin.assign(n, Skin());
  for (int i = 0; i < n; ++i) {
    Surf& a = m.ref[i];
    a.p = mk(rp[3 * i], rp[3 * i + 1], rp[3 * i + 2]);
    a.n = mk(rn[3 * i], rn[3 * i + 1], rn[3 * i + 2]);
    a.r = rr[i];
    a.c = rc[i];
    a.ti = rti[i];
    a.to = rto[i];
    Surf& b = m.live[i];
    b.p = mk(lp[3 * i], lp[3 * i + 1], lp[3 * i + 2]);
    b.n = mk(ln[3 * i], ln[3 * i + 1], ln[3 * i + 2]);
    b.r = lr[i];
    b.c = lc[i];
    b.ti = lti[i];
    b.to = lto[i];
    m.skin[i] = skin_from(si + 8 * i, sw + 8 * i, sc[i]);
  }
}
int32_t or_model_size(const or_state* s) { return int32_t(s->m.size()); }
void or_get_model(const or_state* s, double* rp, double* rn, double* rr, double* rc, int32_t* rti,
                  int32_t* rto, double* lp, double* ln, double* lr, double* lc, int32_t* lti,
                  int32_t* lto, int32_t* si, double* sw, int32_t* sc) {
  const Model& m = s->m;
  for (size_t i = 0; i < m.size(); ++i) {
    const Surf& a = m.ref[i];
    const Surf& b = m.live[i];
    for (int k = 0; k < 3; ++k) {
      rp[3 * i + k] = a.p[k];
      rn[3 * i + k] = a.n[k];
      lp[3 * i + k] = b.p[k];
      ln[3 * i + k] = b.n[k];
    }
    rr[i] = a.r; rc[i] = a.c; rti[i] = a.ti; rto[i] = a.to;
    lr[i] = b.r; lc[i] = b.c; lti[i] = b.ti; lto[i] = b.to;
    const Skin& e = m.skin[i];
    for (int k = 0; k < 8; ++k) {
      si[8 * i + k] = k < e.count ? e.idx[k] : -1;
      sw[8 * i + k] = k < e.count ? e.w[k] : 0.0;
    }
    sc[i] = e.count;
  }
}
void or_set_nodes(or_state* s, int32_t n, const double* pos, const double* sigma,
                  const double* dq, const int32_t* nbr, const int32_t* nbr_count) {
  s->nodes.assign(n, Node());
  for (int j = 0; j < n; ++j) {
    Node& nd = s->nodes[j];
    nd.p = mk(pos[3 * j], pos[3 * j + 1], pos[3 * j + 2]);
    nd.sigma = sigma[j];
    nd.T = dq_from8(dq + 8 * j);
    nd.nbr.assign(nbr + 8 * j, nbr + 8 * j + nbr_count[j]);
  }
}
int32_t or_num_nodes(const or_state* s) { return int32_t(s->nodes.size()); }
void or_get_nodes(const or_state* s, double* pos, double* sigma, double* dq, int32_t* nbr,
                  int32_t* nbr_count) {
  for (size_t j = 0; j < s->nodes.size(); ++j) {
    const Node& nd = s->nodes[j];
    for (int k = 0; k < 3; ++k) pos[3 * j + k] = nd.p[k];
    sigma[j] = nd.sigma;
    dq_to8(nd.T, dq + 8 * j);
    const int c = std::min<int>(8, int(nd.nbr.size()));
    for (int k = 0; k < 8; ++k) nbr[8 * j + k] = k < c ? nd.nbr[k] : -1;
    nbr_count[j] = c;
  }
}

int32_t or_build_frame(or_state* s, const uint16_t* depth, int32_t w, int32_t h, int32_t fi) {
  OR_TRY(s->f = build_frame(depth, w, h, fi, s->cfg));
  return 0;
}
void or_get_frame(const or_state* s, double* vert, double* nrmv, double* conf, double* rad,
                  uint8_t* vv, uint8_t* valid, int32_t* vc) {
  const Frame& f = s->f;
  for (size_t i = 0; i < f.vert.size(); ++i) {
    for (int k = 0; k < 3; ++k) {
      vert[3 * i + k] = f.vert[i][k];
      nrmv[3 * i + k] = f.nrm[i][k];
    }
    conf[i] = f.conf[i];
    rad[i] = f.rad[i];
    vv[i] = f.vvalid[i];
    valid[i] = f.valid[i];
  }
  *vc = f.valid_count;
}
void or_set_frame(or_state* s, int32_t w, int32_t h, int32_t fi, const double* vert,
                  const double* nrmv, const double* conf, const double* rad, const uint8_t* vv,
                  const uint8_t* valid) {
  Frame& f = s->f;
  f.w = w;
  f.h = h;
  f.index = fi;
  const size_t n = size_t(w) * h;
  f.vert = v3s(vert, int(n));
  f.nrm = v3s(nrmv, int(n));
  f.conf.assign(conf, conf + n);
  f.rad.assign(rad, rad + n);
  f.vvalid.assign(vv, vv + n);
  f.valid.assign(valid, valid + n);
  f.valid_count = 0;
  for (size_t i = 0; i < n; ++i) f.valid_count += valid[i] ? 1 : 0;
}
int32_t or_backproject(const uint16_t* depth, int32_t w, int32_t h, const or_config* cfg,
                       double* vert, uint8_t* vvalid) {
  Cfg c;
  std::memcpy(static_cast<or_config*>(&c), cfg, sizeof(or_config));
  std::vector<V3> v;
  std::vector<uint8_t> vv;
  OR_TRY(backproject(depth, w, h, c, v, vv));
  for (size_t i = 0; i < v.size(); ++i) {
    for (int k = 0; k < 3; ++k) vert[3 * i + k] = v[i][k];
    vvalid[i] = vv[i];
  }
  return 0;
}
void or_estimate_normals(const double* vert, const uint8_t* vvalid, int32_t w, int32_t h,
                         double* nrmv, uint8_t* nvalid) {
  const auto v = v3s(vert, w * h);
  std::vector<uint8_t> vv(vvalid, vvalid + size_t(w) * h), nv;
  std::vector<V3> n;
  estimate_normals(v, vv, w, h, n, nv);
  for (size_t i = 0; i < n.size(); ++i) {
    for (int k = 0; k < 3; ++k) nrmv[3 * i + k] = n[i][k];
    nvalid[i] = nv[i];
  }
}
double or_compute_confidence(double px, double py, const or_config* cfg) {
  Cfg c;
  std::memcpy(static_cast<or_config*>(&c), cfg, sizeof(or_config));
  return confidence(px, py, c);
}
double or_compute_radius(double d, double f, double nz) { return radius_of(d, f, nz); }
void or_bilateral_filter(const uint16_t* depth, int32_t w, int32_t h, double ss, double sd,
                         uint16_t* out) {
  bilateral(depth, w, h, ss, sd, out);
}

int32_t or_init_warp_field(or_state* s) {
  OR_TRY(init_warp_field(s->m, s->nodes, s->cfg));
  return 0;
}
void or_compute_node_edges(or_state* s, int32_t k) { node_edges(s->nodes, k); }
int32_t or_forward_warp(or_state* s) { return forward_warp(s->m, s->nodes); }
int32_t or_inverse_warp_surfel(const or_state* s, int32_t i, double* pos, double* nv) {
  const auto r = inv_warp_surfel(s->m.live[i], s->m.skin[i], s->nodes);
  if (!r) return 0;
  for (int k = 0; k < 3; ++k) {
    pos[k] = r->p[k];
    nv[k] = r->n[k];
  }
  return 1;
}
int32_t or_extend_warp_field(or_state* s, int32_t n, const double* positions) {
  std::vector<Surf> app(n);
  for (int i = 0; i < n; ++i) app[i].p = mk(positions[3 * i], positions[3 * i + 1], positions[3 * i + 2]);
  return extend_warp_field(app, s->nodes, s->cfg);
}
void or_update_skinning_incremental(or_state* s, int32_t first_new) {
  update_skinning_incremental(s->m.skin, s->m.ref, s->nodes, first_new, s->cfg);
}
int32_t or_voxel_knn(const double* pts, int32_t n, double cell, const double* q, int32_t k,
                     int32_t* out) {
  Voxels g(cell);
  for (int i = 0; i < n; ++i) g.add(mk(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
  const auto r = g.knn(mk(q[0], q[1], q[2]), k);
  for (size_t i = 0; i < r.size(); ++i) out[i] = r[i].i;
  return int32_t(r.size());
}
int32_t or_voxel_has_point_within(const double* pts, int32_t n, double cell, const double* q,
                                  double radius) {
  Voxels g(cell);
  for (int i = 0; i < n; ++i) g.add(mk(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
  return g.any_within(mk(q[0], q[1], q[2]), radius) ? 1 : 0;
}

void or_render_index_map(const or_state* s, const double* pose, int32_t factor, int32_t* idx,
                         double* depth) {
  const IndexMap im = render_index_map(s->m.live, rig_from12(pose), s->cfg, factor);
  std::memcpy(idx, im.idx.data(), im.idx.size() * sizeof(int32_t));
  std::memcpy(depth, im.depth.data(), im.depth.size() * sizeof(double));
}
void or_render_model_maps(const or_state* s, const double* pose, int32_t t_now, int32_t t_last,
                          int32_t* idx, double* vert, double* nrmv, double* depth,
                          uint8_t* valid) {
  const ModelMaps mm = render_model_maps(s->m.live, rig_from12(pose), s->cfg, t_now, t_last);
  for (size_t i = 0; i < mm.idx.size(); ++i) {
    idx[i] = mm.idx[i];
    for (int k = 0; k < 3; ++k) {
      vert[3 * i + k] = mm.vert[i][k];
      nrmv[3 * i + k] = mm.nrm[i][k];
    }
    depth[i] = mm.depth[i];
    valid[i] = mm.valid[i];
  }
}

int32_t or_find_correspondences(const or_state* s, const int32_t* mi, const double* mv,
                                const double* mn, const uint8_t* mval, int32_t mw, int32_t mh,
                                const double* pose, int32_t cap, int32_t* surfel, int32_t* px,
                                int32_t* py, double* vm, double* vd, double* nd) {
  std::vector<Pair> pairs;
  try {
    pairs = find_correspondences(s->f, maps_from(mi, mv, mn, mval, mw, mh), rig_from12(pose));
  } catch (const Err& e) {
    g_err = e.msg;
    return -e.code;
  }
  const int n = std::min<int>(cap, int(pairs.size()));
  for (int i = 0; i < n; ++i) {
    surfel[i] = pairs[i].s;
    px[i] = pairs[i].px;
    py[i] = pairs[i].py;
    for (int k = 0; k < 3; ++k) {
      vm[3 * i + k] = pairs[i].vm[k];
      vd[3 * i + k] = pairs[i].vd[k];
      nd[3 * i + k] = pairs[i].nd[k];
    }
  }
  return int32_t(pairs.size());
}
int32_t or_normal_equations(or_state* s, const double* pose, int32_t t_now, int32_t t_last,
                            double* h, double* g, uint8_t* touched, double* e_pre,
                            int32_t* n_pairs) {
  const Rig P = rig_from12(pose);
  Model work;
  work.ref = s->m.ref;
  work.skin = s->m.skin;
  work.live.resize(s->m.size());
  forward_warp(work, s->nodes);
  if (s->mirror)  // as solve_nonrigid's own loop: the live state is stored fp32 on the device
    for (auto& sf : work.live) round_surf(sf);
  const ModelMaps mm = render_model_maps(work.live, P, s->cfg, t_now, t_last);
  std::vector<Pair> pairs;
  OR_TRY(pairs = find_correspondences(s->f, mm, P));
  *e_pre = total_energy(pairs, s->m, s->nodes, s->cfg.lambda);
  *n_pairs = int32_t(pairs.size());
  NormalEq ne;
  assemble(pairs, s->m, s->nodes, s->cfg.lambda, ne);
  std::memcpy(h, ne.h.data(), ne.h.size() * sizeof(double));
  std::memcpy(g, ne.g.data(), ne.g.size() * sizeof(double));
  std::memcpy(touched, ne.touched.data(), ne.touched.size());
  return 0;
}
int32_t or_solve_nonrigid(or_state* s, const double* pose, int32_t t_now, int32_t t_last,
                          or_solver_report* out) {
  SolveReport r;
  OR_TRY(r = solve_nonrigid(s->nodes, s->m, s->f, rig_from12(pose), t_now, t_last, s->cfg, s->mirror));
  out->iterations = r.iterations;
  out->correspondences = r.correspondences;
  out->initial_energy = r.e0;
  out->final_energy = r.e1;
  out->mean_residual = r.mean_r;
  return 0;
}
int32_t or_rigid_align(or_state* s, const double* render_pose, const double* init_pose,
                       int32_t t_now, int32_t t_last, or_rigid_result* out) {
  const ModelMaps mm = render_model_maps(s->m.live, rig_from12(render_pose), s->cfg, t_now, t_last);
  const RigidResult r = rigid_align(s->f, mm, rig_from12(init_pose), s->cfg);
  fill_rigid(r, out);
  return 0;
}
double or_data_energy(const or_state* s, int32_t n, const int32_t* surfel, const double* vd,
                      const double* nd) {
  std::vector<Pair> pairs(n);
  for (int i = 0; i < n; ++i) {
    pairs[i].s = surfel[i];
    pairs[i].vd = mk(vd[3 * i], vd[3 * i + 1], vd[3 * i + 2]);
    pairs[i].nd = mk(nd[3 * i], nd[3 * i + 1], nd[3 * i + 2]);
  }
  return data_energy(pairs, s->m, s->nodes);
}
double or_reg_energy(const or_state* s) { return reg_energy(s->nodes); }
int32_t or_blend_jacobian(const or_state* s, int32_t i, double* y3, double* dy_db24,
                          double* node_jac) {
  const Skin& e = s->m.skin[i];
  const BlendState st = blend_state(e, s->nodes);
  if (st.degenerate) return 0;
  const V3 y = warp_point(st, s->m.ref[i].p);
  for (int k = 0; k < 3; ++k) y3[k] = y[k];
  blend_jacobian(st, s->m.ref[i].p, dy_db24);
  for (int m = 0; m < e.count; ++m) node_jacobian(dy_db24, st, e, s->nodes, m, node_jac + 18 * m);
  return e.count;
}
void or_reg_terms(const double* dq_j, const double* dq_i, const double* p_j, double* r3,
                  double* jj18, double* ji18) {
  V3 r;
  reg_terms(dq_to_rig(dq_from8(dq_j)), dq_to_rig(dq_from8(dq_i)), mk(p_j[0], p_j[1], p_j[2]), r,
            jj18, ji18);
  for (int k = 0; k < 3; ++k) r3[k] = r[k];
}
int32_t or_ldlt_solve(int32_t n, const double* a, const double* b, double* x) {
  std::vector<double> A(a, a + size_t(n) * n), B(b, b + n);
  const auto X = ldlt_solve(n, A, B);
  std::memcpy(x, X.data(), sizeof(double) * n);
  return 0;
}
void or_set_dense_solver(or_dense_solver_fn fn) { g_dense_solver = fn; }
int64_t or_dense_solve_count(void) { return g_dense_solves; }
int32_t or_assert_normal_equations(int32_t dim, const double* h) {
  std::vector<double> H(h, h + size_t(dim) * dim);
  OR_TRY(assert_normal_equations(dim, H));
  return 0;
}

int32_t or_fuse_depth(or_state* s, const int32_t* index_map, int32_t factor, const double* pose,
                      int32_t t_now, int32_t cap, int32_t* n_cand, double* cp, double* cn,
                      double* cr, double* cc, int32_t* cx, int32_t* cy) {
  IndexMap im;
  im.factor = factor;
  im.w = s->cfg.width * factor;
  im.h = s->cfg.height * factor;
  im.idx.assign(index_map, index_map + size_t(im.w) * im.h);
  std::vector<Cand> cands;
  const int fused = fuse_depth(s->f, s->m, im, rig_from12(pose), t_now, s->cfg, cands);
  *n_cand = int32_t(cands.size());
  const int n = std::min<int>(cap, int(cands.size()));
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < 3; ++k) {
      cp[3 * i + k] = cands[i].s.p[k];
      cn[3 * i + k] = cands[i].s.n[k];
    }
    cr[i] = cands[i].s.r;
    cc[i] = cands[i].s.c;
    cx[i] = cands[i].px;
    cy[i] = cands[i].py;
  }
  return fused;
}
int32_t or_skin_appended(const or_state* s, const double* x, const double* node_live,
                         int32_t* idx8, double* w8, int32_t* count) {
  const auto nl = v3s(node_live, int(s->nodes.size()));
  const auto e = skin_appended(mk(x[0], x[1], x[2]), nl, s->nodes, s->cfg);
  if (!e) return 0;
  for (int k = 0; k < 8; ++k) {
    idx8[k] = k < e->count ? e->idx[k] : -1;
    w8[k] = k < e->count ? e->w[k] : 0.0;
  }
  *count = e->count;
  return 1;
}
int32_t or_inverse_warp_strain(const or_state* s, const double* x, const int32_t* idx,
                               const double* w, int32_t count, const double* node_live,
                               double* strain9) {
  const auto nl = v3s(node_live, int(s->nodes.size()));
  const auto st = inverse_warp_strain(mk(x[0], x[1], x[2]), skin_from(idx, w, count), s->nodes, nl);
  if (!st) return 0;
  std::memcpy(strain9, st->m, sizeof(double) * 9);
  return 1;
}
int32_t or_check_compressive(const or_state* s, const double* x, const int32_t* idx,
                             const double* w, int32_t count, const double* node_live) {
  const auto nl = v3s(node_live, int(s->nodes.size()));
  return check_compressive(mk(x[0], x[1], x[2]), skin_from(idx, w, count), s->nodes, nl, s->cfg)
             ? 1
             : 0;
}
double or_sigma_max3(const double* m9) {
  M3 m;
  std::memcpy(m.m, m9, sizeof(double) * 9);
  return sigma_max3(m);
}
void or_remove_surfels(const or_state* s, const int32_t* index_map, int32_t factor,
                       const double* pose, int32_t t_now, uint8_t* mask) {
  IndexMap im;
  im.factor = factor;
  im.w = s->cfg.width * factor;
  im.h = s->cfg.height * factor;
  im.idx.assign(index_map, index_map + size_t(im.w) * im.h);
  const auto rm = remove_surfels(s->m, im, rig_from12(pose), t_now, s->cfg);
  std::memcpy(mask, rm.data(), rm.size());
}
int32_t or_apply_fusion(or_state* s, const double* pose, int32_t t_now, or_fusion_outcome* out) {
  Outcome oc;
  OR_TRY(oc = apply_fusion(s->m, s->f, s->nodes, rig_from12(pose), t_now, s->cfg, s->mirror));
  out->fused = oc.fused;
  out->appended = oc.appended;
  out->removed = oc.removed;
  out->compressive_rejected = oc.comp;
  out->low_support_rejected = oc.low;
  out->new_nodes = oc.new_nodes;
  out->degenerate_warps = oc.degen;
  return 0;
}
int32_t or_should_reinitialize(int32_t n, const double* mr, const int32_t* app, int32_t t_now,
                               int32_t t_last, const or_config* cfg) {
  Cfg c;
  std::memcpy(static_cast<or_config*>(&c), cfg, sizeof(or_config));
  return should_reinit(n, mr, app, t_now, t_last, c) ? 1 : 0;
}
int32_t or_clean_and_reset(or_state* s, const double* pose, int32_t* removed, int32_t* survivors) {
  int r = 0, sv = 0;
  OR_TRY(r = clean_and_reset(s->m, s->nodes, s->f, rig_from12(pose), s->cfg, &sv));
  *removed = r;
  *survivors = sv;
  return 0;
}

void or_dq_from_se3(const double* pose, double* dq) { dq_to8(dq_from_rig(rig_from12(pose)), dq); }
void or_dq_to_se3(const double* dq, double* pose) { rig_to12(dq_to_rig(dq_from8(dq)), pose); }
void or_dq_mul(const double* a, const double* b, double* out) {
  dq_to8(dq_mul(dq_from8(a), dq_from8(b)), out);
}
void or_dq_normalized(const double* dq, double* out) { dq_to8(dq_normalized(dq_from8(dq)), out); }
int32_t or_blend(int32_t n, const double* dqs, const double* w, double* out) {
  std::vector<DQ> v(n);
  for (int i = 0; i < n; ++i) v[i] = dq_from8(dqs + 8 * i);
  const auto b = blend(n, v.data(), w);
  if (!b) return 0;
  dq_to8(*b, out);
  return 1;
}
double or_skinning_weight(const double* x, const double* p, double sigma) {
  return skin_weight(mk(x[0], x[1], x[2]), mk(p[0], p[1], p[2]), sigma);
}
void or_se3_increment(const double* om, const double* dt, const double* pose, double* out) {
  rig_to12(se3_increment(mk(om[0], om[1], om[2]), mk(dt[0], dt[1], dt[2]), rig_from12(pose)), out);
}
void or_dq_increment(const double* om, const double* dt, double* out) {
  dq_to8(dq_increment(mk(om[0], om[1], om[2]), mk(dt[0], dt[1], dt[2])), out);
}
void or_quat_from_rotvec(const double* om, double* q) {
  const Q4 r = quat_from_rotvec(mk(om[0], om[1], om[2]));
  for (int i = 0; i < 4; ++i) q[i] = r[i];
}
void or_quat_from_matrix(const double* r9, double* q) {
  M3 m;
  std::memcpy(m.m, r9, sizeof(double) * 9);
  const Q4 r = quat_from_matrix(m);
  for (int i = 0; i < 4; ++i) q[i] = r[i];
}
void or_matrix_from_quat(const double* q, double* r9) {
  const M3 m = matrix_from_quat(mq(q[0], q[1], q[2], q[3]));
  std::memcpy(r9, m.m, sizeof(double) * 9);
}

or_pipeline* or_pipeline_new(const or_config* cfg, int32_t mirror) {
  auto* p = new or_pipeline();
  std::memcpy(static_cast<or_config*>(&p->cfg), cfg, sizeof(or_config));
  p->st.cfg = p->cfg;
  p->mirror = mirror != 0;
  return p;
}
void or_pipeline_free(or_pipeline* p) { delete p; }
int32_t or_pipeline_process_frame(or_pipeline* p, const uint16_t* depth, int32_t w, int32_t h,
                                  int32_t fi, or_frame_stats* out) {
  OR_TRY(process_frame(*p, depth, w, h, fi, out));
  return 0;
}
or_state* or_pipeline_state(or_pipeline* p) { return static_cast<or_state*>(&p->st); }
void or_pipeline_pose(const or_pipeline* p, double* pose) { rig_to12(p->pose, pose); }
int32_t or_pipeline_last_reinit(const or_pipeline* p) { return p->t_last; }

}  // extern "C"
