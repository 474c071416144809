// ds_math.cuh — fp64 rigid / dual-quaternion algebra for the device (and host).
//
// B200 has full-rate-ish FP64 (~45 TFLOP/s), far above what these HBM/latency
// bound kernels need, so every quantity that feeds a discrete decision is
// evaluated in double precision with the reference's operation order
// (geometry.cpp) and sums taken strictly left to right. Surfel state is
// STORED in fp32 (SoA float4); node transforms and frame maps in fp64.
// Compiled with --fmad=false so no FMA contraction changes rounding.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#define DSI __host__ __device__ __forceinline__

namespace ds {

struct V3 {
  double x, y, z;
};
struct Q4 {
  double w, x, y, z;
};
struct DQ {
  Q4 r, d;
};
struct M3 {
  double m[9];  // row-major
};
struct Rig {
  M3 R;
  V3 t;
};

DSI V3 v3(double a, double b, double c) { return V3{a, b, c}; }
DSI V3 add(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
DSI V3 sub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
DSI V3 neg(V3 a) { return v3(-a.x, -a.y, -a.z); }
DSI V3 scl(double s, V3 a) { return v3(s * a.x, s * a.y, s * a.z); }
// x / s, bit-identical to IEEE division for finite nonzero s, but a zero
// numerator returns the signed zero directly: on sm_100 the fp64 division
// fast path sends 0 / s to the slow subroutine (~20x slower), and zeros are
// common here (identity nodes, zero dual parts, unit basis rows).
DSI double ddiv(double x, double s) { return x == 0.0 ? x * s : x / s; }
DSI V3 dvd(V3 a, double s) { return v3(ddiv(a.x, s), ddiv(a.y, s), ddiv(a.z, s)); }
DSI double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
DSI double sqn(V3 a) { return dot(a, a); }
DSI double nrm(V3 a) { return sqrt(sqn(a)); }
DSI V3 cross(V3 a, V3 b) {
  return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
DSI double comp(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

DSI Q4 q4(double w, double x, double y, double z) { return Q4{w, x, y, z}; }
DSI Q4 qadd(Q4 a, Q4 b) { return q4(a.w + b.w, a.x + b.x, a.y + b.y, a.z + b.z); }
DSI Q4 qsub(Q4 a, Q4 b) { return q4(a.w - b.w, a.x - b.x, a.y - b.y, a.z - b.z); }
DSI Q4 qscl(double s, Q4 a) { return q4(s * a.w, s * a.x, s * a.y, s * a.z); }
DSI Q4 qdiv(Q4 a, double s) { return q4(ddiv(a.w, s), ddiv(a.x, s), ddiv(a.y, s), ddiv(a.z, s)); }
DSI Q4 qneg(Q4 a) { return q4(-a.w, -a.x, -a.y, -a.z); }
DSI double qdot(Q4 a, Q4 b) { return ((a.w * b.w + a.x * b.x) + a.y * b.y) + a.z * b.z; }
DSI double qnrm(Q4 a) { return sqrt(qdot(a, a)); }
DSI Q4 qconj(Q4 q) { return q4(q.w, -q.x, -q.y, -q.z); }
// geometry.cpp:7-12
DSI Q4 qmul(Q4 a, Q4 b) {
  return q4(a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z,
            a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
            a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x,
            a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w);
}

DSI M3 m3_identity() {
  M3 r;
  for (int i = 0; i < 9; ++i) r.m[i] = (i % 4 == 0) ? 1.0 : 0.0;
  return r;
}
DSI V3 mulv(const M3& R, V3 p) {
  return v3((R.m[0] * p.x + R.m[1] * p.y) + R.m[2] * p.z,
            (R.m[3] * p.x + R.m[4] * p.y) + R.m[5] * p.z,
            (R.m[6] * p.x + R.m[7] * p.y) + R.m[8] * p.z);
}
DSI M3 mulm(const M3& a, const M3& b) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      o.m[i * 3 + j] = (a.m[i * 3] * b.m[j] + a.m[i * 3 + 1] * b.m[3 + j]) + a.m[i * 3 + 2] * b.m[6 + j];
  return o;
}
DSI M3 transpose(const M3& a) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.m[i * 3 + j] = a.m[j * 3 + i];
  return o;
}

DSI V3 rig_apply(const Rig& T, V3 p) { return add(mulv(T.R, p), T.t); }
DSI V3 rig_rotate(const Rig& T, V3 d) { return mulv(T.R, d); }
DSI Rig rig_inverse(const Rig& T) {
  Rig o;
  o.R = transpose(T.R);
  o.t = neg(mulv(o.R, T.t));
  return o;
}
DSI Rig rig_mul(const Rig& a, const Rig& b) {
  Rig o;
  o.R = mulm(a.R, b.R);
  o.t = add(mulv(a.R, b.t), a.t);
  return o;
}
DSI Rig rig_identity() {
  Rig o;
  o.R = m3_identity();
  o.t = v3(0, 0, 0);
  return o;
}
DSI Rig rig_load(const double* p) {
  Rig o;
  for (int i = 0; i < 9; ++i) o.R.m[i] = p[i];
  o.t = v3(p[9], p[10], p[11]);
  return o;
}
DSI void rig_store(const Rig& o, double* p) {
  for (int i = 0; i < 9; ++i) p[i] = o.R.m[i];
  p[9] = o.t.x;
  p[10] = o.t.y;
  p[11] = o.t.z;
}

// geometry.cpp:32-42
DSI Q4 quat_from_rotvec(V3 om) {
  const double angle = nrm(om);
  if (angle < 1e-12) {
    const Q4 q = q4(1.0, 0.5 * om.x, 0.5 * om.y, 0.5 * om.z);
    return qdiv(q, qnrm(q));
  }
  const double half = 0.5 * angle;
  const V3 axis = dvd(om, angle);
  const double s = sin(half);
  return q4(cos(half), s * axis.x, s * axis.y, s * axis.z);
}
// geometry.cpp:44-50 (Eigen Quaterniond(Matrix3d), normalize, w >= 0)
DSI Q4 quat_from_matrix(const M3& R) {
  const double* m = R.m;
  double q[4];  // w x y z
  double t = (m[0] + m[4]) + m[8];
  if (t > 0.0) {
    t = sqrt(t + 1.0);
    q[0] = 0.5 * t;
    t = 0.5 / t;
    q[1] = (m[7] - m[5]) * t;
    q[2] = (m[2] - m[6]) * t;
    q[3] = (m[3] - m[1]) * t;
  } else {
    int i = 0;
    if (m[4] > m[0]) i = 1;
    if (m[8] > (i == 1 ? m[4] : m[0])) i = 2;
    // the three cases spelled out (j = i+1, k = i+2 mod 3): compile-time
    // indices keep m and q in registers; same operations per case
    if (i == 0) {
      t = sqrt(m[0] - m[4] - m[8] + 1.0);
      q[1] = 0.5 * t;
      t = 0.5 / t;
      q[0] = (m[7] - m[5]) * t;
      q[2] = (m[3] + m[1]) * t;
      q[3] = (m[6] + m[2]) * t;
    } else if (i == 1) {
      t = sqrt(m[4] - m[8] - m[0] + 1.0);
      q[2] = 0.5 * t;
      t = 0.5 / t;
      q[0] = (m[2] - m[6]) * t;
      q[3] = (m[7] + m[5]) * t;
      q[1] = (m[1] + m[3]) * t;
    } else {
      t = sqrt(m[8] - m[0] - m[4] + 1.0);
      q[3] = 0.5 * t;
      t = 0.5 / t;
      q[0] = (m[3] - m[1]) * t;
      q[1] = (m[2] + m[6]) * t;
      q[2] = (m[5] + m[7]) * t;
    }
  }
  Q4 o = q4(q[0], q[1], q[2], q[3]);
  o = qdiv(o, qnrm(o));
  if (o.w < 0) o = qneg(o);
  return o;
}
// geometry.cpp:52-56 (normalize + Quaterniond::toRotationMatrix)
DSI M3 matrix_from_quat(Q4 qin) {
  const Q4 q = qdiv(qin, qnrm(qin));
  const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
  const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  M3 r;
  r.m[0] = 1.0 - (tyy + tzz);
  r.m[1] = txy - twz;
  r.m[2] = txz + twy;
  r.m[3] = txy + twz;
  r.m[4] = 1.0 - (txx + tzz);
  r.m[5] = tyz - twx;
  r.m[6] = txz - twy;
  r.m[7] = tyz + twx;
  r.m[8] = 1.0 - (txx + tyy);
  return r;
}
// geometry.cpp:65-76
DSI Rig se3_increment(V3 om, V3 dt, const Rig& T) {
  Rig inc;
  inc.R = matrix_from_quat(quat_from_rotvec(om));
  inc.t = dt;
  Rig o = rig_mul(inc, T);
  o.R = matrix_from_quat(quat_from_matrix(o.R));
  return o;
}
// geometry.cpp:78-84
DSI DQ dq_from_rig(const Rig& T) {
  DQ q;
  q.r = quat_from_matrix(T.R);
  q.d = qscl(0.5, qmul(q4(0.0, T.t.x, T.t.y, T.t.z), q.r));
  return q;
}
// geometry.cpp:102-109
DSI DQ dq_normalized(const DQ& q) {
  const double a = qnrm(q.r);
  const double b = ddiv(qdot(q.r, q.d), a);
  DQ o;
  o.r = qdiv(q.r, a);
  o.d = qsub(qdiv(q.d, a), qscl(ddiv(b, a * a), q.r));
  return o;
}
// geometry.cpp:86-93
DSI Rig dq_to_rig(const DQ& q) {
  const DQ n = dq_normalized(q);
  Rig T;
  T.R = matrix_from_quat(n.r);
  const Q4 tq = qmul(n.d, qconj(n.r));
  T.t = v3(2.0 * tq.x, 2.0 * tq.y, 2.0 * tq.z);
  return T;
}
// geometry.cpp:95-100
DSI DQ dq_mul(const DQ& a, const DQ& b) {
  DQ o;
  o.r = qmul(a.r, b.r);
  o.d = qadd(qmul(a.r, b.d), qmul(a.d, b.r));
  return o;
}
// geometry.cpp:120-125
DSI DQ dq_increment(V3 om, V3 dt) {
  Rig inc;
  inc.R = matrix_from_quat(quat_from_rotvec(om));
  inc.t = dt;
  return dq_from_rig(inc);
}
DSI DQ dq_identity() {
  DQ q;
  q.r = q4(1, 0, 0, 0);
  q.d = q4(0, 0, 0, 0);
  return q;
}

constexpr double kDegenerateBlend = 1e-8;  // geometry.hpp:89

// geometry.cpp:156-159
DSI double skin_weight(V3 x, V3 p, double sigma) {
  const double d2 = sqn(sub(x, p));
  return exp(-d2 / (2.0 * sigma * sigma));
}

// (d2, index) total order of every KNN in the reference (spatial_grid.hpp:21-23)
DSI bool nb_less(double d2a, int ia, double d2b, int ib) {
  return d2a != d2b ? d2a < d2b : ia < ib;
}

// sorted (d2, index) top-4 insertion (used by every exact 4-NN kernel)
DSI void knn4_insert(double d2, int j, double bd[4], int bi[4]) {
  if (!nb_less(d2, j, bd[3], bi[3])) return;
  double cd = d2;
  int ci = j;
#pragma unroll
  for (int s = 0; s < 4; ++s)
    if (nb_less(cd, ci, bd[s], bi[s])) {
      const double td = bd[s];
      const int ti = bi[s];
      bd[s] = cd;
      bi[s] = ci;
      cd = td;
      ci = ti;
    }
}

// Butterfly merge of the per-lane top-4 lists of an aligned group of LANES
// lanes that scanned disjoint index subsets: afterwards every lane of the group
// holds the group's exact top-4 (strict total order => identical in all lanes).
template <int LANES>
__device__ __forceinline__ void knn4_merge_lanes(double bd[4], int bi[4]) {
#pragma unroll
  for (int off = LANES / 2; off > 0; off >>= 1) {
    double od[4];
    int oi[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      od[s] = __shfl_xor_sync(0xffffffffu, bd[s], off);
      oi[s] = __shfl_xor_sync(0xffffffffu, bi[s], off);
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) knn4_insert(od[s], oi[s], bd, bi);
  }
}

}  // namespace ds
