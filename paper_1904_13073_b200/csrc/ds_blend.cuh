// ds_blend.cuh — device dual-quaternion blending of a K<=4 skinning entry.
//   blend_dual_quaternions  geometry.cpp:127-147 (raw Gaussian weights, sign fix
//                           against slot 0, degenerate if |sum real| < 1e-8)
//   make_blend_state        solver.cpp:31-49 (signed weights kept for Jacobians)
#pragma once
#include "ds_math.cuh"

namespace ds {

struct Blend {
  Q4 rs, ds;
  double sw[4];
  int idx[4];
  int count;
  bool degenerate;
};

__device__ __forceinline__ int entry_count(int4 ki) {
  return ki.x < 0 ? 0 : (ki.y < 0 ? 1 : (ki.z < 0 ? 2 : (ki.w < 0 ? 3 : 4)));
}

__device__ __forceinline__ Q4 ld_q(const double4* __restrict__ p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return q4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ Q4 ld_q_plain(const double4* p) {
  const double4 v = *p;
  return q4(v.x, v.y, v.z, v.w);
}

// node_dq holds 2 double4 per node: real (w,x,y,z), dual (w,x,y,z)
__device__ __forceinline__ Blend blend_entry(int4 ki, float4 kw, const double4* __restrict__ node_dq) {
  Blend b;
  b.rs = q4(0, 0, 0, 0);
  b.ds = q4(0, 0, 0, 0);
  b.idx[0] = ki.x;
  b.idx[1] = ki.y;
  b.idx[2] = ki.z;
  b.idx[3] = ki.w;
  const double w4[4] = {(double)kw.x, (double)kw.y, (double)kw.z, (double)kw.w};
  b.count = entry_count(ki);
  b.degenerate = true;
  if (b.count == 0) return b;
  const Q4 pivot = ld_q(node_dq + 2 * b.idx[0]);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    b.sw[m] = 0.0;
    if (m < b.count) {
      const Q4 r = ld_q(node_dq + 2 * b.idx[m]);
      const Q4 d = ld_q(node_dq + 2 * b.idx[m] + 1);
      const double sign = (qdot(pivot, r) < 0.0) ? -1.0 : 1.0;
      const double w = sign * w4[m];
      b.sw[m] = w;
      b.rs = qadd(b.rs, qscl(w, r));
      b.ds = qadd(b.ds, qscl(w, d));
    }
  }
  b.degenerate = qnrm(b.rs) < kDegenerateBlend;
  return b;
}

// Same rigid transform as blend_rig() up to rounding, with one rsqrt instead of
// the ~24 fp64 divisions of normalized() -> to_se3() -> normalize(): used where
// the result is a continuous quantity (warped positions/normals, residuals).
__device__ __forceinline__ Rig blend_rig_fast(const Blend& b) {
  const double ia = rsqrt(qdot(b.rs, b.rs));
  const Q4 nr = qscl(ia, b.rs);
  const double k = qdot(b.rs, b.ds) * (ia * ia * ia);
  const Q4 nd = qsub(qscl(ia, b.ds), qscl(k, b.rs));
  const double tx = 2.0 * nr.x, ty = 2.0 * nr.y, tz = 2.0 * nr.z;
  const double twx = tx * nr.w, twy = ty * nr.w, twz = tz * nr.w;
  const double txx = tx * nr.x, txy = ty * nr.x, txz = tz * nr.x;
  const double tyy = ty * nr.y, tyz = tz * nr.y, tzz = tz * nr.z;
  Rig T;
  T.R.m[0] = 1.0 - (tyy + tzz);
  T.R.m[1] = txy - twz;
  T.R.m[2] = txz + twy;
  T.R.m[3] = txy + twz;
  T.R.m[4] = 1.0 - (txx + tzz);
  T.R.m[5] = tyz - twx;
  T.R.m[6] = txz - twy;
  T.R.m[7] = tyz + twx;
  T.R.m[8] = 1.0 - (txx + tyy);
  const Q4 tq = qmul(nd, qconj(nr));
  T.t = v3(2.0 * tq.x, 2.0 * tq.y, 2.0 * tq.z);
  return T;
}

// Rigid transform of a non-degenerate blend: normalized() then to_se3()
// (which normalizes again), as blend_dual_quaternions + to_se3 do.
__device__ __forceinline__ Rig blend_rig(const Blend& b) {
  DQ raw;
  raw.r = b.rs;
  raw.d = b.ds;
  return dq_to_rig(dq_normalized(raw));
}

// True when the fp32 rounding of x cannot change if x moves by up to
// 2^m * max(1, |x|): integer test on x's fp64 bits (no FP64-pipe work).
// Within x's binade the fp32 rounding boundaries are where the 29 mantissa
// bits below fp32 precision equal 2^28; x is stable when its low bits are
// farther than the margin, in units of its fp64 ulp 2^(e-52), from that.
// The fast and exact transforms differ by <= ~1e-13 m on positions of a
// <= 5 m scene (R from normalised quaternions a few ulps apart, applied to
// |x| <= 5 m, plus t) and <= ~1.2e-14 on unit normals: margins 2^-40 (9e-13)
// and 2^-43 (1.1e-13) keep a ~10x factor. Tiny |x| (margin >= half an fp32
// ulp) and huge ones take the exact path.
template <int kMarginLog2>
__device__ __forceinline__ bool f32_round_stable(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  const int e = (int)((b >> 52) & 0x7ff) - 1023;
  // margin in fp64 ulps of x: 2^m max(1, |x|) / 2^(e-52) <= 2^(53 + m - min(e, 0))
  const int sh = 53 + kMarginLog2 - (e < 0 ? e : 0);
  if (sh >= 28 || e > 100) return false;
  const long long low = (long long)(b & ((1ull << 29) - 1)) - (1ll << 28);
  return (low < 0 ? -low : low) > (1ll << (sh < 0 ? 0 : sh));
}

// Live state of one surfel under a non-degenerate blend (forward_warp,
// warp_field.cpp:128-140), stored fp32 as the SoA model. The rsqrt transform
// (blend_rig_fast) agrees with the reference's normalized() -> to_se3() chain
// (blend_rig) to a few fp64 ulps; whenever a stored coordinate could round
// differently (f32_round_stable) the exact chain is evaluated instead, so the
// stored live state is the one the reference arithmetic rounds to (bit-exact
// z-buffer inputs). Measured cost: ~2 % of the config-2 frame rate, 12 % of
// the stand-alone warp at config 4 (the exact branch's registers); a fix-up
// kernel for the rare boundary surfels instead measured slower (its launch in
// the GN chain cost 5 %).
__device__ __forceinline__ void warp_surfel(const Blend& b, const float4& rp, const float4& rn,
                                            float4& lp, float4& ln) {
  // a blend of identity transforms (every node before its first solve) gives
  // R = I, t = 0 exactly on both chains: p = x, q = n with no rounding
  const bool ident = b.rs.x == 0.0 && b.rs.y == 0.0 && b.rs.z == 0.0 && b.ds.w == 0.0 &&
                     b.ds.x == 0.0 && b.ds.y == 0.0 && b.ds.z == 0.0;
  const V3 x = v3(rp.x, rp.y, rp.z), nx = v3(rn.x, rn.y, rn.z);
  const Rig T = blend_rig_fast(b);
  V3 p = rig_apply(T, x), q = rig_rotate(T, nx);
#if !defined(DS_WARP_GUARD) || DS_WARP_GUARD != 0
  const bool ok = ident ||
                  (f32_round_stable<-40>(p.x) && f32_round_stable<-40>(p.y) &&
                   f32_round_stable<-40>(p.z) && f32_round_stable<-43>(q.x) &&
                   f32_round_stable<-43>(q.y) && f32_round_stable<-43>(q.z));
  if (!ok) {
    const Rig Te = blend_rig(b);
    p = rig_apply(Te, x);
    q = rig_rotate(Te, nx);
  }
#endif
  lp = make_float4((float)p.x, (float)p.y, (float)p.z, rp.w);
  ln = make_float4((float)q.x, (float)q.y, (float)q.z, rn.w);
}

}  // namespace ds
