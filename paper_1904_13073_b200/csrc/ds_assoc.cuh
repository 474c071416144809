// ds_assoc.cuh — per-pixel model-map resolve and projective association, shared
// by the stand-alone resolve kernel (k_raster.cu) and the fused GN-iteration
// kernel (k_solver.cu).
//   resolve       raster.cpp:104-119: the point channel beats the splat channel
//   associate     solver.cpp:244-271: v_d = pose V, n_d = R N; keep iff
//                 |v_m - v_d| < 0.03 m and n_m . n_d > 0.7 (solver.hpp:14-15)
#pragma once
#include "ds_context.cuh"

namespace ds {

constexpr int kEmptyIdx = 0x7f7f7f7f;

__device__ __forceinline__ int resolve_winner(const int* __restrict__ pidx,
                                              const int* __restrict__ sidx, int c) {
  int win = pidx[c];
  if (win == kEmptyIdx) win = sidx[c];
  return win == kEmptyIdx ? -1 : win;
}

__device__ __forceinline__ int associate_pixel(int c, int win, const ModelBuf& m,
                                               const double4* __restrict__ fvert,
                                               const double4* __restrict__ fnrm,
                                               const uint8_t* __restrict__ fflag, const Rig& pose) {
  if (win < 0 || !(fflag[c] & 2)) return -1;
  const double4 fv = fvert[c], fn = fnrm[c];
  const V3 vd = rig_apply(pose, v3(fv.x, fv.y, fv.z));
  const V3 nd = rig_rotate(pose, v3(fn.x, fn.y, fn.z));
  const float4 lp = m.lp[win], ln = m.ln[win];
  const V3 vm = v3(lp.x, lp.y, lp.z);
  return (nrm(sub(vm, vd)) < 0.03 && dot(v3(ln.x, ln.y, ln.z), nd) > 0.7) ? win : -1;
}

}  // namespace ds
