// ds_pcg.cuh — pieces shared by the PCG kernels (k_solver.cu: cooperative
// grid PCG; k_pcg_cluster.cu: thread-block-cluster PCG).
#pragma once

namespace ds {

// Gauss-Jordan inverse of a 6x6 SPD block by an aligned 8-lane group: lane lr
// (< 6) holds row lr of A in a[] and returns row lr of A^-1 in b[]. A pivot
// that is not > 0 (the block is not SPD in its fp32-rounded form) makes the
// group fall back to the inverse diagonal, like the reference's LDLT guard.
__device__ __forceinline__ void gj_inverse6(double a[6], double b[6], int lr) {
  const int base = (threadIdx.x & 31) & ~7;
  double diag_lr = 1.0;  // a[lr] without a dynamic register-array index (no local memory)
#pragma unroll
  for (int t = 0; t < 6; ++t)
    if (t == lr) diag_lr = a[t];
#pragma unroll
  for (int t = 0; t < 6; ++t) b[t] = (t == lr) ? 1.0 : 0.0;
  bool ok = true;
#pragma unroll
  for (int p = 0; p < 6; ++p) {
    double ap[6], bp[6];
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      ap[t] = __shfl_sync(0xffffffffu, a[t], base + p);
      bp[t] = __shfl_sync(0xffffffffu, b[t], base + p);
    }
    const double piv = ap[p];
    if (!(piv > 0.0)) ok = false;
    // one division per step (pivot > 0 normal); the rows scale by the
    // reciprocal -- dividing the many zero entries would take the slow path
    const double ip = ok ? 1.0 / piv : 0.0;
    if (lr == p) {
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        a[t] = ap[t] * ip;
        b[t] = bp[t] * ip;
      }
    } else {
      const double f = a[p] * ip;
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        a[t] = a[t] - f * ap[t];
        b[t] = b[t] - f * bp[t];
      }
    }
  }
  if (!ok) {
#pragma unroll
    for (int t = 0; t < 6; ++t) b[t] = (t == lr && diag_lr > 0.0) ? 1.0 / diag_lr : 0.0;
  }
}

}  // namespace ds
