// k_rigid.cu — projective point-to-plane rigid pre-alignment (K23).
//   rigid_align  solver.cpp:171-242: stride pyramid 4 -> 2 -> 1 with {3, 3, 4}
//   iterations, association at the lround pixel of the pose-transformed vertex
//   against model maps rendered under the initial pose, J = [v x n, n], 6x6
//   LDLT, se3_increment. Every iteration is ONE kernel: fp64 block reductions
//   of the 21 + 6 + 2 normal-equation terms, and the last block to arrive
//   (ticket) sums the partials in a fixed order and solves on the device, so
//   the whole pyramid runs without a host round trip.
#include <cstdio>

#include "ds_context.cuh"

namespace ds {
namespace {

constexpr int kTerms = 29;  // 21 upper H, 6 g, count, sum |r|
constexpr int kThreads = 256;

// Eigen::LDLT semantics (solver.cpp:225): diagonal pivoting, zero pivots kept,
// pseudo-inverse of D with tolerance DBL_MIN. Register-resident: every index
// is a compile-time constant (unrolled loops); the pivot row/column swaps are
// predicated on the runtime pivot instead of indexing with it. Same operations
// in the same order as the oracle's ldlt_solve.
__device__ __forceinline__ void ldlt_solve6(double A[6][6], const double* b, double* x) {
  int perm[6];
  bool zero_all = false;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    if (zero_all) break;
    int big = k;
    double bv = fabs(A[k][k]);
#pragma unroll
    for (int i = k + 1; i < 6; ++i)
      if (fabs(A[i][i]) > bv) {
        bv = fabs(A[i][i]);
        big = i;
      }
    perm[k] = big;
    if (big != k) {
#pragma unroll
      for (int c = 0; c < k; ++c) {  // swap A[k][c] <-> A[big][c]
        double vb = A[k][c];
#pragma unroll
        for (int i = k + 1; i < 6; ++i)
          if (i == big) vb = A[i][c];
#pragma unroll
        for (int i = k + 1; i < 6; ++i)
          if (i == big) A[i][c] = A[k][c];
        A[k][c] = vb;
      }
#pragma unroll
      for (int r = k + 1; r < 6; ++r) {  // swap A[r][k] <-> A[r][big] for r > big
        double vb = A[r][k];
#pragma unroll
        for (int i = k + 1; i < r; ++i)
          if (i == big) vb = A[r][i];
        if (r > big) {
#pragma unroll
          for (int i = k + 1; i < r; ++i)
            if (i == big) A[r][i] = A[r][k];
          A[r][k] = vb;
        }
      }
      {  // swap diagonal A[k][k] <-> A[big][big]
        double vb = A[k][k];
#pragma unroll
        for (int i = k + 1; i < 6; ++i)
          if (i == big) vb = A[i][i];
#pragma unroll
        for (int i = k + 1; i < 6; ++i)
          if (i == big) A[i][i] = A[k][k];
        A[k][k] = vb;
      }
#pragma unroll
      for (int i = k + 1; i < 6; ++i) {  // swap A[i][k] <-> A[big][i] for k < i < big
        if (i < big) {
          double vb = A[i][k];
#pragma unroll
          for (int j = i + 1; j < 6; ++j)
            if (j == big) vb = A[j][i];
#pragma unroll
          for (int j = i + 1; j < 6; ++j)
            if (j == big) A[j][i] = A[i][k];
          A[i][k] = vb;
        }
      }
    }
    if (k > 0) {
      double temp[6];
#pragma unroll
      for (int c = 0; c < k; ++c) temp[c] = A[c][c] * A[k][c];
      double sacc = 0;
#pragma unroll
      for (int c = 0; c < k; ++c) sacc += A[k][c] * temp[c];
      A[k][k] -= sacc;
#pragma unroll
      for (int r = k + 1; r < 6; ++r) {
        double acc = 0;
#pragma unroll
        for (int c = 0; c < k; ++c) acc += A[r][c] * temp[c];
        A[r][k] -= acc;
      }
    }
    const double akk = A[k][k];
    const bool valid = fabs(akk) > 0.0;
    if (k == 0 && !valid) {
      zero_all = true;
      break;
    }
    if (valid)
#pragma unroll
      for (int r = k + 1; r < 6; ++r) A[r][k] = ddiv(A[r][k], akk);
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) x[i] = zero_all ? 0.0 : b[i];
  if (zero_all) return;
#pragma unroll
  for (int k = 0; k < 6; ++k) {  // x[k] <-> x[perm[k]] (selects, no indexed access)
    const int pk = perm[k];
    const double xk = x[k];
    double vp = xk;
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      const bool hit = i == pk;
      const double xi = x[i];
      vp = hit ? xi : vp;
      x[i] = hit ? xk : xi;
    }
    x[k] = vp;
  }
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    double sacc = x[r];
#pragma unroll
    for (int c = 0; c < r; ++c) sacc -= A[r][c] * x[c];
    x[r] = sacc;
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) x[i] = fabs(A[i][i]) > 2.2250738585072014e-308 ? ddiv(x[i], A[i][i]) : 0.0;
#pragma unroll
  for (int r = 5; r >= 0; --r) {
    double sacc = x[r];
#pragma unroll
    for (int c = r + 1; c < 6; ++c) sacc -= A[c][r] * x[c];
    x[r] = sacc;
  }
#pragma unroll
  for (int k = 5; k >= 0; --k) {  // x[k] <-> x[perm[k]]
    const int pk = perm[k];
    const double xk = x[k];
    double vp = xk;
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      const bool hit = i == pk;
      const double xi = x[i];
      vp = hit ? xi : vp;
      x[i] = hit ? xk : xi;
    }
    x[k] = vp;
  }
}

struct RigidParams {
  Rig render_inv;
  double fx, fy, cx, cy;
  int W, H, stride, sw, sh;
};

__global__ void __launch_bounds__(kThreads) k_rigid_terms(RigidParams rp, const double* __restrict__ cur_pose,
                                                          const int* __restrict__ mm_idx, ModelBuf m,
                                                          const double4* __restrict__ fvert,
                                                          const double4* __restrict__ fnrm,
                                                          const uint8_t* __restrict__ fflag,
                                                          double* __restrict__ part,
                                                          unsigned* __restrict__ ticket, int level,
                                                          double* __restrict__ pose_out,
                                                          DevScalars* __restrict__ sc,
                                                          unsigned long long* __restrict__ trace) {
  __shared__ double sh[kThreads / 32][kTerms];
  __shared__ double tot[kTerms];
  __shared__ bool last;
  pdl_wait();  // programmatic dependent launch: the previous iteration's pose
  if (trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    trace[0] = t_;
  }
  double v[kTerms];
#pragma unroll
  for (int k = 0; k < kTerms; ++k) v[k] = 0.0;
  const int total = rp.sw * rp.sh;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int x = (t % rp.sw) * rp.stride, y = (t / rp.sw) * rp.stride;
    const size_t c = (size_t)y * rp.W + x;
    if (fflag[c] & 2) {
      const Rig cur = rig_load(cur_pose);
      const double4 fv = fvert[c];
      const V3 vw = rig_apply(cur, v3(fv.x, fv.y, fv.z));
      const V3 pr = rig_apply(rp.render_inv, vw);
      if (pr.z > 0) {
        const double u = rp.fx * pr.x / pr.z + rp.cx;
        const double vv = rp.fy * pr.y / pr.z + rp.cy;
        if (fabs(u) < 1e9 && fabs(vv) < 1e9) {
          const int ui = (int)llround(u), vi = (int)llround(vv);
          if (ui >= 0 && ui < rp.W && vi >= 0 && vi < rp.H) {
            const int win = mm_idx[(size_t)vi * rp.W + ui];
            if (win >= 0) {
              const float4 lp = m.lp[win], ln = m.ln[win];
              const V3 vm = v3(lp.x, lp.y, lp.z), nm = v3(ln.x, ln.y, ln.z);
              const double4 fn = fnrm[c];
              if (nrm(sub(vw, vm)) < 0.03 &&
                  dot(rig_rotate(cur, v3(fn.x, fn.y, fn.z)), nm) > 0.7) {
                const double r = dot(nm, sub(vw, vm));
                const V3 cr = cross(vw, nm);
                const double J[6] = {cr.x, cr.y, cr.z, nm.x, nm.y, nm.z};
                int k = 0;
#pragma unroll
                for (int a = 0; a < 6; ++a)
#pragma unroll
                  for (int b = a; b < 6; ++b) v[k++] += J[a] * J[b];
#pragma unroll
                for (int a = 0; a < 6; ++a) v[21 + a] += J[a] * r;
                v[27] += 1.0;
                v[28] += fabs(r);
              }
            }
          }
        }
      }
    }
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < kTerms; ++k) {
    double s = v[k];
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) sh[wid][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < kTerms) {  // term-major partials: the last block reads them coalesced
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += sh[w][threadIdx.x];
    part[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = s;
  }
  // the last block to arrive sums the partials in block order and solves
  // (solver.cpp:214-232) -- the whole ICP iteration is one launch
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  if (trace && threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    trace[1] = t_;
  }
  __threadfence();
  // 8 threads per term (29 x 8 <= 256): each sums every 8th block partial,
  // then an xor butterfly over the 8 (fixed order)
  const int nb = gridDim.x;
  {
    const int term = threadIdx.x >> 3, sub = threadIdx.x & 7;
    double sacc = 0.0;
    if (term < kTerms) {
#pragma unroll 8
      for (int b = sub; b < nb; b += 8) sacc += __ldcg(part + (size_t)term * nb + b);
    }
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, off);
    if (term < kTerms && sub == 0) tot[term] = sacc;
  }
  __syncthreads();
  if (trace && threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    trace[2] = t_;
  }
  if (threadIdx.x != 0) return;
  *ticket = 0u;
  const int pairs = (int)tot[27];
  if (level == 0) {
    sc->rigid_pairs = pairs;
    sc->rigid_abs = tot[28];
  }
  if (pairs < 6) return;
  double A[6][6];  // fully unrolled below: registers, no local memory
  int k = 0;
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = a; b < 6; ++b) {
      A[a][b] = tot[k];
      A[b][a] = tot[k];
      ++k;
    }
  double ng[6], xi[6];
#pragma unroll
  for (int a = 0; a < 6; ++a) ng[a] = -tot[21 + a];
  ldlt_solve6(A, ng, xi);
  if (trace && threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    trace[3] = t_;
  }
#pragma unroll
  for (int a = 0; a < 6; ++a)
    if (!isfinite(xi[a])) return;
  const Rig cur = rig_load(pose_out);
  rig_store(se3_increment(v3(xi[0], xi[1], xi[2]), v3(xi[3], xi[4], xi[5]), cur), pose_out);
  if (trace && threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    trace[4] = t_;
  }
}

}  // namespace

void rigid_align(Ctx& c, const double* render_pose, const double* init_pose, int t_now, int t_last,
                 ds_rigid_result* out) {
  rigid_align_enqueue(c, render_pose, init_pose, t_now, t_last);
  rigid_align_finish(c, init_pose, out);
}

void rigid_align_enqueue(Ctx& c, const double* render_pose, const double* init_pose, int t_now,
                         int t_last) {
  render_model_maps(c, render_pose, t_now, t_last, false, nullptr, true);
  DS_CUDA(cudaMemcpyAsync(c.d_pose, init_pose, 12 * sizeof(double), cudaMemcpyHostToDevice,
                          c.stream));
  DS_CUDA(cudaMemsetAsync(&c.dsc->rigid_pairs, 0, sizeof(int), c.stream));
  DS_CUDA(cudaMemsetAsync(&c.dsc->rigid_abs, 0, sizeof(double), c.stream));
  RigidParams rp;
  rp.render_inv = rig_inverse(rig_load(init_pose));
  rp.fx = c.cfg.fx;
  rp.fy = c.cfg.fy;
  rp.cx = c.cfg.cx;
  rp.cy = c.cfg.cy;
  rp.W = c.W;
  rp.H = c.H;
  static const int kIters[3] = {4, 3, 3};
  for (int level = 2; level >= 0; --level) {
    rp.stride = 1 << level;
    rp.sw = cdiv(c.W, rp.stride);
    rp.sh = cdiv(c.H, rp.stride);
    const int samples = rp.sw * rp.sh;
    // grid-stride, 2 CTAs per SM (DS_RIGID_GRID overrides): one sample per
    // thread measured slower (24.6 -> 32.7 us per level-0 launch at config
    // 2), the last block's reduction over 4x the partials costs more than the
    // shorter per-thread gather chains save
    const int nb = std::min(cdiv(samples, kThreads),
                            c.rigid_grid_cap > 0 ? c.rigid_grid_cap : 2 * c.num_sms);
    for (int it = 0; it < kIters[level]; ++it) {
      DS_LAUNCH_PDL(c, KK_RIGID, 100.0 * samples + 16.0 * kTerms * nb, nb, kThreads, 0, k_rigid_terms,
                rp, c.d_pose, c.mm_idx, c.M(), c.f_vert, c.f_nrm, c.f_flag, c.red_part,
                c.tickets + 3, level, c.d_pose, c.dsc, c.pcg_trace ? c.pcg_trace + 32 : nullptr);
    }
  }
}

void rigid_align_finish(Ctx& c, const double* init_pose, ds_rigid_result* out) {
  double pose[12];
  DS_CUDA(cudaMemcpyAsync(pose, c.d_pose, sizeof pose, cudaMemcpyDeviceToHost, c.stream));
  fetch_scalars(c);  // syncs
  if (c.pcg_trace) {  // last ICP launch: block-0 start -> last block phases (us)
    unsigned long long tr[5];
    DS_CUDA(cudaMemcpy(tr, c.pcg_trace + 32, sizeof tr, cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "rigid_trace last:%.2f reduce:%.2f ldlt:%.2f se3:%.2f\n",
                 (tr[1] - tr[0]) * 1e-3, (tr[2] - tr[1]) * 1e-3, (tr[3] - tr[2]) * 1e-3,
                 (tr[4] - tr[3]) * 1e-3);
  }
  const int pairs = c.hsc->rigid_pairs;
  const double abs_r = c.hsc->rigid_abs;
  ds_rigid_result r{};
  r.correspondences = pairs;
  if (pairs < 100) {  // kRigidMinCorrespondences (solver.hpp:19)
    std::copy(init_pose, init_pose + 12, r.pose);
    r.low_confidence = 1;
    r.mean_residual = pairs > 0 ? abs_r / pairs : 0.0;
  } else {
    std::copy(pose, pose + 12, r.pose);
    r.low_confidence = 0;
    r.mean_residual = abs_r / pairs;
  }
  *out = r;
}

}  // namespace ds
