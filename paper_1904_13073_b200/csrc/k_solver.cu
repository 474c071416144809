// k_solver.cu — Gauss-Newton non-rigid solve (K5-K9) and its LM control.
//
//   pair terms        solver.cpp:330-344 + :58-112: per correspondence pixel, the
//                     blended warp y = W(p_ref), r = n_d . (y - v_d), and the four
//                     1x6 Jacobian rows a_m = n_d^T dy/dxi_m. The 3x8 blend
//                     Jacobian is never formed: u = (dy/db)^T n_d is applied
//                     through the symmetric normalisation derivatives directly.
//   term -> block     the JtJ pattern is a per-frame superset: every surfel's
//                     skinning entry contributes K(K+1)/2 (row<=col) node-pair
//                     records, every directed edge j->i three (solver.cpp:355-369);
//                     records are radix-sorted once per frame by block key.
//   block assembly    warp per upper 6x6 block: lanes walk the block's records,
//                     gather the per-surfel pair lists (pixel order) and
//                     accumulate a_m1 a_m2^T in fp64 registers; a fixed-order
//                     shared-memory reduction makes it bit-deterministic. Blocks
//                     are written as fp32 BSR (both triangles), g in fp64.
//   PCG               one cooperative persistent kernel: block-Jacobi (6x6
//                     Cholesky inverse per node), BSR SpMV with lanes mapped to
//                     (block, row) pairs and a shuffle row reduction, deterministic
//                     grid reductions, two grid.sync per iteration.
//   LM                solver.cpp:371-406 on the host: mu floor from tr(H), <= 8
//                     attempts, accept iff E_post <= E_pre (fp64 energies).
#include <cooperative_groups.h>

#include <algorithm>

#include "ds_blend.cuh"
#include "ds_context.cuh"
#include "ds_reduce.cuh"

namespace cg = cooperative_groups;

namespace ds {

size_t sort_temp_bytes(int n);

namespace {

constexpr int kIntMax = 0x7fffffff;

// ---------------------------------------------------------------- pair terms
// rows 1..3 of quat_right_matrix(q) (geometry.cpp:23-30), row r, col k
__device__ __forceinline__ double Rq(const Q4& q, int r, int k) {
  const double a[4][4] = {{q.w, -q.x, -q.y, -q.z},
                          {q.x, q.w, q.z, -q.y},
                          {q.y, -q.z, q.w, q.x},
                          {q.z, q.y, -q.x, q.w}};
  return a[r][k];
}
__device__ __forceinline__ double Lq(const Q4& q, int r, int k) {  // geometry.cpp:14-21
  const double a[4][4] = {{q.w, -q.x, -q.y, -q.z},
                          {q.x, q.w, -q.z, q.y},
                          {q.y, q.z, q.w, -q.x},
                          {q.z, -q.y, q.x, q.w}};
  return a[r][k];
}

struct PairParams {
  Rig pose;
  int P;
};

// Per correspondence: residual, Jacobian rows (fp32), data energy partials.
__global__ void __launch_bounds__(256) k_pair_terms(const int* __restrict__ pair_s, ModelBuf m,
                                                    const double4* __restrict__ node_dq,
                                                    const double4* __restrict__ fvert,
                                                    const double4* __restrict__ fnrm,
                                                    PairParams pp, uint8_t* __restrict__ pair_ok,
                                                    float* __restrict__ rows,
                                                    double* __restrict__ pair_r,
                                                    int* __restrict__ s_cnt,
                                                    double* __restrict__ part,
                                                    unsigned* __restrict__ ticket,
                                                    double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  double e = 0.0;
  int s = c < pp.P ? pair_s[c] : -1;
  if (s >= 0) {
    const Blend b = blend_entry(m.ki[s], m.kw[s], node_dq);
    if (b.degenerate) {
      pair_ok[c] = 0;
    } else {
      const float4 rp = m.rp[s];
      const V3 p = v3(rp.x, rp.y, rp.z);
      const double4 fv = fvert[c], fn = fnrm[c];
      const V3 vd = rig_apply(pp.pose, v3(fv.x, fv.y, fv.z));
      const V3 nd = rig_rotate(pp.pose, v3(fn.x, fn.y, fn.z));
      const V3 y = rig_apply(blend_rig_fast(b), p);
      const double r = dot(nd, sub(y, vd));
      e = r * r;
      // ---- u = (dy/db)^T n_d  (solver.cpp:58-92)
      const Q4 br = b.rs, bd = b.ds;
      const double a = qnrm(br);
      const double rd = qdot(br, bd);
      const Q4 nr = qdiv(br, a);
      const Q4 ndq = qsub(qdiv(bd, a), qscl(rd / (a * a * a), br));
      const Q4 pq = q4(0.0, p.x, p.y, p.z);
      const Q4 q1 = qmul(pq, qconj(nr)), q2 = qmul(nr, pq);
      const Q4 cn = qconj(nr);
      const double nv[3] = {nd.x, nd.y, nd.z};
      double al[4], be[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double ck = (k == 0) ? 1.0 : -1.0;
        double sa = 0, sb = 0;
#pragma unroll
        for (int rr = 1; rr < 4; ++rr) {
          const double d4r = Rq(q1, rr, k) + Lq(q2, rr, k) * ck + 2.0 * Lq(ndq, rr, k) * ck;
          sa += nv[rr - 1] * d4r;
          sb += nv[rr - 1] * (2.0 * Rq(cn, rr, k));
        }
        al[k] = sa;
        be[k] = sb;
      }
      const Q4 alq = q4(al[0], al[1], al[2], al[3]), beq = q4(be[0], be[1], be[2], be[3]);
      const Q4 rh = qdiv(br, a);
      const double a3 = a * a * a, a5 = a3 * a * a;
      // dnr/dbr al = (al - rh (rh.al)) / a
      const Q4 u_r1 = qdiv(qsub(alq, qscl(qdot(rh, alq), rh)), a);
      // dnd/dbr be = -(bd (br.be) + br (bd.be) + rd be)/a^3 + 3 rd/a^5 br (br.be)
      const double brbe = qdot(br, beq), bdbe = qdot(bd, beq);
      const Q4 t1 = qadd(qadd(qscl(brbe, bd), qscl(bdbe, br)), qscl(rd, beq));
      const Q4 u_r2 = qadd(qscl(-1.0 / a3, t1), qscl(3.0 * rd / a5 * brbe, br));
      const Q4 ur = qadd(u_r1, u_r2);
      // dnd/dbd be = be/a - br (br.be)/a^3
      const Q4 ud = qsub(qdiv(beq, a), qscl(brbe / a3, br));
      const double uv[8] = {ur.w, ur.x, ur.y, ur.z, ud.w, ud.x, ud.y, ud.z};
      float* out = rows + (size_t)c * 24;
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) {
        if (mm < b.count) {
          const Q4 qr = ld_q(node_dq + 2 * b.idx[mm]);
          const Q4 qd = ld_q(node_dq + 2 * b.idx[mm] + 1);
          const double hw = 0.5 * b.sw[mm];
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) {
            double om = 0, tt = 0;
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
              om += uv[rr] * (hw * Rq(qr, rr, cc + 1)) + uv[4 + rr] * (hw * Rq(qd, rr, cc + 1));
              tt += uv[4 + rr] * (hw * Rq(qr, rr, cc + 1));
            }
            out[mm * 6 + cc] = (float)om;
            out[mm * 6 + 3 + cc] = (float)tt;
          }
        }
      }
      pair_r[c] = r;
      pair_ok[c] = 1;
      atomicAdd(s_cnt + s, 1);
    }
  }
  grid_sum<256>(e, part, ticket, out);  // data energy, fixed order
}

// E_data at arbitrary node transforms over the fixed pair set (solver.cpp:132-143);
// mode 0: sum r^2, mode 1: sum |r| and count (final report, solver.cpp:409-420)
__global__ void __launch_bounds__(256) k_pair_energy(const int* __restrict__ pair_s, ModelBuf m,
                                                     const double4* __restrict__ node_dq,
                                                     const double4* __restrict__ fvert,
                                                     const double4* __restrict__ fnrm,
                                                     PairParams pp, int mode,
                                                     double* __restrict__ part,
                                                     int* __restrict__ count,
                                                     unsigned* __restrict__ ticket,
                                                     double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  double e = 0.0;
  int ok = 0;
  const int s = c < pp.P ? pair_s[c] : -1;
  if (s >= 0) {
    const Blend b = blend_entry(m.ki[s], m.kw[s], node_dq);
    if (!b.degenerate) {
      const float4 rp = m.rp[s];
      const double4 fv = fvert[c], fn = fnrm[c];
      const V3 vd = rig_apply(pp.pose, v3(fv.x, fv.y, fv.z));
      const V3 nd = rig_rotate(pp.pose, v3(fn.x, fn.y, fn.z));
      const V3 y = rig_apply(blend_rig_fast(b), v3(rp.x, rp.y, rp.z));
      const double r = dot(nd, sub(y, vd));
      e = mode == 0 ? r * r : fabs(r);
      ok = 1;
    }
  }
  if (count) {
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    if ((threadIdx.x & 31) == 0 && bal) atomicAdd(count, __popc(bal));
  }
  grid_sum<256>(e, part, ticket, out);
}

// E_reg over directed edges j -> i (solver.cpp:145-155)
__global__ void __launch_bounds__(256) k_reg_energy(const double4* __restrict__ pos,
                                                    const int* __restrict__ nbr,
                                                    const double* __restrict__ se3, int N,
                                                    double* __restrict__ part,
                                                    unsigned* __restrict__ ticket,
                                                    double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (e < 8 * N) {
    const int i = nbr[e];
    if (i >= 0) {
      const int j = e >> 3;
      const double4 pj = pos[j];
      const V3 p = v3(pj.x, pj.y, pj.z);
      const Rig Tj = rig_load(se3 + 12 * j), Ti = rig_load(se3 + 12 * i);
      v = sqn(sub(rig_apply(Tj, p), rig_apply(Ti, p)));
    }
  }
  grid_sum<256>(v, part, ticket, out);
}

__global__ void k_any_stable_flag(const float4* __restrict__ ln, int n, double delta_stable,
                                  int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool st = i < n && (double)ln[i].w > delta_stable;
  const unsigned b = __ballot_sync(0xffffffffu, st);
  if ((threadIdx.x & 31) == 0 && b) atomicOr(flag, 1);
}

// ---------------------------------------------------------------- pair lists
__global__ void k_scatter_pairs(const int* __restrict__ pair_s, const uint8_t* __restrict__ pair_ok,
                                int P, const int* __restrict__ s_off, int* __restrict__ s_cur,
                                int* __restrict__ s_list) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P) return;
  const int s = pair_s[c];
  if (s < 0 || !pair_ok[c]) return;
  const int k = atomicAdd(s_cur + s, 1);
  s_list[s_off[s] + k] = c;
}
// Sort each surfel's pair list into pixel order (deterministic summation order)
// and gather the pairs' Jacobian rows / residuals into list order, so the block
// assembly reads one contiguous run per surfel.
__global__ void k_sort_lists(const int* __restrict__ s_cnt, const int* __restrict__ s_off, int n,
                             int* __restrict__ s_list, const float* __restrict__ rows,
                             const double* __restrict__ pair_r, float* __restrict__ rows_l,
                             double* __restrict__ r_l) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int cnt = s_cnt[s];
  if (cnt == 0) return;
  const int off = s_off[s];
  int* l = s_list + off;
  for (int a = 1; a < cnt; ++a) {
    const int v = l[a];
    int b = a;
    while (b > 0 && l[b - 1] > v) {
      l[b] = l[b - 1];
      --b;
    }
    l[b] = v;
  }
  for (int q = 0; q < cnt; ++q) {
    const int pix = l[q];
    const float4* src = reinterpret_cast<const float4*>(rows + (size_t)pix * 24);
    float4* dst = reinterpret_cast<float4*>(rows_l + (size_t)(off + q) * 24);
#pragma unroll
    for (int t = 0; t < 6; ++t) dst[t] = src[t];
    r_l[off + q] = pair_r[pix];
  }
}

// ------------------------------------------------------------ block pattern
__constant__ int kSlotPairs[10][2] = {{0, 0}, {0, 1}, {0, 2}, {0, 3}, {1, 1},
                                      {1, 2}, {1, 3}, {2, 2}, {2, 3}, {3, 3}};

// A surfel can only own correspondence pairs if render_model_maps draws it
// (raster.cpp:42-49, 65-68); eligibility is fixed during one frame's solve.
__global__ void k_elig_flags(const float4* __restrict__ ln, const int2* __restrict__ tt, int n,
                             double delta_stable, int t_now, int delta_recent, int host_boot,
                             const int* __restrict__ any_stable, int* __restrict__ flag) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const bool stable = (double)ln[s].w > delta_stable;
  const bool recent = (t_now - tt[s].y) <= delta_recent;
  const bool boot = host_boot || !(*any_stable);
  flag[s] = (stable || (boot && recent)) ? 1 : 0;
}
__global__ void k_elig_list(const int* __restrict__ flag, const int* __restrict__ scan, int n,
                            int* __restrict__ list) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n && flag[s]) list[scan[s]] = s;
}

__global__ void k_gen_records(const int4* __restrict__ ki, const int* __restrict__ elig, int n,
                              int N, int* __restrict__ key, int* __restrict__ val) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int s = elig[q];
  const int4 e = ki[s];
  const int cnt = entry_count(e);
  const int id[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
  for (int t = 0; t < 10; ++t) {
    const int m1 = kSlotPairs[t][0], m2 = kSlotPairs[t][1];
    int k = kIntMax, v = 0;
    if (m2 < cnt) {
      const int a = id[m1], b = id[m2];
      if (a <= b) {
        k = a * N + b;
        v = (s << 4) | (m1 << 2) | m2;
      } else {
        k = b * N + a;
        v = (s << 4) | (m2 << 2) | m1;
      }
    }
    key[(size_t)q * 10 + t] = k;
    val[(size_t)q * 10 + t] = v;
  }
}
__global__ void k_gen_reg_records(const int* __restrict__ nbr, int N, int* __restrict__ key,
                                  int* __restrict__ val) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 8 * N) return;
  const int i = nbr[e];
  const int j = e >> 3;
  int k0 = kIntMax, k1 = kIntMax, k2 = kIntMax;
  const int base = (int)(0x80000000u | (unsigned)(e << 2));
  int v2 = 0;
  if (i >= 0) {
    k0 = j * N + j;
    k1 = i * N + i;
    if (j < i) {
      k2 = j * N + i;
      v2 = base | 2;
    } else {
      k2 = i * N + j;
      v2 = base | 3;
    }
  }
  key[3 * e] = k0;
  val[3 * e] = base | 0;
  key[3 * e + 1] = k1;
  val[3 * e + 1] = base | 1;
  key[3 * e + 2] = k2;
  val[3 * e + 2] = v2;
}
__global__ void k_mark_unique(const int* __restrict__ key, int n, int* __restrict__ flag) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int v = key[k];
  flag[k] = (v != kIntMax && (k == 0 || key[k - 1] != v)) ? 1 : 0;
}
__global__ void k_write_up(const int* __restrict__ key, const int* __restrict__ scan, int n,
                           int* __restrict__ up_key, int* __restrict__ up_start, int ub_cap,
                           int* __restrict__ err) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int v = key[k];
  if (v == kIntMax) return;
  const int total = scan[n];
  if (total > ub_cap) {
    if (k == 0) atomicOr(err, DERR_BLOCK_CAP);
    return;
  }
  if (k == 0 || key[k - 1] != v) {
    const int ub = scan[k];
    up_key[ub] = v;
    up_start[ub] = k;
  }
  if (k + 1 == n || key[k + 1] == kIntMax) up_start[total] = k + 1;
}
__global__ void k_row_count(const int* __restrict__ up_key, const int* __restrict__ n_up_dev, int N,
                            int* __restrict__ row_cnt) {
  const int ub = blockIdx.x * blockDim.x + threadIdx.x;
  if (ub >= *n_up_dev) return;
  const int k = up_key[ub];
  const int r = k / N, cc = k % N;
  atomicAdd(row_cnt + r, 1);
  if (r != cc) atomicAdd(row_cnt + cc, 1);
}
__global__ void k_row_fill(const int* __restrict__ up_key, const int* __restrict__ n_up_dev, int N,
                           const int* __restrict__ row_ptr, int* __restrict__ row_cur,
                           int* __restrict__ col, int* __restrict__ tag) {
  const int ub = blockIdx.x * blockDim.x + threadIdx.x;
  if (ub >= *n_up_dev) return;
  const int k = up_key[ub];
  const int r = k / N, cc = k % N;
  int p = row_ptr[r] + atomicAdd(row_cur + r, 1);
  col[p] = cc;
  tag[p] = ub << 1;
  if (r != cc) {
    p = row_ptr[cc] + atomicAdd(row_cur + cc, 1);
    col[p] = r;
    tag[p] = (ub << 1) | 1;
  }
}
__global__ void k_row_sort(const int* __restrict__ row_ptr, int N, int* __restrict__ col,
                           int* __restrict__ tag, int* __restrict__ up_pos, int* __restrict__ up_mpos,
                           int* __restrict__ diag_pos) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  const int a0 = row_ptr[r], a1 = row_ptr[r + 1];
  for (int a = a0 + 1; a < a1; ++a) {
    const int vc = col[a], vt = tag[a];
    int b = a;
    while (b > a0 && col[b - 1] > vc) {
      col[b] = col[b - 1];
      tag[b] = tag[b - 1];
      --b;
    }
    col[b] = vc;
    tag[b] = vt;
  }
  diag_pos[r] = -1;
  for (int a = a0; a < a1; ++a) {
    const int t = tag[a];
    if (t & 1) up_mpos[t >> 1] = a;
    else up_pos[t >> 1] = a;
    if (col[a] == r) diag_pos[r] = a;
  }
}

// ------------------------------------------------------------ block assembly
// The sorted records of one upper block are cut into fixed chunks of <= 64;
// an 8-lane group reduces each chunk (lane l takes records l, l+8, ...), then
// one thread per block sums its chunk partials in chunk order. Fixed work
// decomposition + fixed reduction order => bit-deterministic; chunking balances
// the diagonal blocks (hundreds of records) against off-diagonal ones.
constexpr int kChunk = 64;
constexpr int kChunkLanes = 8;

struct AsmArgs {
  const int* up_key;
  const int* up_start;
  const int* up_pos;
  const int* up_mpos;
  const int* chunk_ub;
  const int* chunk_first;
  const int* rec_val;
  const int* s_cnt;
  const int* s_off;
  const float* rows_l;
  const double* r_l;
  const double4* node_pos;
  const int* nbr;
  const double* se3;
  double lambda;
  int N;
  int n_up;
  int n_chunks;
  float* part_h;
  double* part_g;
  int* part_t;
  float* bsr_val;
  uint8_t* bsr_touch;
  double* g;
};

__device__ __forceinline__ void reg_jac(const double4* __restrict__ pos, const int* __restrict__ nbr,
                                        const double* __restrict__ se3, int e, double Jj[3][6],
                                        double Ji[3][6], double rv[3]) {
  const int j = e >> 3, i = nbr[e];
  const double4 pj = pos[j];
  const V3 p = v3(pj.x, pj.y, pj.z);
  const V3 a = rig_apply(rig_load(se3 + 12 * j), p);
  const V3 b = rig_apply(rig_load(se3 + 12 * i), p);
  const V3 r = sub(a, b);
  rv[0] = r.x;
  rv[1] = r.y;
  rv[2] = r.z;
  // reg_jacobian_j = [-[a]x, I], reg_jacobian_i = [[b]x, -I]  (solver.cpp:118-130)
  const double sa[3][3] = {{0, -a.z, a.y}, {a.z, 0, -a.x}, {-a.y, a.x, 0}};
  const double sb[3][3] = {{0, -b.z, b.y}, {b.z, 0, -b.x}, {-b.y, b.x, 0}};
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Jj[k][c] = -sa[k][c];
      Jj[k][3 + c] = (k == c) ? 1.0 : 0.0;
      Ji[k][c] = sb[k][c];
      Ji[k][3 + c] = (k == c) ? -1.0 : 0.0;
    }
}

__global__ void __launch_bounds__(256) k_assemble_chunks(AsmArgs A) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const int chunk = gid / kChunkLanes, l = gid % kChunkLanes;
  const bool valid = chunk < A.n_chunks;  // uniform within a lane group
  float h[36];
  double gg[6];
#pragma unroll
  for (int t = 0; t < 36; ++t) h[t] = 0.f;
#pragma unroll
  for (int t = 0; t < 6; ++t) gg[t] = 0.0;
  int touched = 0;
  if (valid) {
    const int ub = A.chunk_ub[chunk];
    const int key = A.up_key[ub];
    const bool diag = (key / A.N) == (key % A.N);
    const int first = A.chunk_first[ub];
    const int r0 = A.up_start[ub] + (chunk - first) * kChunk;
    const int r1 = min(r0 + kChunk, A.up_start[ub + 1]);
    for (int k = r0 + l; k < r1; k += kChunkLanes) {
      const int v = A.rec_val[k];
      if (v < 0) {
        const int e = (v & 0x7fffffff) >> 2, type = v & 3;
        double Jj[3][6], Ji[3][6], rv[3];
        reg_jac(A.node_pos, A.nbr, A.se3, e, Jj, Ji, rv);
        touched = 1;
        const bool lj = (type == 0 || type == 2), rj = (type == 0 || type == 3);
#pragma unroll
        for (int x = 0; x < 6; ++x) {
#pragma unroll
          for (int y = 0; y < 6; ++y) {
            const double L0 = lj ? Jj[0][x] : Ji[0][x], L1 = lj ? Jj[1][x] : Ji[1][x],
                         L2 = lj ? Jj[2][x] : Ji[2][x];
            const double R0 = rj ? Jj[0][y] : Ji[0][y], R1 = rj ? Jj[1][y] : Ji[1][y],
                         R2 = rj ? Jj[2][y] : Ji[2][y];
            h[x * 6 + y] += (float)(A.lambda * ((L0 * R0 + L1 * R1) + L2 * R2));
          }
          if (type <= 1) {
            const double L0 = lj ? Jj[0][x] : Ji[0][x], L1 = lj ? Jj[1][x] : Ji[1][x],
                         L2 = lj ? Jj[2][x] : Ji[2][x];
            gg[x] += A.lambda * ((L0 * rv[0] + L1 * rv[1]) + L2 * rv[2]);
          }
        }
      } else {
        const int s = v >> 4, mr = (v >> 2) & 3, mc = v & 3;
        const int cnt = A.s_cnt[s];
        if (cnt == 0) continue;
        touched = 1;
        const int off = A.s_off[s];
        for (int q = 0; q < cnt; ++q) {
          const float* rw = A.rows_l + (size_t)(off + q) * 24;
          float a[6], b[6];
#pragma unroll
          for (int t = 0; t < 6; ++t) {
            a[t] = rw[mr * 6 + t];
            b[t] = rw[mc * 6 + t];
          }
#pragma unroll
          for (int x = 0; x < 6; ++x)
#pragma unroll
            for (int y = 0; y < 6; ++y) h[x * 6 + y] += a[x] * b[y];
          if (diag) {
            const double r = A.r_l[off + q];
#pragma unroll
            for (int x = 0; x < 6; ++x) gg[x] += (double)a[x] * r;
          }
        }
      }
    }
  }
  // fixed butterfly over the 8 lanes of the group
#pragma unroll
  for (int off = kChunkLanes / 2; off > 0; off >>= 1) {
#pragma unroll
    for (int t = 0; t < 36; ++t) h[t] += __shfl_xor_sync(0xffffffffu, h[t], off);
#pragma unroll
    for (int t = 0; t < 6; ++t) gg[t] += __shfl_xor_sync(0xffffffffu, gg[t], off);
    touched |= __shfl_xor_sync(0xffffffffu, touched, off);
  }
  if (valid && l == 0) {
    float4* ph = reinterpret_cast<float4*>(A.part_h + (size_t)chunk * 36);
#pragma unroll
    for (int t = 0; t < 9; ++t) ph[t] = make_float4(h[4 * t], h[4 * t + 1], h[4 * t + 2], h[4 * t + 3]);
#pragma unroll
    for (int t = 0; t < 6; ++t) A.part_g[(size_t)chunk * 6 + t] = gg[t];
    A.part_t[chunk] = touched;
  }
}

// thread per upper block: chunk partials in chunk order -> BSR (both triangles), g
__global__ void k_assemble_finish(AsmArgs A) {
  const int ub = blockIdx.x * blockDim.x + threadIdx.x;
  if (ub >= A.n_up) return;
  const int key = A.up_key[ub];
  const int row = key / A.N, colb = key % A.N;
  const int c0 = A.chunk_first[ub], c1 = A.chunk_first[ub + 1];
  int touched = 0;
  for (int c = c0; c < c1; ++c) touched |= A.part_t[c];
  const int pu = A.up_pos[ub];
  const int pm = row != colb ? A.up_mpos[ub] : -1;
  for (int t = 0; t < 36; ++t) {
    double acc = 0.0;
    for (int c = c0; c < c1; ++c) acc += (double)A.part_h[(size_t)c * 36 + t];
    A.bsr_val[(size_t)pu * 36 + t] = (float)acc;
    if (pm >= 0) A.bsr_val[(size_t)pm * 36 + (t % 6) * 6 + t / 6] = (float)acc;
  }
  A.bsr_touch[pu] = touched ? 1 : 0;
  if (pm >= 0) {
    A.bsr_touch[pm] = touched ? 1 : 0;
  } else {
    for (int x = 0; x < 6; ++x) {
      double acc = 0.0;
      for (int c = c0; c < c1; ++c) acc += A.part_g[(size_t)c * 6 + x];
      A.g[6 * row + x] = acc;
    }
  }
}

__global__ void k_chunk_count(const int* __restrict__ up_start, int n_up, int* __restrict__ cnt) {
  const int ub = blockIdx.x * blockDim.x + threadIdx.x;
  if (ub < n_up) cnt[ub] = (up_start[ub + 1] - up_start[ub] + kChunk - 1) / kChunk;
}
__global__ void k_chunk_fill(const int* __restrict__ first, int n_up, int* __restrict__ chunk_ub) {
  const int ub = blockIdx.x * blockDim.x + threadIdx.x;
  if (ub >= n_up) return;
  for (int c = first[ub]; c < first[ub + 1]; ++c) chunk_ub[c] = ub;
}

// ginf, |g|^2, tr(H) (solver.cpp:371, 378)
__global__ void k_g_stats(const double* __restrict__ g, int dim, const float* __restrict__ val,
                          const int* __restrict__ diag_pos, int N, DevScalars* __restrict__ sc) {
  __shared__ double smax[256], ssq[256], str[256];
  double mx = 0, sq = 0, tr = 0;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) {
    const double v = g[i];
    mx = fmax(mx, fabs(v));
    sq += v * v;
  }
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    const int d = diag_pos[j];
    if (d < 0) continue;
    const float* b = val + (size_t)d * 36;
    tr += (((((double)b[0] + (double)b[7]) + (double)b[14]) + (double)b[21]) + (double)b[28]) +
          (double)b[35];
  }
  smax[threadIdx.x] = mx;
  ssq[threadIdx.x] = sq;
  str[threadIdx.x] = tr;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) {
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + k]);
      ssq[threadIdx.x] += ssq[threadIdx.x + k];
      str[threadIdx.x] += str[threadIdx.x + k];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sc->ginf = smax[0];
    sc->g_sq = ssq[0];  // |g|^2
    sc->htrace = str[0];
  }
}

// ------------------------------------------------------------------- PCG
constexpr int kPcgThreads = 256;
constexpr int kPcgWarps = kPcgThreads / 32;

struct PcgArgs {
  const int* row_ptr;
  const int* col;
  const float* val;
  const int* diag_pos;
  const double* g;
  const double* mu_ptr;  // LM damping lives on the device (graph-replay safe)
  int N;
  int max_iters;
  double tol2;
  double* x;
  double* r;
  double* z;
  double* p0;
  double* p1;
  double* q;
  double* minv;
  double* part;
  DevScalars* sc;
};

// 6x6 SPD inverse by Cholesky (row-major, in place into out)
__device__ void spd_inverse6(const double* a, double* out) {
  double L[6][6];
  bool ok = true;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = a[i * 6 + j];
      for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
      if (i == j) {
        if (!(s > 0.0)) {
          ok = false;
          s = 1.0;
        }
        L[i][i] = sqrt(s);
      } else {
        L[i][j] = s / L[j][j];
      }
    }
  if (!ok) {  // not SPD in fp32-rounded form: fall back to the inverse diagonal
    for (int i = 0; i < 36; ++i) out[i] = 0.0;
    for (int i = 0; i < 6; ++i) out[i * 6 + i] = a[i * 6 + i] > 0 ? 1.0 / a[i * 6 + i] : 0.0;
    return;
  }
  double Li[6][6];  // inverse of L (lower)
  for (int i = 0; i < 6; ++i) {
    for (int j = 0; j < 6; ++j) Li[i][j] = 0.0;
    Li[i][i] = 1.0 / L[i][i];
    for (int j = 0; j < i; ++j) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s -= L[i][k] * Li[k][j];
      Li[i][j] = s / L[i][i];
    }
  }
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      double s = 0.0;
      for (int k = max(i, j); k < 6; ++k) s += Li[k][i] * Li[k][j];
      out[i * 6 + j] = s;
    }
}

__device__ __forceinline__ double block_sum_fixed(double v, double* sh) {
  // warp then block sum in a fixed order; result valid in all threads
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int wid = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kPcgWarps; ++w) t += sh[w];
  return t;
}

__device__ __forceinline__ double grid_total(const double* part, int stride, int off, double* sh) {
  // every block sums the per-block partials in the same order
  double v = 0.0;
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) v += part[b * stride + off];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kPcgWarps; ++w) t += sh[w];
  return t;
}

__global__ void __launch_bounds__(kPcgThreads) k_pcg(PcgArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[kPcgWarps];
  __shared__ double hb[kPcgWarps][36];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kPcgWarps + wid, nw = gridDim.x * kPcgWarps;
  const int N = a.N;
  const double mu = *a.mu_ptr;
  // phase 0: block-Jacobi inverse, r = -g, x = 0, z = M^-1 r, p_old = 0
  double prz = 0.0, prr = 0.0;
  for (int j = gw; j < N; j += nw) {
    const int d = a.diag_pos[j];
    for (int t = lane; t < 36; t += 32) {
      double v = d >= 0 ? (double)a.val[(size_t)d * 36 + t] : 0.0;
      if (t % 7 == 0) v += mu;
      hb[wid][t] = v;
    }
    __syncwarp();
    if (lane == 0) spd_inverse6(hb[wid], a.minv + (size_t)36 * j);
    __syncwarp();
    double rv = 0.0;
    if (lane < 6) {
      rv = -a.g[6 * j + lane];
      a.r[6 * j + lane] = rv;
      a.x[6 * j + lane] = 0.0;
      a.p0[6 * j + lane] = 0.0;
    }
    double zv = 0.0;
    for (int k = 0; k < 6; ++k) {
      const double rk = __shfl_sync(0xffffffffu, rv, k);
      if (lane < 6) zv += a.minv[(size_t)36 * j + lane * 6 + k] * rk;
    }
    if (lane < 6) a.z[6 * j + lane] = zv;
    double t1 = lane < 6 ? rv * zv : 0.0, t2 = lane < 6 ? rv * rv : 0.0;
    for (int off = 16; off > 0; off >>= 1) {
      t1 += __shfl_down_sync(0xffffffffu, t1, off);
      t2 += __shfl_down_sync(0xffffffffu, t2, off);
    }
    if (lane == 0) {
      prz += t1;
      prr += t2;
    }
  }
  {
    const double brz = block_sum_fixed(prz, sh);
    const double brr = block_sum_fixed(prr, sh);
    if (threadIdx.x == 0) {
      a.part[blockIdx.x * 4 + 0] = brz;
      a.part[blockIdx.x * 4 + 1] = brr;
    }
  }
  grid.sync();
  double rz = grid_total(a.part, 4, 0, sh);
  const double rr0 = grid_total(a.part, 4, 1, sh);
  double rr = rr0, beta = 0.0;
  double* pold = a.p0;
  double* pnew = a.p1;
  int it = 0;
  const int row6 = lane % 6, blk5 = lane / 6;  // lane -> (block slot, row) of 5 blocks x 6 rows
  for (; it < a.max_iters; ++it) {
    if (rr == 0.0 || (a.tol2 > 0.0 && rr <= a.tol2 * rr0)) break;
    // phase A: q = (H + mu I) p_new, p_new = z + beta p_old computed on the fly
    double ppq = 0.0;
    for (int j = gw; j < N; j += nw) {
      const int b0 = a.row_ptr[j], b1 = a.row_ptr[j + 1];
      double acc = 0.0;
      for (int bb = b0; bb < b1; bb += 5) {
        const int b = bb + blk5;
        if (lane < 30 && b < b1) {
          const int cidx = a.col[b];
          const float* vr = a.val + (size_t)b * 36 + row6 * 6;
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            const double pv = a.z[6 * cidx + k] + beta * pold[6 * cidx + k];
            s += (double)vr[k] * pv;
          }
          acc += s;
        }
      }
      // row total = sum over lanes row6, row6+6, ..., row6+24 (fixed order)
      double tot = 0.0;
#pragma unroll
      for (int k = 0; k < 5; ++k) tot += __shfl_sync(0xffffffffu, acc, (lane % 6) + 6 * k);
      double pq = 0.0;
      if (lane < 6) {
        const double pn = a.z[6 * j + lane] + beta * pold[6 * j + lane];
        const double qv = tot + mu * pn;
        pnew[6 * j + lane] = pn;
        a.q[6 * j + lane] = qv;
        pq = pn * qv;
      }
      for (int off = 16; off > 0; off >>= 1) pq += __shfl_down_sync(0xffffffffu, pq, off);
      if (lane == 0) ppq += pq;
    }
    {
      const double b = block_sum_fixed(ppq, sh);
      if (threadIdx.x == 0) a.part[blockIdx.x * 4 + 2] = b;
    }
    grid.sync();
    const double pqt = grid_total(a.part, 4, 2, sh);
    const double alpha = rz / pqt;
    // phase B: x += alpha p, r -= alpha q, z = M^-1 r
    double prz2 = 0.0, prr2 = 0.0;
    for (int j = gw; j < N; j += nw) {
      double rv = 0.0;
      if (lane < 6) {
        const int i = 6 * j + lane;
        a.x[i] += alpha * pnew[i];
        rv = a.r[i] - alpha * a.q[i];
        a.r[i] = rv;
      }
      double zv = 0.0;
      for (int k = 0; k < 6; ++k) {
        const double rk = __shfl_sync(0xffffffffu, rv, k);
        if (lane < 6) zv += a.minv[(size_t)36 * j + lane * 6 + k] * rk;
      }
      if (lane < 6) a.z[6 * j + lane] = zv;
      double t1 = lane < 6 ? rv * zv : 0.0, t2 = lane < 6 ? rv * rv : 0.0;
      for (int off = 16; off > 0; off >>= 1) {
        t1 += __shfl_down_sync(0xffffffffu, t1, off);
        t2 += __shfl_down_sync(0xffffffffu, t2, off);
      }
      if (lane == 0) {
        prz2 += t1;
        prr2 += t2;
      }
    }
    {
      const double b1 = block_sum_fixed(prz2, sh);
      const double b2 = block_sum_fixed(prr2, sh);
      if (threadIdx.x == 0) {
        a.part[blockIdx.x * 4 + 0] = b1;
        a.part[blockIdx.x * 4 + 1] = b2;
      }
    }
    grid.sync();
    const double rzn = grid_total(a.part, 4, 0, sh);
    rr = grid_total(a.part, 4, 1, sh);
    beta = rzn / rz;
    rz = rzn;
    double* t = pold;
    pold = pnew;
    pnew = t;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.sc->pcg_iters = it;
    a.sc->pcg_rr = rr;
    a.sc->pcg_rr0 = rr0;
  }
}

// Standalone BSR SpMV y = (H + mu I) x, the PCG's SpMV phase as its own kernel
// (warp per block row; lanes = 5 blocks x 6 rows, shuffle row reduction).
// Algorithmic bytes: 144 B per block (fp32 6x6) + 4 B column index + the x
// block (48 B, L1/L2-reused) + row pointers and y (48 B per row).
__global__ void __launch_bounds__(256) k_bsr_spmv(const int* __restrict__ row_ptr,
                                                  const int* __restrict__ col,
                                                  const float* __restrict__ val, int N, double mu,
                                                  const double* __restrict__ x,
                                                  double* __restrict__ y) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= N) return;
  const int row6 = lane % 6, blk5 = lane / 6;
  const int b0 = row_ptr[j], b1 = row_ptr[j + 1];
  double acc = 0.0;
  for (int bb = b0; bb < b1; bb += 5) {
    const int b = bb + blk5;
    if (lane < 30 && b < b1) {
      const int cidx = col[b];
      const float* vr = val + (size_t)b * 36 + row6 * 6;
      const double* xc = x + 6 * cidx;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) s += (double)vr[k] * xc[k];
      acc += s;
    }
  }
  double tot = 0.0;
#pragma unroll
  for (int k = 0; k < 5; ++k) tot += __shfl_sync(0xffffffffu, acc, (lane % 6) + 6 * k);
  if (lane < 6) y[6 * j + lane] = tot + mu * x[6 * j + lane];
}

__global__ void k_check_finite(const double* __restrict__ x, int n, int* __restrict__ finite) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !isfinite(x[i])) atomicAnd(finite, 0);
}

}  // namespace

// ------------------------------------------------------------------ host side
void build_pattern(Ctx& c, int t_now, int t_last) {
  const int n_all = c.n_surfels, N = c.n_nodes;
  if ((long long)N * N >= 0x7fffffffLL) fail(DS_ERR_CAPACITY, "too many nodes for block keys");
  // eligible surfels (the only ones render_model_maps can pair this frame)
  int n = 0;
  if (n_all > 0) {
    DS_CUDA(cudaMemsetAsync(&c.dsc->any_stable, 0, sizeof(int), c.stream));
    DS_LAUNCH(c, KK_PATTERN, 16.0 * n_all, cdiv(n_all, 256), 256, 0, k_any_stable_flag,
              c.M().ln, n_all, c.cfg.delta_stable, &c.dsc->any_stable);
    const int boot = (t_now - t_last <= c.cfg.delta_recent) ? 1 : 0;
    DS_LAUNCH(c, KK_PATTERN, 28.0 * n_all, cdiv(n_all, 256), 256, 0, k_elig_flags, c.M().ln,
              c.M().t, n_all, c.cfg.delta_stable, t_now, c.cfg.delta_recent, boot,
              &c.dsc->any_stable, c.keep);
    scan_exclusive(c, c.keep, c.keep_scan, n_all);
    DS_LAUNCH(c, KK_PATTERN, 12.0 * n_all, cdiv(n_all, 256), 256, 0, k_elig_list, c.keep,
              c.keep_scan, n_all, c.elig);
    DS_CUDA(cudaMemcpyAsync(&n, c.keep_scan + n_all, sizeof(int), cudaMemcpyDeviceToHost,
                            c.stream));
    sync(c);
  }
  c.n_elig = n;
  const int R = n * 10 + N * 24;
  if (R > c.R_cap) fail(DS_ERR_CAPACITY, "term record capacity exceeded");
  int* key = c.rec_key;
  int* val = c.rec_val;
  if (n > 0)
    DS_LAUNCH(c, KK_PATTERN, 60.0 * n, cdiv(n, 256), 256, 0, k_gen_records, c.M().ki, c.elig, n,
              N, key, val);
  if (N > 0)
    DS_LAUNCH(c, KK_PATTERN, 32.0 * 8 * N, cdiv(8 * N, 256), 256, 0, k_gen_reg_records, c.node_nbr,
              N, key + (size_t)n * 10, val + (size_t)n * 10);
  const int end_bit = 31;  // the kIntMax sentinel needs all 31 bits
  int *ks, *vs;
  sort_pairs(c, key, val, c.rec_key2, c.rec_val2, R, end_bit, &ks, &vs);
  // keep the sorted arrays in rec_key/rec_val
  if (ks != c.rec_key) {
    std::swap(c.rec_key, c.rec_key2);
    std::swap(c.rec_val, c.rec_val2);
  }
  DS_LAUNCH(c, KK_PATTERN, 8.0 * R, cdiv(R, 256), 256, 0, k_mark_unique, c.rec_key, R, c.rec_flag);
  scan_exclusive(c, c.rec_flag, c.rec_flag, R);
  DS_CUDA(cudaMemsetAsync(&c.dsc->err, 0, sizeof(int), c.stream));
  DS_LAUNCH(c, KK_PATTERN, 12.0 * R, cdiv(R, 256), 256, 0, k_write_up, c.rec_key, c.rec_flag, R,
            c.up_key, c.up_start, c.UB_cap, &c.dsc->err);
  int* n_up_dev = c.rec_flag + R;
  DS_CUDA(cudaMemsetAsync(c.row_cnt, 0, sizeof(int) * (N + 1), c.stream));
  DS_LAUNCH(c, KK_PATTERN, 4.0 * c.UB_cap, cdiv(c.UB_cap, 256), 256, 0, k_row_count, c.up_key,
            n_up_dev, N, c.row_cnt);
  scan_exclusive(c, c.row_cnt, c.row_ptr, N);
  DS_CUDA(cudaMemsetAsync(c.row_cnt, 0, sizeof(int) * (N + 1), c.stream));
  int host[3] = {0, 0, 0};
  DS_CUDA(cudaMemcpyAsync(&host[0], n_up_dev, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(&host[1], c.row_ptr + N, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(&host[2], &c.dsc->err, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  sync(c);
  if ((host[2] & DERR_BLOCK_CAP) || host[0] > c.UB_cap || host[1] > c.B_cap)
    fail(DS_ERR_CAPACITY, "JtJ block capacity exceeded");
  c.n_up = host[0];
  c.n_full = host[1];
  c.n_records = R;
  if (c.n_up > 0) {
    DS_LAUNCH(c, KK_PATTERN, 16.0 * c.n_up, cdiv(c.n_up, 256), 256, 0, k_row_fill, c.up_key,
              n_up_dev, N, c.row_ptr, c.row_cnt, c.bsr_col, c.bsr_tag);
  }
  DS_LAUNCH(c, KK_PATTERN, 16.0 * c.n_full, cdiv(N, 128), 128, 0, k_row_sort, c.row_ptr, N,
            c.bsr_col, c.bsr_tag, c.up_pos, c.up_mpos, c.diag_pos);
  if (c.n_pairs_ok_est <= 0) c.n_pairs_ok_est = 0.4 * c.P;
  // fixed-size record chunks for the assembly (per frame)
  c.n_chunks = 0;
  if (c.n_up > 0) {
    DS_LAUNCH(c, KK_PATTERN, 12.0 * c.n_up, cdiv(c.n_up, 256), 256, 0, k_chunk_count, c.up_start,
              c.n_up, c.chunk_first);
    scan_exclusive(c, c.chunk_first, c.chunk_first, c.n_up);
    DS_CUDA(cudaMemcpyAsync(&c.n_chunks, c.chunk_first + c.n_up, sizeof(int),
                            cudaMemcpyDeviceToHost, c.stream));
    sync(c);
    if (c.n_chunks > c.CH_cap) fail(DS_ERR_CAPACITY, "assembly chunk capacity exceeded");
    DS_LAUNCH(c, KK_PATTERN, 8.0 * c.n_chunks, cdiv(c.n_up, 256), 256, 0, k_chunk_fill,
              c.chunk_first, c.n_up, c.chunk_ub);
  }
  c.pattern_ready = true;
}

namespace {
PairParams pair_params(Ctx& c, const double* pose) {
  PairParams pp;
  pp.pose = rig_load(pose);
  pp.P = c.P;
  return pp;
}
}  // namespace

// One GN linearisation at the current nodes (solver.cpp:316-369). Leaves e_data,
// e_reg, ginf, |g|^2 (in pcg_rr slot) and tr(H) in DevScalars (no host sync).
void gn_linearize_async(Ctx& c, const double* pose, int t_now, int t_last) {
  const int n = c.n_surfels, N = c.n_nodes, P = c.P;
  // only render-eligible surfels can be drawn / paired during the solve; the
  // post-solve forward_warp (pipeline.cpp:108) rewrites every live surfel
  forward_warp_list(c, c.elig, c.n_elig);
  render_model_maps_list(c, pose, t_now, t_last, pose, c.elig, c.n_elig);
  DS_CUDA(cudaMemsetAsync(c.s_cnt, 0, sizeof(int) * (n + 1), c.stream));
  DS_CUDA(cudaMemsetAsync(c.pair_ok, 0, P, c.stream));
  const int nbp = cdiv(P, 256);
  // per pixel: pair id 4 B, surfel ref + skin 48 B, frame maps 64 B, rows 96 B + r 8 B out
  DS_LAUNCH(c, KK_PAIR_TERMS, 220.0 * P, nbp, 256, 0, k_pair_terms, c.pair_s, c.M(), c.node_dq,
            c.f_vert, c.f_nrm, pair_params(c, pose), c.pair_ok, c.pair_rows, c.pair_r, c.s_cnt,
            c.red_part, c.tickets + 0, &c.dsc->e_data_pre);
  scan_exclusive(c, c.s_cnt, c.s_off, n);
  DS_CUDA(cudaMemsetAsync(c.s_cur, 0, sizeof(int) * n, c.stream));
  DS_LAUNCH(c, KK_PAIR_LISTS, 13.0 * P, nbp, 256, 0, k_scatter_pairs, c.pair_s, c.pair_ok, P,
            c.s_off, c.s_cur, c.s_list);
  DS_LAUNCH(c, KK_PAIR_LISTS, 112.0 * P * 0.5, cdiv(n, 256), 256, 0, k_sort_lists, c.s_cnt,
            c.s_off, n, c.s_list, c.pair_rows, c.pair_r, c.rows_l, c.r_l);
  node_se3(c, c.node_dq, c.node_se3);
  const int nbe = cdiv(8 * N, 256);
  DS_LAUNCH(c, KK_ENERGY, 200.0 * N, nbe, 256, 0, k_reg_energy, c.node_pos, c.node_nbr,
            c.node_se3, N, c.red_part + nbp, c.tickets + 1, &c.dsc->e_reg_pre);
  DS_CUDA(cudaMemsetAsync(c.g, 0, sizeof(double) * 6 * N, c.stream));
  AsmArgs A;
  A.up_key = c.up_key;
  A.up_start = c.up_start;
  A.up_pos = c.up_pos;
  A.up_mpos = c.up_mpos;
  A.chunk_ub = c.chunk_ub;
  A.chunk_first = c.chunk_first;
  A.rec_val = c.rec_val;
  A.s_cnt = c.s_cnt;
  A.s_off = c.s_off;
  A.rows_l = c.rows_l;
  A.r_l = c.r_l;
  A.node_pos = c.node_pos;
  A.nbr = c.node_nbr;
  A.se3 = c.node_se3;
  A.lambda = c.cfg.lambda;
  A.N = N;
  A.n_up = c.n_up;
  A.n_chunks = c.n_chunks;
  A.part_h = c.part_h;
  A.part_g = c.part_g;
  A.part_t = c.part_t;
  A.bsr_val = c.bsr_val;
  A.bsr_touch = c.bsr_touch;
  A.g = c.g;
  if (c.n_up > 0) {
    // algorithmic bytes: records 4 B + (count, offset) 8 B each, the paired
    // surfels' list-ordered rows/residuals (104 B) once, chunk partials out+in,
    // blocks written 144 B (both triangles) + g
    const double bytes = 12.0 * c.n_records + 104.0 * c.n_pairs_ok_est + 200.0 * 2 * c.n_chunks +
                         144.0 * c.n_full + 48.0 * N;
    DS_LAUNCH(c, KK_BLOCK_ASSEMBLY, bytes, cdiv((long long)c.n_chunks * kChunkLanes, 256), 256, 0,
              k_assemble_chunks, A);
    DS_LAUNCH(c, KK_BLOCK_ASSEMBLY, 0.0, cdiv(c.n_up, 128), 128, 0, k_assemble_finish, A);
  }
  DS_LAUNCH(c, KK_REDUCE, 48.0 * N, 1, 256, 0, k_g_stats, c.g, 6 * N, c.bsr_val, c.diag_pos, N,
            c.dsc);
}

void gn_linearize(Ctx& c, const double* pose, int t_now, int t_last, double* e_pre, int* n_pairs) {
  if (!c.pattern_ready) build_pattern(c, t_now, t_last);
  gn_linearize_async(c, pose, t_now, t_last);
  fetch_scalars(c);
  if (e_pre) *e_pre = c.hsc->e_data_pre + c.cfg.lambda * c.hsc->e_reg_pre;
  if (n_pairs) *n_pairs = c.hsc->n_pairs;
}

// PCG on the last assembled system with the damping in dsc->mu
void pcg_solve_async(Ctx& c, int max_iters, double tol) {
  const int N = c.n_nodes;
  PcgArgs a;
  a.row_ptr = c.row_ptr;
  a.col = c.bsr_col;
  a.val = c.bsr_val;
  a.diag_pos = c.diag_pos;
  a.g = c.g;
  a.mu_ptr = &c.dsc->mu;
  a.N = N;
  a.max_iters = max_iters;
  a.tol2 = tol > 0 ? tol * tol : 0.0;
  a.x = c.pcg_x;
  a.r = c.pcg_r;
  a.z = c.pcg_z;
  a.p0 = c.pcg_p0;
  a.p1 = c.pcg_p1;
  a.q = c.pcg_q;
  a.minv = c.pcg_minv;
  a.part = c.pcg_part;
  a.sc = c.dsc;
  const int need = std::max(1, cdiv(N, kPcgWarps));
  const int grid = std::min(c.pcg_grid, need);
  void* args[] = {&a};
  launch_begin(c, KK_PCG);
  DS_CUDA(cudaLaunchCooperativeKernel((void*)k_pcg, dim3(grid), dim3(kPcgThreads), args, 0,
                                      c.stream));
  // algorithmic bytes per PCG: per iteration one BSR SpMV (148 B/block + vectors)
  launch_end(c, KK_PCG, std::max(1, max_iters) * (148.0 * c.n_full + 6.0 * 8 * 8 * N));
  DS_CUDA(cudaMemsetAsync(&c.dsc->finite, 0xff, sizeof(int), c.stream));
  DS_LAUNCH(c, KK_MISC, 48.0 * N, cdiv(6 * N, 256), 256, 0, k_check_finite, c.pcg_x, 6 * N,
            &c.dsc->finite);
}

void pcg_solve(Ctx& c, double mu, int max_iters, double tol, int* iters, double* rel_res) {
  *c.h_mu = mu;
  DS_CUDA(cudaMemcpyAsync(&c.dsc->mu, c.h_mu, sizeof(double), cudaMemcpyHostToDevice, c.stream));
  pcg_solve_async(c, max_iters, tol);
  if (iters || rel_res) {
    fetch_scalars(c);
    if (iters) *iters = c.hsc->pcg_iters;
    if (rel_res) *rel_res = c.hsc->pcg_rr0 > 0 ? std::sqrt(c.hsc->pcg_rr / c.hsc->pcg_rr0) : 0.0;
  }
}

namespace {
// total energy of the pair set at node transforms `dq` (se3 cache in `se3`)
void energy_async(Ctx& c, const double* pose, const double4* dq, double* se3) {
  const int N = c.n_nodes, P = c.P;
  const int nbp = cdiv(P, 256), nbe = cdiv(8 * N, 256);
  DS_LAUNCH(c, KK_ENERGY, 120.0 * P * 0.5, nbp, 256, 0, k_pair_energy, c.pair_s, c.M(), dq,
            c.f_vert, c.f_nrm, pair_params(c, pose), 0, c.red_part, (int*)nullptr, c.tickets + 0,
            &c.dsc->e_data);
  node_se3(c, dq, se3);
  DS_LAUNCH(c, KK_ENERGY, 200.0 * N, nbe, 256, 0, k_reg_energy, c.node_pos, c.node_nbr, se3, N,
            c.red_part + nbp, c.tickets + 1, &c.dsc->e_reg);
}
}  // namespace

namespace {
__global__ void k_lm_prep(DevScalars* sc, int dim) {
  // mu_floor = 1e-6 tr(H) / dim; mu = max(mu, mu_floor)   (solver.cpp:378-379)
  const double floor_ = 1e-6 * sc->htrace / dim;
  sc->mu_floor = floor_;
  sc->mu = fmax(sc->mu, floor_);
}

// one GN iteration up to the first LM attempt: linearise, mu, PCG, candidate, E_post
void gn_step_async(Ctx& c, const double* pose, int t_now, int t_last, int max_pcg, double tol) {
  gn_linearize_async(c, pose, t_now, t_last);
  DS_LAUNCH(c, KK_MISC, 32.0, 1, 1, 0, k_lm_prep, c.dsc, 6 * c.n_nodes);
  pcg_solve_async(c, max_pcg, tol);
  apply_increments(c, c.pcg_x, c.node_dq_cand);
  energy_async(c, pose, c.node_dq_cand, c.node_se3_cand);
}
void attempt_async(Ctx& c, const double* pose, int max_pcg, double tol) {
  pcg_solve_async(c, max_pcg, tol);
  apply_increments(c, c.pcg_x, c.node_dq_cand);
  energy_async(c, pose, c.node_dq_cand, c.node_se3_cand);
}

// Capture `enqueue` into `slot` (update the executable graph in place when the
// topology is unchanged; re-instantiate otherwise). Returns false if the stream
// cannot be captured (the caller then launches directly).
template <class F>
bool capture(Ctx& c, GraphSlot& slot, F&& enqueue) {
  cudaGraph_t graph = nullptr;
  const int64_t l0 = c.total_launches;
  if (cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  try {
    enqueue();
  } catch (...) {
    cudaStreamEndCapture(c.stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    c.total_launches = l0;
    throw;
  }
  if (cudaStreamEndCapture(c.stream, &graph) != cudaSuccess || !graph) {
    cudaGetLastError();
    c.total_launches = l0;
    return false;
  }
  slot.kernels = c.total_launches - l0;
  c.total_launches = l0;
  if (slot.exec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(slot.exec, graph, &info) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphExecDestroy(slot.exec);
      slot.exec = nullptr;
    }
  }
  if (!slot.exec && cudaGraphInstantiate(&slot.exec, graph, 0) != cudaSuccess) {
    cudaGetLastError();
    slot.exec = nullptr;
    cudaGraphDestroy(graph);
    return false;
  }
  cudaGraphDestroy(graph);
  return true;
}
void replay(Ctx& c, GraphSlot& slot) {
  DS_CUDA(cudaGraphLaunch(slot.exec, c.stream));
  c.total_launches += slot.kernels;
}
void set_mu(Ctx& c, double mu) {
  *c.h_mu = mu;
  DS_CUDA(cudaMemcpyAsync(&c.dsc->mu, c.h_mu, sizeof(double), cudaMemcpyHostToDevice, c.stream));
}
}  // namespace

// solve_nonrigid (solver.cpp:296-422). Each GN iteration is one replay of a
// captured graph (linearise + mu floor + PCG + increments + E_post) and one
// host sync for the LM decision; rejected attempts replay the attempt graph.
// The damping mu is kept on the device and mirrored on the host with the same
// arithmetic, so decisions are those of the reference loop.
void solve_nonrigid(Ctx& c, const double* pose, int t_now, int t_last, ds_solver_report* out) {
  ds_solver_report rep{};
  const int N = c.n_nodes, n = c.n_surfels;
  c.lm_attempts = 0;
  c.pcg_iterations = 0;
  if (N == 0 || n == 0) {
    *out = rep;
    return;
  }
  build_pattern(c, t_now, t_last);
  const int max_pcg = c.cfg.pcg_max_iters > 0 ? c.cfg.pcg_max_iters : 10;
  const double tol = c.cfg.pcg_tol;
  const bool graphs = c.use_graphs && !c.cfg.profile;
  bool have_step = false, have_attempt = false;
  double mu = 0.0;
  set_mu(c, 0.0);
  int n_pairs = 0;
  for (int iter = 0; iter < c.cfg.max_gn_iters; ++iter) {
    if (graphs && !have_step)
      have_step = capture(c, c.g_step, [&] { gn_step_async(c, pose, t_now, t_last, max_pcg, tol); });
    if (have_step) replay(c, c.g_step);
    else gn_step_async(c, pose, t_now, t_last, max_pcg, tol);
    fetch_scalars(c);
    const double e_pre = c.hsc->e_data_pre + c.cfg.lambda * c.hsc->e_reg_pre;
    n_pairs = c.hsc->n_pairs;
    c.n_pairs_ok_est = n_pairs;
    if (iter == 0) {
      rep.initial_energy = e_pre;
      rep.final_energy = e_pre;
    }
    if (c.hsc->ginf < 1e-14) break;  // stationary: the speculative attempt is discarded
    const double gnorm = std::sqrt(c.hsc->g_sq);
    const double mu_floor = c.hsc->mu_floor;
    mu = std::max(mu, mu_floor);  // == c.hsc->mu (same arithmetic on the device)
    bool accepted = false;
    double e_post = e_pre;
    for (int attempt = 0; attempt < 8 && !accepted; ++attempt) {
      if (attempt > 0) {
        set_mu(c, mu);
        if (graphs && !have_attempt)
          have_attempt = capture(c, c.g_attempt, [&] { attempt_async(c, pose, max_pcg, tol); });
        if (have_attempt) replay(c, c.g_attempt);
        else attempt_async(c, pose, max_pcg, tol);
        fetch_scalars(c);
      }
      ++c.lm_attempts;
      c.pcg_iterations += c.hsc->pcg_iters;
      const bool finite = c.hsc->finite != 0;
      // residual guard (solver.cpp:387-388) when PCG runs to a tolerance
      const bool guard_fail = tol > 0 && std::sqrt(c.hsc->pcg_rr) > 1e-6 * (gnorm + 1.0) &&
                              std::sqrt(c.hsc->pcg_rr) > tol * std::sqrt(c.hsc->pcg_rr0);
      if (!finite || guard_fail) {
        mu = std::max(mu_floor, mu * 10.0);
        continue;
      }
      e_post = c.hsc->e_data + c.cfg.lambda * c.hsc->e_reg;
      if (e_post <= e_pre) accepted = true;
      else mu = std::max(mu_floor, mu * 10.0);
    }
    if (!accepted) break;
    mu = std::max(mu_floor, mu * 0.1);
    set_mu(c, mu);
    DS_CUDA(cudaMemcpyAsync(c.node_dq, c.node_dq_cand, sizeof(double4) * 2 * N,
                            cudaMemcpyDeviceToDevice, c.stream));
    ++rep.iterations;
    rep.final_energy = e_post;
    if (e_pre - e_post < 1e-4 * std::max(e_pre, 1e-300)) break;
  }
  rep.correspondences = n_pairs;
  // mean |r| at the final nodes over the last pair set (solver.cpp:409-420)
  const int nbp = cdiv(c.P, 256);
  DS_CUDA(cudaMemsetAsync(&c.dsc->mean_cnt, 0, sizeof(int), c.stream));
  DS_LAUNCH(c, KK_ENERGY, 120.0 * c.P * 0.5, nbp, 256, 0, k_pair_energy, c.pair_s, c.M(), c.node_dq,
            c.f_vert, c.f_nrm, pair_params(c, pose), 1, c.red_part, &c.dsc->mean_cnt,
            c.tickets + 0, &c.dsc->mean_abs_r);
  fetch_scalars(c);
  rep.mean_residual = c.hsc->mean_cnt > 0 ? c.hsc->mean_abs_r / c.hsc->mean_cnt : 0.0;
  *out = rep;
}

// y = (H + mu I) x on the assembled BSR system, `reps` times; returns mean ms
double bsr_spmv(Ctx& c, const double* x_dev, double* y_dev, double mu, int reps) {
  const int N = c.n_nodes;
  cudaEvent_t a, b;
  DS_CUDA(cudaEventCreate(&a));
  DS_CUDA(cudaEventCreate(&b));
  const double bytes = 148.0 * c.n_full + 56.0 * N;
  DS_CUDA(cudaEventRecord(a, c.stream));
  for (int r = 0; r < reps; ++r)
    DS_LAUNCH(c, KK_PCG, bytes, cdiv((long long)N * 32, 256), 256, 0, k_bsr_spmv, c.row_ptr,
              c.bsr_col, c.bsr_val, N, mu, x_dev, y_dev);
  DS_CUDA(cudaEventRecord(b, c.stream));
  sync(c);
  float ms = 0;
  DS_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return reps > 0 ? ms / reps : 0.0;
}

int pcg_max_grid(int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg, kPcgThreads, 0);
  return std::max(1, per_sm) * num_sms;
}

}  // namespace ds
