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
#include <chrono>
#include <cstdio>

#include "ds_assoc.cuh"
#include "ds_blend.cuh"
#include "ds_context.cuh"
#include "ds_pcg.cuh"
#include "ds_reduce.cuh"

namespace cg = cooperative_groups;

namespace ds {

size_t sort_temp_bytes(int n);

namespace {


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

// CTA-local compaction of the pixels that carry a correspondence: the CTA's
// ~40 % valid pixels are packed to the low threads, so whole warps retire
// early instead of idling through the fp64 blend with inactive lanes. Returns
// this thread's pixel (or -1) in the packed order (pixel order preserved).
__device__ __forceinline__ int pack_pairs(const int* __restrict__ pair_s, int P, int* s_list,
                                          int* s_wcnt, int& s_out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const bool v = c < P && pair_s[c] >= 0;
  const unsigned bal = __ballot_sync(0xffffffffu, v);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s_wcnt[wid] = __popc(bal);
  __syncthreads();
  int off = 0;
  for (int w = 0; w < wid; ++w) off += s_wcnt[w];
  if (v) s_list[off + __popc(bal & ((1u << lane) - 1u))] = c;
  __syncthreads();
  int tot = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += s_wcnt[w];
  s_out = tot;
  return threadIdx.x < tot ? s_list[threadIdx.x] : -1;
}

// Per correspondence (pixel c, surfel s): residual, Jacobian rows (fp32),
// pair list bookkeeping; returns the data energy term r^2 (0 if degenerate).
__device__ __forceinline__ double pair_term_one(int c, int s, const ModelBuf& m,
                                                const double4* __restrict__ node_dq,
                                                const double4* __restrict__ fvert,
                                                const double4* __restrict__ fnrm,
                                                const PairParams& pp, uint8_t* __restrict__ pair_ok,
                                                float* __restrict__ rows,
                                                double* __restrict__ pair_r,
                                                int* __restrict__ s_cnt,
                                                int* __restrict__ s_head) {
  double e = 0.0;
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
      const Q4 ndq = qsub(qdiv(bd, a), qscl(ddiv(rd, a * a * a), br));
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
      const Q4 u_r2 = qadd(qscl(-1.0 / a3, t1), qscl(ddiv(3.0 * rd, a5) * brbe, br));
      const Q4 ur = qadd(u_r1, u_r2);
      // dnd/dbd be = be/a - br (br.be)/a^3
      const Q4 ud = qsub(qdiv(beq, a), qscl(ddiv(brbe, a3), br));
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
      atomicAdd(s_cnt + s, 1);  // per-surfel pair count and first (lowest) pixel
      atomicMin(s_head + s, c);
    }
  }
  return e;
}

// Fused model-map resolve + association (raster.cpp:104-119, solver.cpp:244-271)
// + per-pair terms: the pixel's winner and correspondence are decided in
// registers, the CTA packs its paired pixels and evaluates their terms.
#ifndef DS_PAIR_PIX
#define DS_PAIR_PIX 1
#endif
constexpr int kPairPix = DS_PAIR_PIX;  // pixels per thread in k_assoc_pair_terms (measured: 1 > 2, 4 -- spills)
#ifndef DS_PAIR_TERMS_MINB
#define DS_PAIR_TERMS_MINB 3
#endif
__global__ void __launch_bounds__(256, DS_PAIR_TERMS_MINB) k_assoc_pair_terms(
    int* __restrict__ pidx, int* __restrict__ sidx, unsigned long long* __restrict__ pkey,
    unsigned long long* __restrict__ skey, const uint8_t* __restrict__ fflag,
    ModelBuf m, const double4* __restrict__ node_dq, const double4* __restrict__ fvert,
    const double4* __restrict__ fnrm, PairParams pp, int* __restrict__ mm_idx,
    int* __restrict__ pair_s, int* __restrict__ n_pairs, uint8_t* __restrict__ pair_ok,
    float* __restrict__ rows, double* __restrict__ pair_r, int* __restrict__ s_cnt,
    int* __restrict__ s_head, double* __restrict__ part, unsigned* __restrict__ ticket,
    double* __restrict__ out) {
  pdl_wait();  // programmatic dependent launch: predecessor results visible
  // kPairPix pixels per thread: the CTA resolves 256 x kPairPix pixels and
  // packs their pairs (~40 %) so that all its warps run pair terms
  __shared__ int s_pix[256 * kPairPix], s_srf[256 * kPairPix];
  __shared__ int s_wcnt[8 * kPairPix];
  __shared__ unsigned s_done;
  __shared__ double s_wsum[8];
  if (threadIdx.x == 0) s_done = 0u;  // visible after the packing barriers below
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tot = 0;
#pragma unroll
  for (int q = 0; q < kPairPix; ++q) {
    const int c = (blockIdx.x * kPairPix + q) * 256 + threadIdx.x;
    int ps = -1;
    if (c < pp.P) {
      // resolve (raster.cpp:104-119), then reset the consumed z-buffer entries
      // so the next GN iteration's splats start from empty maps without memsets
      const int pw = pidx[c], sw = sidx[c];
      const int win = pw != kEmptyIdx ? pw : (sw != kEmptyIdx ? sw : -1);
      if (pw != kEmptyIdx) {
        pidx[c] = kEmptyIdx;
        pkey[c] = ~0ull;
      }
      if (sw != kEmptyIdx) {
        sidx[c] = kEmptyIdx;
        skey[c] = ~0ull;
      }
      mm_idx[c] = win;
      ps = associate_pixel(c, win, m, fvert, fnrm, fflag, pp.pose);
      pair_s[c] = ps;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, ps >= 0);
    if (lane == 0) {
      s_wcnt[q * 8 + wid] = __popc(bal);
      if (bal) atomicAdd(n_pairs, __popc(bal));
    }
    __syncthreads();
    int off = tot;
    for (int w = 0; w < wid; ++w) off += s_wcnt[q * 8 + w];
    if (ps >= 0) {
      const int k = off + __popc(bal & ((1u << lane) - 1u));
      s_pix[k] = c;
      s_srf[k] = ps;
    }
    for (int w = 0; w < 8; ++w) tot += s_wcnt[q * 8 + w];
  }
  __syncthreads();
  double e = 0.0;
  if (kPairPix == 1) {
    const int pc = threadIdx.x < tot ? s_pix[threadIdx.x] : -1;
    const int sc = threadIdx.x < tot ? s_srf[threadIdx.x] : -1;
    e = pair_term_one(pc, sc, m, node_dq, fvert, fnrm, pp, pair_ok, rows, pair_r, s_cnt, s_head);
  } else {
    for (int k = threadIdx.x; k < tot; k += 256)
      e += pair_term_one(s_pix[k], s_srf[k], m, node_dq, fvert, fnrm, pp, pair_ok, rows, pair_r,
                         s_cnt, s_head);
  }
  // data energy, fixed order; warps past the packed pairs finish at once
  grid_sum_warps<256>(e, &s_done, s_wsum, part, ticket, out, blockIdx.x, gridDim.x);
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
  __shared__ int s_list[256];
  __shared__ int s_wcnt[8];
  int n_valid;
  const int c = pack_pairs(pair_s, pp.P, s_list, s_wcnt, n_valid);
  double e = 0.0;
  int ok = 0;
  const int s = c >= 0 ? pair_s[c] : -1;
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
                                                    double* __restrict__ out,
                                                    double* __restrict__ ab_out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (e < 8 * N) {
    const int i = nbr[e];
    if (i >= 0) {
      const int j = e >> 3;
      const double4 pj = pos[j];
      const V3 p = v3(pj.x, pj.y, pj.z);
      const Rig Tj = rig_load(se3 + 12 * j), Ti = rig_load(se3 + 12 * i);
      const V3 a = rig_apply(Tj, p), b = rig_apply(Ti, p);
      v = sqn(sub(a, b));
      if (ab_out) {  // linearisation: T_j p_j and T_i p_j for the Jacobians
        double2* o = reinterpret_cast<double2*>(ab_out + 6 * (size_t)e);
        o[0] = make_double2(a.x, a.y);
        o[1] = make_double2(a.z, b.x);
        o[2] = make_double2(b.y, b.z);
      }
    }
  }
  grid_sum<256>(v, part, ticket, out);
}

#ifndef DS_ENERGY_PIX
#define DS_ENERGY_PIX 2
#endif
constexpr int kEnergyPix = DS_ENERGY_PIX;  // pixels per thread in k_energy (measured: 2 > 1, 4)

// E_post of an LM attempt in one launch: blocks [0, nbp) evaluate E_data over
// the pair set (solver.cpp:132-143), blocks [nbp, nbp + nbe) E_reg over the
// directed edges (solver.cpp:145-155); two independent fixed-order sums.
__global__ void __launch_bounds__(256) k_energy(const int* __restrict__ pair_s, ModelBuf m,
                                                const double4* __restrict__ node_dq,
                                                const double4* __restrict__ fvert,
                                                const double4* __restrict__ fnrm, PairParams pp,
                                                const double4* __restrict__ pos,
                                                const int* __restrict__ nbr,
                                                const double* __restrict__ se3, int N, int nbp,
                                                double* __restrict__ part,
                                                unsigned* __restrict__ tickets,
                                                double* __restrict__ e_data,
                                                double* __restrict__ e_reg) {
  pdl_wait();  // programmatic dependent launch: predecessor results visible
  __shared__ unsigned s_done;
  __shared__ double s_wsum[8];
  if (threadIdx.x == 0) s_done = 0u;  // visible after the next barrier
  if ((int)blockIdx.x < nbp) {
    // kEnergyPix pixels per thread: the CTA packs its ~40 % paired pixels of
    // 256 x kEnergyPix into a list that keeps all its warps busy
    __shared__ int s_list[256 * kEnergyPix];
    __shared__ int s_wcnt[8 * kEnergyPix];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int tot = 0;
#pragma unroll
    for (int q = 0; q < kEnergyPix; ++q) {
      const int c = (blockIdx.x * kEnergyPix + q) * 256 + threadIdx.x;
      const bool v = c < pp.P && pair_s[c] >= 0;
      const unsigned bal = __ballot_sync(0xffffffffu, v);
      if (lane == 0) s_wcnt[q * 8 + wid] = __popc(bal);
      __syncthreads();
      int off = tot;
      for (int w = 0; w < wid; ++w) off += s_wcnt[q * 8 + w];
      if (v) s_list[off + __popc(bal & ((1u << lane) - 1u))] = c;
      for (int w = 0; w < 8; ++w) tot += s_wcnt[q * 8 + w];
    }
    __syncthreads();
    double e = 0.0;
    for (int k = threadIdx.x; k < tot; k += 256) {  // pixel order within the thread
      const int c = s_list[k];
      const int s = pair_s[c];
      const Blend b = blend_entry(m.ki[s], m.kw[s], node_dq);
      if (!b.degenerate) {
        const float4 rp = m.rp[s];
        const double4 fv = fvert[c], fn = fnrm[c];
        const V3 vd = rig_apply(pp.pose, v3(fv.x, fv.y, fv.z));
        const V3 nd = rig_rotate(pp.pose, v3(fn.x, fn.y, fn.z));
        const V3 y = rig_apply(blend_rig_fast(b), v3(rp.x, rp.y, rp.z));
        const double r = dot(nd, sub(y, vd));
        e += r * r;
      }
    }
    grid_sum_warps<256>(e, &s_done, s_wsum, part, tickets + 0, e_data, blockIdx.x, nbp);
  } else {
    __syncthreads();
    const int bid = blockIdx.x - nbp, nbe = gridDim.x - nbp;
    const int e = bid * blockDim.x + threadIdx.x;
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
    grid_sum_warps<256>(v, &s_done, s_wsum, part + nbp, tickets + 1, e_reg, bid, nbe);
  }
}

__global__ void k_any_stable_flag(const float4* __restrict__ ln, int n, double delta_stable,
                                  int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool st = i < n && (double)ln[i].w > delta_stable;
  const unsigned b = __ballot_sync(0xffffffffu, st);
  if ((threadIdx.x & 31) == 0 && b) atomicOr(flag, 1);
}

// ---------------------------------------------------------------- pair lists
// A surfel's correspondence pairs in pixel order (the summation order of the
// assembly) as a chain over the per-pixel rows: s_head[s] = lowest pixel
// (atomicMin in k_pair_terms), p_next[pixel] = next pixel of the same surfel.
// Most surfels own one pair (no chain). For the others: a segment of cnt
// slots is reserved and every pixel of the surfel drops itself into it in
// arrival order (k_pair_fill), and each pixel scans its segment -- independent
// loads, no pointer chasing -- for its successor in pixel order (k_pair_next).
// Slot order is not observable.
// Reservation and fill in one pass: the first of a surfel's pixels to arrive
// claims its segment (CAS on s_base, -1 -> -2), reserves cnt slots and
// publishes the base; the others wait only for that thread, which is already
// running. Every pixel then drops itself into the segment (arrival order).
__global__ void k_pair_fill(const int* __restrict__ pair_s, const uint8_t* __restrict__ pair_ok,
                            int P, const int* __restrict__ s_cnt, int* __restrict__ s_base,
                            int* __restrict__ s_fill, int* __restrict__ p_list,
                            int* __restrict__ counter) {
  pdl_wait();  // programmatic dependent launch: predecessor results visible
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P || !pair_ok[c]) return;
  const int s = pair_s[c];
  const int cnt = s_cnt[s];
  if (cnt < 2) return;
  int b = atomicCAS(s_base + s, -1, -2);
  if (b == -1) {
    b = atomicAdd(counter, cnt);
    atomicExch(s_base + s, b);
  } else {
    while (b < 0) b = *(volatile int*)(s_base + s);
  }
  p_list[b + atomicAdd(s_fill + s, 1)] = c;
}
__global__ void k_pair_next(const int* __restrict__ pair_s, const uint8_t* __restrict__ pair_ok,
                            int P, const int* __restrict__ s_cnt, const int* __restrict__ s_base,
                            const int* __restrict__ p_list, int* __restrict__ p_next) {
  pdl_wait();  // programmatic dependent launch: predecessor results visible
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P || !pair_ok[c]) return;
  const int s = pair_s[c];
  const int cnt = s_cnt[s];
  if (cnt < 2) return;
  const int* seg = p_list + s_base[s];
  int nxt = 0x7fffffff;
#pragma unroll 8
  for (int k = 0; k < cnt; ++k) {
    const int q = seg[k];
    if (q > c && q < nxt) nxt = q;
  }
  p_next[c] = nxt == 0x7fffffff ? -1 : nxt;
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
                              int N, int* __restrict__ key, int* __restrict__ val, int none) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int s = elig[q];
  const int4 e = ki[s];
  const int cnt = entry_count(e);
  const int id[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
  for (int t = 0; t < 10; ++t) {
    const int m1 = kSlotPairs[t][0], m2 = kSlotPairs[t][1];
    int k = none, v = 0;
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
                                  int* __restrict__ val, int none) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 8 * N) return;
  const int i = nbr[e];
  const int j = e >> 3;
  int k0 = none, k1 = none, k2 = none;
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
__global__ void k_mark_unique(const int* __restrict__ key, int n, int* __restrict__ flag, int none) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int v = key[k];
  flag[k] = (v != none && (k == 0 || key[k - 1] != v)) ? 1 : 0;
}
__global__ void k_write_up(const int* __restrict__ key, const int* __restrict__ scan, int n,
                           int* __restrict__ up_key, int* __restrict__ up_start, int ub_cap,
                           int* __restrict__ err, int none) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int v = key[k];
  if (v == none) return;
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
  if (k + 1 == n || key[k + 1] == none) up_start[total] = k + 1;
}
// Regulariser records grouped by upper block (per frame). rec_flag holds the
// exclusive scan of the block-start flags, so record k lies in block
// rec_flag[k + 1] - 1.
__global__ void k_reg_mark(const int* __restrict__ key, const int* __restrict__ val, int n, int none,
                           int* __restrict__ flag) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  flag[k] = (key[k] != none && val[k] < 0) ? 1 : 0;
}
__global__ void k_reg_compact(const int* __restrict__ flag, const int* __restrict__ scan, int n,
                              const int* __restrict__ val, const int* __restrict__ ub_scan,
                              int* __restrict__ reg_rec, int* __restrict__ reg_ub) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || !flag[k]) return;
  const int j = scan[k];
  reg_rec[j] = val[k];  // the record word (edge, type), in sorted order
  reg_ub[j] = ub_scan[k + 1] - 1;
}
__global__ void k_reg_bmark(const int* __restrict__ reg_ub, const int* __restrict__ n_reg_dev,
                            int cap, int* __restrict__ bf) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cap) return;
  bf[j] = (j < *n_reg_dev && (j == 0 || reg_ub[j] != reg_ub[j - 1])) ? 1 : 0;
}
__global__ void k_reg_bfill(const int* __restrict__ reg_ub, const int* __restrict__ bf,
                            const int* __restrict__ bscan, const int* __restrict__ n_reg_dev,
                            int cap, int* __restrict__ blk_start, int* __restrict__ ub_reg) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_reg = *n_reg_dev;
  if (j >= n_reg) return;
  if (bf[j]) {
    blk_start[bscan[j]] = j;
    ub_reg[reg_ub[j]] = bscan[j];
  }
  if (j == n_reg - 1) blk_start[bscan[cap]] = n_reg;
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
                           int* __restrict__ col, int* __restrict__ tag, int ub_cap, int b_cap) {
  const int ub = blockIdx.x * blockDim.x + threadIdx.x;
  if (ub >= min(*n_up_dev, ub_cap) || row_ptr[N] > b_cap) return;  // capacity: reported later
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
// Warp per BSR row: the row's (column, tag) entries are ranked by column
// (columns are distinct within a row) 32 at a time in registers and scattered
// to their sorted slots; rows longer than 32 entries take the serial path.
__global__ void k_row_sort(const int* __restrict__ row_ptr, int N, int* __restrict__ col,
                           int* __restrict__ tag, int* __restrict__ up_pos, int* __restrict__ up_mpos,
                           int* __restrict__ diag_pos, int b_cap) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= N || row_ptr[N] > b_cap) return;  // warp-uniform
  const int a0 = row_ptr[r], a1 = row_ptr[r + 1], len = a1 - a0;
  if (len <= 32) {
    const int vc = lane < len ? col[a0 + lane] : 0x7fffffff;
    const int vt = lane < len ? tag[a0 + lane] : 0;
    int rank = 0;
    for (int q = 0; q < len; ++q) rank += __shfl_sync(0xffffffffu, vc, q) < vc ? 1 : 0;
    __syncwarp();
    if (lane < len) {
      const int a = a0 + rank;
      col[a] = vc;
      tag[a] = vt;
      if (vt & 1) up_mpos[vt >> 1] = a;
      else up_pos[vt >> 1] = a;
    }
    const unsigned d = __ballot_sync(0xffffffffu, lane < len && vc == r);  // warp-uniform
    int dr = -1;
    if (d) dr = __shfl_sync(0xffffffffu, rank, __ffs(d) - 1);  // the diagonal's sorted slot
    if (lane == 0) diag_pos[r] = d ? a0 + dr : -1;
    return;
  }
  if (lane != 0) return;
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
#ifndef DS_CHUNK
#define DS_CHUNK 64
#endif
#ifndef DS_CHUNK_LANES
#define DS_CHUNK_LANES 8
#endif
constexpr int kChunk = DS_CHUNK;            // records per chunk (A/B builds: -DDS_CHUNK=...)
constexpr int kChunkLanes = DS_CHUNK_LANES;  // lanes per chunk

struct AsmArgs {
  const int* up_key;
  const int* up_start;
  const int* up_pos;
  const int* up_mpos;
  const int* chunk_ub;
  const int* chunk_first;
  const int4* chunk_d0;  // per chunk: (record range, BSR position, mirror position)
  const int4* chunk_d1;  // per chunk: (diagonal g row, regulariser block, single-chunk)
  const int* rec_val;
  const int* s_cnt;
  const int* s_head;   // lowest pixel of the surfel's pairs
  const int* p_next;   // next pixel of the same surfel (pixel order)
  const float* rows;   // per-pixel Jacobian rows (4 x 6 fp32)
  const double* pair_r;
  const double4* node_pos;
  const int* nbr;
  const double* se3;
  const double* reg_ab;  // per directed edge: T_j p_j, T_i p_j (k_reg_energy)
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
  const int* ub_reg;   // per upper block: regulariser block or -1
  const double* reg_h;  // per regulariser block: 6x6 sum (k_reg_blocks)
  const double* reg_g;
};

// column x of reg_jacobian_j = [-[a]x, I] (sel 0) or reg_jacobian_i = [[b]x, -I]
// (sel 1) (solver.cpp:118-130), entry by entry as the dense form has them
__device__ __forceinline__ V3 reg_col(int sel, int x, const V3& a, const V3& b) {
  if (sel == 0) {
    switch (x) {
      case 0: return v3(-0.0, -a.z, a.y);
      case 1: return v3(a.z, -0.0, -a.x);
      case 2: return v3(-a.y, a.x, -0.0);
      default: return v3(x == 3 ? 1.0 : 0.0, x == 4 ? 1.0 : 0.0, x == 5 ? 1.0 : 0.0);
    }
  }
  switch (x) {
    case 0: return v3(0.0, b.z, -b.y);
    case 1: return v3(-b.z, 0.0, b.x);
    case 2: return v3(b.y, -b.x, 0.0);
    default: return v3(x == 3 ? -1.0 : 0.0, x == 4 ? -1.0 : 0.0, x == 5 ? -1.0 : 0.0);
  }
}

inline int reg_rb_pad(int N) { return (9 * N + 31) / 32 * 32; }  // reg block bound, warp multiple

// Regulariser blocks (per GN iteration, side branch): thread per (block row
// x, reg block), x uniform across a warp (the reg_col switch on x does not
// diverge); the thread sums row x of the 6x6 block and g[x] of a diagonal
// block over the block's records in order, in fp64. Records: edge e = 8 j +
// slot, type 0: JjtJj / gj, 1: JitJi / gi, 2: JjtJi, 3: JitJj
// (solver.cpp:118-130). Four records per step are loaded together.
__global__ void __launch_bounds__(256) k_reg_blocks(const int* __restrict__ reg_val,
                                                    const int* __restrict__ blk_start,
                                                    const int* __restrict__ n_rb_dev, int rb_pad,
                                                    const double* __restrict__ reg_ab, double lambda,
                                                    double* __restrict__ reg_h,
                                                    double* __restrict__ reg_g) {
  pdl_wait();  // programmatic dependent launch: predecessor results visible
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const int x = gid / rb_pad, rb = gid % rb_pad;
  if (x >= 6 || rb >= *n_rb_dev) return;
  const int j0 = blk_start[rb], j1 = blk_start[rb + 1];
  double acc[6] = {0, 0, 0, 0, 0, 0};
  double gacc = 0.0;
  for (int j = j0; j < j1; j += 4) {
    int v[4];
    double2 u[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = j + q < j1 ? __ldg(reg_val + j + q) : 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (j + q < j1) {
        const double2* ab =
            reinterpret_cast<const double2*>(reg_ab + 6 * (size_t)((v[q] & 0x7fffffff) >> 2));
        u[q][0] = __ldg(ab);
        u[q][1] = __ldg(ab + 1);
        u[q][2] = __ldg(ab + 2);
      }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (j + q >= j1) continue;
      const int type = v[q] & 3;
      const V3 a = v3(u[q][0].x, u[q][0].y, u[q][1].x), b = v3(u[q][1].y, u[q][2].x, u[q][2].y);
      const int ls = (type == 0 || type == 2) ? 0 : 1, rs = (type == 0 || type == 3) ? 0 : 1;
      const V3 L = reg_col(ls, x, a, b);
#pragma unroll
      for (int y = 0; y < 6; ++y) {
        const V3 R = reg_col(rs, y, a, b);
        acc[y] += lambda * ((L.x * R.x + L.y * R.y) + L.z * R.z);
      }
      if (type <= 1) {
        const V3 rv = sub(a, b);
        gacc += lambda * ((L.x * rv.x + L.y * rv.y) + L.z * rv.z);
      }
    }
  }
#pragma unroll
  for (int y = 0; y < 6; ++y) reg_h[(size_t)rb * 36 + x * 6 + y] = acc[y];
  reg_g[(size_t)rb * 6 + x] = gacc;
}

__device__ __forceinline__ void load_rows(const float* __restrict__ rw, int mr, int mc, float a[6],
                                          float b[6]) {
  const float2* ra = reinterpret_cast<const float2*>(rw + mr * 6);
  const float2* rb = reinterpret_cast<const float2*>(rw + mc * 6);
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const float2 x = __ldg(ra + t), y = __ldg(rb + t);
    a[2 * t] = x.x;
    a[2 * t + 1] = x.y;
    b[2 * t] = y.x;
    b[2 * t + 1] = y.y;
  }
}

// explicit fused multiply-adds (one rounding per term; the build's
// --fmad=false only stops implicit contraction, which the fp64 decision
// arithmetic elsewhere relies on)
__device__ __forceinline__ void acc_pair(const float a[6], const float b[6], bool diag, double r,
                                         float h[36], double gg[6]) {
#pragma unroll
  for (int x = 0; x < 6; ++x)
#pragma unroll
    for (int y = 0; y < 6; ++y) h[x * 6 + y] = __fmaf_rn(a[x], b[y], h[x * 6 + y]);
  if (diag) {
#pragma unroll
    for (int x = 0; x < 6; ++x) gg[x] = __fma_rn((double)a[x], r, gg[x]);
  }
}

// A surfel record: its pairs in pixel order (head pixel, then the p_next
// chain), the head pair's rows already loaded into (a, b, r).
__device__ __forceinline__ void acc_surfel_record(const AsmArgs& A, int v, int cnt, int head,
                                                  const float a[6], const float b[6], double r,
                                                  bool diag, float h[36], double gg[6]) {
  const int mr = (v >> 2) & 3, mc = v & 3;
  acc_pair(a, b, diag, r, h, gg);
  int pix = head;
  for (int q = 1; q < cnt; ++q) {
    pix = __ldg(A.p_next + pix);
    float a2[6], b2[6];
    load_rows(A.rows + (size_t)pix * 24, mr, mc, a2, b2);
    acc_pair(a2, b2, diag, diag ? __ldg(A.pair_r + pix) : 0.0, h, gg);
  }
}

// Lane l of a chunk takes records l, l+8, ... in order; two records are in
// flight per step (their count/offset and first-pair rows are loaded before
// either is accumulated), the accumulation order is unchanged.
__global__ void __launch_bounds__(256, 2) k_assemble_chunks(AsmArgs A) {
  pdl_wait();  // programmatic dependent launch: predecessor results visible
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
  int4 d0 = make_int4(0, 0, 0, -1), d1 = make_int4(-1, -1, 0, 0);
  bool diag = false;
  if (valid) {
    d0 = A.chunk_d0[chunk];
    d1 = A.chunk_d1[chunk];
    diag = d1.x >= 0;
    const int r0 = d0.x, r1 = d0.y;
    // Three-stage software pipeline over steps of two records (lane l takes
    // records l, l+8, l+16, ... in order): while step s's Jacobian rows are
    // loaded and accumulated, step s+1's (count, head) and step s+2's record
    // words are already in flight -- one dependent round trip per step instead
    // of three. The accumulation order is unchanged.
    constexpr int kNone = 0x7fffffff;
    const int k0 = r0 + l;
    auto rec_at = [&](int k) { return k < r1 ? __ldg(A.rec_val + k) : kNone; };
    auto info = [&](int v, int& cnt, int& head) {
      cnt = 0;
      head = 0;
      if (v != kNone && v >= 0) {
        cnt = __ldg(A.s_cnt + (v >> 4));
        head = __ldg(A.s_head + (v >> 4));
      }
    };
    int vA0 = rec_at(k0), vA1 = rec_at(k0 + kChunkLanes);
    int vB0 = rec_at(k0 + 2 * kChunkLanes), vB1 = rec_at(k0 + 3 * kChunkLanes);
    int cA0, hA0, cA1, hA1;
    info(vA0, cA0, hA0);
    info(vA1, cA1, hA1);
    for (int ks = k0; ks < r1; ks += 2 * kChunkLanes) {
      const int vC0 = rec_at(ks + 4 * kChunkLanes), vC1 = rec_at(ks + 5 * kChunkLanes);
      int cB0, hB0, cB1, hB1;
      info(vB0, cB0, hB0);
      info(vB1, cB1, hB1);
      float a0[6], b0[6], a1[6], b1[6];
      double rr0 = 0.0, rr1 = 0.0;
      if (cA0 > 0) {
        load_rows(A.rows + (size_t)hA0 * 24, (vA0 >> 2) & 3, vA0 & 3, a0, b0);
        if (diag) rr0 = __ldg(A.pair_r + hA0);
      }
      if (cA1 > 0) {
        load_rows(A.rows + (size_t)hA1 * 24, (vA1 >> 2) & 3, vA1 & 3, a1, b1);
        if (diag) rr1 = __ldg(A.pair_r + hA1);
      }
      // regulariser records (v < 0) are summed by k_reg_blocks
      if (vA0 != kNone) {
        if (vA0 >= 0 && cA0 > 0) {
          acc_surfel_record(A, vA0, cA0, hA0, a0, b0, rr0, diag, h, gg);
          touched = 1;
        }
      }
      if (vA1 != kNone) {
        if (vA1 >= 0 && cA1 > 0) {
          acc_surfel_record(A, vA1, cA1, hA1, a1, b1, rr1, diag, h, gg);
          touched = 1;
        }
      }
      vA0 = vB0;
      vA1 = vB1;
      cA0 = cB0;
      hA0 = hB0;
      cA1 = cB1;
      hA1 = hB1;
      vB0 = vC0;
      vB1 = vC1;
    }
  }
  // fixed reduce-scatter over the 8 lanes of the group: three halving rounds
  // (xor 4, 2, 1); afterwards lane l holds the sums of entries t = l (mod 8)
  static_assert(kChunkLanes == 8, "reduce-scatter is written for 8-lane groups");
  float r1[20];
#pragma unroll
  for (int q = 0; q < 5; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float a = q * 8 + j < 36 ? h[q * 8 + j] : 0.f;
      const float b = q * 8 + j + 4 < 36 ? h[q * 8 + j + 4] : 0.f;
      const bool hi = l & 4;
      r1[q * 4 + j] = (hi ? b : a) + __shfl_xor_sync(0xffffffffu, hi ? a : b, 4);
    }
  float r2[10];
#pragma unroll
  for (int q = 0; q < 5; ++q)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float a = r1[q * 4 + j], b = r1[q * 4 + j + 2];
      const bool hi = l & 2;
      r2[q * 2 + j] = (hi ? b : a) + __shfl_xor_sync(0xffffffffu, hi ? a : b, 2);
    }
  float hs[5];  // hs[q] = entry 8 q + l
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const float a = r2[q * 2], b = r2[q * 2 + 1];
    const bool hi = l & 1;
    hs[q] = (hi ? b : a) + __shfl_xor_sync(0xffffffffu, hi ? a : b, 1);
  }
  double g1[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double a = gg[j], b = j + 4 < 6 ? gg[j + 4] : 0.0;
    const bool hi = l & 4;
    g1[j] = (hi ? b : a) + __shfl_xor_sync(0xffffffffu, hi ? a : b, 4);
  }
  double g2[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double a = g1[j], b = g1[j + 2];
    const bool hi = l & 2;
    g2[j] = (hi ? b : a) + __shfl_xor_sync(0xffffffffu, hi ? a : b, 2);
  }
  double gs;  // entry l of g (lanes 0..5)
  {
    const double a = g2[0], b = g2[1];
    const bool hi = l & 1;
    gs = (hi ? b : a) + __shfl_xor_sync(0xffffffffu, hi ? a : b, 1);
  }
#pragma unroll
  for (int off = 4; off > 0; off >>= 1) touched |= __shfl_xor_sync(0xffffffffu, touched, off);
  if (!valid) return;
  if (d1.z) {
    // single-chunk block (most off-diagonal ones): the partial plus the
    // block's regulariser sum is final; the lanes write it straight into the
    // BSR (both triangles) and g
    const int pu = d0.z, pm = d0.w, rb = d1.y;
    if (rb >= 0) touched = 1;
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int t = 8 * q + l;
      if (t >= 36) continue;
      const float v = rb >= 0 ? (float)((double)hs[q] + __ldg(A.reg_h + (size_t)rb * 36 + t)) : hs[q];
      A.bsr_val[(size_t)pu * 36 + t] = v;
      if (pm >= 0) A.bsr_val[(size_t)pm * 36 + (t % 6) * 6 + t / 6] = v;
    }
    if (l == 0) {
      A.bsr_touch[pu] = touched ? 1 : 0;
      if (pm >= 0) A.bsr_touch[pm] = touched ? 1 : 0;
    }
    if (diag && l < 6)
      A.g[6 * d1.x + l] = rb >= 0 ? gs + __ldg(A.reg_g + (size_t)rb * 6 + l) : gs;
    return;
  }
  // multi-chunk block: the lanes write the partial
#pragma unroll
  for (int q = 0; q < 5; ++q)
    if (8 * q + l < 36) A.part_h[(size_t)chunk * 36 + 8 * q + l] = hs[q];
  if (l < 6) A.part_g[(size_t)chunk * 6 + l] = gs;
  if (l == 0) A.part_t[chunk] = touched;
}

// multi-chunk blocks only: thread per (block, entry) sums the chunk partials in
// chunk order (fp64) -> BSR both triangles; entries 36..41 are g of a diagonal
// block, entry 42 the touched flag
constexpr int kFinishEntries = 43;
__global__ void k_assemble_finish(AsmArgs A, const int* __restrict__ multi, const int* __restrict__ n_multi) {
  pdl_wait();  // programmatic dependent launch: predecessor results visible
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const int mi = gid / kFinishEntries, t = gid % kFinishEntries;
  if (mi >= *n_multi) return;
  const int ub = multi[mi];
  const int key = A.up_key[ub];
  const int row = key / A.N, colb = key % A.N;
  const int c0 = A.chunk_first[ub], c1 = A.chunk_first[ub + 1];
  const int pu = A.up_pos[ub];
  const int pm = row != colb ? A.up_mpos[ub] : -1;
  const int rb = A.ub_reg[ub];
  if (t < 36) {
    double acc = 0.0;
#pragma unroll 4
    for (int c = c0; c < c1; ++c) acc += (double)A.part_h[(size_t)c * 36 + t];
    if (rb >= 0) acc += A.reg_h[(size_t)rb * 36 + t];
    A.bsr_val[(size_t)pu * 36 + t] = (float)acc;
    if (pm >= 0) A.bsr_val[(size_t)pm * 36 + (t % 6) * 6 + t / 6] = (float)acc;
  } else if (t < 42) {
    if (pm >= 0) return;
    double acc = 0.0;
#pragma unroll 4
    for (int c = c0; c < c1; ++c) acc += A.part_g[(size_t)c * 6 + (t - 36)];
    if (rb >= 0) acc += A.reg_g[(size_t)rb * 6 + (t - 36)];
    A.g[6 * row + (t - 36)] = acc;
  } else {
    int touched = rb >= 0 ? 1 : 0;
    for (int c = c0; c < c1; ++c) touched |= A.part_t[c];
    A.bsr_touch[pu] = touched ? 1 : 0;
    if (pm >= 0) A.bsr_touch[pm] = touched ? 1 : 0;
  }
}

// bound >= n_up entries: those past the device count get 0 (the scans run
// over the host-known bound)
__global__ void k_chunk_count(const int* __restrict__ up_start, const int* __restrict__ n_up_dev,
                              int bound, int* __restrict__ cnt, int* __restrict__ multi_flag) {
  const int ub = blockIdx.x * blockDim.x + threadIdx.x;
  if (ub >= bound) return;
  if (ub >= *n_up_dev) {
    cnt[ub] = 0;
    multi_flag[ub] = 0;
    return;
  }
  const int k = (up_start[ub + 1] - up_start[ub] + kChunk - 1) / kChunk;
  cnt[ub] = k;
  multi_flag[ub] = k > 1 ? 1 : 0;
}
__global__ void k_multi_list(const int* __restrict__ flag, const int* __restrict__ scan, int bound,
                             int* __restrict__ list) {
  const int ub = blockIdx.x * blockDim.x + threadIdx.x;
  if (ub < bound && flag[ub]) list[scan[ub]] = ub;
}
// per chunk: its upper block and a descriptor the assembly reads in one go:
// d0 = (first record, end record, BSR position, mirrored position or -1),
// d1 = (g row of a diagonal block or -1, regulariser block or -1, single-chunk)
// Thread 0 also publishes the pattern's counts (and capacity errors) into
// DevScalars for the host, which reads them with the frame's next fetch.
__global__ void k_chunk_fill(const int* __restrict__ first, const int* __restrict__ n_up_dev,
                             const int* __restrict__ up_key, const int* __restrict__ up_start,
                             const int* __restrict__ up_pos, const int* __restrict__ up_mpos,
                             const int* __restrict__ ub_reg, int N, const int* __restrict__ row_ptr,
                             const int* __restrict__ multi_scan, int ub_cap, int b_cap, int ch_cap,
                             const int* __restrict__ err_in, DevScalars* __restrict__ sc,
                             int* __restrict__ chunk_ub, int4* __restrict__ d0,
                             int4* __restrict__ d1) {
  const int ub = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_up = *n_up_dev;
  const bool over = n_up > ub_cap || row_ptr[N] > b_cap || (n_up <= ub_cap && first[n_up] > ch_cap);
  if (ub == 0) {
    sc->pat_n_up = n_up;
    sc->pat_n_full = row_ptr[N];
    sc->pat_n_chunks = n_up <= ub_cap ? first[n_up] : 0;
    sc->pat_n_multi = n_up <= ub_cap ? multi_scan[n_up] : 0;
    sc->pat_err = (over || (*err_in & DERR_BLOCK_CAP)) ? 1 : 0;
  }
  if (ub >= n_up || over) return;
  const int c0 = first[ub], c1 = first[ub + 1];
  const int key = up_key[ub], row = key / N;
  const bool diag = row == key % N;
  const int pu = up_pos[ub], pm = diag ? -1 : up_mpos[ub];
  const int s0 = up_start[ub], s1 = up_start[ub + 1];
  const int rb = ub_reg[ub];
  for (int c = c0; c < c1; ++c) {
    chunk_ub[c] = ub;
    const int r0 = s0 + (c - c0) * kChunk;
    d0[c] = make_int4(r0, min(r0 + kChunk, s1), pu, pm);
    d1[c] = make_int4(diag ? row : -1, rb, c1 - c0 == 1 ? 1 : 0, 0);
  }
}

// ginf, |g|^2, tr(H) (solver.cpp:371, 378), thread per node; the last block
// (ticket) combines the block partials in block order. With lm != 0 it also
// applies the LM floor: mu_floor = 1e-6 tr(H) / dim, mu = max(mu, mu_floor)
// (solver.cpp:378-379).
constexpr int kStatsThreads = 256;
__global__ void __launch_bounds__(kStatsThreads) k_g_stats(
    const double* __restrict__ g, const float* __restrict__ val, const int* __restrict__ diag_pos,
    int N, int lm, double* __restrict__ part, unsigned* __restrict__ ticket,
    DevScalars* __restrict__ sc) {
  pdl_wait();  // programmatic dependent launch: predecessor results visible
  constexpr int kWarps = kStatsThreads / 32;
  __shared__ double wmax[kWarps], wsq[kWarps], wtr[kWarps];
  __shared__ unsigned wdone;
  const int tid = threadIdx.x, j = blockIdx.x * kStatsThreads + tid;
  const int lane = tid & 31, w = tid >> 5;
  if (tid == 0) wdone = 0u;
  double mx = 0, sq = 0, tr = 0;
  if (j < N) {
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const double v = g[6 * j + t];
      mx = fmax(mx, fabs(v));
      sq += v * v;
    }
    const int d = diag_pos[j];
    if (d >= 0) {
      const float* b = val + (size_t)d * 36;
      tr = (((((double)b[0] + (double)b[7]) + (double)b[14]) + (double)b[21]) + (double)b[28]) +
           (double)b[35];
    }
  }
  __syncthreads();  // wdone visible
  // warp xor butterflies, then the last warp of the block combines in warp
  // order and the last block combines the block partials (fixed orders)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    sq += __shfl_xor_sync(0xffffffffu, sq, off);
    tr += __shfl_xor_sync(0xffffffffu, tr, off);
  }
  int lastw = 0;
  if (lane == 0) {
    wmax[w] = mx;
    wsq[w] = sq;
    wtr[w] = tr;
    __threadfence_block();
    lastw = atomicAdd(&wdone, 1u) == (unsigned)kWarps - 1;
  }
  if (!__shfl_sync(0xffffffffu, lastw, 0)) return;
  int lastb = 0;
  if (lane == 0) {
    __threadfence_block();
    const volatile double *vm = wmax, *vq = wsq, *vt = wtr;
    double m = 0, q = 0, t = 0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) {
      m = fmax(m, vm[i]);
      q += vq[i];
      t += vt[i];
    }
    part[3 * blockIdx.x + 0] = m;
    part[3 * blockIdx.x + 1] = q;
    part[3 * blockIdx.x + 2] = t;
    __threadfence();
    lastb = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  if (!__shfl_sync(0xffffffffu, lastb, 0)) return;
  __threadfence();
  double m = 0, q = 0, t = 0;
  for (int b = lane; b < (int)gridDim.x; b += 32) {
    m = fmax(m, __ldcg(part + 3 * b));
    q += __ldcg(part + 3 * b + 1);
    t += __ldcg(part + 3 * b + 2);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    q += __shfl_xor_sync(0xffffffffu, q, off);
    t += __shfl_xor_sync(0xffffffffu, t, off);
  }
  if (lane != 0) return;
  sc->ginf = m;
  sc->g_sq = q;  // |g|^2
  sc->htrace = t;
  if (lm) {
    const double floor_ = 1e-6 * t / (6.0 * N);
    sc->mu_floor = floor_;
    sc->mu = fmax(sc->mu, floor_);
  }
  *ticket = 0u;
}

// ------------------------------------------------------------------- PCG
// Preconditioned pipelined CG (Ghysels & Vanroose 2014, Alg. 3) with the
// block-Jacobi preconditioner of solver.cpp:180-214: in exact arithmetic the
// iterates are those of the reference's PCG; in the kernel each iteration needs
// ONE grid barrier (the dot products and the SpMV input m = M w are published
// together) instead of two.
//
// One cooperative persistent kernel, one CTA per SM. CTA b owns the contiguous
// block rows [r0, r1) whose BSR blocks are [nnzb*b/G, nnzb*(b+1)/G) rounded to
// row boundaries; its matrix slice (fp32 values + columns), the 6x6 inverses
// and all per-row vectors live in shared memory, so an iteration reads global
// memory only for the gathered m of the neighbouring nodes (48 B per block) and
// the grid partials. Slices above the shared-memory budget (very large N) keep
// the same arithmetic on global scratch. Reductions are fixed-order (thread ->
// warp -> CTA -> grid); the decomposition depends only on (N, nnzb, G).
#ifndef DS_PCG_THREADS
#define DS_PCG_THREADS 256
#endif
constexpr int kPcgThreads = DS_PCG_THREADS;  // measured: 256 beats 512 / 384 / 128
constexpr int kPcgWarps = kPcgThreads / 32;
#ifndef DS_PCG_SMEM_KB
#define DS_PCG_SMEM_KB 200
#endif
constexpr int kPcgSmem = DS_PCG_SMEM_KB * 1024;  // A/B builds: -DDS_PCG_SMEM_KB=100 (2 CTAs/SM)
constexpr int kPcgVecs = 10;  // x r u w m n z q s p

struct PcgArgs {
  const int* row_ptr;
  const int* col;
  const float* val;
  const int* diag_pos;
  const double* g;
  const double* mu_ptr;  // LM damping lives on the device (graph-replay safe)
  int N;
  int nnzb;
  int max_iters;
  double tol2;
  double* x;        // solution (6N)
  double* pub0;     // published u0 / m (even iterations) (6N)
  double* pub1;     // published m (odd iterations) / classic p_old (6N)
  double* pub2;     // classic p_new (6N)
  double* minv;     // fallback scratch (36N)
  double* vec;      // fallback scratch (kPcgVecs x 6N)
  double* items;    // fallback SpMV partials (6 nnzb)
  double* part;     // grid partials, 2 x 4 x G
  unsigned long long* trace;  // optional phase timestamps (DS_PCG_TRACE), CTA 0
  const int* slices;  // per CTA (r0, r1, bb0, bb1), k_pcg_slices once per frame
  int smem_cap;       // slice bytes that may live in shared memory (<= kPcgSmem)
  DevScalars* sc;
};

// fixed-order CTA sums of three values; results valid in every thread.
// kLeadSync = false: the caller guarantees that every thread has finished
// reading `sh` from its previous use (a dedicated buffer with barriers in
// between), which saves the leading barrier
template <bool kLeadSync = true>
__device__ __forceinline__ void cta_sum3(double& a, double& b, double& c, double4* sh) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
    c += __shfl_xor_sync(0xffffffffu, c, off);
  }
  if (kLeadSync) __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = make_double4(a, b, c, 0.0);
  __syncthreads();
  double ta = 0.0, tb = 0.0, tc = 0.0;
#pragma unroll
  for (int w = 0; w < kPcgWarps; ++w) {
    const double4 v = sh[w];
    ta += v.x;
    tb += v.y;
    tc += v.z;
  }
  a = ta;
  b = tb;
  c = tc;
}

// grid totals of the 3 partials at part[4 k + 0..2]: thread k < G loads CTA
// k's partials (one coalesced pass), then a fixed warp-shuffle + warp-order
// tree -- identical bits in every CTA
__device__ __forceinline__ double4 grid_sum3(const double* part, double4* sh) {
  double va = 0.0, vb = 0.0, vc = 0.0;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += kPcgThreads) {
    const double2 ab = __ldcg(reinterpret_cast<const double2*>(part + 4 * k));
    va += ab.x;
    vb += ab.y;
    vc += __ldcg(part + 4 * k + 2);
  }
  cta_sum3(va, vb, vc, sh);
  return make_double4(va, vb, vc, 0.0);
}

__device__ __forceinline__ int lower_bound_dev(const int* a, int n, int v) {
  int lo = 0, hi = n;  // first k in [0, n) with a[k] >= v, or n
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// y_own = (H + mu I) v over the CTA's rows, v gathered from the published
// array `pub` at the column nodes; own part of v in `vown`.
__device__ __forceinline__ void slice_spmv(const float* V, const int* C, const int* RP, int bb0,
                                           int nb, int nr, const double* pub, const double* vown,
                                           double mu, double* IT, double* y) {
#pragma unroll 2
  for (int k = threadIdx.x; k < 2 * nb; k += kPcgThreads) {
    const int blk = k >> 1, h3 = 3 * (k & 1);
    const double2* vc = reinterpret_cast<const double2*>(pub + 6 * (size_t)C[blk]);
    double pv[6];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const double2 u = __ldcg(vc + t);
      pv[2 * t] = u.x;
      pv[2 * t + 1] = u.y;
    }
    const float* vr = V + 36 * (size_t)blk + 6 * h3;
#pragma unroll
    for (int rw = 0; rw < 3; ++rw) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < 6; ++t) s += (double)vr[6 * rw + t] * pv[t];
      IT[6 * (size_t)blk + h3 + rw] = s;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 6 * nr; k += kPcgThreads) {
    const int i = k / 6, rw = k - 6 * i;
    const int lb0 = RP[i] - bb0, lb1 = RP[i + 1] - bb0;
    double tot = 0.0;
    for (int b = lb0; b < lb1; ++b) tot += IT[6 * (size_t)b + rw];
    y[k] = tot + mu * vown[k];
  }
}

// y_own = M^-1 v_own (block-diagonal: rows are local); v must be complete
__device__ __forceinline__ void apply_minv(const double* MINV, const double* v, double* y, int nr) {
  for (int k = threadIdx.x; k < 6 * nr; k += kPcgThreads) {
    const int i = k / 6, rw = k - 6 * i;
    const double* mi = MINV + 36 * i + 6 * rw;
    const double* vi = v + 6 * i;
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 6; ++t) s += mi[t] * vi[t];
    y[k] = s;
  }
}

// kPipe = true: pipelined recurrences, one grid barrier per iteration (used
// for a fixed iteration budget, the reference's default). kPipe = false: the
// classic two-barrier recurrences, whose recursive residual stays close to the
// true one -- used when PCG runs to a tolerance (attainable accuracy).
// CTA b of the PCG owns the block rows [r0, r1) whose BSR blocks are
// [nnzb b / G, nnzb (b+1) / G) rounded to row starts; computed once per frame
// (the pattern is fixed for the frame), thread per CTA.
__global__ void k_pcg_slices(const int* __restrict__ row_ptr, int N, int G, int* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= G) return;
  const long long nz = row_ptr[N];
  const int t_lo = (int)(nz * b / G), t_hi = (int)(nz * (b + 1) / G);
  const int r0 = b == 0 ? 0 : min(lower_bound_dev(row_ptr, N + 1, t_lo), N);
  int r1 = b == G - 1 ? N : min(lower_bound_dev(row_ptr, N + 1, t_hi), N);
  r1 = max(r1, r0);
  out[4 * b + 0] = r0;
  out[4 * b + 1] = r1;
  out[4 * b + 2] = row_ptr[r0];
  out[4 * b + 3] = row_ptr[r1];
}

__device__ __forceinline__ void pcg_mark(const PcgArgs& a, int slot) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && slot < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[slot] = t;
  }
}

template <bool kPipe>
__global__ void __launch_bounds__(kPcgThreads, 1) k_pcg(PcgArgs a) {
  cg::grid_group grid = cg::this_grid();
  pcg_mark(a, 0);
  if (blockIdx.x == 0 && threadIdx.x == 0) a.sc->finite = 1;  // before any barrier
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double4 sh[kPcgWarps + 1];
  __shared__ double4 sh2[2][kPcgWarps];  // the pipelined loop's two reductions
  __shared__ int s_rng[4];
  const int tid = threadIdx.x, G = gridDim.x;
  if (tid < 4) s_rng[tid] = a.slices[4 * blockIdx.x + tid];  // (r0, r1, bb0, bb1), per frame
  __syncthreads();
  const int r0 = s_rng[0], r1 = s_rng[1];
  const int nr = r1 - r0, n6 = 6 * nr;
  const int bb0 = s_rng[2], nb = s_rng[3] - bb0;
  const double mu = *a.mu_ptr;
  // ---- slice placement: everything in shared memory when it fits; else the
  // vectors, inverses and SpMV partials in shared memory with the matrix
  // streamed from L2 / HBM (large N); else all on global scratch
  const size_t need_vec = (size_t)nr * (36 + 6 * kPcgVecs) * 8 + (size_t)nb * 6 * 8 +
                          (size_t)(nr + 1) * 4;
  const size_t need = need_vec + (size_t)nb * (36 * 4 + 4);
  const bool fits = need <= (size_t)a.smem_cap;
  const bool fits_vec = !fits && need_vec <= (size_t)a.smem_cap;
  double *MINV, *vb, *IT;
  const float* V;
  const int* C;
  const int* RP;
  if (fits || fits_vec) {
    double* d = reinterpret_cast<double*>(smem);
    MINV = d;
    vb = MINV + 36 * nr;
    IT = vb + kPcgVecs * n6;
    int* srp;
    if (fits) {
      float* sv = reinterpret_cast<float*>(IT + 6 * (size_t)nb);
      int* sc = reinterpret_cast<int*>(sv + 36 * (size_t)nb);
      srp = sc + nb;
      // the slice's blocks and columns stream in asynchronously (cp.async)
      // while the block-Jacobi inverses below are computed; waited for before
      // the first use (the __syncthreads after the r0 initialisation)
      const float4* gv = reinterpret_cast<const float4*>(a.val + 36 * (size_t)bb0);
      float4* sv4 = reinterpret_cast<float4*>(sv);
      for (int k = tid; k < 9 * nb; k += kPcgThreads) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(sv4 + k);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gv + k) : "memory");
      }
      for (int k = tid; k < nb; k += kPcgThreads) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(sc + k);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(a.col + bb0 + k)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      V = sv;
      C = sc;
    } else {
      srp = reinterpret_cast<int*>(IT + 6 * (size_t)nb);
      V = a.val + 36 * (size_t)bb0;
      C = a.col + bb0;
    }
    for (int k = tid; k <= nr; k += kPcgThreads) srp[k] = a.row_ptr[r0 + k];
    RP = srp;
  } else {
    MINV = a.minv + 36 * (size_t)r0;
    vb = a.vec + (size_t)kPcgVecs * 6 * r0;  // CTA-contiguous carve of the scratch
    IT = a.items + 6 * (size_t)bb0;
    V = a.val + 36 * (size_t)bb0;
    C = a.col + bb0;
    RP = a.row_ptr + r0;
  }
  double* X = vb;
  double* R = X + n6;
  double* U = R + n6;  // u (pipelined) / z (classic)
  double* W = U + n6;
  double* Mv = W + n6;
  double* Nv = Mv + n6;
  double* Zv = Nv + n6;
  double* Qv = Zv + n6;
  double* Sv = Qv + n6;
  double* Pv = Sv + n6;
  pcg_mark(a, 1);
  // ---- prologue: block-Jacobi inverses (8-lane Gauss-Jordan per node)
  {
    const int grp = tid >> 3, lr = tid & 7;
    for (int i0 = 0; i0 < nr; i0 += kPcgThreads / 8) {
      const int i = i0 + grp;
      double ar[6], br[6];
      const int d = (i < nr && lr < 6) ? a.diag_pos[r0 + i] : -1;
      if (i0 == 0) pcg_mark(a, 55 + (d >= 0 ? 0 : 4));
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        double v = d >= 0 ? (double)a.val[(size_t)d * 36 + lr * 6 + t] : 0.0;
        if (t == lr) v += mu;
        ar[t] = lr < 6 ? v : 0.0;
      }
      if (i0 == 0) pcg_mark(a, 56 + (ar[0] == 12345.0 ? 1 : 0));
      if (a.trace) {  // diagnostic: a cold and a warm run of the same code
        double a2[6], b2[6];
#pragma unroll
        for (int t = 0; t < 6; ++t) a2[t] = ar[t];
        gj_inverse6(a2, b2, lr);
        if (i0 == 0) pcg_mark(a, 50 + (b2[0] == 12345.0 ? 1 : 0));
      }
      gj_inverse6(ar, br, lr);
      if (i0 == 0) pcg_mark(a, 58 + (br[0] == 12345.0 ? 1 : 0));
      if (i < nr && lr < 6)
#pragma unroll
        for (int t = 0; t < 6; ++t) MINV[36 * i + 6 * lr + t] = br[t];
    }
  }
  pcg_mark(a, 59);
  // r0 = -g, x0 = 0, recurrence vectors 0
  for (int k = tid; k < n6; k += kPcgThreads) {
    R[k] = -a.g[6 * (size_t)r0 + k];
    X[k] = 0.0;
    Zv[k] = 0.0;
    Qv[k] = 0.0;
    Sv[k] = 0.0;
    Pv[k] = 0.0;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");  // the staged slice (no-op if none)
  __syncthreads();
  pcg_mark(a, 60);
  // u0 = M^-1 r0, published (pipelined: in the odd buffer, which iteration 0's
  // m does not overwrite while slower CTAs still gather u0)
  double* u0pub = kPipe ? a.pub1 : a.pub0;
  apply_minv(MINV, R, U, nr);
  pcg_mark(a, 61);
  for (int k = tid; k < n6; k += kPcgThreads) u0pub[6 * (size_t)r0 + k] = U[k];
  pcg_mark(a, 62);
  double rr0 = 0.0, rr = 0.0;
  int it = 0;
  pcg_mark(a, 2);
  if constexpr (kPipe) {
    grid.sync();
    pcg_mark(a, 3);
    slice_spmv(V, C, RP, bb0, nb, nr, u0pub, U, mu, IT, W);  // w0 = A u0
    pcg_mark(a, 4);
    double gamma_old = 0.0, alpha_old = 0.0;
    for (;; ++it) {
      __syncthreads();  // W (and R, U) complete
      // m = M^-1 w (published) + partials (r.u, w.u, r.r)
      double* pub = (it & 1) ? a.pub1 : a.pub0;
      double pg = 0.0, pd = 0.0, pr = 0.0;
      for (int k = tid; k < n6; k += kPcgThreads) {
        const int i = k / 6, rw = k - 6 * i;
        const double* mi = MINV + 36 * i + 6 * rw;
        const double* wi = W + 6 * i;
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < 6; ++t) s += mi[t] * wi[t];
        Mv[k] = s;
        pub[6 * (size_t)r0 + k] = s;
        pg += R[k] * U[k];
        pd += W[k] * U[k];
        pr += R[k] * R[k];
      }
      pcg_mark(a, 5 + 5 * it);
      // own buffers: each is reused only after the grid barrier / the loop-top
      // barrier, so the reductions skip their leading __syncthreads
      cta_sum3<false>(pg, pd, pr, sh2[0]);
      double* part = a.part + 4 * G * (it & 1);
      if (tid == 0) {
        part[4 * blockIdx.x + 0] = pg;
        part[4 * blockIdx.x + 1] = pd;
        part[4 * blockIdx.x + 2] = pr;
      }
      pcg_mark(a, 6 + 5 * it);
      grid.sync();
      pcg_mark(a, 7 + 5 * it);
      // the grid partials (thread k < G holds CTA k's) and the SpMV gathers are
      // in flight together: the partials are only summed after the SpMV
      double qa = 0.0, qb = 0.0, qc = 0.0;
      if (tid < G) {  // G <= kPcgThreads (one CTA per SM)
        const double2 ab = __ldcg(reinterpret_cast<const double2*>(part + 4 * tid));
        qa = ab.x;
        qb = ab.y;
        qc = __ldcg(part + 4 * tid + 2);
      }
      // n = (H + mu I) m  (same k -> thread map in slice_spmv's row pass and below);
      // computed before the stopping test -- unused on the last round
      slice_spmv(V, C, RP, bb0, nb, nr, pub, Mv, mu, IT, Nv);
      pcg_mark(a, 8 + 5 * it);
      cta_sum3<false>(qa, qb, qc, sh2[1]);
      pcg_mark(a, 9 + 5 * it);
      const double gamma = qa, delta = qb;
      rr = qc;
      if (it == 0) rr0 = rr;
      if (it >= a.max_iters || rr == 0.0 || (a.tol2 > 0.0 && rr <= a.tol2 * rr0)) break;
      const double beta = it > 0 ? gamma / gamma_old : 0.0;
      const double alpha = it > 0 ? gamma / (delta - beta * gamma / alpha_old) : gamma / delta;
      for (int k = tid; k < n6; k += kPcgThreads) {
        const double z = Nv[k] + beta * Zv[k];
        const double q = Mv[k] + beta * Qv[k];
        const double sv = W[k] + beta * Sv[k];
        const double p = U[k] + beta * Pv[k];
        Zv[k] = z;
        Qv[k] = q;
        Sv[k] = sv;
        Pv[k] = p;
        X[k] = X[k] + alpha * p;
        R[k] = R[k] - alpha * sv;
        U[k] = U[k] - alpha * q;
        W[k] = W[k] - alpha * z;
      }
      gamma_old = gamma;
      alpha_old = alpha;
    }
  } else {
    // classic: z = U (published in pub0), p_old / p_new published in pub1 /
    // pub2; consumers form p = z + beta p_old on the fly
    double* zpub = a.pub0;
    double* pold = a.pub1;
    double* pnew = a.pub2;
    double pz = 0.0, pr = 0.0, dz = 0.0;
    for (int k = tid; k < n6; k += kPcgThreads) {
      pz += R[k] * U[k];
      pr += R[k] * R[k];
      pold[6 * (size_t)r0 + k] = 0.0;
    }
    cta_sum3(pz, pr, dz, sh);
    if (tid == 0) {
      a.part[4 * blockIdx.x + 0] = pz;
      a.part[4 * blockIdx.x + 1] = pr;
    }
    grid.sync();
    double4 tot = grid_sum3(a.part, sh);
    double rz = tot.x, beta = 0.0;
    rr0 = rr = tot.y;
    for (; it < a.max_iters; ++it) {
      if (rr == 0.0 || (a.tol2 > 0.0 && rr <= a.tol2 * rr0)) break;
      // q = (H + mu I) p with p = z + beta p_old gathered at the column nodes
      for (int k = tid; k < 2 * nb; k += kPcgThreads) {
        const int blk = k >> 1, h3 = 3 * (k & 1);
        const int cidx = C[blk];
        const double2* zc = reinterpret_cast<const double2*>(zpub + 6 * (size_t)cidx);
        const double2* pc = reinterpret_cast<const double2*>(pold + 6 * (size_t)cidx);
        double pv[6];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const double2 zz = __ldcg(zc + t), pp = __ldcg(pc + t);
          pv[2 * t] = zz.x + beta * pp.x;
          pv[2 * t + 1] = zz.y + beta * pp.y;
        }
        const float* vr = V + 36 * (size_t)blk + 6 * h3;
#pragma unroll
        for (int rw = 0; rw < 3; ++rw) {
          double s = 0.0;
#pragma unroll
          for (int t = 0; t < 6; ++t) s += (double)vr[6 * rw + t] * pv[t];
          IT[6 * (size_t)blk + h3 + rw] = s;
        }
      }
      __syncthreads();
      double ppq = 0.0, d1 = 0.0, d2 = 0.0;
      for (int k = tid; k < n6; k += kPcgThreads) {
        const int i = k / 6, rw = k - 6 * i;
        const int lb0 = RP[i] - bb0, lb1 = RP[i + 1] - bb0;
        double t = 0.0;
        for (int b = lb0; b < lb1; ++b) t += IT[6 * (size_t)b + rw];
        const double pn = U[k] + beta * Pv[k];
        const double qv = t + mu * pn;
        Pv[k] = pn;
        pnew[6 * (size_t)r0 + k] = pn;
        Qv[k] = qv;
        ppq += pn * qv;
      }
      cta_sum3(ppq, d1, d2, sh);
      if (tid == 0) a.part[4 * blockIdx.x + 2] = ppq;
      grid.sync();
      tot = grid_sum3(a.part, sh);
      const double alpha = rz / tot.z;
      for (int k = tid; k < n6; k += kPcgThreads) {
        X[k] += alpha * Pv[k];
        R[k] = R[k] - alpha * Qv[k];
      }
      __syncthreads();
      double prz = 0.0, prr = 0.0, d3 = 0.0;
      apply_minv(MINV, R, U, nr);
      for (int k = tid; k < n6; k += kPcgThreads) {
        zpub[6 * (size_t)r0 + k] = U[k];
        prz += R[k] * U[k];
        prr += R[k] * R[k];
      }
      cta_sum3(prz, prr, d3, sh);
      if (tid == 0) {
        a.part[4 * blockIdx.x + 0] = prz;
        a.part[4 * blockIdx.x + 1] = prr;
      }
      grid.sync();
      tot = grid_sum3(a.part, sh);
      beta = tot.x / rz;
      rz = tot.x;
      rr = tot.y;
      double* t = pold;
      pold = pnew;
      pnew = t;
    }
  }
  bool bad = false;  // non-finite increment -> LM reject (solver.cpp:387)
  for (int k = tid; k < n6; k += kPcgThreads) {
    a.x[6 * (size_t)r0 + k] = X[k];
    bad |= !isfinite(X[k]);
  }
  if (bad) atomicExch(&a.sc->finite, 0);
  pcg_mark(a, 63);
  if (blockIdx.x == 0 && tid == 0) {
    a.sc->pcg_iters = it;
    a.sc->pcg_rr = rr;
    a.sc->pcg_rr0 = rr0;
  }
}

// Standalone BSR SpMV y = (H + mu I) x (the PCG's SpMV as its own kernel, for
// systems streamed from HBM). Warp per block row: one coalesced load brings
// the column indices of up to 5 G blocks of the row (lane i <- block i), then
// lanes = 5 blocks x 6 rows issue, for G groups of 5 blocks at once, the fp32
// value rows (float2) and the gathered x blocks (double2) before any product.
// Shuffle row reduction; block order within a lane is fixed (deterministic).
// Algorithmic bytes: 144 B per block + 4 B column index; row pointers + own x
// + y = 56 B per row; neighbour x blocks are L2-resident gathers.
// Measured (ncu, cold L2, N = 16k, 254k blocks): G = 2 beats G = 3, 4 (register
// growth costs more occupancy than the extra loads in flight buy) and beats
// TMA-staged tiles (the per-tile row search / staging adds a dependent round
// trip per row).
template <int kSpmvGroups>
__global__ void __launch_bounds__(256) k_bsr_spmv_rows(const int* __restrict__ row_ptr,
                                                       const int* __restrict__ col,
                                                       const float* __restrict__ val, int N,
                                                       double mu, const double* __restrict__ x,
                                                       double* __restrict__ y) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= N) return;
  const int rw = lane % 6, blk5 = lane / 6;
  const int b0 = row_ptr[j], b1 = row_ptr[j + 1];
  double acc = 0.0;
  for (int w0 = b0; w0 < b1; w0 += 5 * kSpmvGroups) {
    const int nbw = min(5 * kSpmvGroups, b1 - w0);
    const int cl = lane < nbw ? __ldcs(col + w0 + lane) : 0;
    float2 f[kSpmvGroups][3];
    double2 xv[kSpmvGroups][3];
#pragma unroll
    for (int g = 0; g < kSpmvGroups; ++g) {
      const int bi = g * 5 + blk5;
      const bool ok = lane < 30 && bi < nbw;
      const int cidx = __shfl_sync(0xffffffffu, cl, bi);
      const float2* vr = reinterpret_cast<const float2*>(val + (size_t)(w0 + bi) * 36 + rw * 6);
      const double2* xc = reinterpret_cast<const double2*>(x + 6 * (size_t)cidx);
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        f[g][t] = ok ? __ldcs(vr + t) : make_float2(0.f, 0.f);
        xv[g][t] = ok ? __ldg(xc + t) : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int g = 0; g < kSpmvGroups; ++g) {
      double sg = 0.0;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        sg += (double)f[g][t].x * xv[g][t].x;
        sg += (double)f[g][t].y * xv[g][t].y;
      }
      acc += sg;
    }
  }
  double tot = 0.0;
#pragma unroll
  for (int k = 0; k < 5; ++k) tot += __shfl_sync(0xffffffffu, acc, rw + 6 * k);
  if (lane < 6) y[6 * j + lane] = tot + mu * x[6 * j + lane];
}


}  // namespace

// ------------------------------------------------------------------ host side
// the "no record" block key: 2^bits - 1 with 2^bits > N^2 (sorts after every block)
int none_key(int N) {
  int bits = 1;
  while (bits < 31 && ((long long)1 << bits) <= (long long)N * N) ++bits;
  return (int)(((long long)1 << bits) - 1);
}

// a CTA per SM; small systems use fewer CTAs
int pcg_ctas(const Ctx& c) { return std::min(c.pcg_grid, std::max(1, cdiv(c.n_full, 64))); }

void build_pattern_enqueue(Ctx& c, int t_now, int t_last) {
  const int n_all = c.n_surfels, N = c.n_nodes;
  if ((long long)N * N >= 0x7fffffffLL) fail(DS_ERR_CAPACITY, "too many nodes for block keys");
  // eligible surfels (the only ones render_model_maps can pair this frame)
  int n = 0;
  if (n_all > 0) {
    // own flag: the pattern may be built concurrently with the rigid ICP, whose
    // model-map render computes dsc->any_stable
    const int* any_stable = c.any_stable_ready ? c.any_stable_pre : &c.dsc->any_stable_pat;
    if (!c.any_stable_ready) {
      DS_CUDA(cudaMemsetAsync(&c.dsc->any_stable_pat, 0, sizeof(int), c.stream));
      DS_LAUNCH(c, KK_PATTERN, 16.0 * n_all, cdiv(n_all, 256), 256, 0, k_any_stable_flag,
                c.M().ln, n_all, c.cfg.delta_stable, &c.dsc->any_stable_pat);
    }
    const int boot = (t_now - t_last <= c.cfg.delta_recent) ? 1 : 0;
    DS_LAUNCH(c, KK_PATTERN, 28.0 * n_all, cdiv(n_all, 256), 256, 0, k_elig_flags, c.M().ln,
              c.M().t, n_all, c.cfg.delta_stable, t_now, c.cfg.delta_recent, boot, any_stable,
              c.keep);
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
              N, key, val, none_key(N));
  if (N > 0)
    DS_LAUNCH(c, KK_PATTERN, 32.0 * 8 * N, cdiv(8 * N, 256), 256, 0, k_gen_reg_records, c.node_nbr,
              N, key + (size_t)n * 10, val + (size_t)n * 10, none_key(N));
  // block keys row * N + col < N^2; the "no record" key (2^bits - 1) sorts last.
  // Sorting only `bits` key bits saves radix passes (23 bits at N = 2.6k: 3 of 4)
  int end_bit = 1;
  while (end_bit < 31 && ((long long)1 << end_bit) <= (long long)N * N) ++end_bit;
  const int none = (int)(((long long)1 << end_bit) - 1);
  int *ks, *vs;
  sort_pairs(c, key, val, c.rec_key2, c.rec_val2, R, end_bit, &ks, &vs, KK_PATTERN);
  // keep the sorted arrays in rec_key/rec_val
  if (ks != c.rec_key) {
    std::swap(c.rec_key, c.rec_key2);
    std::swap(c.rec_val, c.rec_val2);
  }
  DS_LAUNCH(c, KK_PATTERN, 8.0 * R, cdiv(R, 256), 256, 0, k_mark_unique, c.rec_key, R, c.rec_flag,
            none);
  scan_exclusive(c, c.rec_flag, c.rec_flag, R);
  DS_CUDA(cudaMemsetAsync(&c.dsc->err, 0, sizeof(int), c.stream));
  DS_LAUNCH(c, KK_PATTERN, 12.0 * R, cdiv(R, 256), 256, 0, k_write_up, c.rec_key, c.rec_flag, R,
            c.up_key, c.up_start, c.UB_cap, &c.dsc->err, none);
  int* n_up_dev = c.rec_flag + R;
  DS_CUDA(cudaMemsetAsync(c.row_cnt, 0, sizeof(int) * (N + 1), c.stream));
  DS_LAUNCH(c, KK_PATTERN, 4.0 * c.UB_cap, cdiv(c.UB_cap, 256), 256, 0, k_row_count, c.up_key,
            n_up_dev, N, c.row_cnt);
  scan_exclusive(c, c.row_cnt, c.row_ptr, N);
  DS_CUDA(cudaMemsetAsync(c.row_cnt, 0, sizeof(int) * (N + 1), c.stream));
  // No host sync from here on: kernels take the device counts and run over
  // host-known bounds (ubb >= n_up); k_chunk_fill publishes the counts, which
  // pattern_adopt reads (capacity errors included) before the solve uses them.
  const int ubb = std::max(1, std::min(R, c.UB_cap));
  c.n_records = R;
  // regulariser records grouped by upper block (k_reg_blocks sums them per
  // GN iteration; the assembly adds the sums)
  c.reg_cap_now = 24 * N;
  if (N > 0) {
    DS_LAUNCH(c, KK_PATTERN, 12.0 * R, cdiv(R, 256), 256, 0, k_reg_mark, c.rec_key, c.rec_val, R,
              none, c.rec_key2);
    scan_exclusive(c, c.rec_key2, c.rec_val2, R);
    DS_LAUNCH(c, KK_PATTERN, 12.0 * R, cdiv(R, 256), 256, 0, k_reg_compact, c.rec_key2, c.rec_val2,
              R, c.rec_val, c.rec_flag, c.reg_rec, c.reg_ub);
    DS_LAUNCH(c, KK_PATTERN, 12.0 * c.reg_cap_now, cdiv(c.reg_cap_now, 256), 256, 0, k_reg_bmark,
              c.reg_ub, c.rec_val2 + R, c.reg_cap_now, c.reg_bf);
    scan_exclusive(c, c.reg_bf, c.reg_bscan, c.reg_cap_now);
    DS_CUDA(cudaMemsetAsync(c.ub_reg, 0xff, sizeof(int) * ubb, c.stream));
    DS_LAUNCH(c, KK_PATTERN, 16.0 * c.reg_cap_now, cdiv(c.reg_cap_now, 256), 256, 0, k_reg_bfill,
              c.reg_ub, c.reg_bf, c.reg_bscan, c.rec_val2 + R, c.reg_cap_now, c.reg_blk_start,
              c.ub_reg);
  }
  DS_LAUNCH(c, KK_PATTERN, 16.0 * ubb, cdiv(ubb, 256), 256, 0, k_row_fill, c.up_key, n_up_dev, N,
            c.row_ptr, c.row_cnt, c.bsr_col, c.bsr_tag, c.UB_cap, c.B_cap);
  DS_LAUNCH(c, KK_PATTERN, 32.0 * ubb, cdiv((long long)N * 32, 256), 256, 0, k_row_sort, c.row_ptr, N,
            c.bsr_col, c.bsr_tag, c.up_pos, c.up_mpos, c.diag_pos, c.B_cap);
  if (c.n_pairs_ok_est <= 0) c.n_pairs_ok_est = 0.4 * c.P;
  // fixed-size record chunks for the assembly (per frame)
  DS_LAUNCH(c, KK_PATTERN, 12.0 * ubb, cdiv(ubb, 256), 256, 0, k_chunk_count, c.up_start, n_up_dev,
            ubb, c.chunk_first, c.multi_flag);
  scan_exclusive(c, c.chunk_first, c.chunk_first, ubb);
  scan_exclusive(c, c.multi_flag, c.multi_scan, ubb);
  DS_LAUNCH(c, KK_PATTERN, 8.0 * ubb, cdiv(ubb, 256), 256, 0, k_multi_list, c.multi_flag,
            c.multi_scan, ubb, c.multi_list);
  DS_LAUNCH(c, KK_PATTERN, 40.0 * ubb, cdiv(ubb, 256), 256, 0, k_chunk_fill, c.chunk_first, n_up_dev,
            c.up_key, c.up_start, c.up_pos, c.up_mpos, c.ub_reg, N, c.row_ptr, c.multi_scan,
            c.UB_cap, c.B_cap, c.CH_cap, &c.dsc->err, c.dsc, c.chunk_ub, c.chunk_d0, c.chunk_d1);
  c.pattern_pending = true;
}

// Adopt the enqueued pattern's counts: from the scalars the caller already
// fetched (have_scalars, e.g. the rigid ICP's fetch after the side branch
// joined), else with a fetch here. Then the PCG slices for its grid.
void pattern_adopt(Ctx& c, bool have_scalars) {
  if (!c.pattern_pending) return;
  if (!have_scalars) fetch_scalars(c);
  c.pattern_pending = false;
  const DevScalars& h = *c.hsc;
  if (h.pat_err) fail(DS_ERR_CAPACITY, "JtJ block / assembly chunk capacity exceeded");
  c.n_up = h.pat_n_up;
  c.n_full = h.pat_n_full;
  c.n_chunks = h.pat_n_chunks;
  c.n_multi = h.pat_n_multi;
  DS_LAUNCH(c, KK_PATTERN, 16.0 * pcg_ctas(c), cdiv(pcg_ctas(c), 128), 128, 0, k_pcg_slices,
            c.row_ptr, c.n_nodes, pcg_ctas(c), c.pcg_slices);
  c.pattern_ready = true;
}

void build_pattern(Ctx& c, int t_now, int t_last) {
  build_pattern_enqueue(c, t_now, t_last);
  pattern_adopt(c, false);
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
void gn_linearize_async(Ctx& c, const double* pose, int t_now, int t_last, bool lm_floor,
                        bool maps_clean = false) {
  const int n = c.n_surfels, N = c.n_nodes, P = c.P;
  // fork: the pair-list resets (needed by the association kernel) and the node
  // transforms + E_reg (needed only by the assembly) run on a side branch,
  // concurrently with the warp + splat passes
  const int nbp = cdiv(P, 256);
  DS_CUDA(cudaEventRecord(c.ev_fork, c.stream));
  DS_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
  {
    cudaStream_t main_stream = c.stream;
    c.stream = c.side;
    try {
      DS_CUDA(cudaMemsetAsync(c.s_cnt, 0, sizeof(int) * (n + 1), c.stream));
      DS_CUDA(cudaMemsetAsync(c.s_head, 0x7f, sizeof(int) * (n + 1), c.stream));
      DS_CUDA(cudaMemsetAsync(c.s_fill, 0, sizeof(int) * (n + 1), c.stream));
      DS_CUDA(cudaMemsetAsync(c.s_base, 0xff, sizeof(int) * (n + 1), c.stream));
      DS_CUDA(cudaMemsetAsync(&c.dsc->pair_list_n, 0, sizeof(int), c.stream));
      DS_CUDA(cudaMemsetAsync(&c.dsc->n_pairs, 0, sizeof(int), c.stream));
      DS_CUDA(cudaMemsetAsync(c.pair_ok, 0, P, c.stream));
      DS_CUDA(cudaEventRecord(c.ev_mid, c.stream));
      DS_CUDA(cudaMemsetAsync(c.g, 0, sizeof(double) * 6 * N, c.stream));  // assembly output
      node_se3(c, c.node_dq, c.node_se3);
      DS_LAUNCH(c, KK_ENERGY, 200.0 * N, cdiv(8 * N, 256), 256, 0, k_reg_energy, c.node_pos,
                c.node_nbr, c.node_se3, N, c.red_part + nbp, c.tickets + 1, &c.dsc->e_reg_pre,
                c.reg_ab);
      if (N > 0)
        DS_LAUNCH(c, KK_ENERGY, 48.0 * c.reg_cap_now, cdiv(6LL * reg_rb_pad(N), 256), 256, 0,
                  k_reg_blocks, c.reg_rec, c.reg_blk_start, c.reg_bscan + c.reg_cap_now,
                  reg_rb_pad(N), c.reg_ab, c.cfg.lambda, c.reg_h, c.reg_g);
    } catch (...) {
      c.stream = main_stream;
      throw;
    }
    c.stream = main_stream;
    DS_CUDA(cudaEventRecord(c.ev_join, c.side));
  }
  // only render-eligible surfels can be drawn / paired during the solve (the
  // post-solve forward_warp, pipeline.cpp:108, rewrites every live surfel):
  // warp + splat pass 1 fused, splat pass 2, then resolve + associate + terms
  render_model_maps_list(c, pose, t_now, t_last, pose, c.elig, c.n_elig, c.node_dq, false,
                         !maps_clean);
  DS_CUDA(cudaStreamWaitEvent(c.stream, c.ev_mid, 0));  // pair-list resets done
  // per pixel: 2 x 4 B winner ids, frame maps 65 B, winner live 32 B, ids out 8 B; per pair:
  // surfel ref + skin 48 B, rows 96 B + r 8 B out
  DS_LAUNCH_PDL(c, KK_PAIR_TERMS, 113.0 * P + 152.0 * c.n_pairs_ok_est, cdiv(P, 256 * kPairPix), 256, 0,
            k_assoc_pair_terms, c.mm_pidx, c.mm_sidx, c.mm_pkey, c.mm_skey, c.f_flag, c.M(), c.node_dq, c.f_vert,
            c.f_nrm, pair_params(c, pose), c.mm_idx, c.pair_s, &c.dsc->n_pairs, c.pair_ok,
            c.pair_rows, c.pair_r, c.s_cnt, c.s_head, c.red_part, c.tickets + 0,
            &c.dsc->e_data_pre);
  c.mm_clean = true;  // k_assoc_pair_terms resets the z-buffer entries it consumed
  DS_LAUNCH_PDL(c, KK_PAIR_LISTS, 9.0 * P, nbp, 256, 0, k_pair_fill, c.pair_s, c.pair_ok, P, c.s_cnt,
                c.s_base, c.s_fill, c.p_list, &c.dsc->pair_list_n);
  DS_LAUNCH_PDL(c, KK_PAIR_LISTS, 13.0 * P, nbp, 256, 0, k_pair_next, c.pair_s, c.pair_ok, P, c.s_cnt,
            c.s_base, c.p_list, c.p_next);
  DS_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));  // join
  AsmArgs A;
  A.up_key = c.up_key;
  A.up_start = c.up_start;
  A.up_pos = c.up_pos;
  A.up_mpos = c.up_mpos;
  A.chunk_ub = c.chunk_ub;
  A.chunk_first = c.chunk_first;
  A.chunk_d0 = c.chunk_d0;
  A.chunk_d1 = c.chunk_d1;
  A.rec_val = c.rec_val;
  A.s_cnt = c.s_cnt;
  A.s_head = c.s_head;
  A.p_next = c.p_next;
  A.rows = c.pair_rows;
  A.pair_r = c.pair_r;
  A.node_pos = c.node_pos;
  A.nbr = c.node_nbr;
  A.se3 = c.node_se3;
  A.reg_ab = c.reg_ab;
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
  A.ub_reg = c.ub_reg;
  A.reg_h = c.reg_h;
  A.reg_g = c.reg_g;
  if (c.n_up > 0) {
    // algorithmic bytes: 80 B per pair (pair 32 + reference
    // position 16 + skinning ids 16 + weights 16) + 144 B per 6x6 block written
    // + 24 B per node (g). (Round 1 counted this kernel's own intermediates --
    // 12 B per record, 104 B rows per pair, 400 B per chunk partial -- which
    // overstated its roofline fraction ~3x.)
    const double bytes = 80.0 * c.n_pairs_ok_est + 144.0 * c.n_full + 24.0 * N;
    DS_LAUNCH_PDL(c, KK_BLOCK_ASSEMBLY, bytes, cdiv((long long)c.n_chunks * kChunkLanes, 256), 256, 0,
              k_assemble_chunks, A);
    if (c.n_multi > 0)
      DS_LAUNCH_PDL(c, KK_REDUCE, 0.0, cdiv((long long)c.n_multi * kFinishEntries, 256), 256, 0,
                k_assemble_finish, A, c.multi_list, c.multi_scan + c.n_up);
  }
  DS_LAUNCH_PDL(c, KK_REDUCE, 48.0 * N + 24.0 * N, std::max(1, cdiv(N, kStatsThreads)), kStatsThreads, 0,
            k_g_stats, c.g, c.bsr_val, c.diag_pos, N, lm_floor ? 1 : 0, c.gst_part, c.tickets + 2,
            c.dsc);
  if (c.check_ne) check_normal_equations_async(c);  // DS_CHECK_NE (debug)
}

void gn_linearize(Ctx& c, const double* pose, int t_now, int t_last, double* e_pre, int* n_pairs) {
  if (!c.pattern_ready) build_pattern(c, t_now, t_last);
  gn_linearize_async(c, pose, t_now, t_last, false);
  fetch_scalars(c);
  if (e_pre) *e_pre = c.hsc->e_data_pre + c.cfg.lambda * c.hsc->e_reg_pre;
  if (n_pairs) *n_pairs = c.hsc->n_pairs;
}

// PCG on the last assembled system with the damping in dsc->mu
void pcg_solve_async(Ctx& c, int max_iters, double tol) {
  // one thread-block cluster when the system is small enough (k_pcg_cluster.cu)
  if (pcg_cluster_launch(c, max_iters, tol)) return;
  const int N = c.n_nodes;
  PcgArgs a;
  a.row_ptr = c.row_ptr;
  a.col = c.bsr_col;
  a.val = c.bsr_val;
  a.diag_pos = c.diag_pos;
  a.g = c.g;
  a.mu_ptr = &c.dsc->mu;
  a.N = N;
  a.nnzb = c.n_full;
  a.max_iters = max_iters;
  a.tol2 = tol > 0 ? tol * tol : 0.0;
  a.x = c.pcg_x;
  a.pub0 = c.pcg_p0;
  a.pub1 = c.pcg_p1;
  a.pub2 = c.pcg_p2;
  a.minv = c.pcg_minv;
  a.vec = c.pcg_vec;
  a.items = c.pcg_items;
  a.part = c.pcg_part;
  a.slices = c.pcg_slices;
  a.smem_cap = std::min(c.pcg_smem_cap, kPcgSmem);
  a.trace = c.pcg_trace;
  a.sc = c.dsc;
  const int grid = pcg_ctas(c);
  void* args[] = {&a};
  launch_begin(c, KK_PCG);
  void* fn = a.tol2 > 0.0 ? (void*)k_pcg<false> : (void*)k_pcg<true>;
  DS_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kPcgThreads), args, kPcgSmem, c.stream));
  // algorithmic bytes per PCG: per iteration one BSR SpMV
  // (148 B/block + 4 B row pointers + 48 B x/y per node) + ~10 vector passes
  // (240 B per node)
  launch_end(c, KK_PCG, std::max(1, max_iters) * (148.0 * c.n_full + 292.0 * N + 4.0));

}

namespace {
// ---- assert_normal_equations (solver.cpp:157-167) on the device
// scale = max(1, max|H|): |H| as fp32 bits (non-negative floats order as ints)
__global__ void k_ne_scale(const float* __restrict__ val, long long n, unsigned* __restrict__ bits) {
  pdl_wait();
  unsigned m = 0u;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x)
    m = max(m, __float_as_uint(fabsf(val[k])));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(bits, m);
}
// symmetry: block (r, c) against its mirror (c, r), thread per block
__global__ void k_ne_symmetry(const int* __restrict__ row_ptr, const int* __restrict__ col,
                              const float* __restrict__ val, int N, DevScalars* sc) {
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (r >= N) return;
  const double scale = fmax(1.0, (double)__uint_as_float(sc->ne_scale_bits));
  bool bad = false;
  for (int a = row_ptr[r] + lane; a < row_ptr[r + 1]; a += 32) {
    const int cc = col[a];
    int lo = row_ptr[cc], hi = row_ptr[cc + 1];  // rows are column-sorted
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (col[mid] < r) lo = mid + 1;
      else hi = mid;
    }
    if (lo >= row_ptr[cc + 1] || col[lo] != r) {
      bad = true;  // the mirror block is missing
      continue;
    }
    for (int t = 0; t < 36; ++t) {
      const double d = (double)val[(size_t)a * 36 + t] - (double)val[(size_t)lo * 36 + (t % 6) * 6 + t / 6];
      if (fabs(d) > 1e-9 * scale) bad = true;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&sc->ne_err, NE_ASYMMETRIC);
}
// diagonal blocks PSD: smallest eigenvalue (cyclic Jacobi, fp64) >= -1e-8 scale
__global__ void k_ne_psd(const int* __restrict__ diag_pos, const float* __restrict__ val, int N,
                         DevScalars* sc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  const int d = diag_pos[j];
  double a[6][6];
  for (int x = 0; x < 6; ++x)
    for (int y = 0; y < 6; ++y) a[x][y] = d >= 0 ? (double)val[(size_t)d * 36 + x * 6 + y] : 0.0;
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 6; ++p)
      for (int q = p + 1; q < 6; ++q) off += a[p][q] * a[p][q];
    if (off < 1e-30) break;
    for (int p = 0; p < 6; ++p)
      for (int q = p + 1; q < 6; ++q) {
        if (a[p][q] == 0.0) continue;
        const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < 6; ++k) {
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = cs * akp - sn * akq;
          a[k][q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < 6; ++k) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = cs * apk - sn * aqk;
          a[q][k] = sn * apk + cs * aqk;
        }
      }
  }
  double mn = a[0][0];
  for (int k = 1; k < 6; ++k) mn = fmin(mn, a[k][k]);
  const double scale = fmax(1.0, (double)__uint_as_float(sc->ne_scale_bits));
  if (mn < -1e-8 * scale) atomicOr(&sc->ne_err, NE_NOT_PSD);
}
}  // namespace

void check_normal_equations_async(Ctx& c) {
  const int N = c.n_nodes;
  DS_CUDA(cudaMemsetAsync(&c.dsc->ne_scale_bits, 0, sizeof(unsigned), c.stream));
  DS_LAUNCH(c, KK_MISC, 144.0 * c.n_full, 2 * c.num_sms, 256, 0, k_ne_scale, c.bsr_val,
            36LL * c.n_full, &c.dsc->ne_scale_bits);
  DS_LAUNCH(c, KK_MISC, 288.0 * c.n_full, cdiv(N, 8), 256, 0, k_ne_symmetry, c.row_ptr, c.bsr_col,
            c.bsr_val, N, c.dsc);
  DS_LAUNCH(c, KK_MISC, 144.0 * N, cdiv(N, 128), 128, 0, k_ne_psd, c.diag_pos, c.bsr_val, N, c.dsc);
}

void check_normal_equations(Ctx& c) {
  DS_CUDA(cudaMemsetAsync(&c.dsc->ne_err, 0, sizeof(int), c.stream));
  check_normal_equations_async(c);
  fetch_scalars(c);
  if (c.hsc->ne_err & NE_ASYMMETRIC) fail(DS_ERR_NUMERICAL, "normal equations lost symmetry");
  if (c.hsc->ne_err & NE_NOT_PSD) fail(DS_ERR_NUMERICAL, "normal equations diagonal block not PSD");
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
  const int nbp = cdiv(P, 256 * kEnergyPix), nbe = cdiv(8 * N, 256);
  // the node transforms `se3` of `dq` are written by apply_increments (fused)
  DS_LAUNCH_PDL(c, KK_ENERGY, 120.0 * c.n_pairs_ok_est + 200.0 * N, nbp + nbe, 256, 0, k_energy,
            c.pair_s, c.M(), dq, c.f_vert, c.f_nrm, pair_params(c, pose), c.node_pos, c.node_nbr,
            se3, N, nbp, c.red_part, c.tickets, &c.dsc->e_data, &c.dsc->e_reg);
}
}  // namespace

namespace {
// one GN iteration up to the first LM attempt: linearise, mu, PCG, candidate, E_post
void gn_step_async(Ctx& c, const double* pose, int t_now, int t_last, int max_pcg, double tol) {
  gn_linearize_async(c, pose, t_now, t_last, true);  // + LM floor on mu
  pcg_solve_async(c, max_pcg, tol);
  apply_increments(c, c.pcg_x, c.node_dq_cand, c.node_se3_cand);
  energy_async(c, pose, c.node_dq_cand, c.node_se3_cand);
}
void attempt_async(Ctx& c, const double* pose, int max_pcg, double tol) {
  pcg_solve_async(c, max_pcg, tol);
  apply_increments(c, c.pcg_x, c.node_dq_cand, c.node_se3_cand);
  energy_async(c, pose, c.node_dq_cand, c.node_se3_cand);
}

// ------------------------------------------------------ device-resident LM
// The LM loop of solver.cpp:296-406 as device state, one decision per attempt
// (same arithmetic as the host loop below): a WHILE graph node repeats
// [IF(relinearise) {linearise + mu floor}; PCG; candidate; E_post; decide].
struct LmParams {
  double lambda, tol;
  int max_gn_iters, N;
  cudaGraphConditionalHandle h_loop, h_relin;
};

__global__ void k_lm_init(DevScalars* sc) {
  sc->mu = 0.0;  // solver.cpp:313
  sc->lm_iter = 0;
  sc->lm_attempt = 0;
  sc->lm_relin = 1;
  sc->lm_done = 0;
  sc->lm_accepted = 0;
  sc->lm_attempts_total = 0;
  sc->pcg_iter_total = 0;
  sc->lm_rounds = 0;
  sc->lm_relins = 0;
  sc->lm_pairs = 0;
  sc->lm_initial = 0.0;
  sc->lm_final = 0.0;
}

__global__ void __launch_bounds__(1024) k_lm_decide(DevScalars* sc, LmParams lp,
                                                   double4* __restrict__ node_dq,
                                                   const double4* __restrict__ node_dq_cand) {
  pdl_wait();  // programmatic dependent launch: predecessor results visible
  __shared__ int s_acc;
  if (threadIdx.x == 0) {
    ++sc->lm_rounds;
    bool done = false, accepted = false;
    double mu = sc->mu;
    const double floor_ = sc->mu_floor;
    if (sc->lm_relin) {  // a GN iteration started this round (solver.cpp:316-379)
      ++sc->lm_relins;
      const double e_pre = sc->e_data_pre + lp.lambda * sc->e_reg_pre;
      sc->lm_e_pre = e_pre;
      sc->lm_pairs = sc->n_pairs;
      if (sc->lm_iter == 0) {
        sc->lm_initial = e_pre;
        sc->lm_final = e_pre;
      }
      sc->lm_gnorm = sqrt(sc->g_sq);
      sc->lm_attempt = 0;
      if (sc->ginf < 1e-14) done = true;  // stationary: the attempt is discarded
    }
    if (!done) {
      ++sc->lm_attempts_total;
      sc->pcg_iter_total += sc->pcg_iters;
      const bool finite = sc->finite != 0;
      const double rr = sqrt(sc->pcg_rr), rr0 = sqrt(sc->pcg_rr0);
      const bool guard_fail = lp.tol > 0 && rr > 1e-6 * (sc->lm_gnorm + 1.0) && rr > lp.tol * rr0;
      double e_post = 0.0;
      if (!finite || guard_fail) {
        mu = fmax(floor_, mu * 10.0);
      } else {
        e_post = sc->e_data + lp.lambda * sc->e_reg;
        if (e_post <= sc->lm_e_pre) accepted = true;
        else mu = fmax(floor_, mu * 10.0);
      }
      ++sc->lm_attempt;
      if (accepted) {
        mu = fmax(floor_, mu * 0.1);
        ++sc->lm_accepted;
        sc->lm_final = e_post;
        ++sc->lm_iter;
        const double e_pre = sc->lm_e_pre;
        done = (e_pre - e_post < 1e-4 * fmax(e_pre, 1e-300)) || sc->lm_iter >= lp.max_gn_iters;
      } else if (sc->lm_attempt >= 8) {
        done = true;  // no acceptable step (solver.cpp:403)
      }
    }
    sc->mu = mu;
    sc->lm_relin = accepted ? 1 : 0;
    sc->lm_done = done ? 1 : 0;
    cudaGraphSetConditional(lp.h_loop, done ? 0u : 1u);
    cudaGraphSetConditional(lp.h_relin, accepted ? 1u : 0u);
    s_acc = accepted ? 1 : 0;
  }
  __syncthreads();
  if (s_acc)  // T <- T_cand (solver.cpp:399)
    for (int k = threadIdx.x; k < 2 * lp.N; k += blockDim.x) node_dq[k] = node_dq_cand[k];
}

// Build the per-frame solve graph: WHILE(loop) { IF(relin) {linearise}; attempt; decide }.
// mean |r| at the final nodes over the last pair set (solver.cpp:409-420)
void report_async(Ctx& c, const double* pose) {
  const int nbp = cdiv(c.P, 256);
  DS_CUDA(cudaMemsetAsync(&c.dsc->mean_cnt, 0, sizeof(int), c.stream));
  DS_LAUNCH(c, KK_ENERGY, 120.0 * c.P * 0.5, nbp, 256, 0, k_pair_energy, c.pair_s, c.M(), c.node_dq,
            c.f_vert, c.f_nrm, pair_params(c, pose), 1, c.red_part, &c.dsc->mean_cnt,
            c.tickets + 0, &c.dsc->mean_abs_r);
}

bool build_solve_graph(Ctx& c, const double* pose, int t_now, int t_last, int max_pcg,
                       double tol) {
  cudaGraph_t g = nullptr;
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return false;
  bool ok = true;
  const int64_t l0 = c.total_launches;
  auto fail_ = [&]() {
    cudaGetLastError();
    c.total_launches = l0;
    if (g) cudaGraphDestroy(g);
    return false;
  };
  cudaGraphConditionalHandle h_loop, h_relin;
  if (cudaGraphConditionalHandleCreate(&h_loop, g, 1, cudaGraphCondAssignDefault) != cudaSuccess)
    return fail_();
  cudaGraphNodeParams pw = {};
  pw.type = cudaGraphNodeTypeConditional;
  pw.conditional.handle = h_loop;
  pw.conditional.type = cudaGraphCondTypeWhile;
  pw.conditional.size = 1;
  cudaGraphNode_t wnode;
  if (cudaGraphAddNode(&wnode, g, nullptr, 0, &pw) != cudaSuccess) return fail_();
  cudaGraph_t body = pw.conditional.phGraph_out[0];
  if (cudaGraphConditionalHandleCreate(&h_relin, body, 1, cudaGraphCondAssignDefault) != cudaSuccess)
    return fail_();
  cudaGraphNodeParams pi = {};
  pi.type = cudaGraphNodeTypeConditional;
  pi.conditional.handle = h_relin;
  pi.conditional.type = cudaGraphCondTypeIf;
  pi.conditional.size = 1;
  cudaGraphNode_t inode;
  if (cudaGraphAddNode(&inode, body, nullptr, 0, &pi) != cudaSuccess) return fail_();
  cudaGraph_t lin = pi.conditional.phGraph_out[0];
  cudaGraph_t tmp = nullptr;
  // linearisation round
  if (cudaStreamBeginCaptureToGraph(c.stream, lin, nullptr, nullptr, 0,
                                    cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return fail_();
  try {
    // maps are cleared before the graph launch and reset by their consumer
    gn_linearize_async(c, pose, t_now, t_last, true, true);
  } catch (...) {
    cudaStreamEndCapture(c.stream, &tmp);
    fail_();
    throw;
  }
  ok = cudaStreamEndCapture(c.stream, &tmp) == cudaSuccess;
  const int64_t k_lin = c.total_launches - l0;
  if (!ok) return fail_();
  // attempt + decision
  if (cudaStreamBeginCaptureToGraph(c.stream, body, &inode, nullptr, 1,
                                    cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return fail_();
  LmParams lp;
  lp.lambda = c.cfg.lambda;
  lp.tol = tol;
  lp.max_gn_iters = c.cfg.max_gn_iters;
  lp.N = c.n_nodes;
  lp.h_loop = h_loop;
  lp.h_relin = h_relin;
  try {
    pcg_solve_async(c, max_pcg, tol);
    apply_increments(c, c.pcg_x, c.node_dq_cand, c.node_se3_cand);
    energy_async(c, pose, c.node_dq_cand, c.node_se3_cand);
    DS_LAUNCH_PDL(c, KK_MISC, 64.0 * 2 * c.n_nodes, 1, 1024, 0, k_lm_decide, c.dsc, lp, c.node_dq,
              c.node_dq_cand);
  } catch (...) {
    cudaStreamEndCapture(c.stream, &tmp);
    fail_();
    throw;
  }
  ok = cudaStreamEndCapture(c.stream, &tmp) == cudaSuccess;
  if (!ok) return fail_();
  const int64_t k_round = c.total_launches - l0 - k_lin;
  // the report as the graph's last node, after the loop: one host sync per solve
  if (cudaStreamBeginCaptureToGraph(c.stream, g, &wnode, nullptr, 1,
                                    cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return fail_();
  try {
    report_async(c, pose);
  } catch (...) {
    cudaStreamEndCapture(c.stream, &tmp);
    fail_();
    throw;
  }
  ok = cudaStreamEndCapture(c.stream, &tmp) == cudaSuccess;
  if (!ok) return fail_();
  c.g_solve.kernels_lin = k_lin;
  c.g_solve.kernels = k_round;
  c.g_solve.kernels_tail = c.total_launches - l0 - k_lin - k_round;
  c.total_launches = l0;
  if (c.g_solve.exec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(c.g_solve.exec, g, &info) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphExecDestroy(c.g_solve.exec);
      c.g_solve.exec = nullptr;
    }
  }
  if (!c.g_solve.exec && cudaGraphInstantiate(&c.g_solve.exec, g, 0) != cudaSuccess) {
    cudaGetLastError();
    c.g_solve.exec = nullptr;
    cudaGraphDestroy(g);
    return false;
  }
  cudaGraphDestroy(g);
  return true;
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
  const auto tp0 = std::chrono::steady_clock::now();
  if (c.pattern_frame != t_now) build_pattern(c, t_now, t_last);
  c.pattern_frame = -1;
  if (c.check_ne) DS_CUDA(cudaMemsetAsync(&c.dsc->ne_err, 0, sizeof(int), c.stream));
  if (c.trace_host)
    std::fprintf(stderr, "build_pattern %.1f us\n",
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tp0)
                     .count());
  const int max_pcg = c.cfg.pcg_max_iters > 0 ? c.cfg.pcg_max_iters : 10;
  const double tol = c.cfg.pcg_tol;
  const bool graphs = c.use_graphs && !c.cfg.profile;
  int n_pairs = 0;
  bool report_done = false;
  if (graphs && c.device_lm && c.cfg.max_gn_iters > 0) {
    // the whole LM loop on the device: one graph launch, one host sync
    DS_LAUNCH(c, KK_MISC, 64.0, 1, 1, 0, k_lm_init, c.dsc);
    const auto tb0 = std::chrono::steady_clock::now();
    const bool clean_before = c.mm_clean;  // the capture's bookkeeping is not the stream's
    const bool built = build_solve_graph(c, pose, t_now, t_last, max_pcg, tol);
    c.mm_clean = clean_before;
    if (c.trace_host)
      std::fprintf(stderr, "solve graph build %.1f us\n",
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tb0)
                       .count());
    if (built) {
      if (!c.mm_clean) clear_model_maps(c);
      DS_CUDA(cudaGraphLaunch(c.g_solve.exec, c.stream));
      c.mm_clean = true;  // every linearisation's consumer resets the maps
      fetch_scalars(c);
      const DevScalars& h = *c.hsc;
      c.total_launches += c.g_solve.kernels_lin * h.lm_relins + c.g_solve.kernels * h.lm_rounds +
                          c.g_solve.kernels_tail;
      report_done = true;  // captured as the graph's last node
      c.lm_attempts = h.lm_attempts_total;
      c.pcg_iterations = h.pcg_iter_total;
      rep.iterations = h.lm_accepted;
      rep.initial_energy = h.lm_initial;
      rep.final_energy = h.lm_final;
      n_pairs = h.lm_pairs;
      c.n_pairs_ok_est = n_pairs;
      goto report;
    }
  }
  {
  bool have_step = false, have_attempt = false;
  double mu = 0.0;
  set_mu(c, 0.0);
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
  }
report:
  rep.correspondences = n_pairs;
  if (!report_done) {  // host LM path
    report_async(c, pose);
    fetch_scalars(c);
  }
  if (c.check_ne && c.hsc->ne_err) {  // assert_normal_equations (solver.cpp:375)
    if (c.hsc->ne_err & NE_ASYMMETRIC) fail(DS_ERR_NUMERICAL, "normal equations lost symmetry");
    fail(DS_ERR_NUMERICAL, "normal equations diagonal block not PSD");
  }
  rep.mean_residual = c.hsc->mean_cnt > 0 ? c.hsc->mean_abs_r / c.hsc->mean_cnt : 0.0;
  *out = rep;
}

// y = (H + mu I) x on the assembled BSR system, `reps` times; returns mean ms
// HBM-streaming BSR SpMV y = (H + mu I) x with the matrix staged by the TMA
// engine: CTA b owns block rows [16 b, 16 b + 16); one thread issues bulk
// async copies of the rows' contiguous fp32 blocks (144 B each) and column
// indices into shared memory (mbarrier completion), so the matrix streams at
// copy-engine bandwidth with 4 CTAs per SM in flight; then warp per row (lane
// = 5 blocks x 6 rows, as k_bsr_spmv_rows) from shared memory, x gathered
// through L1/L2. Blocks past the staging capacity (very dense rows) are read
// from global memory. Algorithmic bytes: 148 B per block + 56 B per row.
// Opt-in (DS_SPMV_TMA=1): measured at config 4 (16k nodes, 254k blocks, cold
// L2) 31.3 us against 22.0 us for k_bsr_spmv_rows -- each CTA serialises row
// pointers -> bulk copy -> compute, and 1.2 waves leave the copy engine idle
// in the compute phases (a persistent double-buffered variant would be next).
constexpr int kSpmvTmaRows = 16;
constexpr int kSpmvTmaCap = 320;  // staged blocks per CTA (46 KB + columns)
constexpr int kSpmvTmaSmem = kSpmvTmaCap * 144 + (kSpmvTmaCap + 8) * 4;
__global__ void __launch_bounds__(256, 4) k_bsr_spmv_tma(const int* __restrict__ row_ptr,
                                                        const int* __restrict__ col,
                                                        const float* __restrict__ val, int N,
                                                        double mu, const double* __restrict__ x,
                                                        double* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) unsigned long long s_bar;
  float* V = reinterpret_cast<float*>(smem);
  int* Cs = reinterpret_cast<int*>(smem + kSpmvTmaCap * 144);
  const int r0 = blockIdx.x * kSpmvTmaRows, r1 = min(N, r0 + kSpmvTmaRows);
  const int bb0 = __ldg(row_ptr + r0), bb1 = __ldg(row_ptr + r1);
  const int staged = min(bb1 - bb0, kSpmvTmaCap);
  // the column copy starts on a 16 B boundary (bulk copies need it)
  const int c0 = bb0 & ~3, c1 = (bb0 + staged + 3) & ~3;
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&s_bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const unsigned vbytes = 144u * (unsigned)staged, cbytes = 4u * (unsigned)(c1 - c0);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar),
                 "r"(vbytes + cbytes)
                 : "memory");
    if (vbytes)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              (unsigned)__cvta_generic_to_shared(V)),
          "l"(val + 36 * (size_t)bb0), "r"(vbytes), "r"(bar)
          : "memory");
    if (cbytes)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              (unsigned)__cvta_generic_to_shared(Cs)),
          "l"(col + c0), "r"(cbytes), "r"(bar)
          : "memory");
  }
  __syncthreads();  // barrier initialised before anyone waits on it
  {
    unsigned done = 0;
    while (!done)
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(bar)
          : "memory");
  }
  const int* Cl = Cs + (bb0 - c0);
  const int lane = threadIdx.x & 31, rw = lane % 6, blk5 = lane / 6;
  for (int j = r0 + (threadIdx.x >> 5); j < r1; j += 8) {
    const int b0 = __ldg(row_ptr + j) - bb0, b1 = __ldg(row_ptr + j + 1) - bb0;
    double acc = 0.0;
    for (int w0 = b0; w0 < b1; w0 += 10) {
      float2 f[2][3];
      double2 xv[2][3];
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int bi = w0 + g * 5 + blk5;
        const bool ok = lane < 30 && bi < b1;
        const int cidx = ok ? (bi < staged ? Cl[bi] : __ldg(col + bb0 + bi)) : 0;
        const float2* vr = reinterpret_cast<const float2*>(
            (bi < staged ? V + 36 * bi : val + 36 * ((size_t)bb0 + bi)) + 6 * rw);
        const double2* xc = reinterpret_cast<const double2*>(x + 6 * (size_t)cidx);
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          f[g][t] = ok ? vr[t] : make_float2(0.f, 0.f);
          xv[g][t] = ok ? __ldg(xc + t) : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        double sg = 0.0;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          sg += (double)f[g][t].x * xv[g][t].x;
          sg += (double)f[g][t].y * xv[g][t].y;
        }
        acc += sg;
      }
    }
    double tot = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) tot += __shfl_sync(0xffffffffu, acc, rw + 6 * k);
    if (lane < 6) y[6 * j + lane] = tot + mu * x[6 * j + lane];
  }
}

// Persistent, double-buffered variant (DS_SPMV_TMA=2): 2 CTAs per SM, each
// walking tiles of kSpmvTmaRows block rows (tile t = blockIdx + k gridDim);
// while a tile is multiplied, the bulk copy of the CTA's next tile is in
// flight into the other buffer (mbarrier per buffer, phase parity per use).
// Measured (ncu, config 4, 16k nodes): 20.5-22.0 us against 17.4-18.7 us for
// k_bsr_spmv_rows -- the per-row x gathers, not the matrix stream, set the
// time: the compute phase of a tile outlasts the next tile's copy.
constexpr int kSpmvPCap = 320;  // staged blocks per buffer
constexpr int kSpmvPBuf = kSpmvPCap * 144 + (kSpmvPCap + 8) * 4;
constexpr int kSpmvPSmem = 2 * kSpmvPBuf;
__device__ __forceinline__ void spmv_issue_tile(const int* __restrict__ col,
                                                const float* __restrict__ val, int bb0, int bb1,
                                                unsigned char* buf, unsigned bar) {
  const int staged = min(bb1 - bb0, kSpmvPCap);
  const int c0 = bb0 & ~3, c1 = (bb0 + staged + 3) & ~3;
  const unsigned vbytes = 144u * (unsigned)staged, cbytes = 4u * (unsigned)(c1 - c0);
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(vbytes + cbytes)
               : "memory");
  if (vbytes)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (unsigned)__cvta_generic_to_shared(buf)),
        "l"(val + 36 * (size_t)bb0), "r"(vbytes), "r"(bar)
        : "memory");
  if (cbytes)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (unsigned)__cvta_generic_to_shared(buf + kSpmvPCap * 144)),
        "l"(col + c0), "r"(cbytes), "r"(bar)
        : "memory");
}
__global__ void __launch_bounds__(256, 2) k_bsr_spmv_pipe(const int* __restrict__ row_ptr,
                                                         const int* __restrict__ col,
                                                         const float* __restrict__ val, int N,
                                                         double mu, const double* __restrict__ x,
                                                         double* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) unsigned long long s_bar[2];
  const int ntiles = (N + kSpmvTmaRows - 1) / kSpmvTmaRows;
  const unsigned bar0 = (unsigned)__cvta_generic_to_shared(&s_bar[0]);
  const unsigned bar1 = (unsigned)__cvta_generic_to_shared(&s_bar[1]);
  auto tile_rows = [&](int t, int& r0, int& r1) {
    r0 = t * kSpmvTmaRows;
    r1 = min(N, r0 + kSpmvTmaRows);
  };
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar0));
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < 2; ++q) {
      const int t = blockIdx.x + q * gridDim.x;
      if (t < ntiles) {
        int r0, r1;
        tile_rows(t, r0, r1);
        spmv_issue_tile(col, val, __ldg(row_ptr + r0), __ldg(row_ptr + r1), smem + q * kSpmvPBuf,
                        q ? bar1 : bar0);
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, rw = lane % 6, blk5 = lane / 6;
  unsigned phases = 0u;  // bit q: parity of buffer q's next completion
  int k = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int q = k & 1;
    const unsigned bar = q ? bar1 : bar0;
    unsigned char* buf = smem + q * kSpmvPBuf;
    int r0, r1;
    tile_rows(t, r0, r1);
    const int bb0 = __ldg(row_ptr + r0);
    const int staged = min(__ldg(row_ptr + r1) - bb0, kSpmvPCap);
    {
      unsigned done = 0;
      while (!done)
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar), "r"((phases >> q) & 1u)
            : "memory");
    }
    phases ^= 1u << q;
    const float* V = reinterpret_cast<const float*>(buf);
    const int* Cl = reinterpret_cast<const int*>(buf + kSpmvPCap * 144) + (bb0 - (bb0 & ~3));
    for (int j = r0 + (threadIdx.x >> 5); j < r1; j += 8) {
      const int b0 = __ldg(row_ptr + j) - bb0, b1 = __ldg(row_ptr + j + 1) - bb0;
      double acc = 0.0;
      for (int w0 = b0; w0 < b1; w0 += 10) {
        float2 f[2][3];
        double2 xv[2][3];
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const int bi = w0 + g * 5 + blk5;
          const bool ok = lane < 30 && bi < b1;
          const int cidx = ok ? (bi < staged ? Cl[bi] : __ldg(col + bb0 + bi)) : 0;
          const float2* vr = reinterpret_cast<const float2*>(
              (bi < staged ? V + 36 * bi : val + 36 * ((size_t)bb0 + bi)) + 6 * rw);
          const double2* xc = reinterpret_cast<const double2*>(x + 6 * (size_t)cidx);
#pragma unroll
          for (int u = 0; u < 3; ++u) {
            f[g][u] = ok ? vr[u] : make_float2(0.f, 0.f);
            xv[g][u] = ok ? __ldg(xc + u) : make_double2(0.0, 0.0);
          }
        }
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          double sg = 0.0;
#pragma unroll
          for (int u = 0; u < 3; ++u) {
            sg += (double)f[g][u].x * xv[g][u].x;
            sg += (double)f[g][u].y * xv[g][u].y;
          }
          acc += sg;
        }
      }
      double tot = 0.0;
#pragma unroll
      for (int kk = 0; kk < 5; ++kk) tot += __shfl_sync(0xffffffffu, acc, rw + 6 * kk);
      if (lane < 6) y[6 * j + lane] = tot + mu * x[6 * j + lane];
    }
    __syncthreads();  // the buffer is free again
    const int tn = t + 2 * gridDim.x;
    if (threadIdx.x == 0 && tn < ntiles) {
      int n0, n1;
      tile_rows(tn, n0, n1);
      spmv_issue_tile(col, val, __ldg(row_ptr + n0), __ldg(row_ptr + n1), buf, bar);
    }
  }
}

double bsr_spmv(Ctx& c, const double* x_dev, double* y_dev, double mu, int reps) {
  const int N = c.n_nodes;
  cudaEvent_t a, b;
  DS_CUDA(cudaEventCreate(&a));
  DS_CUDA(cudaEventCreate(&b));
  const double bytes = 148.0 * c.n_full + 56.0 * N;
  DS_CUDA(cudaEventRecord(a, c.stream));
  static bool attr = [] {
    return cudaFuncSetAttribute(k_bsr_spmv_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSpmvTmaSmem) == cudaSuccess &&
           cudaFuncSetAttribute(k_bsr_spmv_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSpmvPSmem) == cudaSuccess;
  }();
  const int mode = attr ? c.spmv_tma : 0;
  for (int r = 0; r < reps; ++r) {
    if (mode == 1)
      DS_LAUNCH(c, KK_PCG, bytes, cdiv(N, kSpmvTmaRows), 256, kSpmvTmaSmem, k_bsr_spmv_tma,
                c.row_ptr, c.bsr_col, c.bsr_val, N, mu, x_dev, y_dev);
    else if (mode == 2)
      DS_LAUNCH(c, KK_PCG, bytes, std::min(2 * c.num_sms, cdiv(N, kSpmvTmaRows)), 256, kSpmvPSmem,
                k_bsr_spmv_pipe, c.row_ptr, c.bsr_col, c.bsr_val, N, mu, x_dev, y_dev);
    else
      DS_LAUNCH(c, KK_PCG, bytes, cdiv((long long)N * 32, 256), 256, 0, k_bsr_spmv_rows<2>,
                c.row_ptr, c.bsr_col, c.bsr_val, N, mu, x_dev, y_dev);
  }
  DS_CUDA(cudaEventRecord(b, c.stream));
  sync(c);
  float ms = 0;
  DS_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return reps > 0 ? ms / reps : 0.0;
}

int pcg_max_grid(int num_sms) {
  DS_CUDA(cudaFuncSetAttribute(k_pcg<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcgSmem));
  DS_CUDA(cudaFuncSetAttribute(k_pcg<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcgSmem));
  int per_sm = 0, per_sm2 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg<true>, kPcgThreads, kPcgSmem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_pcg<false>, kPcgThreads, kPcgSmem);
  per_sm = std::min(per_sm, per_sm2);
  // <= kPcgThreads: the pipelined loop holds one CTA partial per thread
  return std::min(std::max(1, per_sm) * num_sms, kPcgThreads);
}

}  // namespace ds
