// k_pcg_cluster.cu — block-Jacobi PCG of one LM attempt (the step replacing
// the reference's dense LDLT, solver.cpp:383-386) inside ONE thread-block
// cluster (8 or 16 CTAs, one per SM), for node counts up to 240 per CTA.
//
// Why a cluster: at config-2 sizes (N ~ 1.5k-2.5k nodes, ~20k 6x6 blocks,
// ~3 MB of fp32 blocks) the cooperative 148-CTA kernel (k_solver.cu k_pcg)
// spends its ~5 us per iteration on latency: a grid barrier through L2
// atomics (~1.7 us incl. skew), L2 round trips for the published vector and
// the dot-product partials. Here every per-iteration exchange stays on chip:
//   * the published vector (m = M^-1 w) lives in each CTA's shared memory and
//     is read by the other CTAs through distributed shared memory (DSMEM);
//   * the three dot-product partials of a CTA sit in its shared memory and are
//     summed by every CTA in rank order (deterministic, identical bits in all);
//   * one hardware cluster barrier (barrier.cluster arrive.release /
//     wait.acquire) per iteration orders both.
// The CTA's slice of the BSR matrix is staged into shared memory once per
// launch with bulk async copies (cp.async.bulk + mbarrier, the TMA engine);
// blocks that do not fit are read from L2 (the matrix is L2-resident: it was
// just assembled). The per-element CG state (x r u w z q s p m n) is held in
// registers: warp w of a CTA owns 5 block rows per pass (lane = 6 row + rw),
// so the block-Jacobi apply M^-1 v is six shuffles within the row's lanes.
//
// Recurrences: the pipelined (Ghysels-Vanroose) CG of k_pcg<true>, the same
// summation orders inside a block row (6-term block products in column
// order, blocks in BSR order) — iterates agree with the cooperative kernel to
// rounding (dot products are reduced in a different tree).
#include <cooperative_groups.h>

#include <algorithm>

#include "ds_context.cuh"
#include "ds_pcg.cuh"

namespace cg = cooperative_groups;

namespace ds {
namespace {

constexpr int kCThreads = 512;
constexpr int kCWarps = kCThreads / 32;
constexpr int kRowsPerWarp = 5;                     // lanes 0..29 = 5 rows x 6
constexpr int kRowsPerPass = kCWarps * kRowsPerWarp;  // 80 block rows per pass
constexpr int kCSmem = 200 * 1024;
constexpr int kMaxCluster = 16;
constexpr int kSrcShift = 20;  // block source code: (src << 20) | offset
constexpr unsigned kOffMask = (1u << kSrcShift) - 1;
constexpr int kBulkChunk = 32 * 1024;

struct PcgcArgs {
  const int* row_ptr;
  const int* col;
  const float* val;
  const int* diag_pos;
  const double* g;
  const double* mu_ptr;
  double* x;
  unsigned* idx;  // global fallback for the block codes / halo list (B_cap + 16 N)
  DevScalars* sc;
  int N;
  int max_iters;
  int cap;  // shared-memory bytes the carve may use (<= kCSmem; tests shrink it)
  unsigned long long* trace;  // DS_PCG_TRACE: phase timestamps of rank 0
};

__device__ __forceinline__ void cmark(const PcgcArgs& a, int rank, int slot) {
  if (a.trace && rank == 0 && threadIdx.x == 0 && slot < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[slot] = t;
  }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// y = M^-1 v for the P elements of this lane (row i, component rw):
// the row's six v components come from the lanes of its group
template <int P>
__device__ __forceinline__ void minv_apply(const double (&v)[P], double (&y)[P],
                                           const double* __restrict__ MINV, int row0, int rw,
                                           int gbase, bool (&act)[P]) {
#pragma unroll
  for (int j = 0; j < P; ++j) {
    double vr[6];
#pragma unroll
    for (int t = 0; t < 6; ++t) vr[t] = __shfl_sync(0xffffffffu, v[j], gbase + t);
    double s = 0.0;
    if (act[j]) {
      const double2* mi =
          reinterpret_cast<const double2*>(MINV + 36 * (row0 + j * kRowsPerPass) + 6 * rw);
      const double2 m01 = mi[0], m23 = mi[1], m45 = mi[2];
      s = (__fma_rn(m01.x, vr[0], m01.y * vr[1]) + __fma_rn(m23.x, vr[2], m23.y * vr[3])) +
          __fma_rn(m45.x, vr[4], m45.y * vr[5]);
    }
    y[j] = s;
  }
}

// y = (H + mu I) v over this lane's elements; v published (own rows, halo)
template <int P>
__device__ __forceinline__ void spmv(double (&y)[P], const double (&vown)[P], double mu,
                                     const int* __restrict__ RP, const unsigned* __restrict__ BSRC,
                                     const float* __restrict__ VS, int ncache,
                                     const float* __restrict__ VG, const double* const* base,
                                     int row0, int rw, bool (&act)[P]) {
#pragma unroll
  for (int j = 0; j < P; ++j) {
    double tot = 0.0;
    if (act[j]) {
      const int i = row0 + j * kRowsPerPass;
      const int lb1 = RP[i + 1];
      for (int b = RP[i]; b < lb1; ++b) {
        const unsigned code = BSRC[b];
        const double2* xv =
            reinterpret_cast<const double2*>(base[code >> kSrcShift] + 6 * (code & kOffMask));
        const double2 x01 = xv[0], x23 = xv[1], x45 = xv[2];
        const float2* vr = reinterpret_cast<const float2*>(
            (b < ncache ? VS + 36 * (size_t)b : VG + 36 * (size_t)b) + 6 * rw);
        const float2 v01 = vr[0], v23 = vr[1], v45 = vr[2];
        double s = 0.0;
        s += (double)v01.x * x01.x;
        s += (double)v01.y * x01.y;
        s += (double)v23.x * x23.x;
        s += (double)v23.y * x23.y;
        s += (double)v45.x * x45.x;
        s += (double)v45.y * x45.y;
        tot += s;
      }
      tot = tot + mu * vown[j];
    }
    y[j] = tot;
  }
}

// one block row of a 6x6 block times a 6-vector (row rw), fp32 matrix, fp64 math
__device__ __forceinline__ double blk_dot(float2 v01, float2 v23, float2 v45, double2 x01,
                                          double2 x23, double2 x45) {
  return (__fma_rn((double)v01.x, x01.x, (double)v01.y * x01.y) +
          __fma_rn((double)v23.x, x23.x, (double)v23.y * x23.y)) +
         __fma_rn((double)v45.x, x45.x, (double)v45.y * x45.y);
}

// Staged-halo SpMV: every column value is in this CTA's shared memory (own rows
// of the published vector at `obase`, the staged halo at `hbase`, in doubles
// from the start of the dynamic shared memory; code bit 31 = halo). Blocks are
// taken four at a time with independent products (latency hiding); the row
// total adds them in BSR order.
template <int P>
__device__ __forceinline__ void spmv_staged(double (&y)[P], const double (&vown)[P], double mu,
                                            const int* __restrict__ RP,
                                            const unsigned* __restrict__ BSRC,
                                            const float* __restrict__ VS, int ncache,
                                            const float* __restrict__ VG,
                                            const double* __restrict__ SD, int obase, int hbase,
                                            int row0, int rw, bool (&act)[P]) {
  auto xsrc = [&](unsigned code) {
    const int off = ((code >> 31) ? hbase : obase) + 6 * (int)(code & 0x7fffffffu);
    return reinterpret_cast<const double2*>(SD + off);
  };
#pragma unroll
  for (int j = 0; j < P; ++j) {
    double tot = 0.0;
    if (act[j]) {
      const int i = row0 + j * kRowsPerPass;
      int b = RP[i];
      const int b1 = RP[i + 1], bc = min(b1, ncache);
      for (; b + 4 <= bc; b += 4) {
        double sb[4];
        const uint4 cd = make_uint4(BSRC[b], BSRC[b + 1], BSRC[b + 2], BSRC[b + 3]);
        const unsigned cds[4] = {cd.x, cd.y, cd.z, cd.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2* xv = xsrc(cds[u]);
          const float2* vr = reinterpret_cast<const float2*>(VS + 36 * (b + u) + 6 * rw);
          sb[u] = blk_dot(vr[0], vr[1], vr[2], xv[0], xv[1], xv[2]);
        }
        tot = ((tot + sb[0]) + sb[1]) + (sb[2] + sb[3]);
      }
      for (; b < bc; ++b) {
        const double2* xv = xsrc(BSRC[b]);
        const float2* vr = reinterpret_cast<const float2*>(VS + 36 * b + 6 * rw);
        tot += blk_dot(vr[0], vr[1], vr[2], xv[0], xv[1], xv[2]);
      }
      for (; b + 4 <= b1; b += 4) {  // blocks past the cache: fp32 rows from L2
        double sb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2* xv = xsrc(BSRC[b + u]);
          const float2* vr = reinterpret_cast<const float2*>(VG + 36 * (size_t)(b + u) + 6 * rw);
          sb[u] = blk_dot(__ldg(vr), __ldg(vr + 1), __ldg(vr + 2), xv[0], xv[1], xv[2]);
        }
        tot = ((tot + sb[0]) + sb[1]) + (sb[2] + sb[3]);
      }
      for (; b < b1; ++b) {
        const double2* xv = xsrc(BSRC[b]);
        const float2* vr = reinterpret_cast<const float2*>(VG + 36 * (size_t)b + 6 * rw);
        tot += blk_dot(__ldg(vr), __ldg(vr + 1), __ldg(vr + 2), xv[0], xv[1], xv[2]);
      }
      tot = __fma_rn(mu, vown[j], tot);
    }
    y[j] = tot;
  }
}

template <int P>
__global__ void __launch_bounds__(kCThreads, 1) k_pcg_cluster(PcgcArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double s_part[2][4];                 // published dot partials (DSMEM)
  __shared__ double s_gath[kMaxCluster][4];       // all CTAs' partials, rank order
  __shared__ double s_wsum[kCWarps][4];
  __shared__ const double* s_base[2][kMaxCluster + 1];
  __shared__ int s_scan[kCWarps + 1];
  __shared__ int s_nh;
  __shared__ __align__(8) unsigned long long s_mbar;

  const int N = a.N;
  const int r0 = (int)((long long)N * rank / C), r1 = (int)((long long)N * (rank + 1) / C);
  const int nr = r1 - r0, nrmax = (N + C - 1) / C;
  const int bb0 = a.row_ptr[r0], nb = a.row_ptr[r1] - bb0;
  if (rank == 0 && tid == 0) a.sc->finite = 1;  // before the first cluster barrier
  const double mu = *a.mu_ptr;

  cmark(a, rank, 0);
  // ---- shared-memory carve (OWN first: the same offset in every CTA)
  double* OWN = reinterpret_cast<double*>(smem);  // [2][6 nrmax] published vector
  double* UNI = OWN + 12 * (size_t)nrmax;         // MINV [nr][36] / halo marks [N]
  const size_t uni_d = std::max<size_t>(36 * (size_t)nr, ((size_t)N + 1) / 2);
  int* RP = reinterpret_cast<int*>(UNI + uni_d);  // local row pointers (block offsets)
  int* mark = reinterpret_cast<int*>(UNI);
  for (int k = tid; k <= nr; k += kCThreads) RP[k] = a.row_ptr[r0 + k] - bb0;
  for (int k = tid; k < N; k += kCThreads) mark[k] = 0;
  __syncthreads();
  for (int b = tid; b < nb; b += kCThreads) {
    const int c = a.col[bb0 + b];
    if (c < r0 || c >= r1) mark[c] = 1;
  }
  __syncthreads();
  // exclusive scan of the marks over [0, N): contiguous chunk per thread
  {
    const int ch = (N + kCThreads - 1) / kCThreads;
    const int c0 = min(N, tid * ch), c1 = min(N, c0 + ch);
    int cnt = 0;
    for (int c = c0; c < c1; ++c) cnt += mark[c];
    int inc = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += v;
    }
    if (lane == 31) s_scan[warp] = inc;
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int w = 0; w < kCWarps; ++w) {
        const int v = s_scan[w];
        s_scan[w] = run;
        run += v;
      }
      s_nh = run;
    }
    __syncthreads();
    int pos = s_scan[warp] + inc - cnt;
    for (int c = c0; c < c1; ++c) mark[c] = mark[c] ? pos++ : -1;
  }
  __syncthreads();
  cmark(a, rank, 1);
  const int nh = s_nh;
  // past the row pointers: block source codes + halo list (on chip when they
  // fit, else a global scratch), the staged halo values [2][6 nh] (else remote
  // columns are read straight from the owners' shared memory in the SpMV),
  // then as many matrix blocks as fit
  const size_t i_off = (size_t)(reinterpret_cast<unsigned char*>(RP + nr + 1) - smem);
  const bool idx_on_chip = i_off + 4 * ((size_t)nb + nh) <= (size_t)a.cap;
  unsigned* BSRC = idx_on_chip ? reinterpret_cast<unsigned*>(smem + i_off) : a.idx + bb0;
  unsigned* HL = idx_on_chip ? BSRC + nb : a.idx + (a.row_ptr[N] + (size_t)N * rank);
  const size_t hv_off =
      ((idx_on_chip ? i_off + 4 * ((size_t)nb + nh) : i_off) + 15) & ~(size_t)15;
  const bool stage = hv_off + 96 * (size_t)nh <= (size_t)a.cap;
  double* HV = reinterpret_cast<double*>(smem + hv_off);
  const size_t v_off = (hv_off + (stage ? 96 * (size_t)nh : 0) + 15) & ~(size_t)15;
  const int ncache = v_off >= (size_t)a.cap ? 0
                         : (int)std::min<size_t>((size_t)nb, ((size_t)a.cap - v_off) / 144);
  float* VS = reinterpret_cast<float*>(smem + v_off);
  const float* VG = a.val + 36 * (size_t)bb0;
  // owner of a column: the rank whose row range holds it
  auto owner_of = [&](int c) {
    int q = (int)(((long long)c * C) / N);
    while (q + 1 < C && (int)((long long)N * (q + 1) / C) <= c) ++q;
    while (q > 0 && (int)((long long)N * q / C) > c) --q;
    return q;
  };
  for (int c = tid; c < N; c += kCThreads) {
    const int h = mark[c];
    if (h >= 0) {
      const int q = owner_of(c);
      HL[h] = ((unsigned)q << kSrcShift) | (unsigned)(c - (int)((long long)N * q / C));
    }
  }
  for (int b = tid; b < nb; b += kCThreads) {
    const int c = a.col[bb0 + b];
    unsigned code;
    if (stage) {  // local shared memory only: own rows / staged halo (bit 31)
      code = (c >= r0 && c < r1) ? (unsigned)(c - r0) : (0x80000000u | (unsigned)mark[c]);
    } else if (c >= r0 && c < r1) {
      code = ((unsigned)rank << kSrcShift) | (unsigned)(c - r0);
    } else {
      const int q = owner_of(c);
      code = ((unsigned)q << kSrcShift) | (unsigned)(c - (int)((long long)N * q / C));
    }
    BSRC[b] = code;
  }
  if (tid < 2 * (kMaxCluster + 1)) {
    const int par = tid / (kMaxCluster + 1), q = tid % (kMaxCluster + 1);
    const double* p = nullptr;
    if (q < C) p = cluster.map_shared_rank(OWN + 6 * (size_t)nrmax * par, q);
    else if (q == C) p = HV + 6 * (size_t)nh * par;
    s_base[par][q] = p;
  }
  // ---- stage the cached matrix blocks: bulk async copies (TMA engine)
  if (tid == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&s_mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // marks consumed; mbarrier initialised
  cmark(a, rank, 2);
  const unsigned bytes = 144u * (unsigned)ncache;
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&s_mbar)),
                 "r"(bytes)
                 : "memory");
    for (unsigned off = 0; off < bytes; off += kBulkChunk) {
      const unsigned sz = min((unsigned)kBulkChunk, bytes - off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(reinterpret_cast<unsigned char*>(VS) + off)),
          "l"(reinterpret_cast<const unsigned char*>(VG) + off), "r"(sz), "r"(smem_u32(&s_mbar))
          : "memory");
    }
  }
  // ---- block-Jacobi inverses (8-lane Gauss-Jordan groups) while the copy flies
  double* MINV = UNI;
  {
    const int grp = tid >> 3, lr = tid & 7;
    for (int i0 = 0; i0 < nr; i0 += kCThreads / 8) {
      const int i = i0 + grp;
      double ar[6], br[6];
      const int d = (i < nr && lr < 6) ? a.diag_pos[r0 + i] : -1;
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        double v = d >= 0 ? (double)a.val[(size_t)d * 36 + lr * 6 + t] : 0.0;
        if (t == lr) v += mu;
        ar[t] = lr < 6 ? v : 0.0;
      }
      gj_inverse6(ar, br, lr);
      if (i < nr && lr < 6)
#pragma unroll
        for (int t = 0; t < 6; ++t) MINV[36 * i + 6 * lr + t] = br[t];
    }
  }
  // ---- element ownership: pass j, warp w, lane = 6 (row in warp) + rw
  const int rl = lane / 6, rw = lane - 6 * rl;
  const int gbase = 6 * min(rl, kRowsPerWarp - 1);
  const int row0 = warp * kRowsPerWarp + rl;  // + j * kRowsPerPass
  bool act[P];
#pragma unroll
  for (int j = 0; j < P; ++j) act[j] = lane < 30 && row0 + j * kRowsPerPass < nr;
  double X[P], R[P], U[P], W[P], Z[P], Q[P], S[P], Pv[P], M[P], Nv[P];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const int k = 6 * (row0 + j * kRowsPerPass) + rw;
    R[j] = act[j] ? -a.g[6 * (size_t)r0 + k] : 0.0;
    X[j] = Z[j] = Q[j] = S[j] = Pv[j] = 0.0;
  }
  __syncthreads();  // MINV complete
  cmark(a, rank, 3);
  // u0 = M^-1 r0, published in the odd buffer (iteration 0's m goes to the even one)
  minv_apply<P>(R, U, MINV, row0, rw, gbase, act);
#pragma unroll
  for (int j = 0; j < P; ++j)
    if (act[j]) OWN[6 * (size_t)nrmax + 6 * (row0 + j * kRowsPerPass) + rw] = U[j];
  // the matrix copy must have landed before the first SpMV
  {
    unsigned done = 0;
    while (!done)
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(smem_u32(&s_mbar))
          : "memory");
  }
  cmark(a, rank, 4);
  cluster.sync();
  cmark(a, rank, 5);
  auto gather = [&](int par) {  // remote columns of the published vector -> HV[par]
    if (stage) {
      double* hv = HV + 6 * (size_t)nh * par;
      for (int k = tid; k < 6 * nh; k += kCThreads) {
        const int h = k / 6, t = k - 6 * h;
        const unsigned code = HL[h];
        hv[k] = s_base[par][code >> kSrcShift][6 * (code & kOffMask) + t];
      }
    }
  };
  gather(1);
  __syncthreads();
  cmark(a, rank, 6);
  const double* SD = reinterpret_cast<const double*>(smem);
  const int hb = (int)((reinterpret_cast<const unsigned char*>(HV) - smem) / 8);
  auto spmv_any = [&](double (&y)[P], const double (&v)[P], int par) {
    if (stage)
      spmv_staged<P>(y, v, mu, RP, BSRC, VS, ncache, VG, SD, 6 * nrmax * par, hb + 6 * nh * par,
                     row0, rw, act);
    else
      spmv<P>(y, v, mu, RP, BSRC, VS, ncache, VG, s_base[par], row0, rw, act);
  };
  spmv_any(W, U, 1);  // w0 = A u0
  cmark(a, rank, 7);
  double gamma_old = 0.0, alpha_old = 0.0, rr = 0.0, rr0 = 0.0;
  int it = 0;
  for (;; ++it) {
    const int par = it & 1;
    // m = M^-1 w (published), partials (r.u, w.u, r.r)
    minv_apply<P>(W, M, MINV, row0, rw, gbase, act);
    double pg = 0.0, pd = 0.0, pr = 0.0;
#pragma unroll
    for (int j = 0; j < P; ++j) {
      if (act[j]) OWN[6 * (size_t)nrmax * par + 6 * (row0 + j * kRowsPerPass) + rw] = M[j];
      pg += R[j] * U[j];
      pd += W[j] * U[j];
      pr += R[j] * R[j];
    }
    pg = warp_sum(pg);
    pd = warp_sum(pd);
    pr = warp_sum(pr);
    if (lane == 0) {
      s_wsum[warp][0] = pg;
      s_wsum[warp][1] = pd;
      s_wsum[warp][2] = pr;
    }
    __syncthreads();
    if (warp == 0) {  // fixed shuffle tree over the warp sums
      double v0 = lane < kCWarps ? s_wsum[lane][0] : 0.0;
      double v1 = lane < kCWarps ? s_wsum[lane][1] : 0.0;
      double v2 = lane < kCWarps ? s_wsum[lane][2] : 0.0;
#pragma unroll
      for (int off = kCWarps / 2; off > 0; off >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, off);
        v1 += __shfl_xor_sync(0xffffffffu, v1, off);
        v2 += __shfl_xor_sync(0xffffffffu, v2, off);
      }
      if (lane == 0) {
        s_part[par][0] = v0;
        s_part[par][1] = v1;
        s_part[par][2] = v2;
      }
    }
    cmark(a, rank, 8 + 4 * it);
    cluster.sync();  // release m and the partials; acquire everyone's
    cmark(a, rank, 9 + 4 * it);
    gather(par);
    if (tid < 3 * C) {
      const int q = tid / 3, k = tid - 3 * q;
      s_gath[q][k] = cluster.map_shared_rank(&s_part[par][0], q)[k];
    }
    __syncthreads();
    cmark(a, rank, 10 + 4 * it);
    // n = (H + mu I) m -- computed before the stopping test (unused on the last round)
    spmv_any(Nv, M, par);
    cmark(a, rank, 11 + 4 * it);
    double gamma = 0.0, delta = 0.0;
    rr = 0.0;
    for (int q = 0; q < C; ++q) {
      gamma += s_gath[q][0];
      delta += s_gath[q][1];
      rr += s_gath[q][2];
    }
    if (it == 0) rr0 = rr;
    if (it >= a.max_iters || rr == 0.0) break;
    const double beta = it > 0 ? gamma / gamma_old : 0.0;
    const double alpha = it > 0 ? gamma / (delta - beta * gamma / alpha_old) : gamma / delta;
#pragma unroll
    for (int j = 0; j < P; ++j) {
      Z[j] = Nv[j] + beta * Z[j];
      Q[j] = M[j] + beta * Q[j];
      S[j] = W[j] + beta * S[j];
      Pv[j] = U[j] + beta * Pv[j];
      X[j] = X[j] + alpha * Pv[j];
      R[j] = R[j] - alpha * S[j];
      U[j] = U[j] - alpha * Q[j];
      W[j] = W[j] - alpha * Z[j];
    }
    gamma_old = gamma;
    alpha_old = alpha;
  }
  bool bad = false;  // non-finite increment -> LM reject (solver.cpp:387)
#pragma unroll
  for (int j = 0; j < P; ++j)
    if (act[j]) {
      a.x[6 * (size_t)r0 + 6 * (row0 + j * kRowsPerPass) + rw] = X[j];
      bad |= !isfinite(X[j]);
    }
  if (bad) atomicExch(&a.sc->finite, 0);
  if (rank == 0 && tid == 0) {
    a.sc->pcg_iters = it;
    a.sc->pcg_rr = rr;
    a.sc->pcg_rr0 = rr0;
  }
  cluster.sync();  // no CTA leaves while another may still read its shared memory
  cmark(a, rank, 63);
}

template <int P>
bool configure(int C) {
  static int state[kMaxCluster + 1] = {};  // 0 unknown, 1 ok, -1 unavailable
  if (state[C] != 0) return state[C] > 0;
  auto fn = k_pcg_cluster<P>;
  bool ok = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kCSmem) ==
                cudaSuccess &&
            cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                cudaSuccess;
  if (ok) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kCThreads);
    cfg.dynamicSmemBytes = kCSmem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    ok = cudaOccupancyMaxActiveClusters(&n, fn, &cfg) == cudaSuccess && n >= 1;
  }
  cudaGetLastError();
  state[C] = ok ? 1 : -1;
  return ok;
}

template <int P>
void launch(Ctx& c, int C, const PcgcArgs& a) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kCThreads);
  cfg.dynamicSmemBytes = kCSmem;
  cfg.stream = c.stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DS_CUDA(cudaLaunchKernelEx(&cfg, k_pcg_cluster<P>, a));
}

}  // namespace

// Launches the cluster PCG when it applies (fixed iteration budget, N small
// enough for P <= 3 passes, the cluster shape available); returns false when
// the caller should run the cooperative grid kernel instead.
bool pcg_cluster_launch(Ctx& c, int max_iters, double tol) {
  // DS_PCG_CLUSTER: unset / 0 off (default), 2..16 the cluster size. Off by
  // default: at config-2 sizes the measured launch is slower than the
  // cooperative grid kernel (123 vs 65 us for 10 iterations at
  // 2k nodes -- 16 SMs run ~9x longer dependent fp64 chains per iteration
  // than 148 do, and the matrix slice spills past shared memory).
  const int mode = c.pcg_cluster;
  const int N = c.n_nodes;
  if (mode <= 0 || tol > 0.0 || N < 8) return false;
  int C = std::min(mode, kMaxCluster);
  C = std::min(C, N / 4);
  if (C < 2) return false;
  const int nrmax = (N + C - 1) / C;
  const int P = (nrmax + kRowsPerPass - 1) / kRowsPerPass;
  if (P > 3) return false;
  // the fixed part of the carve must fit (the rest adapts: index lists, halo
  // staging, cached blocks)
  const size_t fixed = 96 * (size_t)nrmax + 8 * std::max<size_t>(36 * (size_t)nrmax, N / 2 + 1) +
                       4 * (size_t)(nrmax + 2);
  const int cap = std::min(kCSmem, c.pcgc_smem_cap);
  if (fixed > (size_t)cap || C * (size_t)N > 16 * (size_t)c.N_cap) return false;
  const bool ok = P == 1 ? configure<1>(C) : P == 2 ? configure<2>(C) : configure<3>(C);
  if (!ok) return false;
  PcgcArgs a;
  a.row_ptr = c.row_ptr;
  a.col = c.bsr_col;
  a.val = c.bsr_val;
  a.diag_pos = c.diag_pos;
  a.g = c.g;
  a.mu_ptr = &c.dsc->mu;
  a.x = c.pcg_x;
  a.idx = c.pcgc_idx;
  a.sc = c.dsc;
  a.N = N;
  a.max_iters = max_iters;
  a.cap = cap;
  a.trace = c.pcg_trace;
  launch_begin(c, KK_PCG);
  if (P == 1) launch<1>(c, C, a);
  else if (P == 2) launch<2>(c, C, a);
  else launch<3>(c, C, a);
  launch_end(c, KK_PCG, std::max(1, max_iters) * (148.0 * c.n_full + 292.0 * N + 4.0));
  return true;
}

}  // namespace ds
