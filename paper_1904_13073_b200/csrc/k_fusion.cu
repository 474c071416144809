// k_fusion.cu — geometry update (K11-K16, K2) and reinitialisation cleaning.
//   fuse_depth         fusion.cpp:9-75: per valid pixel, scan the f x f block of
//                      the supersampled index map, best = (confidence desc, d2
//                      asc, index asc) within the 1 mm / 0.85 gates, Eq. 5 update
//                      (each surfel lives in exactly one block, so pixels are
//                      independent writers), else an append candidate.
//   candidates         row-major stable compaction (fusion.cpp:46-57)
//   skin_appended      fusion.cpp:77-122 (brute-force live-frame K-NN over nodes,
//                      Eq. 6 ratio test, delta_nn support)
//   check_compressive  fusion.cpp:128-177 (1 mm re-weighted inverse-warp strain,
//                      sigma_max <= 1 + epsilon)
//   remove_surfels     fusion.cpp:179-218 (unstable rule, 3x3 duplicate rule on the
//                      pre-append index map)
//   compaction + inverse warp  fusion.cpp:264-294 fused in one pass: stable scatter
//                      of the survivors into the alternate SoA buffer while the
//                      reference pose is rebuilt from the live one.
//   clean_and_reset    reinit.cpp:28-89
#include "ds_blend.cuh"
#include "ds_context.cuh"
#include "ds_knn.cuh"

namespace ds {

void init_warp_field(Ctx& c);

namespace {

constexpr int kEmptyIdx = 0x7f7f7f7f;

struct FuseParams {
  Rig pose;
  int W, H, f;
  int t_now;
  double dd2, dn;
};

__global__ void __launch_bounds__(256) k_fuse(const int* __restrict__ im_idx, ModelBuf m,
                                              const double4* __restrict__ fvert,
                                              const double4* __restrict__ fnrm,
                                              const uint8_t* __restrict__ fflag, FuseParams fp,
                                              int* __restrict__ cand_flag, int* __restrict__ fused) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= fp.W * fp.H) return;
  if (!(fflag[c] & 2)) {
    cand_flag[c] = 0;
    return;
  }
  const int x = c % fp.W, y = c / fp.W;
  const double4 fv = fvert[c], fn = fnrm[c];
  const V3 vd = rig_apply(fp.pose, v3(fv.x, fv.y, fv.z));
  const V3 nd = rig_rotate(fp.pose, v3(fn.x, fn.y, fn.z));
  int best = -1;
  double bc = 0, bd2 = 0;
  const int Wf = fp.W * fp.f;
  for (int sy = fp.f * y; sy < fp.f * (y + 1); ++sy)
    for (int sx = fp.f * x; sx < fp.f * (x + 1); ++sx) {
      const int id = im_idx[(size_t)sy * Wf + sx];
      if (id == kEmptyIdx) continue;
      const float4 lp = m.lp[id], ln = m.ln[id];
      const double d2 = sqn(sub(v3(lp.x, lp.y, lp.z), vd));
      if (d2 >= fp.dd2) continue;
      if (dot(nd, v3(ln.x, ln.y, ln.z)) < fp.dn) continue;
      const double sc = ln.w;
      const bool better = best < 0 || sc > bc || (sc == bc && (d2 < bd2 || (d2 == bd2 && id < best)));
      if (better) {
        best = id;
        bc = sc;
        bd2 = d2;
      }
    }
  if (best < 0) {
    cand_flag[c] = 1;
    return;
  }
  cand_flag[c] = 0;
  const float4 lp = m.lp[best], ln = m.ln[best];
  const double c_old = ln.w, c_d = fn.w, c_new = c_old + c_d;
  const V3 sp = v3(lp.x, lp.y, lp.z), sn = v3(ln.x, ln.y, ln.z);
  const V3 np = dvd(add(scl(c_old, sp), scl(c_d, vd)), c_new);
  const V3 nn = dvd(add(scl(c_old, sn), scl(c_d, nd)), c_new);
  const V3 nu = dvd(nn, nrm(nn));
  const double r = (c_old * (double)lp.w + c_d * fv.w) / c_new;
  m.lp[best] = make_float4((float)np.x, (float)np.y, (float)np.z, (float)r);
  m.ln[best] = make_float4((float)nu.x, (float)nu.y, (float)nu.z, (float)c_new);
  m.t[best].y = fp.t_now;
  atomicAdd(fused, 1);
}

__global__ void k_write_cands(const int* __restrict__ flag, const int* __restrict__ scan, int P,
                              const double4* __restrict__ fvert, const double4* __restrict__ fnrm,
                              Rig pose, int* __restrict__ cand_pix, float4* __restrict__ cp,
                              float4* __restrict__ cn) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P || !flag[c]) return;
  const int k = scan[c];
  const double4 fv = fvert[c], fn = fnrm[c];
  const V3 vd = rig_apply(pose, v3(fv.x, fv.y, fv.z));
  const V3 nd = rig_rotate(pose, v3(fn.x, fn.y, fn.z));
  cand_pix[k] = c;
  cp[k] = make_float4((float)vd.x, (float)vd.y, (float)vd.z, (float)fv.w);
  cn[k] = make_float4((float)nd.x, (float)nd.y, (float)nd.z, (float)fn.w);
}

// 3x3 symmetric eigenvalues by cyclic Jacobi; returns sqrt(max eig of S^T S).
// Fully unrolled over the (p, q) pairs so the matrix stays in registers; the
// arithmetic (and its order) is the oracle's.
__device__ double sigma_max3(const double S[3][3]) {
  double a[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double acc = 0;
#pragma unroll
      for (int k = 0; k < 3; ++k) acc += S[k][i] * S[k][j];
      a[i][j] = acc;
    }
  for (int sweep = 0; sweep < 30; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    if (off < 1e-300) break;
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double theta = ddiv(a[q][q] - a[p][p], 2.0 * a[p][q]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = cs * akp - sn * akq;
          a[k][q] = sn * akp + cs * akq;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = cs * apk - sn * aqk;
          a[q][k] = sn * apk + cs * aqk;
        }
      }
  }
  const double m = fmax(fmax(a[0][0], a[1][1]), fmax(a[2][2], 0.0));
  return sqrt(m);
}

// sigma_max3(S) <= 1 + eps, deciding from cheap bounds on lambda_max(S^T S)
// when they are clear of the threshold by a relative 1e-9 (Rayleigh: max
// diagonal <= lambda_max <= max Gershgorin row sum; the Jacobi result is
// within ~1e-15 of lambda_max), else by the Jacobi sweep itself.
__device__ bool strain_within(const double S[3][3], double eps) {
  double a[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double acc = 0;
#pragma unroll
      for (int k = 0; k < 3; ++k) acc += S[k][i] * S[k][j];
      a[i][j] = acc;
    }
  const double g0 = a[0][0] + fabs(a[0][1]) + fabs(a[0][2]);
  const double g1 = a[1][1] + fabs(a[1][0]) + fabs(a[1][2]);
  const double g2 = a[2][2] + fabs(a[2][0]) + fabs(a[2][1]);
  const double gmax = fmax(g0, fmax(g1, g2));
  const double thr = (1.0 + eps) * (1.0 + eps);
  if (gmax < thr * (1.0 - 1e-9)) return true;  // false for NaN
  if (gmax == gmax && fmax(a[0][0], fmax(a[1][1], a[2][2])) > thr * (1.0 + 1e-9)) return false;
  return sigma_max3(S) <= 1.0 + eps;
}

struct ScreenParams {
  int N, K, compressive;
  double eps, delta_nn;
};

// inverse warp with weights re-evaluated at x over the entry's node set
__device__ bool inv_warp_reweighted(V3 x, const int* ids, int cnt, const double4* __restrict__ node_dq,
                                    const double4* __restrict__ node_live, V3& out) {
  Q4 rs = q4(0, 0, 0, 0), ds_ = q4(0, 0, 0, 0);
  const Q4 pivot = ld_q(node_dq + 2 * ids[0]);
  for (int m = 0; m < cnt; ++m) {
    const double4 nl = node_live[ids[m]];
    const double w = skin_weight(x, v3(nl.x, nl.y, nl.z), nl.w);
    const Q4 r = ld_q(node_dq + 2 * ids[m]);
    const Q4 d = ld_q(node_dq + 2 * ids[m] + 1);
    const double sign = (qdot(pivot, r) < 0.0) ? -1.0 : 1.0;
    const double ww = sign * w;
    rs = qadd(rs, qscl(ww, r));
    ds_ = qadd(ds_, qscl(ww, d));
  }
  if (qnrm(rs) < kDegenerateBlend) return false;
  DQ raw;
  raw.r = rs;
  raw.d = ds_;
  out = rig_apply(rig_inverse(dq_to_rig(dq_normalized(raw))), x);
  return true;
}

// skin_appended + check_compressive for candidate k (fusion.cpp:77-177).
// result: 0 = low support, 1 = compressive reject, 2 = accepted
// Eq. 6 ratio test, weights, delta_nn, compressive check on a K-NN list.
__device__ int screen_one(V3 x, const double bd[4], const int bi[4],
                          const double4* __restrict__ node_pos,
                          const double4* __restrict__ node_live, const double4* __restrict__ node_dq,
                          const ScreenParams& sp, int ids[4], float ws[4], int& cnt) {
  (void)bd;
  const int k = min(sp.K, sp.N);
  const int n0 = bi[0];
  const double4 l0 = node_live[n0], p0 = node_pos[n0];
  double w[4];
  cnt = 0;
  ids[cnt] = n0;
  w[cnt] = skin_weight(x, v3(l0.x, l0.y, l0.z), l0.w);
  ++cnt;
  for (int m = 1; m < k; ++m) {
    const int j = bi[m];
    const double4 lj = node_live[j], pj = node_pos[j];
    const double lpair = nrm(sub(v3(lj.x, lj.y, lj.z), v3(l0.x, l0.y, l0.z)));
    const double rpair = nrm(sub(v3(pj.x, pj.y, pj.z), v3(p0.x, p0.y, p0.z)));
    if (rpair <= 0) continue;
    const double ratio = lpair / rpair;
    if (ratio <= 1.0 - sp.eps || ratio >= 1.0 + sp.eps) continue;
    ids[cnt] = j;
    w[cnt] = skin_weight(x, v3(lj.x, lj.y, lj.z), lj.w);
    ++cnt;
  }
  double wsum = 0;
  for (int m = 0; m < cnt; ++m) wsum += w[m];
  for (int m = 0; m < 4; ++m) ws[m] = m < cnt ? (float)w[m] : 0.f;
  for (int m = cnt; m < 4; ++m) ids[m] = -1;
  if (wsum < sp.delta_nn) return 0;
  if (sp.compressive) {
    V3 c0;
    if (!inv_warp_reweighted(x, ids, cnt, node_dq, node_live, c0)) return 1;
    double S[3][3];
    for (int a = 0; a < 3; ++a) {
      V3 pr = x;
      if (a == 0) pr.x += 1e-3;
      else if (a == 1) pr.y += 1e-3;
      else pr.z += 1e-3;
      V3 sh;
      if (!inv_warp_reweighted(pr, ids, cnt, node_dq, node_live, sh)) return 1;
      const V3 col = dvd(sub(sh, c0), 1e-3);
      S[0][a] = col.x;
      S[1][a] = col.y;
      S[2][a] = col.z;
    }
    if (!strain_within(S, sp.eps)) return 1;
  }
  return 2;
}

// kScreenLanes lanes per candidate (>= 4: the compressive check's four
// inverse warps run on lanes 0-3), each scanning a strided subset of the node
// tiles / grid cells; the per-lane top-4 lists are merged by shuffles.
#ifndef DS_SCREEN_LANES
#define DS_SCREEN_LANES 4
#endif
constexpr int kScreenLanes = DS_SCREEN_LANES;
static_assert(kScreenLanes >= 4 && (kScreenLanes & (kScreenLanes - 1)) == 0, "lanes: 4, 8, 16 or 32");

// screen_one for an aligned kScreenLanes group (all lanes call it): the Eq. 6 entry
// is built redundantly, the four inverse warps of the compressive check
// (x and the three 1 mm probes, fusion.cpp:151-176) run on lanes 0-3 and
// meet in lane 0 for the strain's sigma_max. Same arithmetic as screen_one.
__device__ int screen_group(V3 x, const double bd[4], const int bi[4],
                            const double4* __restrict__ node_pos,
                            const double4* __restrict__ node_live,
                            const double4* __restrict__ node_dq, const ScreenParams& sp, int ids[4],
                            float ws[4], int& cnt, int lane_k) {
  (void)bd;
  const unsigned gmask = kScreenLanes >= 32 ? 0xffffffffu
                        : ((1u << kScreenLanes) - 1u) << ((threadIdx.x & 31) & ~(unsigned)(kScreenLanes - 1));
  const int k = min(sp.K, sp.N);
  const int n0 = bi[0];
  const double4 l0 = node_live[n0], p0 = node_pos[n0];
  double w[4];
  cnt = 0;
  ids[cnt] = n0;
  w[cnt] = skin_weight(x, v3(l0.x, l0.y, l0.z), l0.w);
  ++cnt;
  for (int m = 1; m < k; ++m) {
    const int j = bi[m];
    const double4 lj = node_live[j], pj = node_pos[j];
    const double lpair = nrm(sub(v3(lj.x, lj.y, lj.z), v3(l0.x, l0.y, l0.z)));
    const double rpair = nrm(sub(v3(pj.x, pj.y, pj.z), v3(p0.x, p0.y, p0.z)));
    if (rpair <= 0) continue;
    const double ratio = lpair / rpair;
    if (ratio <= 1.0 - sp.eps || ratio >= 1.0 + sp.eps) continue;
    ids[cnt] = j;
    w[cnt] = skin_weight(x, v3(lj.x, lj.y, lj.z), lj.w);
    ++cnt;
  }
  double wsum = 0;
  for (int m = 0; m < cnt; ++m) wsum += w[m];
  for (int m = 0; m < 4; ++m) ws[m] = m < cnt ? (float)w[m] : 0.f;
  for (int m = cnt; m < 4; ++m) ids[m] = -1;
  if (wsum < sp.delta_nn) return 0;  // uniform across the group
  if (!sp.compressive) return 2;
  V3 pr = x, r = v3(0, 0, 0);
  if (lane_k == 1) pr.x += 1e-3;
  else if (lane_k == 2) pr.y += 1e-3;
  else if (lane_k == 3) pr.z += 1e-3;
  int okw = 1;
  if (lane_k < 4) okw = inv_warp_reweighted(pr, ids, cnt, node_dq, node_live, r) ? 1 : 0;
  double rx[4], ry[4], rz[4];
  int oks = 1;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int src = ((threadIdx.x & 31) & ~(kScreenLanes - 1)) + a;
    rx[a] = __shfl_sync(gmask, r.x, src);
    ry[a] = __shfl_sync(gmask, r.y, src);
    rz[a] = __shfl_sync(gmask, r.z, src);
    oks &= __shfl_sync(gmask, okw, src);
  }
  if (!oks) return 1;  // a degenerate probe blend (fusion.cpp:174)
  const V3 c0 = v3(rx[0], ry[0], rz[0]);
  double S[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const V3 col = dvd(sub(v3(rx[a + 1], ry[a + 1], rz[a + 1]), c0), 1e-3);
    S[0][a] = col.x;
    S[1][a] = col.y;
    S[2][a] = col.z;
  }
  if (lane_k != 0) return 2;  // only lane 0's verdict is used
  return strain_within(S, sp.eps) ? 2 : 1;
}

// (kScreenLanes: see above)
constexpr int kScreenThreads = 256;

// one block's group of kScreenThreads / kScreenLanes candidates from `kb`
__device__ __forceinline__ void screen_block(
    int kb, int n, float4* tile, const float4* __restrict__ cp,
    const double4* __restrict__ node_pos, const double4* __restrict__ node_live,
    const float4* __restrict__ node_live_f, const int* __restrict__ rmax_bits,
    const double4* __restrict__ node_dq, const ScreenParams& sp, int4* __restrict__ cki,
    float4* __restrict__ ckw, int* __restrict__ ok, int* __restrict__ res_out,
    int* __restrict__ low, int* __restrict__ comp, const KnnGridView& grid, int use_grid) {
  const int k = kb + threadIdx.x / kScreenLanes, lane_k = threadIdx.x % kScreenLanes;
  const bool active = k < n;
  double bd[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
  int bi[4] = {0x7fffffff, 0x7fffffff, 0x7fffffff, 0x7fffffff};
  if (use_grid) {  // exact 4-NN on the live-node grid (ds_knn.cuh), group of 8 lanes
    if (!active) return;  // whole 8-lane group
    const float4 p = cp[k];
    const V3 x = v3(p.x, p.y, p.z);
    double md[4];
    int mi[4];
    if (!knn_grid_query<4, kScreenLanes>(grid, node_live, x, [](int) { return true; }, md, mi)) {
      for (int t = lane_k; t < sp.N; t += kScreenLanes) {
        const double4 nl = node_live[t];
        knnk_insert<4>(sqn(sub(v3(nl.x, nl.y, nl.z), x)), t, bd, bi);
      }
      knnk_merged<4, kScreenLanes>(bd, bi, md, mi);
    }
    int ids[4];
    float ws[4];
    int cnt = 0;
    const int res = screen_group(x, md, mi, node_pos, node_live, node_dq, sp, ids, ws, cnt, lane_k);
    if (lane_k != 0) return;
    ok[k] = res == 2 ? 1 : 0;
    res_out[k] = res;
    if (res == 0) atomicAdd(low, 1);
    if (res == 1) atomicAdd(comp, 1);
    cki[k] = make_int4(ids[0], ids[1], ids[2], ids[3]);
    ckw[k] = make_float4(ws[0], ws[1], ws[2], ws[3]);
    return;
  }
  V3 x = v3(0, 0, 0);
  float xf = 0.f, yf = 0.f, zf = 0.f;
  if (active) {
    const float4 p = cp[k];  // candidate positions are fp32 values: exact in both
    x = v3(p.x, p.y, p.z);
    xf = p.x;
    yf = p.y;
    zf = p.z;
  }
  // Exact live-frame K-NN by (d2, idx) in two passes over shared-memory tiles.
  // Rounding model: node coordinates rounded to fp32 move each |difference| by
  // <= u*R (+ u of the difference), so |sqrt(d2f) - sqrt(d2)| <= delta = 1.8 u R
  // up to a relative 1e-5 for the fp32 arithmetic.
  // Pass 1 (fp32 only, branch-free): T32 = 4th smallest d2f of the candidate.
  // The 4 nodes realising T32 have d2 <= B = (sqrt(T32 (1+2e-5)) + delta)^2, so
  // the exact 4th-smallest d2 is <= B and every node of the exact top-4 has
  // d2f <= T' = (sqrt(B) + delta)^2 (1+2e-5). Pass 2 evaluates the exact fp64
  // (d2, idx) order only for nodes with d2f <= T' (a handful per candidate).
  const double delta = 1.8 * 5.9604644775390625e-8 * (double)__int_as_float(*rmax_bits);
  float t0 = INFINITY, t1 = INFINITY, t2 = INFINITY, t3 = INFINITY;
  for (int base = 0; base < sp.N; base += kScreenThreads) {
    __syncthreads();
    if (base + threadIdx.x < sp.N) tile[threadIdx.x] = node_live_f[base + threadIdx.x];
    __syncthreads();
    const int lim = min(kScreenThreads, sp.N - base);
    if (active)
      for (int t = lane_k; t < lim; t += kScreenLanes) {
        const float4 q = tile[t];
        const float dx = q.x - xf, dy = q.y - yf, dz = q.z - zf;
        float v = (dx * dx + dy * dy) + dz * dz, m;
        m = fminf(t0, v); v = fmaxf(t0, v); t0 = m;
        m = fminf(t1, v); v = fmaxf(t1, v); t1 = m;
        m = fminf(t2, v); v = fmaxf(t2, v); t2 = m;
        t3 = fminf(t3, v);
      }
  }
#pragma unroll
  for (int off = kScreenLanes / 2; off > 0; off >>= 1) {
    const float o0 = __shfl_xor_sync(0xffffffffu, t0, off), o1 = __shfl_xor_sync(0xffffffffu, t1, off),
                o2 = __shfl_xor_sync(0xffffffffu, t2, off), o3 = __shfl_xor_sync(0xffffffffu, t3, off);
    const float ov[4] = {o0, o1, o2, o3};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float v = ov[u], m;
      m = fminf(t0, v); v = fmaxf(t0, v); t0 = m;
      m = fminf(t1, v); v = fmaxf(t1, v); t1 = m;
      m = fminf(t2, v); v = fmaxf(t2, v); t2 = m;
      t3 = fminf(t3, v);
    }
  }
  float thr = INFINITY;
  if (t3 < INFINITY) {
    const double B = sqrt((double)t3 * (1.0 + 2e-5)) + delta;
    const double tp = B + delta;
    thr = (float)(tp * tp * (1.0 + 2e-5)) + 1e-37f;
  }
  for (int base = 0; base < sp.N; base += kScreenThreads) {
    __syncthreads();
    if (base + threadIdx.x < sp.N) tile[threadIdx.x] = node_live_f[base + threadIdx.x];
    __syncthreads();
    const int lim = min(kScreenThreads, sp.N - base);
    if (active)
      for (int t = lane_k; t < lim; t += kScreenLanes) {
        const float4 q = tile[t];
        const float dx = q.x - xf, dy = q.y - yf, dz = q.z - zf;
        if ((dx * dx + dy * dy) + dz * dz > thr) continue;
        const double4 nl = node_live[base + t];
        knn4_insert(sqn(sub(v3(nl.x, nl.y, nl.z), x)), base + t, bd, bi);
      }
  }
  knn4_merge_lanes<kScreenLanes>(bd, bi);
  if (!active || lane_k != 0) return;
  int ids[4];
  float ws[4];
  int cnt = 0;
  int res = 0;
  if (sp.N > 0) res = screen_one(x, bd, bi, node_pos, node_live, node_dq, sp, ids, ws, cnt);
  if (sp.N == 0) {
    for (int m = 0; m < 4; ++m) {
      ids[m] = -1;
      ws[m] = 0.f;
    }
  }
  ok[k] = res == 2 ? 1 : 0;
  res_out[k] = res;
  if (res == 0) atomicAdd(low, 1);
  if (res == 1) atomicAdd(comp, 1);
  cki[k] = make_int4(ids[0], ids[1], ids[2], ids[3]);
  ckw[k] = make_float4(ws[0], ws[1], ws[2], ws[3]);
}

// Persistent grid (the candidate count is on the device): blocks stride over
// candidate groups; every thread of a block runs the same rounds (the tiled
// fallback synchronises the block).
__global__ void __launch_bounds__(kScreenThreads, 2) k_screen(
    const float4* __restrict__ cp, const int* __restrict__ n_cand_dev,
    const double4* __restrict__ node_pos, const double4* __restrict__ node_live,
    const float4* __restrict__ node_live_f, const int* __restrict__ rmax_bits,
    const double4* __restrict__ node_dq, ScreenParams sp, int4* __restrict__ cki,
    float4* __restrict__ ckw, int* __restrict__ ok, int* __restrict__ res_out,
    int* __restrict__ low, int* __restrict__ comp, KnnGridView grid, int use_grid) {
  __shared__ float4 tile[kScreenThreads];
  const int n = *n_cand_dev;
  constexpr int kPerBlock = kScreenThreads / kScreenLanes;
  for (int kb = blockIdx.x * kPerBlock; kb < n; kb += gridDim.x * kPerBlock)
    screen_block(kb, n, tile, cp, node_pos, node_live, node_live_f, rmax_bits, node_dq, sp, cki,
                 ckw, ok, res_out, low, comp, grid, use_grid);
}

__global__ void k_append(const int* __restrict__ ok, const int* __restrict__ scan,
                         const int* __restrict__ n_cand_dev, const float4* __restrict__ cp,
                         const float4* __restrict__ cn, const int4* __restrict__ cki,
                         const float4* __restrict__ ckw, int n_old, int cap, int t_now, ModelBuf m,
                         int* __restrict__ err) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= *n_cand_dev || !ok[k]) return;
  const int o = n_old + scan[k];
  if (o >= cap) {
    atomicOr(err, 16);
    return;
  }
  m.rp[o] = cp[k];
  m.lp[o] = cp[k];
  m.rn[o] = cn[k];
  m.ln[o] = cn[k];
  m.t[o] = make_int2(t_now, t_now);
  m.ki[o] = cki[k];
  m.kw[o] = ckw[k];
}

struct RemoveParams {
  Rig w2c;
  double fx, fy, cx, cy;
  int W, H, f, t_now, t_low;
  double delta_stable, delta_distance, delta_normal;
};

__global__ void __launch_bounds__(256) k_remove(ModelBuf m, const int* __restrict__ n_dev, int n_old,
                                                const int* __restrict__ im_idx, RemoveParams rp,
                                                int* __restrict__ keep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = n_old + *n_dev;
  if (i >= n) {
    if (i < n_old + rp.W * rp.H) keep[i] = 0;
    return;
  }
  const float4 lp = m.lp[i], ln = m.ln[i];
  const int2 t = m.t[i];
  const double ci = ln.w;
  int rm = 0;
  if (rp.t_now - t.x > rp.t_low && ci < rp.delta_stable) {
    rm = 1;
  } else {
    const V3 sp = v3(lp.x, lp.y, lp.z), sn = v3(ln.x, ln.y, ln.z);
    const V3 pc = rig_apply(rp.w2c, sp);
    if (pc.z > 0) {
      const double u = rp.fx * pc.x / pc.z + rp.cx;
      const double v = rp.fy * pc.y / pc.z + rp.cy;
      const double fsx = floor(rp.f * (u + 0.5)), fsy = floor(rp.f * (v + 0.5));
      const int Wf = rp.W * rp.f, Hf = rp.H * rp.f;
      if (fabs(fsx) < 1e9 && fabs(fsy) < 1e9) {
        // the 3x3 neighbourhood's ids, then their surfels three at a time: the
        // verdict is an OR over the neighbours, so all loads can be in flight
        const int sx = (int)fsx, sy = (int)fsy;
        int js[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) {
          const int nx = sx + q % 3 - 1, ny = sy + q / 3 - 1;
          js[q] = (nx < 0 || nx >= Wf || ny < 0 || ny >= Hf) ? kEmptyIdx
                                                             : __ldg(im_idx + (size_t)ny * Wf + nx);
        }
#pragma unroll
        for (int g = 0; g < 9; g += 3) {
          float4 op[3], on[3];
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const int j = js[g + q];
            if (j != kEmptyIdx && j != i) {
              op[q] = m.lp[j];
              on[q] = m.ln[j];
            }
          }
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const int j = js[g + q];
            if (j == kEmptyIdx || j == i) continue;
            const double oc = on[q].w;
            if (oc <= rp.delta_stable) continue;
            if (oc <= ci) continue;
            if (nrm(sub(v3(op[q].x, op[q].y, op[q].z), sp)) >= rp.delta_distance) continue;
            if (dot(v3(on[q].x, on[q].y, on[q].z), sn) < rp.delta_normal) continue;
            rm = 1;
          }
        }
      }
    }
  }
  keep[i] = rm ? 0 : 1;
}

// stable scatter of survivors into the alternate buffer + inverse warp (K2, K16)
// Also flags "some survivor is stable" (the next frame's render eligibility
// bootstrap test, raster.cpp:65-68) so that frame needs no extra pass.
__global__ void __launch_bounds__(256) k_compact_inverse(ModelBuf src, ModelBuf dst, int limit,
                                                         const int* __restrict__ keep,
                                                         const int* __restrict__ scan,
                                                         const double4* __restrict__ node_dq,
                                                         int* __restrict__ degenerate,
                                                         double delta_stable,
                                                         int* __restrict__ any_stable) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool kept = i < limit && keep[i];
  const bool st = kept && (double)src.ln[i].w > delta_stable;
  if (__ballot_sync(0xffffffffu, st) && (threadIdx.x & 31) == 0) atomicOr(any_stable, 1);
  if (!kept) return;
  const int o = scan[i];
  const float4 lp = src.lp[i], ln = src.ln[i];
  const int4 ki = src.ki[i];
  const float4 kw = src.kw[i];
  const Blend b = blend_entry(ki, kw, node_dq);
  float4 rp = lp, rn = ln;
  if (!b.degenerate) {
    const Rig inv = rig_inverse(blend_rig_fast(b));
    const V3 p = rig_apply(inv, v3(lp.x, lp.y, lp.z));
    const V3 q = rig_rotate(inv, v3(ln.x, ln.y, ln.z));
    rp = make_float4((float)p.x, (float)p.y, (float)p.z, lp.w);
    rn = make_float4((float)q.x, (float)q.y, (float)q.z, ln.w);
  } else {
    atomicAdd(degenerate, 1);
  }
  dst.lp[o] = lp;
  dst.ln[o] = ln;
  dst.rp[o] = rp;
  dst.rn[o] = rn;
  dst.t[o] = src.t[i];
  dst.ki[o] = ki;
  dst.kw[o] = kw;
}

// clean_and_reset keep rule (reinit.cpp:37-75)
struct CleanParams {
  Rig pose, w2c;
  double fx, fy, cx, cy, gate, delta_normal;
  int W, H;
};
__global__ void k_clean(ModelBuf m, int n, const double4* __restrict__ fvert,
                        const double4* __restrict__ fnrm, const uint8_t* __restrict__ fflag,
                        CleanParams cp, int* __restrict__ keep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 lp = m.lp[i], ln = m.ln[i];
  const V3 sp = v3(lp.x, lp.y, lp.z), sn = v3(ln.x, ln.y, ln.z);
  const V3 pc = rig_apply(cp.w2c, sp);
  bool kp = true;
  if (pc.z > 0 && dot(rig_rotate(cp.w2c, sn), pc) < 0) {
    const double u = cp.fx * pc.x / pc.z + cp.cx;
    const double v = cp.fy * pc.y / pc.z + cp.cy;
    if (fabs(u) < 1e9 && fabs(v) < 1e9) {
      const int ui = (int)llround(u), vi = (int)llround(v);
      if (ui >= 0 && ui < cp.W && vi >= 0 && vi < cp.H) {
        bool corr = false, occl = false, anym = false;
        for (int dy = -1; dy <= 2 && !corr; ++dy)
          for (int dx = -1; dx <= 2; ++dx) {
            const int x = ui + dx, y = vi + dy;
            if (x < 0 || x >= cp.W || y < 0 || y >= cp.H) continue;
            const size_t c = (size_t)y * cp.W + x;
            const uint8_t fl = fflag[c];
            if (!(fl & 1)) continue;
            anym = true;
            const double4 fv = fvert[c];
            if (fv.z < pc.z - cp.gate) occl = true;
            if (!(fl & 2)) continue;
            const V3 vd = rig_apply(cp.pose, v3(fv.x, fv.y, fv.z));
            if (nrm(sub(vd, sp)) >= cp.gate) continue;
            const double4 fn = fnrm[c];
            if (dot(rig_rotate(cp.pose, v3(fn.x, fn.y, fn.z)), sn) < cp.delta_normal) continue;
            corr = true;
            break;
          }
        kp = corr || occl || !anym;
      }
    }
  }
  keep[i] = kp ? 1 : 0;
}
__global__ void k_compact_reset(ModelBuf src, ModelBuf dst, int n, const int* __restrict__ keep,
                                const int* __restrict__ scan) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !keep[i]) return;
  const int o = scan[i];
  const float4 lp = src.lp[i], ln = src.ln[i];
  dst.lp[o] = lp;
  dst.ln[o] = ln;
  dst.rp[o] = lp;
  dst.rn[o] = ln;
  dst.t[o] = src.t[i];
  dst.ki[o] = make_int4(-1, -1, -1, -1);
  dst.kw[o] = make_float4(0, 0, 0, 0);
}

FuseParams fuse_params(Ctx& c, const double* pose, int t_now) {
  FuseParams fp;
  fp.pose = rig_load(pose);
  fp.W = c.W;
  fp.H = c.H;
  fp.f = c.im_factor;
  fp.t_now = t_now;
  fp.dd2 = c.cfg.delta_distance * c.cfg.delta_distance;
  fp.dn = c.cfg.delta_normal;
  return fp;
}

ScreenParams screen_params(Ctx& c) {
  ScreenParams sp;
  sp.N = c.n_nodes;
  sp.K = std::min(4, c.cfg.knn_k);
  sp.compressive = c.cfg.compressive_check ? 1 : 0;
  sp.eps = c.cfg.epsilon;
  sp.delta_nn = c.cfg.delta_nn;
  return sp;
}

}  // namespace

// fuse_depth + candidate compaction; counts stay on the device (dsc)
void fuse_depth_async(Ctx& c, const double* pose, int t_now) {
  if (!c.im_ready) fail(DS_ERR_INVALID_ARGUMENT, "fuse_depth: no index map rendered");
  DS_CUDA(cudaMemsetAsync(&c.dsc->fused, 0, sizeof(int), c.stream));
  const int P = c.P;
  // per pixel: frame maps 65 B, 16 index cells x 4 B, winner read+write 64 B, flag 4 B
  DS_LAUNCH(c, KK_FUSE, 197.0 * P, cdiv(P, 256), 256, 0, k_fuse, c.im_idx, c.M(), c.f_vert, c.f_nrm,
            c.f_flag, fuse_params(c, pose, t_now), c.cand_flag, &c.dsc->fused);
  scan_exclusive(c, c.cand_flag, c.cand_scan, P);
  DS_LAUNCH(c, KK_FUSE, 40.0 * P, cdiv(P, 256), 256, 0, k_write_cands, c.cand_flag, c.cand_scan, P,
            c.f_vert, c.f_nrm, rig_load(pose), c.cand_pix, c.cand_p, c.cand_n);
  DS_CUDA(cudaMemcpyAsync(&c.dsc->n_cand, c.cand_scan + P, sizeof(int), cudaMemcpyDeviceToDevice,
                          c.stream));
}

void fuse_depth(Ctx& c, const double* pose, int t_now, int* fused, int* n_cand) {
  fuse_depth_async(c, pose, t_now);
  fetch_scalars(c);
  *fused = c.hsc->fused;
  *n_cand = c.hsc->n_cand;
}

// Live node positions + their K-NN grid depend only on the solved nodes: the
// frame loop launches them on the side stream right after the solve, so they
// overlap the full-model warp, the index map and the depth fusion.
void prepare_live_nodes_async(Ctx& c) {
  DS_CUDA(cudaEventRecord(c.ev_fork, c.stream));
  DS_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
  cudaStream_t main_stream = c.stream;
  c.stream = c.side;
  try {
    node_live_positions(c);
    c.live_grid = c.screen_grid &&
                  build_knn_grid(c, c.grid_live, c.node_live, c.n_nodes, c.live_cell * c.cfg.node_sigma);
  } catch (...) {
    c.stream = main_stream;
    throw;
  }
  c.stream = main_stream;
  DS_CUDA(cudaEventRecord(c.ev_live, c.side));
  c.live_pending = true;
}

void screen_candidates_async(Ctx& c) {
  DS_CUDA(cudaMemsetAsync(&c.dsc->low_support, 0, sizeof(int), c.stream));
  DS_CUDA(cudaMemsetAsync(&c.dsc->comp_rejected, 0, sizeof(int), c.stream));
  DS_CUDA(cudaMemsetAsync(c.cand_ok, 0, sizeof(int) * c.P, c.stream));
  bool grid;
  if (c.live_pending) {
    DS_CUDA(cudaStreamWaitEvent(c.stream, c.ev_live, 0));
    grid = c.live_grid;
    c.live_pending = false;
  } else {
    node_live_positions(c);
    grid = c.screen_grid &&
           build_knn_grid(c, c.grid_live, c.node_live, c.n_nodes, c.live_cell * c.cfg.node_sigma);
  }
  DS_LAUNCH(c, KK_SKIN_APPEND, 64.0 * c.P * 0.02,
            std::min(cdiv((long long)c.P * kScreenLanes, kScreenThreads), 2 * c.num_sms),
            kScreenThreads, 0, k_screen, c.cand_p,
            &c.dsc->n_cand, c.node_pos, c.node_live, c.node_live_f, &c.dsc->rmax_bits, c.node_dq,
            screen_params(c), c.cand_ki,
            c.cand_kw, c.cand_ok, c.cand_flag, &c.dsc->low_support, &c.dsc->comp_rejected,
            knn_view(c.grid_live, 3), grid ? 1 : 0);
}

void screen_candidates(Ctx& c, int n_cand, int* low_support, int* comp_rejected, int* accepted) {
  DS_CUDA(cudaMemcpyAsync(&c.dsc->n_cand, &n_cand, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  screen_candidates_async(c);
  fetch_scalars(c);
  *low_support = c.hsc->low_support;
  *comp_rejected = c.hsc->comp_rejected;
  *accepted = n_cand - c.hsc->low_support - c.hsc->comp_rejected;
}

void removal_mask(Ctx& c, const double* pose, int t_now, int n) {
  RemoveParams rp;
  rp.w2c = rig_inverse(rig_load(pose));
  rp.fx = c.cfg.fx;
  rp.fy = c.cfg.fy;
  rp.cx = c.cfg.cx;
  rp.cy = c.cfg.cy;
  rp.W = c.W;
  rp.H = c.H;
  rp.f = c.im_factor;
  rp.t_now = t_now;
  rp.t_low = c.cfg.t_low_confid;
  rp.delta_stable = c.cfg.delta_stable;
  rp.delta_distance = c.cfg.delta_distance;
  rp.delta_normal = c.cfg.delta_normal;
  int zero = 0;
  DS_CUDA(cudaMemcpyAsync(&c.dsc->n_accept, &zero, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  DS_LAUNCH(c, KK_REMOVE, 76.0 * n, cdiv(n, 256), 256, 0, k_remove, c.M(), &c.dsc->n_accept, n,
            c.im_idx, rp, c.keep);
}

// apply_fusion (fusion.cpp:220-307)
void apply_fusion(Ctx& c, const double* pose, int t_now, ds_fusion_outcome* out) {
  ds_fusion_outcome oc{};
  const int P = c.P;
  render_index_map(c, pose, c.cfg.supersample_factor, c.warp_in_index_map ? c.node_dq : nullptr);
  c.warp_in_index_map = false;
  fuse_depth_async(c, pose, t_now);
  screen_candidates_async(c);
  // accepted candidates keep row-major order (fusion.cpp:235-257)
  scan_exclusive(c, c.cand_ok, c.cand_ok_scan, P);
  DS_CUDA(cudaMemcpyAsync(&c.dsc->n_accept, c.cand_ok_scan + P, sizeof(int),
                          cudaMemcpyDeviceToDevice, c.stream));
  const int n_old = c.n_surfels;
  DS_CUDA(cudaMemsetAsync(&c.dsc->err, 0, sizeof(int), c.stream));
  DS_LAUNCH(c, KK_FUSE, 64.0 * P * 0.02, cdiv(P, 256), 256, 0, k_append, c.cand_ok, c.cand_ok_scan,
            &c.dsc->n_cand, c.cand_p, c.cand_n, c.cand_ki, c.cand_kw, n_old, c.S_cap, t_now, c.M(),
            &c.dsc->err);
  // removal over old + appended (upper bound n_old + P, exact count on device)
  RemoveParams rp;
  rp.w2c = rig_inverse(rig_load(pose));
  rp.fx = c.cfg.fx;
  rp.fy = c.cfg.fy;
  rp.cx = c.cfg.cx;
  rp.cy = c.cfg.cy;
  rp.W = c.W;
  rp.H = c.H;
  rp.f = c.im_factor;
  rp.t_now = t_now;
  rp.t_low = c.cfg.t_low_confid;
  rp.delta_stable = c.cfg.delta_stable;
  rp.delta_distance = c.cfg.delta_distance;
  rp.delta_normal = c.cfg.delta_normal;
  const int limit = std::min(n_old + P, c.S_cap);
  DS_LAUNCH(c, KK_REMOVE, 76.0 * limit, cdiv(limit, 256), 256, 0, k_remove, c.M(), &c.dsc->n_accept,
            n_old, c.im_idx, rp, c.keep);
  scan_exclusive(c, c.keep, c.keep_scan, limit);
  DS_CUDA(cudaMemsetAsync(&c.dsc->degenerate, 0, sizeof(int), c.stream));
  DS_CUDA(cudaMemsetAsync(c.any_stable_pre, 0, sizeof(int), c.stream));
  DS_LAUNCH(c, KK_COMPACT_INVERSE_WARP, 104.0 * 2 * limit, cdiv(limit, 256), 256, 0,
            k_compact_inverse, c.M(), c.Malt(), limit, c.keep, c.keep_scan, c.node_dq,
            &c.dsc->degenerate, c.cfg.delta_stable, c.any_stable_pre);
  DS_CUDA(cudaMemcpyAsync(&c.dsc->n_keep, c.keep_scan + limit, sizeof(int),
                          cudaMemcpyDeviceToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(&c.dsc->surv_old, c.keep_scan + n_old, sizeof(int),
                          cudaMemcpyDeviceToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(&c.dsc->fuse_err, &c.dsc->err, sizeof(int), cudaMemcpyDeviceToDevice,
                          c.stream));
  c.cur ^= 1;
  // extend the warp field over the appended survivors (compacted order):
  // positions rp[surv_old, n_keep) of the compacted model, counts on the
  // device -- no host sync here; the greedy pass's fetch brings every count
  const int first_new = c.n_nodes;
  oc.new_nodes = extend_warp_field_dev(c, c.M().rp, &c.dsc->surv_old, &c.dsc->n_keep,
                                       std::min(P, c.S_cap));
  if (c.hsc->fuse_err & 16) fail(DS_ERR_CAPACITY, "surfel capacity exceeded while appending");
  const int n_acc = c.hsc->n_accept;
  const int n_new = c.hsc->n_keep;
  oc.fused = c.hsc->fused;
  oc.appended = n_acc;
  oc.low_support_rejected = c.hsc->low_support;
  oc.compressive_rejected = c.hsc->comp_rejected;
  oc.removed = n_old + n_acc - n_new;
  oc.degenerate_warps = c.hsc->degenerate;
  c.n_surfels = n_new;
  if (oc.new_nodes > 0) update_skinning_incremental(c, first_new);
  // (seeds, edges and the incremental reskin stay on the side stream: joined
  // by the next API call or after the next frame's rigid ICP is launched;
  // DS_NO_DEFER=1 joins here)
  if (c.no_defer) join_node_updates(c);
  c.any_stable_ready = true;  // computed by the compaction for this model
  c.pattern_ready = false;
  *out = oc;
}

int clean_and_reset(Ctx& c, const double* pose, int* survivors) {
  const int n = c.n_surfels;
  CleanParams cp;
  cp.pose = rig_load(pose);
  cp.w2c = rig_inverse(cp.pose);
  cp.fx = c.cfg.fx;
  cp.fy = c.cfg.fy;
  cp.cx = c.cfg.cx;
  cp.cy = c.cfg.cy;
  cp.gate = c.cfg.delta_distance_reinit;
  cp.delta_normal = c.cfg.delta_normal;
  cp.W = c.W;
  cp.H = c.H;
  if (n > 0) {
    DS_LAUNCH(c, KK_MISC, 40.0 * n, cdiv(n, 256), 256, 0, k_clean, c.M(), n, c.f_vert, c.f_nrm,
              c.f_flag, cp, c.keep);
  }
  scan_exclusive(c, c.keep, c.keep_scan, n);
  int kept = 0;
  DS_CUDA(cudaMemcpyAsync(&kept, c.keep_scan + n, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  sync(c);
  if (kept == 0) fail(DS_ERR_EMPTY_GEOMETRY, "clean_and_reset: no surfel survived");
  DS_LAUNCH(c, KK_MISC, 72.0 * n, cdiv(n, 256), 256, 0, k_compact_reset, c.M(), c.Malt(), n, c.keep,
            c.keep_scan);
  c.cur ^= 1;
  c.n_surfels = kept;
  if (survivors) *survivors = kept;
  init_warp_field(c);
  c.pattern_ready = false;
  return n - kept;
}

}  // namespace ds
