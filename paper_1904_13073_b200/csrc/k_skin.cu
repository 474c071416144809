// k_skin.cu — node graph construction and skinning (K17-K21).
//   greedy sigma-sampling   warp_field.cpp:88-97 (init) / :151-157 (extension):
//       exact ordered greedy (lexicographic-first maximal independent set) in
//       one persistent CTA: candidates are tested 1024 at a time against a
//       sigma-cell hash of accepted nodes (27 cells, strict d2 < sigma^2,
//       spatial_grid.hpp:46-60); the uncovered ones of a chunk are resolved in
//       index order, one accepted node per block-wide round.
//   node edges (k=8)        warp_field.cpp:42-56, warp per node, (d2, idx) order
//   skinning KNN (K=4)      warp_field.cpp:60-79 (VoxelGrid::knn is exact, so a
//       brute-force (d2, idx) scan over shared-memory node tiles is identical)
//   extension seeds         warp_field.cpp:159-178
//   incremental skinning    warp_field.cpp:186-236
#include "ds_blend.cuh"
#include "ds_context.cuh"
#include "ds_knn.cuh"

namespace ds {
namespace {

constexpr long long kEmptyKey = -1;

struct HashView {
  long long* key;
  int* cnt;
  int* ids;
  int mask;
  double inv_cell;
};

__device__ __forceinline__ long long pack_cell(int x, int y, int z) {
  const long long b = 1LL << 20;
  return ((x + b) << 42) | ((y + b) << 21) | (z + b);
}
__device__ __forceinline__ unsigned hash_cell(long long k) {
  unsigned long long h = (unsigned long long)k * 0x9E3779B97F4A7C15ULL;
  return (unsigned)(h >> 32);
}
__device__ __forceinline__ void cell_of(const HashView& h, V3 p, int& x, int& y, int& z) {
  x = (int)floor(p.x * h.inv_cell);
  y = (int)floor(p.y * h.inv_cell);
  z = (int)floor(p.z * h.inv_cell);
}
__device__ __forceinline__ double4 ldcg_d4(const double4* p) {
  const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}
__device__ int ht_find(const HashView& h, long long k) {
  unsigned s = hash_cell(k) & h.mask;
  for (int probe = 0; probe <= h.mask; ++probe) {
    const long long v = __ldcg(h.key + s);
    if (v == k) return (int)s;
    if (v == kEmptyKey) return -1;
    s = (s + 1) & h.mask;
  }
  return -1;
}
// single-writer insert (only one thread of the greedy CTA mutates the table)
__device__ void ht_insert_single(const HashView& h, long long k, int id, int* err) {
  unsigned s = hash_cell(k) & h.mask;
  for (int probe = 0; probe <= h.mask; ++probe) {
    const long long v = __ldcg(h.key + s);
    if (v == k || v == kEmptyKey) {
      if (v == kEmptyKey) {
        h.key[s] = k;
        h.cnt[s] = 0;
      }
      const int c = __ldcg(h.cnt + s);
      if (c >= 8) {
        atomicOr(err, DERR_HASH_CELL);
        return;
      }
      h.ids[8 * s + c] = id;
      h.cnt[s] = c + 1;
      return;
    }
    s = (s + 1) & h.mask;
  }
  atomicOr(err, DERR_HASH_FULL);
}
__device__ bool ht_any_within(const HashView& h, const double4* node_pos, V3 p, double r2) {
  int cx, cy, cz;
  cell_of(h, p, cx, cy, cz);
  // centre cell first: a covered point usually exits on its own cell
  for (int o = 0; o < 27; ++o) {
        const int oc = (o + 13) % 27;  // 13 = (0,0,0)
        const int dx = oc % 3 - 1, dy = (oc / 3) % 3 - 1, dz = oc / 9 - 1;
        const int s = ht_find(h, pack_cell(cx + dx, cy + dy, cz + dz));
        if (s < 0) continue;
        const int c = __ldcg(h.cnt + s);
        for (int q = 0; q < c; ++q) {
          const int id = __ldcg(h.ids + 8 * s + q);
          const double4 np = ldcg_d4(node_pos + id);
          if (sqn(sub(v3(np.x, np.y, np.z), p)) < r2) return true;
        }
  }
  return false;
}

__global__ void k_ht_prefill(HashView h, const double4* __restrict__ node_pos, int n, int* err) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double4 np = node_pos[j];
  int cx, cy, cz;
  cell_of(h, v3(np.x, np.y, np.z), cx, cy, cz);
  const long long k = pack_cell(cx, cy, cz);
  unsigned s = hash_cell(k) & h.mask;
  for (int probe = 0; probe <= h.mask; ++probe) {
    const long long prev = (long long)atomicCAS((unsigned long long*)(h.key + s),
                                                (unsigned long long)kEmptyKey, (unsigned long long)k);
    if (prev == kEmptyKey || prev == k) {
      const int c = atomicAdd(h.cnt + s, 1);
      if (c < 8) h.ids[8 * s + c] = j;
      else atomicOr(err, DERR_HASH_CELL);
      return;
    }
    s = (s + 1) & h.mask;
  }
  atomicOr(err, DERR_HASH_FULL);
}

constexpr int kGreedyThreads = 1024;
constexpr int kListNodes = 1024;  // extension: new nodes kept in shared memory

// list_mode = 0 (init): coverage tested against the sigma-cell hash of all
// accepted nodes. list_mode = 1 (extension, after k_uncovered removed every
// candidate covered by a pre-existing node): only the nodes accepted by this
// launch can cover a candidate; they are tested from shared memory.
// M_dev != nullptr: the candidate count is read from the device (no host
// round trip between the pre-filter's compaction and the greedy pass)
__global__ void __launch_bounds__(kGreedyThreads) k_greedy_nodes(
    const float4* __restrict__ cand, int M, const int* __restrict__ M_dev, double sigma, HashView h,
    double4* node_pos, int* n_nodes, int N_cap, int list_mode, int* err) {
  if (M_dev) M = *M_dev;
  __shared__ int s_first;
  __shared__ int s_count;
  __shared__ int s_nlist;
  __shared__ double s_new[3];
  __shared__ double s_list[kListNodes][3];
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_count = *n_nodes;
    s_nlist = 0;
  }
  __syncthreads();
  const double r2 = sigma * sigma;
  for (int base = 0; base < M; base += kGreedyThreads) {
    const int i = base + tid;
    V3 p = v3(0, 0, 0);
    bool covered = true;
    if (i < M) {
      const float4 cp = cand[i];
      p = v3(cp.x, cp.y, cp.z);
      if (list_mode) {
        covered = false;
        for (int q = 0; q < s_nlist && !covered; ++q)
          covered = sqn(sub(v3(s_list[q][0], s_list[q][1], s_list[q][2]), p)) < r2;
      } else {
        covered = ht_any_within(h, node_pos, p, r2);
      }
    }
    for (;;) {
      if (tid == 0) s_first = 0x7fffffff;
      __syncthreads();
      if (!covered) atomicMin(&s_first, tid);
      __syncthreads();
      const int f = s_first;
      if (f == 0x7fffffff) break;
      if (tid == f) {
        const int id = s_count;
        if (id < N_cap) {
          node_pos[id] = make_double4(p.x, p.y, p.z, sigma);
          if (list_mode) {
            if (s_nlist < kListNodes) {
              s_list[s_nlist][0] = p.x;
              s_list[s_nlist][1] = p.y;
              s_list[s_nlist][2] = p.z;
              ++s_nlist;
            } else {
              atomicOr(err, DERR_HASH_FULL);  // host re-runs in hash mode
            }
          } else {
            int cx, cy, cz;
            cell_of(h, p, cx, cy, cz);
            ht_insert_single(h, pack_cell(cx, cy, cz), id, err);
          }
        } else {
          atomicOr(err, DERR_NODE_CAP);
        }
        s_count = id + 1;
        s_new[0] = p.x;
        s_new[1] = p.y;
        s_new[2] = p.z;
        covered = true;
      }
      __syncthreads();
      if (!covered && sqn(sub(v3(s_new[0], s_new[1], s_new[2]), p)) < r2) covered = true;
    }
  }
  if (tid == 0) *n_nodes = min(s_count, N_cap);
}

// Exact pre-filter for extension: a candidate within sigma of a pre-existing
// node is skipped by the ordered greedy whatever happens before it, so only the
// uncovered ones (kept in order) need the sequential pass.
// kUncLanes lanes per candidate split the 27 cells; a covered candidate
// (the common case) stops after the first round, where lane 0 holds its own cell.
constexpr int kUncLanes = 8;
// candidate i of cand: flag[i] = 1 when no node lies within sigma (kUncLanes
// lanes per candidate, all of the group call it)
__device__ __forceinline__ void uncovered_one(const float4* __restrict__ cand, int i, double sigma,
                                              HashView h, const double4* __restrict__ node_pos,
                                              int* __restrict__ flag) {
  const int lane = (blockIdx.x * blockDim.x + threadIdx.x) % kUncLanes;
  const unsigned gmask = 0xffu << ((threadIdx.x & 31) & ~(unsigned)(kUncLanes - 1));
  const float4 cp = cand[i];
  const V3 p = v3(cp.x, cp.y, cp.z);
  const double r2 = sigma * sigma;
  int cx, cy, cz;
  cell_of(h, p, cx, cy, cz);
  bool found = false;
  for (int base = 0; base < 27; base += kUncLanes) {
    const int o = base + lane;
    if (o < 27 && !found) {
      const int oc = (o + 13) % 27;  // 13 = (0,0,0): lane 0 of round 0 takes the own cell
      const int dx = oc % 3 - 1, dy = (oc / 3) % 3 - 1, dz = oc / 9 - 1;
      const int s = ht_find(h, pack_cell(cx + dx, cy + dy, cz + dz));
      if (s >= 0) {
        const int c = __ldcg(h.cnt + s);
        for (int q = 0; q < c && !found; ++q) {
          const int id = __ldcg(h.ids + 8 * s + q);
          const double4 np = ldcg_d4(node_pos + id);
          if (sqn(sub(v3(np.x, np.y, np.z), p)) < r2) found = true;
        }
      }
    }
    if (__any_sync(gmask, found)) {
      found = true;
      break;
    }
  }
  if (lane == 0) flag[i] = found ? 0 : 1;
}
__global__ void k_uncovered(const float4* __restrict__ cand, int M, double sigma, HashView h,
                            const double4* __restrict__ node_pos, int* __restrict__ flag) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = gt / kUncLanes;
  if (i >= M) return;  // whole group
  uncovered_one(cand, i, sigma, h, node_pos, flag);
}
__global__ void k_gather_uncovered(const float4* __restrict__ cand, const int* __restrict__ flag,
                                   const int* __restrict__ scan, int M, float4* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M && flag[i]) out[scan[i]] = cand[i];
}
// device-count variants: candidates base[*off, *end), flags zero past the count
__global__ void k_uncovered_dev(const float4* __restrict__ base, const int* __restrict__ off,
                                const int* __restrict__ end, int bound, double sigma, HashView h,
                                const double4* __restrict__ node_pos, int* __restrict__ flag) {
  const int o = *off, M = *end - o;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = gt / kUncLanes;
  if (i >= bound) return;
  if (i >= M) {
    if (gt % kUncLanes == 0) flag[i] = 0;
    return;  // whole group
  }
  uncovered_one(base + o, i, sigma, h, node_pos, flag);
}
__global__ void k_gather_uncovered_dev(const float4* __restrict__ base, const int* __restrict__ off,
                                       const int* __restrict__ end, const int* __restrict__ flag,
                                       const int* __restrict__ scan, int bound,
                                       float4* __restrict__ out) {
  const int o = *off, M = *end - o;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < bound && i < M && flag[i]) out[scan[i]] = base[o + i];
}

__global__ void k_identity_dq(double4* dq, int from, int to) {
  const int j = from + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= to) return;
  dq[2 * j] = make_double4(1, 0, 0, 0);
  dq[2 * j + 1] = make_double4(0, 0, 0, 0);
}

// Warp per node: k nearest other nodes by (d2, index).
__global__ void k_node_edges(const double4* __restrict__ pos, int n, int k, int* __restrict__ nbr) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const int j = warp;
  const double4 pj = pos[j];
  double bd[8];
  int bi[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    bd[t] = INFINITY;
    bi[t] = 0x7fffffff;
  }
#pragma unroll 4
  for (int i = lane; i < n; i += 32) {
    const double4 pi = pos[i];
    const double d2 = sqn(sub(v3(pi.x, pi.y, pi.z), v3(pj.x, pj.y, pj.z)));
    if (i == j || !nb_less(d2, i, bd[7], bi[7])) continue;
    // insert keeping ascending (d2, idx) order
    double cd = d2;
    int ci = i;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (nb_less(cd, ci, bd[t], bi[t])) {
        const double td = bd[t];
        const int ti = bi[t];
        bd[t] = cd;
        bi[t] = ci;
        cd = td;
        ci = ti;
      }
    }
  }
  for (int r = 0; r < 8; ++r) {
    double md = bd[0];
    int mi = bi[0];
    for (int off = 16; off > 0; off >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, md, off);
      const int oi = __shfl_xor_sync(0xffffffffu, mi, off);
      if (nb_less(od, oi, md, mi)) {
        md = od;
        mi = oi;
      }
    }
    if (lane == 0) nbr[8 * j + r] = (r < k && mi != 0x7fffffff) ? mi : -1;
    if (bi[0] == mi && mi != 0x7fffffff) {  // winner pops its head
#pragma unroll
      for (int t = 0; t < 7; ++t) {
        bd[t] = bd[t + 1];
        bi[t] = bi[t + 1];
      }
      bd[7] = INFINITY;
      bi[7] = 0x7fffffff;
    }
  }
}

// Grid versions (ds_knn.cuh): same exact (d2, index) results as the brute-force
// kernels, visiting only the Chebyshev shells the distance bound requires;
// queries that exhaust the shell limit fall back to the full scan.
constexpr int kKnnRing = 3;

constexpr int kEdgeLanes = 8;  // lanes per node query

__global__ void k_node_edges_grid(const double4* __restrict__ pos, int n, int k, KnnGridView g,
                                  int* __restrict__ nbr) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) / kEdgeLanes;
  const int lane = threadIdx.x & (kEdgeLanes - 1);
  if (j >= n) return;  // whole group
  const double4 pj = pos[j];
  const V3 x = v3(pj.x, pj.y, pj.z);
  double md[8];
  int mi[8];
  if (!knn_grid_query<8, kEdgeLanes>(g, pos, x, [j](int id) { return id != j; }, md, mi)) {
    double bd[8];
    int bi[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      bd[t] = INFINITY;
      bi[t] = 0x7fffffff;
    }
    for (int i = lane; i < n; i += kEdgeLanes) {
      if (i == j) continue;
      const double4 pi = pos[i];
      knnk_insert<8>(sqn(sub(v3(pi.x, pi.y, pi.z), x)), i, bd, bi);
    }
    knnk_merged<8, kEdgeLanes>(bd, bi, md, mi);
  }
  if (lane == 0)
#pragma unroll
    for (int r = 0; r < 8; ++r) nbr[8 * j + r] = (r < k && mi[r] != 0x7fffffff) ? mi[r] : -1;
}

constexpr int kTile = 256;

// Thread per surfel: exact K nearest nodes by (d2, idx), Gaussian weights.
__global__ void __launch_bounds__(kTile) k_skin_knn(ModelBuf m, int n, const double4* __restrict__ pos,
                                                    int N, int K) {
  __shared__ double4 tile[kTile];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  V3 p = v3(0, 0, 0);
  if (i < n) {
    const float4 rp = m.rp[i];
    p = v3(rp.x, rp.y, rp.z);
  }
  double bd[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
  int bi[4] = {0x7fffffff, 0x7fffffff, 0x7fffffff, 0x7fffffff};
  float thr = INFINITY;
  for (int base = 0; base < N; base += kTile) {
    __syncthreads();
    if (base + threadIdx.x < N) tile[threadIdx.x] = pos[base + threadIdx.x];
    __syncthreads();
    const int lim = min(kTile, N - base);
    if (i < n) {
      for (int t = 0; t < lim; ++t) {
        const double4 q = tile[t];
        // fp32 pre-test (see k_screen): never rejects a node of the exact top-K
        const float fx = (float)(q.x - p.x), fy = (float)(q.y - p.y), fz = (float)(q.z - p.z);
        if ((fx * fx + fy * fy) + fz * fz > thr) continue;
        const double d2 = sqn(sub(v3(q.x, q.y, q.z), p));
        const int id = base + t;
        if (!nb_less(d2, id, bd[3], bi[3])) continue;
        double cd = d2;
        int ci = id;
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
        if (bd[3] < INFINITY) thr = (float)(bd[3] * (1.0 + 1e-5)) + 1e-37f;
      }
    }
  }
  if (i >= n) return;
  int ids[4];
  float w[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const bool ok = s < K && bi[s] != 0x7fffffff;
    ids[s] = ok ? bi[s] : -1;
    if (ok) {
      const double4 q = pos[bi[s]];
      w[s] = (float)skin_weight(p, v3(q.x, q.y, q.z), q.w);
    } else {
      w[s] = 0.f;
    }
  }
  m.ki[i] = make_int4(ids[0], ids[1], ids[2], ids[3]);
  m.kw[i] = make_float4(w[0], w[1], w[2], w[3]);
}

// Thread per surfel on the node grid (init_warp_field's skin_positions_bulk,
// warp_field.cpp:60-79): exact 4-NN by (d2, idx), Gaussian weights.
__global__ void __launch_bounds__(256) k_skin_knn_grid(ModelBuf m, int n,
                                                       const double4* __restrict__ pos, int N,
                                                       int K, KnnGridView g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 rp = m.rp[i];
  const V3 p = v3(rp.x, rp.y, rp.z);
  double bd[4], md[4];
  int bi[4], mi[4];
  if (!knn_grid_query<4, 1>(g, pos, p, [](int) { return true; }, md, mi)) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      bd[s] = INFINITY;
      bi[s] = 0x7fffffff;
    }
    for (int j = 0; j < N; ++j) {
      const double4 q = pos[j];
      knn4_insert(sqn(sub(v3(q.x, q.y, q.z), p)), j, bd, bi);
    }
  } else {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      bd[s] = md[s];
      bi[s] = mi[s];
    }
  }
  int ids[4];
  float w[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const bool ok = s < K && bi[s] != 0x7fffffff;
    ids[s] = ok ? bi[s] : -1;
    if (ok) {
      const double4 q = pos[bi[s]];
      w[s] = (float)skin_weight(p, v3(q.x, q.y, q.z), q.w);
    } else {
      w[s] = 0.f;
    }
  }
  m.ki[i] = make_int4(ids[0], ids[1], ids[2], ids[3]);
  m.kw[i] = make_float4(w[0], w[1], w[2], w[3]);
}

// Seeds of appended nodes from their K nearest pre-existing nodes
// (warp_field.cpp:163-177). A CTA per new node: 8 warps scan strided subsets of
// the N0 pre-existing nodes (or one grid query for large node sets), warp
// shuffle merges, then warp 0 merges the 8 warp lists and lane 0 blends the DQs.
constexpr int kSeedThreads = 256;
__global__ void __launch_bounds__(kSeedThreads) k_seed_dq(const double4* __restrict__ pos,
                                                         double4* dq, int N0, int N, int K,
                                                         KnnGridView g, int use_grid) {
  __shared__ double s_d[kSeedThreads / 32][4];
  __shared__ int s_i[kSeedThreads / 32][4];
  const int jn = N0 + blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (jn >= N) return;  // block-uniform
  DQ out = dq_identity();
  if (N0 > 0) {
    const double4 pn = pos[jn];
    const V3 p = v3(pn.x, pn.y, pn.z);
    double bd[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
    int bi[4] = {0x7fffffff, 0x7fffffff, 0x7fffffff, 0x7fffffff};
    if (use_grid) {
      if (wid == 0) {
        double md[4];
        int mi[4];
        if (knn_grid_query<4, 32>(g, pos, p, [N0](int id) { return id < N0; }, md, mi)) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            bd[t] = md[t];
            bi[t] = mi[t];
          }
        } else {
          for (int i = lane; i < N0; i += 32) {
            const double4 q = pos[i];
            knn4_insert(sqn(sub(v3(q.x, q.y, q.z), p)), i, bd, bi);
          }
          knn4_merge_lanes<32>(bd, bi);
        }
      }
    } else {
#pragma unroll 4
      for (int i = threadIdx.x; i < N0; i += kSeedThreads) {
        const double4 q = pos[i];
        knn4_insert(sqn(sub(v3(q.x, q.y, q.z), p)), i, bd, bi);
      }
      knn4_merge_lanes<32>(bd, bi);
      if (lane == 0)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          s_d[wid][t] = bd[t];
          s_i[wid][t] = bi[t];
        }
      __syncthreads();
      if (wid == 0) {  // lane w < 8 holds warp w's list, then a butterfly over 8 lanes
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          bd[t] = lane < kSeedThreads / 32 ? s_d[lane][t] : INFINITY;
          bi[t] = lane < kSeedThreads / 32 ? s_i[lane][t] : 0x7fffffff;
        }
        knn4_merge_lanes<32>(bd, bi);
      }
    }
    if (threadIdx.x != 0) return;
    Q4 rs = q4(0, 0, 0, 0), ds_ = q4(0, 0, 0, 0);
    const int cnt = min(K, N0);
    const Q4 pivot = ld_q_plain(dq + 2 * bi[0]);
    for (int s = 0; s < cnt; ++s) {
      const double4 q = pos[bi[s]];
      const double w = skin_weight(p, v3(q.x, q.y, q.z), q.w);
      const Q4 r = ld_q_plain(dq + 2 * bi[s]);
      const Q4 d = ld_q_plain(dq + 2 * bi[s] + 1);
      const double sign = (qdot(pivot, r) < 0.0) ? -1.0 : 1.0;
      rs = qadd(rs, qscl(sign * w, r));
      ds_ = qadd(ds_, qscl(sign * w, d));
    }
    if (!(qnrm(rs) < kDegenerateBlend)) {
      DQ raw;
      raw.r = rs;
      raw.d = ds_;
      out = dq_normalized(raw);
    }
  }
  if (threadIdx.x != 0) return;
  dq[2 * jn] = make_double4(out.r.w, out.r.x, out.r.y, out.r.z);
  dq[2 * jn + 1] = make_double4(out.d.w, out.d.x, out.d.y, out.d.z);
}

// update_skinning_incremental (warp_field.cpp:186-236), thread per surfel.
// Slots live in registers (every index compile-time; insertions are
// predicated). A full entry can only change if some new node is closer than
// its worst slot: the new nodes' bounding box (bbox, 6 doubles) gives a lower
// bound on their distance, so surfels far from every new node exit after one
// test -- exact (strict >: equal distances still take the index tie-break path).
__device__ __forceinline__ void slot_swap(double sd[4], int si[4], double sw[4], int b) {
#pragma unroll
  for (int t = 1; t < 4; ++t)
    if (t == b) {
      const double td = sd[t];
      sd[t] = sd[t - 1];
      sd[t - 1] = td;
      const int ti = si[t];
      si[t] = si[t - 1];
      si[t - 1] = ti;
      const double tw = sw[t];
      sw[t] = sw[t - 1];
      sw[t - 1] = tw;
    }
}

__global__ void k_skin_incremental(ModelBuf m, int n, const double4* __restrict__ pos, int first,
                                   int N, int K, const double* __restrict__ bbox, KnnGridView gnew,
                                   int use_grid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 rp = m.rp[i];
  const V3 p = v3(rp.x, rp.y, rp.z);
  const int4 ki = m.ki[i];
  const float4 kw = m.kw[i];
  int count = entry_count(ki);
  double sd[4];
  int si[4];
  double sw[4];
  const int ids[4] = {ki.x, ki.y, ki.z, ki.w};
  const double ws[4] = {kw.x, kw.y, kw.z, kw.w};
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s < count) {
      const double4 q = pos[ids[s]];
      sd[s] = sqn(sub(v3(q.x, q.y, q.z), p));
      si[s] = ids[s];
      sw[s] = ws[s];
    } else {
      sd[s] = INFINITY;
      si[s] = 0x7fffffff;
      sw[s] = 0;
    }
  }
  double worst = sd[0];
  if (count >= K) {  // full entry: skip unless a new node can come closer than the worst slot
#pragma unroll
    for (int s = 1; s < 4; ++s)
      if (s < count) worst = fmax(worst, sd[s]);
    const double dx = fmax(fmax(bbox[0] - p.x, p.x - bbox[3]), 0.0);
    const double dy = fmax(fmax(bbox[1] - p.y, p.y - bbox[4]), 0.0);
    const double dz = fmax(fmax(bbox[2] - p.z, p.z - bbox[5]), 0.0);
    if ((dx * dx + dy * dy + dz * dz) * (1.0 - 1e-12) > worst) return;
  }
  // insertion sort of the first `count` slots (registers)
#pragma unroll
  for (int a = 1; a < 4; ++a)
#pragma unroll
    for (int b2 = 3; b2 >= 1; --b2)
      if (a < count && b2 <= a && nb_less(sd[b2], si[b2], sd[b2 - 1], si[b2 - 1]))
        slot_swap(sd, si, sw, b2);
  bool changed = false;
  // streaming top-K over the new nodes (oracle loop, warp_field.cpp:186-236);
  // the final slots are the (d2, index) top K of old + new, independent of the
  // order the candidates arrive in
  auto consider = [&](int j, const double4 q) {
    const double d2 = sqn(sub(v3(q.x, q.y, q.z), p));
    int slot;
    double ld = sd[0];  // worst slot (count - 1) without a dynamic index
    int li = si[0];
#pragma unroll
    for (int t = 1; t < 4; ++t)
      if (t == count - 1) {
        ld = sd[t];
        li = si[t];
      }
    if (count < K) {
      slot = count++;
    } else if (nb_less(d2, j, ld, li)) {
      slot = count - 1;
    } else {
      return;
    }
    const double w = skin_weight(p, v3(q.x, q.y, q.z), q.w);
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (t == slot) {
        sd[t] = d2;
        si[t] = j;
        sw[t] = w;
      }
#pragma unroll
    for (int b2 = 3; b2 >= 1; --b2)
      if (b2 <= slot && nb_less(sd[b2], si[b2], sd[b2 - 1], si[b2 - 1])) slot_swap(sd, si, sw, b2);
    changed = true;
  };
  bool done = false;
  if (use_grid && count >= K) {
    // only new nodes with d2 <= worst can enter: the grid cells (over the new
    // nodes) meeting the box |x - p|_inf <= sqrt(worst) (margin for rounding)
    const double lox = gnew.prm[0], loy = gnew.prm[1], loz = gnew.prm[2], ih = gnew.prm[4];
    const double r = sqrt(worst) * (1.0 + 1e-9);
    const int x0 = (int)floor((p.x - r - lox) * ih), x1 = (int)floor((p.x + r - lox) * ih);
    const int y0 = (int)floor((p.y - r - loy) * ih), y1 = (int)floor((p.y + r - loy) * ih);
    const int z0 = (int)floor((p.z - r - loz) * ih), z1 = (int)floor((p.z + r - loz) * ih);
    if ((x1 - x0 + 1) * (y1 - y0 + 1) * (z1 - z0 + 1) <= 64) {
      for (int cz = z0; cz <= z1; ++cz)
        for (int cy = y0; cy <= y1; ++cy)
          for (int cx = x0; cx <= x1; ++cx) {
            const int2 rg = knn_find(gnew, knn_pack(cx, cy, cz));
            for (int k = rg.x; k < rg.x + rg.y; ++k)
              consider(first + __ldg(gnew.ids + k), ldg_d4(gnew.cpos + k));
          }
      done = true;
    }
  }
  if (!done)
    for (int j = first; j < N; ++j) consider(j, pos[j]);
  if (!changed) return;
  int o[4];
  float w[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    o[s] = s < count ? si[s] : -1;
    w[s] = s < count ? (float)sw[s] : 0.f;
  }
  m.ki[i] = make_int4(o[0], o[1], o[2], o[3]);
  m.kw[i] = make_float4(w[0], w[1], w[2], w[3]);
}

// bounding box of pos[first, N) -> bbox (min xyz, max xyz); one CTA
__global__ void k_bbox(const double4* __restrict__ pos, int first, int N, double* __restrict__ bbox) {
  __shared__ double red[6][8];
  double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int j = first + threadIdx.x; j < N; j += blockDim.x) {
    const double4 q = pos[j];
    v[0] = fmin(v[0], q.x);
    v[1] = fmin(v[1], q.y);
    v[2] = fmin(v[2], q.z);
    v[3] = fmax(v[3], q.x);
    v[4] = fmax(v[4], q.y);
    v[5] = fmax(v[5], q.z);
  }
#pragma unroll
  for (int a = 0; a < 6; ++a)
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, v[a], off);
      v[a] = a < 3 ? fmin(v[a], o) : fmax(v[a], o);
    }
  if ((threadIdx.x & 31) == 0)
    for (int a = 0; a < 6; ++a) red[a][threadIdx.x >> 5] = v[a];
  __syncthreads();
  if (threadIdx.x < 6) {
    double r = red[threadIdx.x][0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      r = threadIdx.x < 3 ? fmin(r, red[threadIdx.x][w]) : fmax(r, red[threadIdx.x][w]);
    bbox[threadIdx.x] = r;
  }
}

HashView hash_view(Ctx& c) {
  HashView h;
  h.key = c.ht_key;
  h.cnt = c.ht_cnt;
  h.ids = c.ht_ids;
  h.mask = c.HT - 1;
  h.inv_cell = 1.0 / c.cfg.node_sigma;
  return h;
}

void clear_hash(Ctx& c) {
  DS_CUDA(cudaMemsetAsync(c.ht_key, 0xff, sizeof(long long) * c.HT, c.stream));
  DS_CUDA(cudaMemsetAsync(c.ht_cnt, 0, sizeof(int) * c.HT, c.stream));
}

// runs the greedy CTA over `cand` starting at node count n0; returns new count
int greedy(Ctx& c, const float4* cand, int M, int n0, int list_mode, const int* M_dev = nullptr) {
  *c.h_int = n0;
  DS_CUDA(cudaMemcpyAsync(&c.dsc->n_nodes, c.h_int, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemsetAsync(&c.dsc->err, 0, sizeof(int), c.stream));
  DS_LAUNCH(c, KK_GREEDY_NODES, 16.0 * M, 1, kGreedyThreads, 0, k_greedy_nodes, cand, M, M_dev,
            c.cfg.node_sigma, hash_view(c), c.node_pos, &c.dsc->n_nodes, c.N_cap, list_mode,
            &c.dsc->err);
  // one full scalar fetch (the caller may also read its other counts)
  fetch_scalars(c);
  const int res[2] = {c.hsc->n_nodes, c.hsc->err};
  if (res[1] & DERR_NODE_CAP) fail(DS_ERR_CAPACITY, "node capacity exceeded");
  if (list_mode && (res[1] & DERR_HASH_FULL)) {
    // more than kListNodes new nodes: redo in hash mode (existing nodes are
    // already in the hash; the rerun re-accepts the same nodes in order)
    return greedy(c, cand, M, n0, 0, M_dev);
  }
  if (res[1] & (DERR_HASH_CELL | DERR_HASH_FULL))
    fail(DS_ERR_CAPACITY, "node hash overflow (nodes closer than node_sigma?)");
  return res[0];
}

}  // namespace

// grid over the reference node positions, cell 2 sigma (nodes are >= sigma apart)
bool build_ref_grid(Ctx& c) {
  return build_knn_grid(c, c.grid_ref, c.node_pos, c.n_nodes, c.ref_cell * c.cfg.node_sigma);
}

// Node edges stay a brute-force warp-per-node scan up to the grid capacity: at
// a few thousand nodes 32 lanes x ~100 distances beat 2-3 grid shells of a
// top-8 query (measured); the grid takes over beyond c.knn_edges_grid nodes
// (8192; DS_KNN_EDGES_GRID overrides, used by the parity test).
void compute_node_edges(Ctx& c, bool build_grid) {
  const int n = c.n_nodes;
  if (n == 0) return;
  const int k = std::min(8, std::max(0, c.cfg.node_neighbor_k));
  const bool big = n > c.knn_edges_grid;
  const bool grid = big && (build_grid ? build_ref_grid(c) : c.grid_ref.valid);
  if (grid)
    DS_LAUNCH(c, KK_NODE_EDGES, 32.0 * n + 32.0 * n, cdiv((long long)n * kEdgeLanes, 256), 256, 0,
              k_node_edges_grid, c.node_pos, n, k, knn_view(c.grid_ref, kKnnRing), c.node_nbr);
  else
    DS_LAUNCH(c, KK_NODE_EDGES, 32.0 * n + 32.0 * n, cdiv((long long)n * 32, 256), 256, 0,
              k_node_edges, c.node_pos, n, k, c.node_nbr);
}

void init_warp_field(Ctx& c) {
  if (c.n_surfels == 0) fail(DS_ERR_EMPTY_GEOMETRY, "init_warp_field: no reference surfels");
  clear_hash(c);
  const int n = greedy(c, c.M().rp, c.n_surfels, 0, 0);
  c.n_nodes = n;
  DS_LAUNCH(c, KK_MISC, 64.0 * n, cdiv(n, 128), 128, 0, k_identity_dq, c.node_dq, 0, n);
  const bool grid = build_ref_grid(c);  // current node set (also used by the edges if large)
  compute_node_edges(c, false);
  if (grid)
    DS_LAUNCH(c, KK_SKIN_KNN, 48.0 * c.n_surfels, cdiv(c.n_surfels, 256), 256, 0, k_skin_knn_grid,
              c.M(), c.n_surfels, c.node_pos, n, std::min(4, c.cfg.knn_k),
              knn_view(c.grid_ref, kKnnRing));
  else
    DS_LAUNCH(c, KK_SKIN_KNN, 48.0 * c.n_surfels, cdiv(c.n_surfels, kTile), kTile, 0, k_skin_knn,
              c.M(), c.n_surfels, c.node_pos, n, std::min(4, c.cfg.knn_k));
}

int extend_tail(Ctx& c, int n0, int total);

int extend_warp_field(Ctx& c, const float4* positions, int n) {
  if (n == 0) return 0;
  const int n0 = c.n_nodes;
  clear_hash(c);
  const float4* cand = positions;
  int m = n;
  const int* m_dev = nullptr;
  if (n0 > 0) {
    DS_CUDA(cudaMemsetAsync(&c.dsc->err, 0, sizeof(int), c.stream));
    DS_LAUNCH(c, KK_GREEDY_NODES, 32.0 * n0, cdiv(n0, 256), 256, 0, k_ht_prefill, hash_view(c),
              c.node_pos, n0, &c.dsc->err);
    DS_LAUNCH(c, KK_GREEDY_NODES, 20.0 * n, cdiv((long long)n * kUncLanes, 256), 256, 0, k_uncovered, positions, n,
              c.cfg.node_sigma, hash_view(c), c.node_pos, c.keep);
    scan_exclusive(c, c.keep, c.keep_scan, n);
    DS_LAUNCH(c, KK_GREEDY_NODES, 24.0 * n, cdiv(n, 256), 256, 0, k_gather_uncovered, positions,
              c.keep, c.keep_scan, n, c.ext_pos);
    cand = c.ext_pos;
    m_dev = c.keep_scan + n;  // the uncovered count stays on the device
  }
  const int total = greedy(c, cand, m, n0, n0 > 0 ? 1 : 0, m_dev);
  return extend_tail(c, n0, total);
}

// the new nodes' seeds and edges (side stream), after the greedy pass
int extend_tail(Ctx& c, int n0, int total) {
  const int added = total - n0;
  c.n_nodes = total;
  if (added > 0) {
    // the new nodes' seeds and the edges (warp_field.cpp:163-182) only touch
    // node DQs / neighbour lists: they run on the side stream, concurrently with
    // the caller's incremental reskinning of the surfels (joined at frame end)
    DS_CUDA(cudaEventRecord(c.ev_fork, c.stream));
    DS_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
    cudaStream_t main_stream = c.stream;
    c.stream = c.side;
    try {
      const bool grid = total > c.knn_edges_grid && build_ref_grid(c);
      DS_LAUNCH(c, KK_GREEDY_NODES, 64.0 * added, added, kSeedThreads, 0, k_seed_dq, c.node_pos,
                c.node_dq, n0, total, std::min(4, c.cfg.knn_k), knn_view(c.grid_ref, kKnnRing),
                grid ? 1 : 0);
      compute_node_edges(c, false);
    } catch (...) {
      c.stream = main_stream;
      throw;
    }
    c.stream = main_stream;
    DS_CUDA(cudaEventRecord(c.ev_nodes, c.side));
    c.nodes_pending = true;
  }
  return added;
}

int extend_warp_field_dev(Ctx& c, const float4* base, const int* off_dev, const int* end_dev,
                          int bound) {
  if (bound <= 0) return 0;
  const int n0 = c.n_nodes;
  clear_hash(c);
  DS_CUDA(cudaMemsetAsync(&c.dsc->err, 0, sizeof(int), c.stream));
  if (n0 > 0)
    DS_LAUNCH(c, KK_GREEDY_NODES, 32.0 * n0, cdiv(n0, 256), 256, 0, k_ht_prefill, hash_view(c),
              c.node_pos, n0, &c.dsc->err);
  DS_LAUNCH(c, KK_GREEDY_NODES, 20.0 * bound, cdiv((long long)bound * kUncLanes, 256), 256, 0,
            k_uncovered_dev, base, off_dev, end_dev, bound, c.cfg.node_sigma, hash_view(c),
            c.node_pos, c.keep);
  scan_exclusive(c, c.keep, c.keep_scan, bound);
  DS_LAUNCH(c, KK_GREEDY_NODES, 24.0 * bound, cdiv(bound, 256), 256, 0, k_gather_uncovered_dev, base,
            off_dev, end_dev, c.keep, c.keep_scan, bound, c.ext_pos);
  const int total = greedy(c, c.ext_pos, bound, n0, n0 > 0 ? 1 : 0, c.keep_scan + bound);
  return extend_tail(c, n0, total);
}

void update_skinning_incremental(Ctx& c, int first_new) {
  if (first_new >= c.n_nodes || c.n_surfels == 0) return;
  // side stream, after the new nodes' seeds and edges: only the next solve (and
  // fusion) read the skinning, so it overlaps the next frame's rigid ICP; the
  // main stream joins at the next API call / after the next frame's ICP launch
  DS_CUDA(cudaEventRecord(c.ev_fork, c.stream));
  DS_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
  cudaStream_t main_stream = c.stream;
  c.stream = c.side;
  try {
    DS_LAUNCH(c, KK_SKIN_INCREMENTAL, 32.0 * (c.n_nodes - first_new), 1, 256, 0, k_bbox,
              c.node_pos, first_new, c.n_nodes, c.new_bbox);
    // a grid over the new nodes restricts each full entry to the cells within
    // its worst slot distance (worthwhile once there are more than a few new
    // nodes; sparse cells: large, and a table at load <= 1/8 so that most
    // probes of an empty cell end at the first slot)
    const int added = c.n_nodes - first_new;
    const bool grid = added > c.incr_grid_min &&
                      build_knn_grid(c, c.grid_new, c.node_pos + first_new, added,
                                     c.incr_cell * c.cfg.node_sigma, 8);
    DS_LAUNCH(c, KK_SKIN_INCREMENTAL, 48.0 * c.n_surfels, cdiv(c.n_surfels, 256), 256, 0,
              k_skin_incremental, c.M(), c.n_surfels, c.node_pos, first_new, c.n_nodes,
              std::min(4, c.cfg.knn_k), (const double*)c.new_bbox, knn_view(c.grid_new, 0),
              grid ? 1 : 0);
  } catch (...) {
    c.stream = main_stream;
    throw;
  }
  c.stream = main_stream;
  DS_CUDA(cudaEventRecord(c.ev_nodes, c.side));
  c.nodes_pending = true;
}

}  // namespace ds
