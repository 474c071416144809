// k_knn.cu — builds the uniform-grid index of ds_knn.cuh (VoxelGrid,
// spatial_grid.hpp:16-136) for the node set: one CTA computes the bounding box,
// inserts every point's cell into the open-addressing table with counts, scans
// the counts and scatters the ids by cell. Rebuilt whenever the node set or the live node
// positions change; queries are in k_skin.cu / k_fusion.cu.
#include "ds_context.cuh"
#include "ds_knn.cuh"

namespace ds {
namespace {

constexpr int kBuildThreads = 1024;

// scratch: per point slot (n ints) + per slot fill counter (slots ints)
__global__ void __launch_bounds__(kBuildThreads) k_knn_build(const double4* __restrict__ pos, int n,
                                                             double h, KnnGrid g,
                                                             int* __restrict__ pslot,
                                                             int* __restrict__ fill) {
  __shared__ double red[6][kBuildThreads / 32];
  __shared__ double lo[3];
  __shared__ int wsum[kBuildThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int S = g.mask + 1;
  // bounding box (min/max are exact: order-independent)
  double mn[3] = {INFINITY, INFINITY, INFINITY};
  for (int i = tid; i < n; i += kBuildThreads) {
    const double4 p = pos[i];
    mn[0] = fmin(mn[0], p.x);
    mn[1] = fmin(mn[1], p.y);
    mn[2] = fmin(mn[2], p.z);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
    for (int off = 16; off > 0; off >>= 1) mn[a] = fmin(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], off));
  if (lane == 0)
    for (int a = 0; a < 3; ++a) red[a][wid] = mn[a];
  // clear the cell table
  for (int s = tid; s < S; s += kBuildThreads) {
    g.key[s] = kKnnEmpty;
    g.range[s] = make_int2(0, 0);
    fill[s] = 0;
  }
  __syncthreads();
  if (tid == 0) {
    for (int a = 0; a < 3; ++a) {
      double m = INFINITY;
      for (int w = 0; w < kBuildThreads / 32; ++w) m = fmin(m, red[a][w]);
      lo[a] = (n > 0 ? m : 0.0) - h;
    }
    g.prm[0] = lo[0];
    g.prm[1] = lo[1];
    g.prm[2] = lo[2];
    g.prm[3] = h;
    g.prm[4] = 1.0 / h;
  }
  __syncthreads();
  // cell of every point -> table slot (insert-or-find), per-cell counts
  const double ih = 1.0 / h;
  for (int i = tid; i < n; i += kBuildThreads) {
    const double4 p = pos[i];
    const long long k = knn_pack((int)floor((p.x - lo[0]) * ih), (int)floor((p.y - lo[1]) * ih),
                                 (int)floor((p.z - lo[2]) * ih));
    unsigned s = knn_hash(k) & g.mask;
    for (int probe = 0; probe <= g.mask; ++probe) {
      const long long prev = (long long)atomicCAS((unsigned long long*)(g.key + s),
                                                  (unsigned long long)kKnnEmpty,
                                                  (unsigned long long)k);
      if (prev == kKnnEmpty || prev == k) break;
      s = (s + 1) & g.mask;
    }
    pslot[i] = (int)s;
    atomicAdd(&g.range[s].y, 1);
  }
  __syncthreads();
  // exclusive scan of the counts over the slots (block-wide, contiguous chunks)
  const int per = (S + kBuildThreads - 1) / kBuildThreads;
  const int s0 = tid * per, s1 = min(s0 + per, S);
  int local = 0;
  for (int s = s0; s < s1; ++s) local += g.range[s].y;
  int incl = local;
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  int base = incl - local;
  for (int w = 0; w < wid; ++w) base += wsum[w];
  for (int s = s0; s < s1; ++s) {
    g.range[s].x = base;
    base += g.range[s].y;
  }
  __syncthreads();
  // scatter ids by cell (order within a cell is irrelevant: queries rank by (d2, id))
  for (int i = tid; i < n; i += kBuildThreads) {
    const int s = pslot[i];
    const int k = g.range[s].x + atomicAdd(fill + s, 1);
    g.ids[k] = i;
    g.cpos[k] = pos[i];
  }
}

}  // namespace

// (Re)build `g` over pos[0..n) with cell size h. Returns false when n exceeds
// the shared-memory sort capacity (callers then use the brute-force kernels).
bool build_knn_grid(Ctx& c, KnnGrid& g, const double4* pos, int n, double h, int load_inv) {
  if (n <= 0 || n > kKnnMaxPoints) {
    g.valid = false;
    return false;
  }
  // table sized to the point count (load <= 1/load_inv): the build clears only these slots
  int slots = 1;
  while (slots < load_inv * n) slots <<= 1;
  g.mask = std::min(slots - 1, g.cap_mask);
  DS_LAUNCH(c, KK_SKIN_KNN, 40.0 * n, 1, kBuildThreads, 0, k_knn_build, pos, n, h, g, g.pslot,
            g.fill);
  g.valid = true;
  return true;
}

}  // namespace ds
