// ds_knn.cuh — exact K-nearest-node queries on a uniform grid (the device
// counterpart of VoxelGrid, spatial_grid.hpp:16-136).
//
// The grid is rebuilt whenever the point set changes (k_knn_build, one CTA):
// cell size h, cells keyed by packed integer coordinates, node ids sorted by
// cell, an open-addressing table cell -> (start, count). A query walks
// Chebyshev shells r = 0, 1, 2, ... around its cell; every point outside the
// shells walked so far lies in a cell at Chebyshev distance >= r + 1, hence at
// Euclidean distance >= r h from the query (the query lies inside its own
// cell). Once the K-th best squared distance is below (r h)^2 (with a rounding
// margin) no unvisited point can enter the top K, so the result is the exact
// (d^2, index) top K of the brute-force scan -- same fp64 distances, same total
// order (spatial_grid.hpp:21-23).
#pragma once
#include "ds_context.cuh"
#include "ds_math.cuh"

namespace ds {

constexpr long long kKnnEmpty = -1LL;
constexpr int kKnnOff = 1 << 20;  // coordinate offset (queries may lie outside the box)

struct KnnGridView {
  const long long* key;  // slot -> packed cell key, kKnnEmpty if free
  const int2* range;     // slot -> (start, count) into ids
  const int* ids;        // point ids sorted by cell
  const double4* cpos;   // their positions, same order
  const double* prm;     // lo.x, lo.y, lo.z, h, 1/h
  int mask;              // slots - 1
  int max_ring;          // shells walked before giving up (then brute force)
};

inline KnnGridView knn_view(const KnnGrid& g, int max_ring) {
  KnnGridView v;
  v.key = g.key;
  v.range = g.range;
  v.ids = g.ids;
  v.cpos = g.cpos;
  v.prm = g.prm;
  v.mask = g.mask;
  v.max_ring = max_ring;
  return v;
}

__device__ __forceinline__ double4 ldg_d4(const double4* p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ long long knn_pack(int cx, int cy, int cz) {
  return ((long long)(cx + kKnnOff) << 42) | ((long long)(cy + kKnnOff) << 21) |
         (long long)(cz + kKnnOff);
}
__device__ __forceinline__ unsigned knn_hash(long long k) {
  unsigned long long x = (unsigned long long)k * 0x9E3779B97F4A7C15ull;
  return (unsigned)(x >> 32);
}
__device__ __forceinline__ int2 knn_find(const KnnGridView& g, long long k) {
  unsigned s = knn_hash(k) & g.mask;
  for (int probe = 0; probe <= g.mask; ++probe) {
    const long long v = __ldg(g.key + s);
    if (v == k) return __ldg(g.range + s);
    if (v == kKnnEmpty) return make_int2(0, 0);
    s = (s + 1) & g.mask;
  }
  return make_int2(0, 0);
}

// sorted (d2, index) insertion into a top-K list
template <int K>
__device__ __forceinline__ void knnk_insert(double d2, int j, double bd[K], int bi[K]) {
  if (!nb_less(d2, j, bd[K - 1], bi[K - 1])) return;
  double cd = d2;
  int ci = j;
#pragma unroll
  for (int s = 0; s < K; ++s)
    if (nb_less(cd, ci, bd[s], bi[s])) {
      const double td = bd[s];
      const int ti = bi[s];
      bd[s] = cd;
      bi[s] = ci;
      cd = td;
      ci = ti;
    }
}

// Top K of two sorted (d2, index) lists a and b (K a power of two), into a:
// c[s] = min(a[s], b[K-1-s]) holds exactly the K smallest of the union and is
// bitonic; a bitonic merge sorts it (K/2 log K compare-exchanges, static
// register indices).
template <int K>
__device__ __forceinline__ void knnk_merge2(double ad[K], int ai[K], const double bd[K],
                                            const int bi[K]) {
  static_assert((K & (K - 1)) == 0, "K must be a power of two");
#pragma unroll
  for (int s = 0; s < K; ++s)
    if (nb_less(bd[K - 1 - s], bi[K - 1 - s], ad[s], ai[s])) {
      ad[s] = bd[K - 1 - s];
      ai[s] = bi[K - 1 - s];
    }
#pragma unroll
  for (int j = K / 2; j > 0; j >>= 1)
#pragma unroll
    for (int s = 0; s < K; ++s)
      if ((s & j) == 0 && nb_less(ad[s + j], ai[s + j], ad[s], ai[s])) {
        const double td = ad[s];
        const int ti = ai[s];
        ad[s] = ad[s + j];
        ai[s] = ai[s + j];
        ad[s + j] = td;
        ai[s + j] = ti;
      }
}

// top-K of the union of the per-lane lists of an aligned LANES group (disjoint
// point subsets), written to (md, mi) in every lane; the per-lane lists stay.
template <int K, int LANES>
__device__ __forceinline__ void knnk_merged(const double bd[K], const int bi[K], double md[K],
                                            int mi[K]) {
#pragma unroll
  for (int s = 0; s < K; ++s) {
    md[s] = bd[s];
    mi[s] = bi[s];
  }
  // only the group's lanes take part: groups of a warp may be at different
  // shells of their own queries
  const unsigned gmask =
      LANES >= 32 ? 0xffffffffu
                  : (((1u << LANES) - 1u) << ((threadIdx.x & 31) & ~(unsigned)(LANES - 1)));
#pragma unroll
  for (int off = LANES / 2; off > 0; off >>= 1) {
    double od[K];
    int oi[K];
#pragma unroll
    for (int s = 0; s < K; ++s) {
      od[s] = __shfl_xor_sync(gmask, md[s], off);
      oi[s] = __shfl_xor_sync(gmask, mi[s], off);
    }
    knnk_merge2<K>(md, mi, od, oi);
  }
}

// Exact top-K of the points `pos` (x, y, z in double4) around x by (d2, id),
// ids accepted by `keep(id)`; LANES lanes of an aligned group cooperate (every
// lane of the group must call it). Shells are walked outwards; once the group
// holds K points with K-th best d2 = B, a cell whose box is farther than
// sqrt(B) from x is skipped, and the walk stops when every face of the walked
// cube is farther than sqrt(B) (unvisited points lie outside the cube). The
// distances carry a margin of 1e-9 h (cell assignment rounding) and the
// comparisons are strict, so ties on d2 are still visited for the index
// tie-break. Returns false if the shell limit was hit before the result was
// certain (caller falls back to brute force).
template <int K, int LANES, class Keep>
__device__ bool knn_grid_query(const KnnGridView& g, const double4* __restrict__ pos, V3 x,
                               Keep keep, double md[K], int mi[K]) {
  const int lane = threadIdx.x & (LANES - 1);
  const double lox = g.prm[0], loy = g.prm[1], loz = g.prm[2], h = g.prm[3], ih = g.prm[4];
  const int cx = (int)floor((x.x - lox) * ih), cy = (int)floor((x.y - loy) * ih),
            cz = (int)floor((x.z - loz) * ih);
  const double eps = 1e-9 * h;
  // x relative to its cell's low corner (per axis, in [0, h) up to rounding)
  const double ox = x.x - (lox + cx * h), oy = x.y - (loy + cy * h), oz = x.z - (loz + cz * h);
  double bd[K];
  int bi[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    bd[s] = INFINITY;
    bi[s] = 0x7fffffff;
  }
  double bound = INFINITY;  // K-th best d2 of the group after the last shell
  for (int r = 0; r <= g.max_ring; ++r) {
    const int side = 2 * r + 1, ncell = side * side * side;
    for (int q = lane; q < ncell; q += LANES) {
      const int dx = q % side - r, dy = (q / side) % side - r, dz = q / (side * side) - r;
      if (max(abs(dx), max(abs(dy), abs(dz))) != r) continue;  // interior: done before
      if (bound < INFINITY) {
        // distance from x to the cell box [d h, (d + 1) h) relative to x's cell
        const double ax = dx > 0 ? dx * h - ox : (dx < 0 ? ox - (dx + 1) * h : 0.0);
        const double ay = dy > 0 ? dy * h - oy : (dy < 0 ? oy - (dy + 1) * h : 0.0);
        const double az = dz > 0 ? dz * h - oz : (dz < 0 ? oz - (dz + 1) * h : 0.0);
        const double ex = fmax(ax - eps, 0.0), ey = fmax(ay - eps, 0.0), ez = fmax(az - eps, 0.0);
        if ((ex * ex + ey * ey + ez * ez) * (1.0 - 1e-9) > bound) continue;
      }
      const int2 rg = knn_find(g, knn_pack(cx + dx, cy + dy, cz + dz));
      // points four at a time: their (id, position) loads are in flight together
      for (int k0 = rg.x; k0 < rg.x + rg.y; k0 += 4) {
        int id[4];
        double4 p[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (k0 + u < rg.x + rg.y) {
            id[u] = __ldg(g.ids + k0 + u);
            p[u] = ldg_d4(g.cpos + k0 + u);
          }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (k0 + u < rg.x + rg.y && keep(id[u]))
            knnk_insert<K>(sqn(sub(v3(p[u].x, p[u].y, p[u].z), x)), id[u], bd, bi);
      }
    }
    knnk_merged<K, LANES>(bd, bi, md, mi);
    bound = md[K - 1];
    // nearest face of the walked cube [c - r, c + r + 1) h
    const double f = fmin(fmin(fmin(ox, h - ox), fmin(oy, h - oy)), fmin(oz, h - oz)) + r * h - eps;
    if (f > 0.0 && f * f * (1.0 - 1e-9) > bound) return true;
  }
  return false;
}

}  // namespace ds
