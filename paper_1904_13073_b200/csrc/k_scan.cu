// k_scan.cu — deterministic scan / reduction utilities used for stream compaction
// (order-preserving, fusion.cpp:264-284) and fixed-order fp64 reductions.
#include <cub/block/block_load.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/block/block_store.cuh>
#include <cub/device/device_radix_sort.cuh>

#include "ds_context.cuh"

namespace ds {

namespace {
// Single-pass exclusive scan with decoupled look-back: tile t publishes its
// aggregate (flag A), sums its predecessors' published values back to the
// first inclusive prefix (flag P), publishes its own inclusive prefix and
// adds the exclusive prefix to its locally scanned items. Integer sums: the
// result does not depend on the order. Status words (flag << 32 | value) are
// cleared by a memset before each scan (graph-replay safe).
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
#define kFlagA (1ull << 32)
#define kFlagP (2ull << 32)

__global__ void __launch_bounds__(kScanThreads) k_scan_lookback(const int* in, int n, int* out,
                                                                unsigned long long* status) {
  using BL = cub::BlockLoad<int, kScanThreads, kScanItems, cub::BLOCK_LOAD_WARP_TRANSPOSE>;
  using BS = cub::BlockScan<int, kScanThreads>;
  using BST = cub::BlockStore<int, kScanThreads, kScanItems, cub::BLOCK_STORE_WARP_TRANSPOSE>;
  __shared__ union {
    typename BL::TempStorage load;
    typename BS::TempStorage scan;
    typename BST::TempStorage store;
  } tmp;
  __shared__ int s_prefix;
  const int tile = blockIdx.x;
  const long long base = (long long)tile * kScanTile;
  const int valid = (int)min((long long)kScanTile, (long long)n - base);
  int v[kScanItems];
  BL(tmp.load).Load(in + base, v, valid, 0);  // in == out allowed: read before written
  __syncthreads();
  int agg;
  BS(tmp.scan).ExclusiveSum(v, v, agg);
  if (threadIdx.x < 32) {  // warp 0: publish, then look back 32 predecessors at a time
    volatile unsigned long long* st = status;
    const int lane = threadIdx.x;
    int prefix = 0;
    if (tile == 0) {
      if (lane == 0) st[0] = kFlagP | (unsigned)agg;
    } else {
      if (lane == 0) st[tile] = kFlagA | (unsigned)agg;
      int hi = tile - 1;  // window [hi - 31, hi], lane l reads hi - l
      while (true) {
        const int j = hi - lane;
        unsigned long long w = j >= 0 ? st[j] : kFlagP;  // before tile 0: prefix 0
        while (__any_sync(0xffffffffu, (w & (3ull << 32)) == 0))
          if ((w & (3ull << 32)) == 0) w = st[j];
        const unsigned pmask = __ballot_sync(0xffffffffu, (w & (3ull << 32)) == kFlagP);
        // lanes up to the nearest inclusive prefix contribute
        const int stop = pmask ? __ffs(pmask) - 1 : 31;
        int val = (lane <= stop && j >= 0) ? (int)(unsigned)w : 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) val += __shfl_xor_sync(0xffffffffu, val, off);
        prefix += val;
        if (pmask) break;
        hi -= 32;
      }
      if (lane == 0) {
        __threadfence();
        st[tile] = kFlagP | (unsigned)(prefix + agg);
      }
    }
    if (lane == 0) {
      s_prefix = prefix;
      if (tile == gridDim.x - 1) out[n] = prefix + agg;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) v[k] += s_prefix;
  BST(tmp.store).Store(out + base, v, valid);
}

}  // namespace

void scan_exclusive(Ctx& c, const int* in, int* out, int n) {
  if (n <= 0) {
    DS_CUDA(cudaMemsetAsync(out, 0, sizeof(int), c.stream));
    return;
  }
  const int nb = cdiv(n, kScanTile);
  if (nb > c.scan_tmp_n) fail(DS_ERR_CAPACITY, "scan scratch too small");
  DS_CUDA(cudaMemsetAsync(c.scan_status, 0, sizeof(unsigned long long) * nb, c.stream));
  DS_LAUNCH(c, KK_SCAN, 8.0 * n, nb, kScanThreads, 0, k_scan_lookback, in, n, out, c.scan_status);
}

void sort_pairs(Ctx& c, int* keys, int* vals, int* keys_alt, int* vals_alt, int n, int end_bit,
                int** keys_out, int** vals_out, int kind) {
  cub::DoubleBuffer<int> dk(keys, keys_alt), dv(vals, vals_alt);
  size_t bytes = c.cub_tmp_bytes;
  launch_begin(c, kind);
  DS_CUDA(cub::DeviceRadixSort::SortPairs(c.cub_tmp, bytes, dk, dv, n, 0, end_bit, c.stream));
  launch_end(c, kind, 16.0 * n * ((end_bit + 7) / 8));
  *keys_out = dk.Current();
  *vals_out = dv.Current();
}

size_t sort_temp_bytes(int n) {
  cub::DoubleBuffer<int> dk(nullptr, nullptr), dv(nullptr, nullptr);
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, n, 0, 32);
  return bytes;
}


}  // namespace ds
