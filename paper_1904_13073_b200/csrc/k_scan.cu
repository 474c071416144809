// k_scan.cu — deterministic scan / reduction utilities used for stream compaction
// (order-preserving, fusion.cpp:264-284) and fixed-order fp64 reductions.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>

#include "ds_context.cuh"

namespace ds {

namespace {
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) k_scan_tile_sums(const int* __restrict__ in, int n,
                                                                 int* __restrict__ sums) {
  using BR = cub::BlockReduce<int, kScanThreads>;
  __shared__ typename BR::TempStorage tmp;
  const long long base = (long long)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) s += in[base + k];
  const int tot = BR(tmp).Sum(s);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_sums(int* __restrict__ sums, int nb,
                                                            int* __restrict__ total) {
  using BS = cub::BlockScan<int, kScanThreads>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += kScanThreads) {
    const int i = base + threadIdx.x;
    const int v = i < nb ? sums[i] : 0;
    int ex, agg;
    BS(tmp).ExclusiveSum(v, ex, agg);
    if (i < nb) sums[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const int* in, int n,
                                                             const int* __restrict__ sums,
                                                             int* out) {
  using BS = cub::BlockScan<int, kScanThreads>;
  __shared__ typename BS::TempStorage tmp;
  const long long base = (long long)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  int v[kScanItems];
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (base + k < n) ? in[base + k] : 0;
    s += v[k];
  }
  int ex;
  BS(tmp).ExclusiveSum(s, ex);
  int run = ex + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

}  // namespace

void scan_exclusive(Ctx& c, const int* in, int* out, int n) {
  if (n <= 0) {
    DS_CUDA(cudaMemsetAsync(out, 0, sizeof(int), c.stream));
    return;
  }
  const int nb = cdiv(n, kScanTile);
  if (nb > c.scan_tmp_n) fail(DS_ERR_CAPACITY, "scan scratch too small");
  DS_LAUNCH(c, KK_SCAN, 4.0 * n, nb, kScanThreads, 0, k_scan_tile_sums, in, n, c.scan_tmp);
  DS_LAUNCH(c, KK_SCAN, 8.0 * nb, 1, kScanThreads, 0, k_scan_sums, c.scan_tmp, nb, out + n);
  DS_LAUNCH(c, KK_SCAN, 8.0 * n, nb, kScanThreads, 0, k_scan_apply, in, n, c.scan_tmp, out);
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
