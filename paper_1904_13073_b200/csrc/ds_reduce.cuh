// ds_reduce.cuh — deterministic grid-wide fp64 sums fused into the producing kernel.
// Each block reduces in a fixed tree order and publishes its partial; the last
// block to arrive (threadfence + ticket) sums all partials in block order and
// writes the result, then re-arms the ticket. Same launch config => same bits.
#pragma once
#include <cuda_runtime.h>

namespace ds {

// Blocks [0, nblocks) of a sub-range of the grid (block id `bid`) reduce into
// `out`; the plain overload uses the whole grid.
template <int kBlock>
__device__ __forceinline__ void grid_sum_part(double v, double* __restrict__ part,
                                              unsigned* __restrict__ ticket,
                                              double* __restrict__ out, int bid, int nblocks) {
  __shared__ double sh[kBlock];
  __shared__ bool last;
  const int tid = threadIdx.x;
  sh[tid] = v;
  __syncthreads();
#pragma unroll
  for (int k = kBlock / 2; k > 0; k >>= 1) {
    if (tid < k) sh[tid] += sh[tid + k];
    __syncthreads();
  }
  if (tid == 0) {
    part[bid] = sh[0];
    __threadfence();
    last = atomicAdd(ticket, 1u) == (unsigned)nblocks - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double acc = 0.0;
#pragma unroll 8
  for (int b = tid; b < nblocks; b += kBlock) acc += __ldcg(part + b);
  sh[tid] = acc;
  __syncthreads();
#pragma unroll
  for (int k = kBlock / 2; k > 0; k >>= 1) {
    if (tid < k) sh[tid] += sh[tid + k];
    __syncthreads();
  }
  if (tid == 0) {
    *out = sh[0];
    *ticket = 0u;
  }
}

// Barrier-free variant: each warp reduces (xor butterfly) and publishes its
// sum; the last warp of the block to arrive adds the warp sums in warp order,
// the last block adds the block partials in block order (one warp). Warps may
// exit right after the call, so idle warps do not wait for the busy ones.
// Requires *wcnt == 0 on entry, made visible by a __syncthreads before the call
// (the caller zeroes it at kernel start); every warp of the block calls it once.
template <int kBlock>
__device__ __forceinline__ void grid_sum_warps(double v, unsigned* wcnt, double* wsum,
                                               double* __restrict__ part,
                                               unsigned* __restrict__ ticket,
                                               double* __restrict__ out, int bid, int nblocks) {
  constexpr int kWarps = kBlock / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  int lastw = 0;
  if (lane == 0) {
    wsum[w] = v;
    __threadfence_block();
    lastw = atomicAdd(wcnt, 1u) == (unsigned)kWarps - 1;
  }
  if (!__shfl_sync(0xffffffffu, lastw, 0)) return;
  int lastb = 0;
  if (lane == 0) {
    __threadfence_block();
    const volatile double* ws = wsum;
    double b = 0.0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) b += ws[i];
    part[bid] = b;
    __threadfence();
    lastb = atomicAdd(ticket, 1u) == (unsigned)nblocks - 1;
  }
  if (!__shfl_sync(0xffffffffu, lastb, 0)) return;
  __threadfence();
  double acc = 0.0;
  for (int b = lane; b < nblocks; b += 32) acc += __ldcg(part + b);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    *out = acc;
    *ticket = 0u;
  }
}

template <int kBlock>
__device__ __forceinline__ void grid_sum(double v, double* __restrict__ part,
                                         unsigned* __restrict__ ticket, double* __restrict__ out) {
  grid_sum_part<kBlock>(v, part, ticket, out, blockIdx.x, gridDim.x);
}

}  // namespace ds
