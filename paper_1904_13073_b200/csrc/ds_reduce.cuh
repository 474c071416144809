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

template <int kBlock>
__device__ __forceinline__ void grid_sum(double v, double* __restrict__ part,
                                         unsigned* __restrict__ ticket, double* __restrict__ out) {
  grid_sum_part<kBlock>(v, part, ticket, out, blockIdx.x, gridDim.x);
}

}  // namespace ds
