// Why is the PCG prologue slow? Time a 6x6 Gauss-Jordan (8-lane groups) and a
// 6x6 smem mat-vec in CTA 0 of a cooperative 148x512 launch with 200 KB of
// dynamic smem, against variants (no coop, small smem, fmad on/off via build).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void gj_inverse6(double a[6], double b[6], int lr) {
  const int base = (threadIdx.x & 31) & ~7;
#pragma unroll
  for (int t = 0; t < 6; ++t) b[t] = (t == lr) ? 1.0 : 0.0;
#pragma unroll
  for (int p = 0; p < 6; ++p) {
    double ap[6], bp[6];
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      ap[t] = __shfl_sync(0xffffffffu, a[t], base + p);
      bp[t] = __shfl_sync(0xffffffffu, b[t], base + p);
    }
    const double piv = ap[p];
#ifdef RCP
    const double ip = 1.0 / piv;
#endif
    if (lr == p) {
#pragma unroll
      for (int t = 0; t < 6; ++t) {
#ifdef RCP
        a[t] = ap[t] * ip;
        b[t] = bp[t] * ip;
#else
        a[t] = ap[t] / piv;
        b[t] = bp[t] / piv;
#endif
      }
    } else {
#ifdef RCP
      const double f = a[p] * ip;
#else
      const double f = a[p] / piv;
#endif
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        a[t] = a[t] - f * ap[t];
        b[t] = b[t] - f * bp[t];
      }
    }
  }
}

template <bool kCoop>
__global__ void __launch_bounds__(512, 1) k_test(const double* __restrict__ in, double* out,
                                                 unsigned long long* tr, int reps) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* M = reinterpret_cast<double*>(smem);
  double* R = M + 36 * 64;
  double* U = R + 6 * 64;
  const int tid = threadIdx.x, grp = tid >> 3, lr = tid & 7;
  if (tid == 0 && blockIdx.x == 0) tr[0] = gt();
  for (int rep = 0; rep < reps; ++rep) {
    double ar[6], br[6];
#pragma unroll
    for (int t = 0; t < 6; ++t) ar[t] = (lr < 6) ? in[(grp % 7) * 36 + lr * 6 + t] + (t == lr ? 10.0 : 0.0) : (t == lr ? 1.0 : 0.0);
    gj_inverse6(ar, br, lr);
    if (lr < 6 && grp < 64)
#pragma unroll
      for (int t = 0; t < 6; ++t) M[36 * grp + 6 * lr + t] = br[t];
    if (tid < 384) R[tid] = in[tid % 252];
    __syncthreads();
    if (tid == 0 && blockIdx.x == 0) tr[1 + 2 * rep] = gt();
    for (int k = tid; k < 384; k += 512) {
      const int i = k / 6, rw = k % 6;
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < 6; ++t) s += M[36 * i + 6 * rw + t] * R[6 * i + t];
      U[k] = s;
    }
    __syncthreads();
    if (tid == 0 && blockIdx.x == 0) tr[2 + 2 * rep] = gt();
  }
  if (kCoop) cg::this_grid().sync();
  if (tid < 384) out[blockIdx.x * 384 + tid] = U[tid];
}

int main() {
  double *in, *out;
  unsigned long long* tr;
  cudaMalloc(&in, 4096 * 8);
  cudaMalloc(&out, 148 * 384 * 8);
  cudaMalloc(&tr, 64 * 8);
  cudaMemset(in, 0, 4096 * 8);
  const int reps = 3;
  for (int variant = 0; variant < 4; ++variant) {
    const bool coop = variant & 1;
    const int smemb = (variant & 2) ? 200 * 1024 : 48 * 1024;
    cudaFuncSetAttribute(k_test<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_test<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int rr = 0; rr < 3; ++rr) {
      int rp = reps;
      void* args[] = {&in, &out, &tr, &rp};
      if (coop) cudaLaunchCooperativeKernel((void*)k_test<true>, 148, 512, args, smemb, 0);
      else k_test<false><<<148, 512, smemb>>>(in, out, tr, reps);
      cudaDeviceSynchronize();
    }
    unsigned long long h[8];
    cudaMemcpy(h, tr, sizeof h, cudaMemcpyDeviceToHost);
    printf("coop=%d smem=%dKB: ", coop, smemb / 1024);
    for (int k = 1; k <= 2 * reps; ++k) printf(" %.2f", (h[k] - h[0]) * 1e-3);
    printf("  [%s]\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
