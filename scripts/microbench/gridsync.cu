// Grid-barrier cost on this GPU: cooperative-groups grid.sync() vs a
// hand-rolled arrive/spin barrier, and the PCG's reduce+barrier+total round.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync gridsync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void k_own(int iters, unsigned* ctr) {
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      red_release(ctr, 1u);
      const unsigned target = (unsigned)(i + 1) * gridDim.x;
      while (ld_acquire(ctr) < target) {
      }
    }
    __syncthreads();
  }
}

// hierarchical: hardware cluster barrier, then one CTA per cluster on the
// global counter, then the cluster barrier again (cooperative + cluster launch)
__global__ void k_hier(int iters, unsigned* ctr) {
  cg::cluster_group cl = cg::this_cluster();
  const unsigned ncl = gridDim.x / cl.num_blocks();
  for (int i = 0; i < iters; ++i) {
    cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
      red_release(ctr, 1u);
      const unsigned target = (unsigned)(i + 1) * ncl;
      while (ld_acquire(ctr) < target) {
      }
    }
    cl.sync();
  }
}

__global__ void k_round(int iters, double* part) {
  cg::grid_group g = cg::this_grid();
  __shared__ double2 sh[33];
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    double a = threadIdx.x * 1e-3 + i, b = a * 2;
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, off);
      b += __shfl_xor_sync(0xffffffffu, b, off);
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = make_double2(a, b);
    __syncthreads();
    double ta = 0, tb = 0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) ta += sh[w].x, tb += sh[w].y;
    if (threadIdx.x == 0) part[4 * blockIdx.x] = ta, part[4 * blockIdx.x + 1] = tb;
    g.sync();
    if (threadIdx.x < 32) {
      double va = 0, vb = 0;
      for (int k = threadIdx.x; k < gridDim.x; k += 32) va += __ldcg(part + 4 * k), vb += __ldcg(part + 4 * k + 1);
      for (int off = 16; off > 0; off >>= 1) {
        va += __shfl_xor_sync(0xffffffffu, va, off);
        vb += __shfl_xor_sync(0xffffffffu, vb, off);
      }
      if (threadIdx.x == 0) sh[32] = make_double2(va, vb);
    }
    __syncthreads();
    acc += sh[32].x;
    g.sync();  // keep part stable before the next round overwrites it
  }
  if (acc == -1) part[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* ctr;
  double* part;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&part, 4 * 8 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2000;
  for (int G : {16, 74, 144, 148}) {
    for (int T : {256, 512, 1024}) {
      float ms[3];
      for (int v = 0; v < 3; ++v) {
        int it = iters;
        void* args_cg[] = {&it};
        void* args_own[] = {&it, &ctr};
        void* args_r[] = {&it, &part};
        for (int rep = 0; rep < 2; ++rep) {
          cudaMemset(ctr, 0, 4);
          cudaEventRecord(a);
          if (v == 0) cudaLaunchCooperativeKernel((void*)k_cg, G, T, args_cg, 0, 0);
          if (v == 1) cudaLaunchCooperativeKernel((void*)k_own, G, T, args_own, 0, 0);
          if (v == 2) cudaLaunchCooperativeKernel((void*)k_round, G, T, args_r, 0, 0);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          cudaEventElapsedTime(&ms[v], a, b);
        }
      }
      float mh[3] = {0, 0, 0};
      const int cls[3] = {2, 4, 8};
      for (int q = 0; q < 3; ++q) {
        if (G % cls[q]) continue;
        int it = iters;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = cls[q];
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(T);
        cfg.attrs = at;
        cfg.numAttrs = 2;
        for (int rep = 0; rep < 2; ++rep) {
          cudaMemset(ctr, 0, 4);
          cudaEventRecord(a);
          cudaLaunchKernelEx(&cfg, k_hier, it, ctr);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          cudaEventElapsedTime(&mh[q], a, b);
        }
      }
      printf("G=%3d T=%4d  cg.sync %.3f us  own %.3f us  round(2 sync) %.3f us  hier c2 %.3f c4 %.3f c8 %.3f us [%s]\n", G, T,
             ms[0] * 1e3 / iters, ms[1] * 1e3 / iters, ms[2] * 1e3 / iters, mh[0] * 1e3 / iters,
             mh[1] * 1e3 / iters, mh[2] * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
