// k_warp.cu — dual-quaternion surfel warp (K1) and per-node transforms.
//   forward_warp            warp_field.cpp:104-114, 128-140
//   node to_se3 cache       solver.cpp:355 (node_se3), geometry.cpp:86-93
//   WarpNode::live_position warp_field.hpp:21
//   apply_increments        solver.cpp:277-286
// forward_warp is HBM-bound: per surfel it streams 64 B in (reference pos+r,
// nrm+c, 4 node ids, 4 weights) and 32 B out (live pos+r, nrm+c) = 96 B; the
// <=4 node dual quaternions per surfel are gathered from L1/L2 (N x 64 B).
#include "ds_blend.cuh"
#include "ds_context.cuh"

namespace ds {
namespace {

// Thread per surfel, streaming loads/stores (__ldcs/__stcs: read-once data).
// (A two-surfels-per-thread variant measured slower: 80 registers cost more
// occupancy than the extra memory-level parallelism bought.)
__global__ void __launch_bounds__(256) k_forward_warp(ModelBuf m, int n,
                                                      const double4* __restrict__ node_dq,
                                                      int* __restrict__ degenerate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 rp = __ldcs(m.rp + i);
  const float4 rn = __ldcs(m.rn + i);
  const int4 ki = __ldcs(m.ki + i);
  const float4 kw = __ldcs(m.kw + i);
  const Blend b = blend_entry(ki, kw, node_dq);
  float4 lp = rp, ln = rn;
  if (!b.degenerate) {
    warp_surfel(b, rp, rn, lp, ln);
  } else if (degenerate) {
    atomicAdd(degenerate, 1);
  }
  __stcs(m.lp + i, lp);
  __stcs(m.ln + i, ln);
}

__global__ void k_node_se3(const double4* __restrict__ dq, int n, double* __restrict__ se3) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  DQ q;
  q.r = ld_q_plain(dq + 2 * j);
  q.d = ld_q_plain(dq + 2 * j + 1);
  rig_store(dq_to_rig(q), se3 + 12 * j);
}

// live positions (fp64 + an fp32 copy for K-NN pre-tests) and the largest
// |coordinate| (bound for the fp32 rounding margin, as float bits)
__global__ void k_node_live(const double4* __restrict__ pos, const double4* __restrict__ dq, int n,
                            double4* __restrict__ live, float4* __restrict__ live_f,
                            int* __restrict__ rmax_bits) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  DQ q;
  q.r = ld_q_plain(dq + 2 * j);
  q.d = ld_q_plain(dq + 2 * j + 1);
  const double4 p = pos[j];
  const V3 l = rig_apply(dq_to_rig(q), v3(p.x, p.y, p.z));
  live[j] = make_double4(l.x, l.y, l.z, p.w);
  live_f[j] = make_float4((float)l.x, (float)l.y, (float)l.z, 0.f);
  const double m = fmax(fmax(fabs(l.x), fabs(l.y)), fabs(l.z));
  atomicMax(rmax_bits, __float_as_int(__double2float_ru(m)));
}

// se3 (optional): the new transforms' to_se3 cache (geometry.cpp:86-93) for
// the energy evaluation, fused here instead of a separate k_node_se3 launch
__global__ void k_apply_increments(const double4* __restrict__ dq, const double* __restrict__ delta,
                                   int n, double4* __restrict__ out, double* __restrict__ se3) {
  pdl_wait();  // programmatic dependent launch: predecessor results visible
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double* d = delta + 6 * j;
  const DQ inc = dq_increment(v3(d[0], d[1], d[2]), v3(d[3], d[4], d[5]));
  DQ q;
  q.r = ld_q_plain(dq + 2 * j);
  q.d = ld_q_plain(dq + 2 * j + 1);
  const DQ o = dq_normalized(dq_mul(inc, q));
  out[2 * j] = make_double4(o.r.w, o.r.x, o.r.y, o.r.z);
  out[2 * j + 1] = make_double4(o.d.w, o.d.x, o.d.y, o.d.z);
  if (se3) rig_store(dq_to_rig(o), se3 + 12 * j);
}

}  // namespace

void apply_increments(Ctx& c, const double* delta, double4* out, double* se3) {
  if (c.n_nodes == 0) return;
  DS_LAUNCH_PDL(c, KK_NODE_UPDATE, (se3 ? 208.0 : 112.0) * c.n_nodes, cdiv(c.n_nodes, 128), 128, 0,
            k_apply_increments, c.node_dq, delta, c.n_nodes, out, se3);
}

int forward_warp(Ctx& c, bool count_degenerate) {
  const int n = c.n_surfels;
  if (n == 0) return 0;
  if (count_degenerate) DS_CUDA(cudaMemsetAsync(&c.dsc->degenerate, 0, sizeof(int), c.stream));
  DS_LAUNCH(c, KK_FORWARD_WARP, 96.0 * n, cdiv(n, 256), 256, 0, k_forward_warp, c.M(), n,
            c.node_dq, count_degenerate ? &c.dsc->degenerate : nullptr);
  if (!count_degenerate) return 0;
  int deg = 0;
  DS_CUDA(cudaMemcpyAsync(&deg, &c.dsc->degenerate, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  sync(c);
  return deg;
}

void node_se3(Ctx& c, const double4* dq, double* se3) {
  if (c.n_nodes == 0) return;
  DS_LAUNCH(c, KK_NODE_UPDATE, 160.0 * c.n_nodes, cdiv(c.n_nodes, 128), 128, 0, k_node_se3, dq,
            c.n_nodes, se3);
}

void node_live_positions(Ctx& c) {
  if (c.n_nodes == 0) return;
  DS_CUDA(cudaMemsetAsync(&c.dsc->rmax_bits, 0, sizeof(int), c.stream));
  DS_LAUNCH(c, KK_NODE_UPDATE, 144.0 * c.n_nodes, cdiv(c.n_nodes, 128), 128, 0, k_node_live,
            c.node_pos, c.node_dq, c.n_nodes, c.node_live, c.node_live_f, &c.dsc->rmax_bits);
}

}  // namespace ds
