// k_raster.cu — compute-side rasterisation (K3, K4, K10) replacing the paper's
// OpenGL index maps.
//   render_model_maps   raster.cpp:32-121: eligibility (stable, or recent in the
//                       bootstrap window), back-face cull, point channel at the
//                       lround pixel, opaque disk splats, point beats splat
//   find_correspondences solver.cpp:244-271: gates |v_m - v_d| < 3 cm and
//                       n_m . n_d > 0.7, pair per pixel in row-major order
//   render_index_map    raster.cpp:8-30: supersampled point z-buffer
// Exact z-buffer semantics (nearest fp64 depth wins, ties -> lower surfel index)
// in two atomic passes: pass 1 atomicMin on the fp64 depth bits (positive
// doubles order like unsigned ints), pass 2 atomicMin on the index among the
// writers whose depth equals the stored minimum.
#include "ds_assoc.cuh"
#include "ds_blend.cuh"
#include "ds_context.cuh"

namespace ds {
namespace {

// z-buffer updates are fire-and-forget reductions (RED.MIN: the result is not
// read, nothing waits). A load-then-atomic pre-test measured 2.5x slower: the
// load blocks the thread for an L2 round trip, the RED does not.
__device__ __forceinline__ void zmin(unsigned long long* p, unsigned long long v) { atomicMin(p, v); }
__device__ __forceinline__ void imin(int* p, int v) { atomicMin(p, v); }

struct CamParams {
  Rig w2c;
  double fx, fy, cx, cy, focal;
  int W, H;
};

#ifndef DS_SPLAT_LANES1
#define DS_SPLAT_LANES1 1
#endif
#ifndef DS_SPLAT_LANES2
#define DS_SPLAT_LANES2 4
#endif
// lanes per surfel in the solve-loop splats: pass 1 (with the fp64 warp, done
// redundantly per lane) and pass 2 (depth-test loads, the latency-bound one)
constexpr int kSplatLanes1 = DS_SPLAT_LANES1, kSplatLanes2 = DS_SPLAT_LANES2;

struct SplatParams {
  CamParams cam;
  int t_now, delta_recent, host_bootstrap;
  double delta_stable;
};

__global__ void k_any_stable(const float4* __restrict__ ln, int n, double delta_stable,
                             int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool st = i < n && (double)ln[i].w > delta_stable;
  const unsigned b = __ballot_sync(0xffffffffu, st);
  if ((threadIdx.x & 31) == 0 && b) atomicOr(flag, 1);
}

// list == nullptr: every surfel, eligibility tested here (raster.cpp:65-68);
// list != nullptr: a precomputed render-eligible surfel list (solve loop)
// kWarp (pass 1 over a list): the surfel is first forward-warped
// (warp_field.cpp:128-140, as k_forward_warp) and its live state written,
// so the solve loop's warp + first splat pass are one launch.
// The splat of one surfel (raster.cpp:70-101): point channel at its centre
// pixel, splat channel over its disk; kL lanes share the disk pixels.
template <bool kPass2, int kL>
__device__ __forceinline__ void model_splat_surfel(const float4& lp, const float4& ln, int i,
                                                   int lane, const SplatParams& sp,
                                                   unsigned long long* pkey,
                                                   unsigned long long* skey, int* pidx,
                                                   int* sidx) {
  const CamParams& k = sp.cam;
  const V3 pc = rig_apply(k.w2c, v3(lp.x, lp.y, lp.z));
  if (pc.z <= 0) return;
  const V3 nc = rig_rotate(k.w2c, v3(ln.x, ln.y, ln.z));
  if (dot(nc, pc) >= 0) return;
  const double u = k.fx * pc.x / pc.z + k.cx;
  const double v = k.fy * pc.y / pc.z + k.cy;
  const unsigned long long zb = (unsigned long long)__double_as_longlong(pc.z);
  const bool sane = fabs(u) < 1e9 && fabs(v) < 1e9;
  const int ccx = sane ? (int)llround(u) : -1, ccy = sane ? (int)llround(v) : -1;
  const bool cin = ccx >= 0 && ccx < k.W && ccy >= 0 && ccy < k.H;
  if (cin && lane == 0) {
    const size_t c = (size_t)ccy * k.W + ccx;
    if (!kPass2) zmin(pkey + c, zb);
    else if (pkey[c] == zb) imin(pidx + c, i);
  }
  const double rpx = (double)lp.w * k.focal / pc.z;
  const double r2 = rpx * rpx;
  if (sane && rpx < 1e6) {
    const int y0 = max((int)ceil(v - rpx), 0), y1 = min((int)floor(v + rpx), k.H - 1);
    const int x0 = max((int)ceil(u - rpx), 0), x1 = min((int)floor(u + rpx), k.W - 1);
    if (y1 >= y0 && x1 >= x0) {
      const int bw = x1 - x0 + 1, total = bw * (y1 - y0 + 1);
      if (!kPass2) {
        for (int idx = lane; idx < total; idx += kL) {
          const int y = y0 + idx / bw, x = x0 + idx % bw;
          const double dx = x - u, dy = y - v;
          if (dx * dx + dy * dy <= r2) zmin(skey + (size_t)y * k.W + x, zb);
        }
      } else {
        // pass 2 must read the stored depth before its RED: four disk pixels'
        // loads per lane are issued together instead of one blocking load each
        for (int base = 0; base < total; base += 4 * kL) {
          unsigned long long kv[4];
          size_t cc[4];
          bool in[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int idx = base + q * kL + lane;
            const int y = y0 + idx / bw, x = x0 + idx % bw;
            const double dx = x - u, dy = y - v;
            in[q] = idx < total && dx * dx + dy * dy <= r2;
            cc[q] = (size_t)y * k.W + x;
            kv[q] = in[q] ? skey[cc[q]] : 0ull;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (in[q] && kv[q] == zb) imin(sidx + cc[q], i);
        }
      }
    }
  }
  if (cin && lane == 0) {  // sub-pixel splats keep their own pixel (raster.cpp:101)
    const size_t c = (size_t)ccy * k.W + ccx;
    if (!kPass2) zmin(skey + c, zb);
    else if (skey[c] == zb) imin(sidx + c, i);
  }
}

template <bool kPass2, bool kWarp = false, int kL = 1>
__global__ void __launch_bounds__(256) k_model_splat(ModelBuf m, int n, const int* __restrict__ list,
                                                     SplatParams sp,
                                                     const int* __restrict__ any_stable,
                                                     unsigned long long* pkey,
                                                     unsigned long long* skey, int* pidx,
                                                     int* sidx,
                                                     const double4* __restrict__ warp_dq = nullptr) {
  pdl_wait();  // programmatic dependent launch: predecessor results visible
  // kL lanes per surfel: each computes the surfel's projection (bit-identical
  // in every lane) and takes every kL-th pixel of its splat disk
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int k0 = gt / kL, lane = gt % kL;
  if (k0 >= n) return;
  const int i = list ? list[k0] : k0;
  float4 lp, ln;
  if (kWarp) {
    const float4 rp = m.rp[i], rn = m.rn[i];
    const int4 ki = m.ki[i];
    const float4 kw = m.kw[i];
    const Blend b = blend_entry(ki, kw, warp_dq);
    lp = rp;
    ln = rn;
    if (!b.degenerate) warp_surfel(b, rp, rn, lp, ln);
    if (lane == 0) {
      m.lp[i] = lp;
      m.ln[i] = ln;
    }
  } else {
    lp = m.lp[i];
    ln = m.ln[i];
  }
  if (!list) {
    const int2 t = m.t[i];
    const bool stable = (double)ln.w > sp.delta_stable;
    const bool recent = (sp.t_now - t.y) <= sp.delta_recent;
    const bool bootstrap = sp.host_bootstrap || !(*any_stable);
    if (!stable && !(bootstrap && recent)) return;
  }
  model_splat_surfel<kPass2, kL>(lp, ln, i, lane, sp, pkey, skey, pidx, sidx);
}

struct AssocParams {
  Rig pose;
  int P;
  int associate;
  int reset;  // reset the consumed z-buffer entries (the maps end up cleared)
};

__global__ void k_resolve_associate(int* __restrict__ pidx, int* __restrict__ sidx,
                                    unsigned long long* __restrict__ pkey,
                                    unsigned long long* __restrict__ skey,
                                    ModelBuf m, const double4* __restrict__ fvert,
                                    const double4* __restrict__ fnrm,
                                    const uint8_t* __restrict__ fflag, AssocParams ap,
                                    int* __restrict__ mm_idx, int* __restrict__ pair_s,
                                    int* __restrict__ n_pairs) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ap.P) return;
  const int win = resolve_winner(pidx, sidx, c);
  mm_idx[c] = win;
  if (ap.reset) {
    if (pidx[c] != kEmptyIdx) {
      pidx[c] = kEmptyIdx;
      pkey[c] = ~0ull;
    }
    if (sidx[c] != kEmptyIdx) {
      sidx[c] = kEmptyIdx;
      skey[c] = ~0ull;
    }
  }
  if (!ap.associate) return;
  const int ps = associate_pixel(c, win, m, fvert, fnrm, fflag, ap.pose);
  pair_s[c] = ps;
  const unsigned b = __ballot_sync(0xffffffffu, ps >= 0);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(n_pairs, __popc(b));
}

// kWarp (pass 1): the full-model forward warp (warp_field.cpp:104-140,
// pipeline.cpp:108) is done here, the live state written, then splatted.
// Index-map splat of one surfel (raster.cpp:8-30): its supersampled cell.
template <bool kPass2>
__device__ __forceinline__ void index_splat_surfel(const float4& lp, int i, const CamParams& k,
                                                   int factor, unsigned long long* key, int* idx) {
  const V3 pc = rig_apply(k.w2c, v3(lp.x, lp.y, lp.z));
  if (pc.z <= 0) return;
  const double u = k.fx * pc.x / pc.z + k.cx;
  const double v = k.fy * pc.y / pc.z + k.cy;
  const double fu = floor(factor * (u + 0.5)), fv = floor(factor * (v + 0.5));
  const int Wf = k.W * factor, Hf = k.H * factor;
  if (!(fu >= 0 && fu < Wf && fv >= 0 && fv < Hf)) return;
  const size_t c = (size_t)fv * Wf + (size_t)fu;
  const unsigned long long zb = (unsigned long long)__double_as_longlong(pc.z);
  if (!kPass2) zmin(key + c, zb);
  else if (key[c] == zb) imin(idx + c, i);
}

template <bool kPass2, bool kWarp = false>
__global__ void __launch_bounds__(256) k_index_splat(ModelBuf m, int n, CamParams k, int factor,
                                                     unsigned long long* key, int* idx,
                                                     const double4* __restrict__ warp_dq = nullptr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float4 lp;
  if (kWarp) {
    const float4 rp = __ldcs(m.rp + i), rn = __ldcs(m.rn + i);
    const int4 ki = __ldcs(m.ki + i);
    const float4 kw = __ldcs(m.kw + i);
    const Blend b = blend_entry(ki, kw, warp_dq);
    float4 ln = rn;
    lp = rp;
    if (!b.degenerate) warp_surfel(b, rp, rn, lp, ln);
    m.lp[i] = lp;
    m.ln[i] = ln;
  } else {
    lp = m.lp[i];
  }
  index_splat_surfel<kPass2>(lp, i, k, factor, key, idx);
}

CamParams cam_params(Ctx& c, const double* pose) {
  CamParams k;
  k.w2c = rig_inverse(rig_load(pose));
  k.fx = c.cfg.fx;
  k.fy = c.cfg.fy;
  k.cx = c.cfg.cx;
  k.cy = c.cfg.cy;
  k.focal = 0.5 * (c.cfg.fx + c.cfg.fy);
  k.W = c.W;
  k.H = c.H;
  return k;
}

}  // namespace

// consume_reset: the resolve pass resets the entries it consumed, leaving the
// z-buffers cleared for the next render (no memsets there)
void render_model_maps(Ctx& c, const double* pose, int t_now, int t_last, bool associate,
                       const double* assoc_pose, bool consume_reset) {
  const int n = c.n_surfels;
  if (!c.mm_clean) clear_model_maps(c);
  c.mm_clean = false;
  // the bootstrap flag: from the last compaction when valid, else a pass here
  const int* any_stable = c.any_stable_ready ? c.any_stable_pre : &c.dsc->any_stable;
  if (!c.any_stable_ready) DS_CUDA(cudaMemsetAsync(&c.dsc->any_stable, 0, sizeof(int), c.stream));
  DS_CUDA(cudaMemsetAsync(&c.dsc->n_pairs, 0, sizeof(int), c.stream));
  SplatParams sp;
  sp.cam = cam_params(c, pose);
  sp.t_now = t_now;
  sp.delta_recent = c.cfg.delta_recent;
  sp.delta_stable = c.cfg.delta_stable;
  sp.host_bootstrap = (t_now - t_last <= c.cfg.delta_recent) ? 1 : 0;
  if (n > 0) {
    if (!c.any_stable_ready)
      DS_LAUNCH(c, KK_MODEL_MAP_SPLAT, 16.0 * n, cdiv(n, 256), 256, 0, k_any_stable, c.M().ln, n,
                c.cfg.delta_stable, &c.dsc->any_stable);
    DS_LAUNCH(c, KK_MODEL_MAP_SPLAT, 40.0 * n, cdiv(n, 256), 256, 0, k_model_splat<false>, c.M(), n,
              (const int*)nullptr, sp, any_stable, c.mm_pkey, c.mm_skey, c.mm_pidx, c.mm_sidx,
              (const double4*)nullptr);
    DS_LAUNCH(c, KK_MODEL_MAP_SPLAT, 40.0 * n, cdiv(n, 256), 256, 0, k_model_splat<true>, c.M(), n,
              (const int*)nullptr, sp, any_stable, c.mm_pkey, c.mm_skey, c.mm_pidx, c.mm_sidx,
              (const double4*)nullptr);
  }
  AssocParams ap;
  ap.pose = rig_load(associate ? assoc_pose : pose);
  ap.P = c.P;
  ap.associate = associate ? 1 : 0;
  ap.reset = consume_reset ? 1 : 0;
  // per pixel: 2 x 4 B winner ids, frame maps 65 B, winner live 32 B, 2 x 4 B out
  DS_LAUNCH(c, KK_ASSOCIATE, (associate ? 113.0 : 12.0) * c.P, cdiv(c.P, 256), 256, 0,
            k_resolve_associate, c.mm_pidx, c.mm_sidx, c.mm_pkey, c.mm_skey, c.M(), c.f_vert,
            c.f_nrm, c.f_flag, ap, c.mm_idx, c.pair_s, &c.dsc->n_pairs);
  c.mm_clean = consume_reset;
  std::copy(pose, pose + 12, c.mm_pose);
  c.mm_ready = true;
}

void clear_model_maps(Ctx& c) {
  const size_t P = c.P;
  DS_CUDA(cudaMemsetAsync(c.mm_pkey, 0xff, 8 * P, c.stream));
  DS_CUDA(cudaMemsetAsync(c.mm_skey, 0xff, 8 * P, c.stream));
  DS_CUDA(cudaMemsetAsync(c.mm_pidx, 0x7f, 4 * P, c.stream));
  DS_CUDA(cudaMemsetAsync(c.mm_sidx, 0x7f, 4 * P, c.stream));
  c.mm_clean = true;
}

// clear = false: the z-buffers are known to be empty (reset by their last
// consumer, k_assoc_pair_terms, inside the device LM loop)
void render_model_maps_list(Ctx& c, const double* pose, int t_now, int t_last,
                            const double* assoc_pose, const int* list, int n,
                            const double4* warp_dq, bool resolve, bool clear) {
  if (clear && !c.mm_clean) clear_model_maps(c);
  c.mm_clean = false;  // the consumer (k_assoc_pair_terms) resets what it reads
  // the pair counter of the resolve pass (without it, the caller's consumer
  // counts and the caller resets it)
  if (resolve) DS_CUDA(cudaMemsetAsync(&c.dsc->n_pairs, 0, sizeof(int), c.stream));
  SplatParams sp;
  sp.cam = cam_params(c, pose);
  sp.t_now = t_now;
  sp.delta_recent = c.cfg.delta_recent;
  sp.delta_stable = c.cfg.delta_stable;
  sp.host_bootstrap = (t_now - t_last <= c.cfg.delta_recent) ? 1 : 0;
  if (n > 0) {
    // several lanes per listed surfel (the solve loop's short lists)
    auto k_warp_splat = k_model_splat<false, true, kSplatLanes1>;
    auto k_pass1 = k_model_splat<false, false, kSplatLanes1>;
    auto k_pass2 = k_model_splat<true, false, kSplatLanes2>;
    const int nb = cdiv((long long)n * kSplatLanes1, 256), nb2 = cdiv((long long)n * kSplatLanes2, 256);
    if (warp_dq)  // warp (96 B) + pass 1 (36 B) per listed surfel
      DS_LAUNCH_PDL(c, KK_MODEL_MAP_SPLAT, 132.0 * n, nb, 256, 0, k_warp_splat, c.M(), n, list, sp,
                    &c.dsc->any_stable, c.mm_pkey, c.mm_skey, c.mm_pidx, c.mm_sidx, warp_dq);
    else
      DS_LAUNCH_PDL(c, KK_MODEL_MAP_SPLAT, 36.0 * n, nb, 256, 0, k_pass1, c.M(), n, list, sp,
                    &c.dsc->any_stable, c.mm_pkey, c.mm_skey, c.mm_pidx, c.mm_sidx,
                    (const double4*)nullptr);
    DS_LAUNCH_PDL(c, KK_MODEL_MAP_SPLAT, 36.0 * n, nb2, 256, 0, k_pass2, c.M(), n, list, sp,
                  &c.dsc->any_stable, c.mm_pkey, c.mm_skey, c.mm_pidx, c.mm_sidx,
                  (const double4*)nullptr);
  }
  if (resolve) {
    AssocParams ap;
    ap.pose = rig_load(assoc_pose);
    ap.P = c.P;
    ap.associate = 1;
    ap.reset = 0;
    DS_LAUNCH(c, KK_ASSOCIATE, 113.0 * c.P, cdiv(c.P, 256), 256, 0, k_resolve_associate, c.mm_pidx,
              c.mm_sidx, c.mm_pkey, c.mm_skey, c.M(), c.f_vert, c.f_nrm, c.f_flag, ap, c.mm_idx,
              c.pair_s, &c.dsc->n_pairs);
  }
  std::copy(pose, pose + 12, c.mm_pose);
  c.mm_ready = true;
}

void render_index_map(Ctx& c, const double* pose, int factor, const double4* warp_dq) {
  const int n = c.n_surfels;
  const size_t cells = (size_t)c.P * factor * factor;
  if (factor != c.cfg.supersample_factor && factor > c.cfg.supersample_factor)
    fail(DS_ERR_CAPACITY, "index map factor larger than the configured supersample_factor");
  DS_CUDA(cudaMemsetAsync(c.im_key, 0xff, 8 * cells, c.stream));
  DS_CUDA(cudaMemsetAsync(c.im_idx, 0x7f, 4 * cells, c.stream));
  const CamParams k = cam_params(c, pose);
  if (n > 0) {
    auto k_warp_index = k_index_splat<false, true>;
    if (warp_dq)  // full forward warp (96 B) + index pass 1 (16 B) per surfel
      DS_LAUNCH(c, KK_INDEX_MAP, 112.0 * n, cdiv(n, 256), 256, 0, k_warp_index, c.M(), n, k, factor,
                c.im_key, c.im_idx, warp_dq);
    else
      DS_LAUNCH(c, KK_INDEX_MAP, 16.0 * n, cdiv(n, 256), 256, 0, k_index_splat<false>, c.M(), n, k,
                factor, c.im_key, c.im_idx, (const double4*)nullptr);
    DS_LAUNCH(c, KK_INDEX_MAP, 16.0 * n, cdiv(n, 256), 256, 0, k_index_splat<true>, c.M(), n, k,
              factor, c.im_key, c.im_idx, (const double4*)nullptr);
  }
  c.im_factor = factor;
  std::copy(pose, pose + 12, c.im_pose);
  c.im_ready = true;
}

}  // namespace ds
