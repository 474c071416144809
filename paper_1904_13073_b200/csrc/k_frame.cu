// k_frame.cu — depth -> frame maps (K22) and frame-0 surfel initialisation.
//   build_frame_maps   depth_processing.cpp:103-138 (backproject :14-32,
//                      estimate_normals :34-57, confidence/radius :59-69)
//   bilateral filter   depth_processing.cpp:71-101 (off by default)
//   initialize_from_frame surfels  pipeline.cpp:42-59
// One thread per pixel; the 4 neighbour vertices are re-derived from the u16
// depth in registers (same fp64 expressions) instead of a second pass.
#include "ds_context.cuh"

namespace ds {
namespace {

struct FrameParams {
  int W, H;
  double fx, fy, cx, cy, dmin, dmax, focal, max_radial, min_abs_nz;
};

__device__ __forceinline__ bool vert_at(const uint16_t* __restrict__ depth, const FrameParams& p,
                                        int x, int y, V3& v) {
  const uint16_t raw = depth[(size_t)y * p.W + x];
  if (raw == 0) return false;
  const double d = raw * 1e-3;
  if (d < p.dmin || d > p.dmax) return false;
  v = v3(d * (x - p.cx) / p.fx, d * (y - p.cy) / p.fy, d);
  return true;
}

__global__ void k_frame_maps(const uint16_t* __restrict__ depth, FrameParams p,
                             double4* __restrict__ vert, double4* __restrict__ nrmv,
                             uint8_t* __restrict__ flag, int* __restrict__ valid_count) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= p.W) return;
  const size_t i = (size_t)y * p.W + x;
  V3 v;
  const bool vv = vert_at(depth, p, x, y, v);
  uint8_t f = vv ? 1 : 0;
  double4 outv = make_double4(0, 0, 0, 0), outn = make_double4(0, 0, 0, 0);
  if (vv) outv = make_double4(v.x, v.y, v.z, 0.0);
  if (vv && x >= 1 && y >= 1 && x + 1 < p.W && y + 1 < p.H) {
    V3 xm, xp, ym, yp;
    if (vert_at(depth, p, x - 1, y, xm) && vert_at(depth, p, x + 1, y, xp) &&
        vert_at(depth, p, x, y - 1, ym) && vert_at(depth, p, x, y + 1, yp)) {
      const V3 tu = sub(xp, xm), tv = sub(yp, ym);
      V3 c = cross(tu, tv);
      const double len = nrm(c);
      if (!(len < 1e-12)) {
        c = dvd(c, len);
        if (dot(c, v) > 0) c = neg(c);
        const double g = p.max_radial > 0 ? hypot(x - p.cx, y - p.cy) / p.max_radial : 0.0;
        const double conf = exp(-(g * g) / (2.0 * 0.6 * 0.6));
        const double a = fmax(fabs(c.z), p.min_abs_nz);
        const double rad = sqrt(2.0) * v.z / (p.focal * a);
        outv.w = rad;
        outn = make_double4(c.x, c.y, c.z, conf);
        f |= 2;
        atomicAdd(valid_count, 1);
      }
    }
  }
  vert[i] = outv;
  nrmv[i] = outn;
  flag[i] = f;
}

__global__ void k_bilateral(const uint16_t* __restrict__ in, int W, int H, double i2s,
                            double i2d, uint16_t* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= W) return;
  const uint16_t c = in[(size_t)y * W + x];
  uint16_t res = 0;
  if (c != 0) {
    double ws = 0, vs = 0;
    for (int dy = -2; dy <= 2; ++dy)
      for (int dx = -2; dx <= 2; ++dx) {
        const int nx = x + dx, ny = y + dy;
        if (nx < 0 || nx >= W || ny < 0 || ny >= H) continue;
        const uint16_t s = in[(size_t)ny * W + nx];
        if (s == 0) continue;
        const double dd = double(s) - double(c);
        const double wb = exp(-(dx * dx + dy * dy) * i2s - dd * dd * i2d);
        ws += wb;
        vs += wb * s;
      }
    res = (uint16_t)llround(vs / ws);
  }
  out[(size_t)y * W + x] = res;
}

__global__ void k_valid_flags(const uint8_t* __restrict__ flag, int n, int* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (flag[i] & 2) ? 1 : 0;
}

__global__ void k_init_surfels(const double4* __restrict__ vert, const double4* __restrict__ nrmv,
                               const uint8_t* __restrict__ flag, const int* __restrict__ pos,
                               int n, Rig pose, int frame_index, ModelBuf m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !(flag[i] & 2)) return;
  const int o = pos[i];
  const double4 a = vert[i], b = nrmv[i];
  const V3 p = rig_apply(pose, v3(a.x, a.y, a.z));
  const V3 nn = rig_rotate(pose, v3(b.x, b.y, b.z));
  const float4 pr = make_float4((float)p.x, (float)p.y, (float)p.z, (float)a.w);
  const float4 nc = make_float4((float)nn.x, (float)nn.y, (float)nn.z, (float)b.w);
  m.rp[o] = pr;
  m.lp[o] = pr;
  m.rn[o] = nc;
  m.ln[o] = nc;
  m.t[o] = make_int2(frame_index, frame_index);
  m.ki[o] = make_int4(-1, -1, -1, -1);
  m.kw[o] = make_float4(0, 0, 0, 0);
}
}  // namespace

void frame_maps(Ctx& c, const uint16_t* depth_dev, int frame_index) {
  const ds_config& k = c.cfg;
  FrameParams p;
  p.W = c.W;
  p.H = c.H;
  p.fx = k.fx;
  p.fy = k.fy;
  p.cx = k.cx;
  p.cy = k.cy;
  p.dmin = k.depth_min;
  p.dmax = k.depth_max;
  p.focal = 0.5 * (k.fx + k.fy);
  double best = 0;  // CameraIntrinsics::max_radial_distance (types.hpp:31-38)
  for (int corner = 0; corner < 4; ++corner) {
    const double x = (corner & 1) ? double(c.W - 1) : 0.0;
    const double y = (corner & 2) ? double(c.H - 1) : 0.0;
    best = std::max(best, std::hypot(x - k.cx, y - k.cy));
  }
  p.max_radial = best;
  p.min_abs_nz = std::cos(75.0 * M_PI / 180.0);
  const uint16_t* src = depth_dev;
  const dim3 grid(cdiv(c.W, 128), c.H);
  if (k.bilateral_filter) {
    const double i2s = 1.0 / (2.0 * k.bilateral_sigma_space * k.bilateral_sigma_space);
    const double i2d = 1.0 / (2.0 * k.bilateral_sigma_depth * k.bilateral_sigma_depth);
    DS_LAUNCH(c, KK_FRAME_MAPS, 4.0 * c.P, grid, 128, 0, k_bilateral, depth_dev, c.W, c.H, i2s,
              i2d, c.depth_f);
    src = c.depth_f;
  }
  DS_CUDA(cudaMemsetAsync(&c.dsc->valid_count, 0, sizeof(int), c.stream));
  // algorithmic bytes: 2 B depth in, 2 x 32 B maps + 1 B flags out
  DS_LAUNCH(c, KK_FRAME_MAPS, 67.0 * c.P, grid, 128, 0, k_frame_maps, src, p, c.f_vert, c.f_nrm,
            c.f_flag, &c.dsc->valid_count);
  c.frame_index = frame_index;
  c.frame_ready = true;
}

void init_surfels_from_frame(Ctx& c) {
  DS_LAUNCH(c, KK_MISC, 5.0 * c.P, cdiv(c.P, 256), 256, 0, k_valid_flags, c.f_flag, c.P,
            c.cand_flag);
  scan_exclusive(c, c.cand_flag, c.cand_scan, c.P);
  int n = 0;
  DS_CUDA(cudaMemcpyAsync(&n, c.cand_scan + c.P, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  sync(c);
  if (n == 0) fail(DS_ERR_EMPTY_GEOMETRY, "initialization frame has no valid depth pixels");
  ensure_surfel_capacity(c, n);
  DS_LAUNCH(c, KK_MISC, 70.0 * c.P, cdiv(c.P, 256), 256, 0, k_init_surfels, c.f_vert, c.f_nrm,
            c.f_flag, c.cand_scan, c.P, rig_load(c.pose), c.frame_index, c.M());
  c.n_surfels = n;
}

}  // namespace ds
