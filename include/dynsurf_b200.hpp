// dynsurf_b200.hpp — C++ host mirror of the reference's dynsurf API over the C ABI.
//
// Same names, argument meaning and error behaviour as the reference core
// (/root/reference/proj/core/include/dynsurf): Pipeline (pipeline.hpp:38-62),
// PipelineConfig (config.hpp:11-50), Surfel / SkinningEntry / SurfelModel
// (types.hpp:41-80), WarpNode (warp_field.hpp:15-22), FrameStats
// (pipeline.hpp:16-33), the exception hierarchy (errors.hpp:8-38), and the
// stage functions used by the reference tests through dynsurf_b200::Stages.
// All compute runs on the B200 through libdynsurf_b200.so; this header only
// converts host types and rethrows C-ABI statuses as exceptions.
#pragma once

#include <array>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "dynsurf_b200.h"
#include "dynsurf_synth.h"

namespace dynsurf_b200 {

// ------------------------------------------------------------ errors.hpp
struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct DimensionMismatch : Error { using Error::Error; };
struct EmptyGeometry : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct UnknownScenario : Error { using Error::Error; };
struct CapacityExceeded : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };
struct InvalidArgument : Error { using Error::Error; };
struct IoFailure : Error { using Error::Error; };

inline void check(ds_status s) {
  if (s == DS_OK) return;
  const std::string m = ds_last_error();
  switch (s) {
    case DS_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(m);
    case DS_ERR_EMPTY_GEOMETRY: throw EmptyGeometry(m);
    case DS_ERR_CONFIG: throw ConfigError(m);
    case DS_ERR_CAPACITY: throw CapacityExceeded(m);
    case DS_ERR_CUDA: throw CudaError(m);
    case DS_ERR_INVALID_ARGUMENT: throw InvalidArgument(m);
    case DS_ERR_UNKNOWN_SCENARIO: throw UnknownScenario(m);
    default: throw Error(m);
  }
}

// ------------------------------------------------------------ types.hpp
using Vec3 = std::array<double, 3>;
using Quat = std::array<double, 4>;  // (w, x, y, z)

struct CameraIntrinsics {
  double fx = 0, fy = 0, cx = 0, cy = 0;
  int width = 0, height = 0;
  bool is_valid() const { return fx > 0 && fy > 0 && width > 0 && height > 0; }
};

struct PipelineConfig {
  ds_config c;
  PipelineConfig() { ds_default_config(&c); }
  CameraIntrinsics intrinsics() const { return {c.fx, c.fy, c.cx, c.cy, c.width, c.height}; }
  void set_intrinsics(const CameraIntrinsics& k) {
    c.fx = k.fx; c.fy = k.fy; c.cx = k.cx; c.cy = k.cy; c.width = k.width; c.height = k.height;
  }
  void validate() const { check(ds_validate_config(&c)); }
};

struct Surfel {
  Vec3 position{0, 0, 0};
  Vec3 normal{0, 0, 1};
  double radius = 0, confidence = 0;
  int32_t t_init = 0, t_observed = 0;
};

inline constexpr int kMaxSkinNeighbors = 8;
struct SkinningEntry {
  std::array<int32_t, kMaxSkinNeighbors> node_indices{};
  std::array<double, kMaxSkinNeighbors> weights{};
  int count = 0;
};

struct SurfelModel {
  std::vector<Surfel> reference, live;
  std::vector<SkinningEntry> skinning;
  size_t size() const { return reference.size(); }
  bool consistent() const { return reference.size() == live.size() && live.size() == skinning.size(); }
};

struct DualQuaternion {
  Quat real{1, 0, 0, 0};
  Quat dual{0, 0, 0, 0};
};
struct WarpNode {
  Vec3 position{0, 0, 0};
  double sigma = 0.025;
  DualQuaternion transform;
  std::vector<int32_t> neighbors;
};
struct Se3 {
  std::array<double, 9> rotation{1, 0, 0, 0, 1, 0, 0, 0, 1};
  Vec3 translation{0, 0, 0};
  static Se3 identity() { return {}; }
  void to12(double* p) const {
    std::memcpy(p, rotation.data(), 9 * sizeof(double));
    std::memcpy(p + 9, translation.data(), 3 * sizeof(double));
  }
  static Se3 from12(const double* p) {
    Se3 s;
    std::memcpy(s.rotation.data(), p, 9 * sizeof(double));
    std::memcpy(s.translation.data(), p + 9, 3 * sizeof(double));
    return s;
  }
};

struct DepthImage {  // image.hpp:39-45 (row-major mm, 0 = invalid)
  int width = 0, height = 0, frame_index = 0;
  std::vector<uint16_t> data;
};

using SolverReport = ds_solver_report;
using RigidAlignResult = ds_rigid_result;
using FusionOutcome = ds_fusion_outcome;
struct FrameStats : ds_frame_stats {
  Se3 pose_se3() const { return Se3::from12(pose); }
};

// ----------------------------------------------------------- device state
class Stages;

// Owns one ds_context (one sequence on one GPU / stream).
class DeviceState {
 public:
  explicit DeviceState(const PipelineConfig& cfg, int device = 0, void* stream = nullptr) {
    check(ds_create(&cfg.c, device, stream, &ctx_));
  }
  ~DeviceState() { ds_destroy(ctx_); }
  DeviceState(const DeviceState&) = delete;
  DeviceState& operator=(const DeviceState&) = delete;
  ds_context* get() const { return ctx_; }

  void upload(const SurfelModel& m) {
    if (!m.consistent()) throw InvalidArgument("SurfelModel arrays are not aligned");
    const size_t n = m.size();
    std::vector<double> rp(3 * n), rn(3 * n), lp(3 * n), ln(3 * n), r(n), c(n), w(8 * n);
    std::vector<int32_t> ti(n), to(n), idx(8 * n), cnt(n);
    for (size_t i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) {
        rp[3 * i + a] = m.reference[i].position[a];
        rn[3 * i + a] = m.reference[i].normal[a];
        lp[3 * i + a] = m.live[i].position[a];
        ln[3 * i + a] = m.live[i].normal[a];
      }
      r[i] = m.live[i].radius;
      c[i] = m.live[i].confidence;
      ti[i] = m.live[i].t_init;
      to[i] = m.live[i].t_observed;
      for (int k = 0; k < 8; ++k) {
        idx[8 * i + k] = m.skinning[i].node_indices[k];
        w[8 * i + k] = m.skinning[i].weights[k];
      }
      cnt[i] = m.skinning[i].count;
    }
    check(ds_upload_model(ctx_, int32_t(n), rp.data(), rn.data(), lp.data(), ln.data(), r.data(),
                          c.data(), ti.data(), to.data(), idx.data(), w.data(), cnt.data()));
  }
  SurfelModel download() const {
    int32_t n = 0;
    check(ds_model_size(ctx_, &n));
    std::vector<double> rp(3 * n), rn(3 * n), lp(3 * n), ln(3 * n), r(n), c(n), w(8 * n);
    std::vector<int32_t> ti(n), to(n), idx(8 * n), cnt(n);
    check(ds_download_model(ctx_, rp.data(), rn.data(), lp.data(), ln.data(), r.data(), c.data(),
                            ti.data(), to.data(), idx.data(), w.data(), cnt.data()));
    SurfelModel m;
    m.reference.resize(n);
    m.live.resize(n);
    m.skinning.resize(n);
    for (int32_t i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) {
        m.reference[i].position[a] = rp[3 * i + a];
        m.reference[i].normal[a] = rn[3 * i + a];
        m.live[i].position[a] = lp[3 * i + a];
        m.live[i].normal[a] = ln[3 * i + a];
      }
      for (Surfel* s : {&m.reference[i], &m.live[i]}) {
        s->radius = r[i];
        s->confidence = c[i];
        s->t_init = ti[i];
        s->t_observed = to[i];
      }
      m.skinning[i].count = cnt[i];
      for (int k = 0; k < 8; ++k) {
        m.skinning[i].node_indices[k] = idx[8 * i + k];
        m.skinning[i].weights[k] = w[8 * i + k];
      }
    }
    return m;
  }
  void upload(const std::vector<WarpNode>& nodes) {
    const size_t n = nodes.size();
    std::vector<double> pos(3 * n), sig(n), dq(8 * n);
    std::vector<int32_t> nb(8 * n, -1), nc(n);
    for (size_t j = 0; j < n; ++j) {
      for (int a = 0; a < 3; ++a) pos[3 * j + a] = nodes[j].position[a];
      sig[j] = nodes[j].sigma;
      for (int a = 0; a < 4; ++a) {
        dq[8 * j + a] = nodes[j].transform.real[a];
        dq[8 * j + 4 + a] = nodes[j].transform.dual[a];
      }
      nc[j] = int32_t(nodes[j].neighbors.size());
      if (nc[j] > 8) throw InvalidArgument("device keeps at most 8 node edges");
      for (int k = 0; k < nc[j]; ++k) nb[8 * j + k] = nodes[j].neighbors[k];
    }
    check(ds_upload_nodes(ctx_, int32_t(n), pos.data(), sig.data(), dq.data(), nb.data(), nc.data()));
  }
  std::vector<WarpNode> download_nodes() const {
    int32_t n = 0;
    check(ds_num_nodes(ctx_, &n));
    std::vector<double> pos(3 * n), sig(n), dq(8 * n);
    std::vector<int32_t> nb(8 * n), nc(n);
    check(ds_download_nodes(ctx_, pos.data(), sig.data(), dq.data(), nb.data(), nc.data()));
    std::vector<WarpNode> out(n);
    for (int32_t j = 0; j < n; ++j) {
      for (int a = 0; a < 3; ++a) out[j].position[a] = pos[3 * j + a];
      out[j].sigma = sig[j];
      for (int a = 0; a < 4; ++a) {
        out[j].transform.real[a] = dq[8 * j + a];
        out[j].transform.dual[a] = dq[8 * j + 4 + a];
      }
      out[j].neighbors.assign(nb.begin() + 8 * j, nb.begin() + 8 * j + nc[j]);
    }
    return out;
  }

 private:
  ds_context* ctx_ = nullptr;
};

// ------------------------------------------------------------ pipeline.hpp
class Pipeline {
 public:
  explicit Pipeline(const PipelineConfig& cfg, int device = 0, void* stream = nullptr)
      : cfg_(cfg), dev_((cfg.validate(), cfg), device, stream) {}

  FrameStats process_frame(const DepthImage& depth) {
    if (depth.data.size() != size_t(depth.width) * depth.height)
      throw DimensionMismatch("depth buffer size does not match width x height");
    FrameStats st;
    check(ds_process_frame(dev_.get(), depth.data.data(), depth.width, depth.height,
                           depth.frame_index, &st));
    return st;
  }

  const PipelineConfig& config() const { return cfg_; }
  SurfelModel model() const { return dev_.download(); }            // lazy download
  std::vector<WarpNode> nodes() const { return dev_.download_nodes(); }
  Se3 pose() const {
    double p[12];
    check(ds_get_pose(dev_.get(), p));
    return Se3::from12(p);
  }
  bool initialized() const {
    int32_t i = 0, t = 0;
    check(ds_is_initialized(dev_.get(), &i, &t));
    return i != 0;
  }
  int last_reinit_frame() const {
    int32_t i = 0, t = 0;
    check(ds_is_initialized(dev_.get(), &i, &t));
    return t;
  }
  DeviceState& device_state() { return dev_; }

 private:
  PipelineConfig cfg_;
  DeviceState dev_;
};

// ------------------------------------------------- stage functions (tests)
// The reference's free functions take host containers; on the device they run
// against a DeviceState that holds the model / nodes between calls.
class Stages {
 public:
  explicit Stages(const PipelineConfig& cfg, int device = 0) : dev_(cfg, device) {}
  DeviceState& state() { return dev_; }

  // init_warp_field (warp_field.hpp:31-32)
  std::pair<std::vector<WarpNode>, std::vector<SkinningEntry>> init_warp_field(
      const std::vector<Surfel>& reference) {
    SurfelModel m;
    m.reference = reference;
    m.live = reference;
    m.skinning.resize(reference.size());
    dev_.upload(m);
    check(ds_init_warp_field(dev_.get()));
    return {dev_.download_nodes(), dev_.download().skinning};
  }
  // forward_warp (warp_field.hpp:56): rewrites model.live, returns #degenerate
  int forward_warp(SurfelModel& model, const std::vector<WarpNode>& nodes) {
    dev_.upload(model);
    dev_.upload(nodes);
    int32_t deg = 0;
    check(ds_forward_warp(dev_.get(), &deg));
    model = dev_.download();
    return deg;
  }
  // solve_nonrigid (solver.hpp:61-63) on frame maps built from `depth`
  SolverReport solve_nonrigid(std::vector<WarpNode>& nodes, const SurfelModel& model,
                              const DepthImage& depth, const Se3& pose, int t_now,
                              int t_last_reinit) {
    dev_.upload(model);
    dev_.upload(nodes);
    check(ds_frame_maps(dev_.get(), depth.data.data(), depth.width, depth.height,
                        depth.frame_index, nullptr));
    double p[12];
    pose.to12(p);
    SolverReport r{};
    check(ds_solve_nonrigid(dev_.get(), p, t_now, t_last_reinit, &r));
    nodes = dev_.download_nodes();
    return r;
  }
  // apply_fusion (fusion.hpp:76-78)
  FusionOutcome apply_fusion(SurfelModel& model, const DepthImage& depth,
                             std::vector<WarpNode>& nodes, const Se3& pose, int t_now) {
    dev_.upload(model);
    dev_.upload(nodes);
    check(ds_frame_maps(dev_.get(), depth.data.data(), depth.width, depth.height,
                        depth.frame_index, nullptr));
    double p[12];
    pose.to12(p);
    FusionOutcome o{};
    check(ds_apply_fusion(dev_.get(), p, t_now, &o));
    model = dev_.download();
    nodes = dev_.download_nodes();
    return o;
  }

 private:
  DeviceState dev_;
};

// --------------------------------------------------------------- synth.hpp
class SyntheticSequence {
 public:
  SyntheticSequence(const std::string& scenario, int frames, const PipelineConfig& cfg,
                    double noise_sigma_mm = 0.0, uint32_t seed = 20240901)
      : kind_(ds_synth_scenario(scenario.c_str())), cfg_(cfg), noise_(noise_sigma_mm), seed_(seed) {
    if (kind_ < 0) throw UnknownScenario("unknown scenario: " + scenario);
    frames_ = frames > 0 ? frames : ds_synth_default_frames(kind_);
  }
  int frame_count() const { return frames_; }
  DepthImage render_depth(int t) const {
    DepthImage d;
    d.width = cfg_.c.width;
    d.height = cfg_.c.height;
    d.frame_index = t;
    d.data.resize(size_t(d.width) * d.height);
    check(ds_synth_render_depth(kind_, frames_, &cfg_.c, noise_, seed_, t, d.data.data()));
    return d;
  }

 private:
  int kind_;
  int frames_ = 0;
  PipelineConfig cfg_;
  double noise_;
  uint32_t seed_;
};

// ------------------------------------------- ply_io.hpp / pipeline.cpp logs
// Same bytes as the reference's writers: export_pointcloud (ply_io.cpp:16-37)
// and the metrics / timings lines of process_sequence (pipeline.cpp:144-188,
// nlohmann::ordered_json::dump number layout). Python twin: sequence_io.py.
enum class ModelSide { kReference, kLive };

inline void export_pointcloud(const SurfelModel& model, ModelSide side, const std::string& path) {
  if (model.size() == 0) throw EmptyGeometry("export_pointcloud: empty model");
  const std::vector<Surfel>& surfels = side == ModelSide::kReference ? model.reference : model.live;
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoFailure("cannot create PLY: " + path);
  out << "ply\nformat binary_little_endian 1.0\nelement vertex " << surfels.size() << "\n";
  for (const char* p : {"x", "y", "z", "nx", "ny", "nz", "radius", "confidence"})
    out << "property double " << p << "\n";
  out << "end_header\n";
  for (const Surfel& s : surfels) {
    const double rec[8] = {s.position[0], s.position[1], s.position[2], s.normal[0],
                           s.normal[1],   s.normal[2],   s.radius,      s.confidence};
    out.write(reinterpret_cast<const char*>(rec), sizeof(rec));
  }
  if (!out) throw IoFailure("failed writing PLY: " + path);
}

namespace detail {
// nlohmann's double layout: shortest round-trip digits, format_buffer with
// min_exp = -4, max_exp = 15; non-finite values serialise as null.
inline std::string json_double(double x) {
  if (!std::isfinite(x)) return "null";
  if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof(buf), std::fabs(x), std::chars_format::scientific);
  const std::string sci(buf, r.ptr);
  const size_t e = sci.find('e');
  std::string digits = sci.substr(0, 1) + (e > 1 ? sci.substr(2, e - 2) : "");
  const int n = std::stoi(sci.substr(e + 1)) + 1;  // decimal point position
  const int k = int(digits.size());
  std::string out = x < 0 ? "-" : "";
  if (k <= n && n <= 15) {
    out += digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(-n, '0') + digits;
  } else {
    const int ex = n - 1;
    out += (k == 1 ? digits : digits.substr(0, 1) + "." + digits.substr(1)) + "e" +
           (ex < 0 ? "-" : "+") + (std::abs(ex) < 10 ? "0" : "") + std::to_string(std::abs(ex));
  }
  return out;
}
// quat_from_matrix (geometry.cpp:44-50): Eigen's branch order, normalised, w >= 0.
inline std::array<double, 4> quat_from_matrix(const std::array<double, 9>& m) {
  auto M = [&](int r, int c) { return m[r * 3 + c]; };
  std::array<double, 4> q{0, 0, 0, 0};
  double t = (M(0, 0) + M(1, 1)) + M(2, 2);
  if (t > 0.0) {
    t = std::sqrt(t + 1.0);
    q[0] = 0.5 * t;
    t = 0.5 / t;
    q[1] = (M(2, 1) - M(1, 2)) * t;
    q[2] = (M(0, 2) - M(2, 0)) * t;
    q[3] = (M(1, 0) - M(0, 1)) * t;
  } else {
    int i = 0;
    if (M(1, 1) > M(0, 0)) i = 1;
    if (M(2, 2) > M(i, i)) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    t = std::sqrt(M(i, i) - M(j, j) - M(k, k) + 1.0);
    q[1 + i] = 0.5 * t;
    t = 0.5 / t;
    q[0] = (M(k, j) - M(j, k)) * t;
    q[1 + j] = (M(j, i) + M(i, j)) * t;
    q[1 + k] = (M(k, i) + M(i, k)) * t;
  }
  const double nrm = std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
  for (double& c : q) c /= nrm;
  if (q[0] < 0)
    for (double& c : q) c = -c;
  return q;
}
}  // namespace detail

inline std::string frame_stats_to_json(const FrameStats& s) {
  using detail::json_double;
  auto b = [](int v) { return std::string(v ? "true" : "false"); };
  std::string o = "{\"frame\":" + std::to_string(s.frame) + ",\"skipped\":" + b(s.skipped);
  if (s.skipped) return o + "}";
  auto i = [&](const char* k, long v) { o += std::string(",\"") + k + "\":" + std::to_string(v); };
  auto d = [&](const char* k, double v) { o += std::string(",\"") + k + "\":" + json_double(v); };
  i("valid_pixels", s.valid_pixels); i("surfel_count", s.surfel_count);
  i("node_count", s.node_count); i("fused", s.fusion.fused); i("appended", s.fusion.appended);
  i("removed", s.fusion.removed); i("compressive_rejected", s.fusion.compressive_rejected);
  i("low_support_rejected", s.fusion.low_support_rejected); i("new_nodes", s.fusion.new_nodes);
  i("degenerate_warps", s.fusion.degenerate_warps); i("gn_iters", s.solver.iterations);
  i("correspondences", s.solver.correspondences); d("initial_energy", s.solver.initial_energy);
  d("final_energy", s.solver.final_energy); d("mean_residual", s.solver.mean_residual);
  i("rigid_pairs", s.rigid.correspondences); d("rigid_residual", s.rigid.mean_residual);
  o += ",\"rigid_low_confidence\":" + b(s.rigid.low_confidence) + ",\"reinit\":" + b(s.reinit);
  i("reinit_removed", s.reinit_removed);
  std::array<double, 9> rot;
  std::memcpy(rot.data(), s.pose, sizeof(rot));
  const auto q = detail::quat_from_matrix(rot);
  o += ",\"pose\":[" + json_double(q[0]) + "," + json_double(q[1]) + "," + json_double(q[2]) +
       "," + json_double(q[3]) + "," + json_double(s.pose[9]) + "," + json_double(s.pose[10]) +
       "," + json_double(s.pose[11]) + "]}";
  return o;
}

inline std::string timings_to_json(const FrameStats& s) {
  using detail::json_double;
  return "{\"frame\":" + std::to_string(s.frame) + ",\"depth_ms\":" + json_double(s.depth_ms) +
         ",\"rigid_ms\":" + json_double(s.rigid_ms) + ",\"solve_ms\":" + json_double(s.solve_ms) +
         ",\"fusion_ms\":" + json_double(s.fusion_ms) + ",\"reinit_ms\":" +
         json_double(s.reinit_ms) + ",\"total_ms\":" + json_double(s.total_ms) + "}";
}

}  // namespace dynsurf_b200
