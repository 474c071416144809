// ref_capi.cpp -- TEST INFRASTRUCTURE (oracle/_ref build only).
//
// A C ABI over the UNMODIFIED reference dynsurf::Pipeline, compiled from
// /root/reference/proj/core/src against the shims in ref_shim/ into
// oracle/_ref/libdynsurf_ref.so (oracle/Makefile, target `ref`). Used only by
// tests/ (oracle-vs-reference and device-vs-reference parity) and by the
// bench's CPU reference arm (`bench.py --impl reference`, `cpu_baseline` with
// kind "reference"). The product path never loads it.
//
// Reference interface: pipeline.hpp:35-61 (Pipeline, FrameStats),
// config.cpp apply_config_entry (the key/value names of the config file),
// types.hpp:41-80 (Surfel, SkinningEntry, SurfelModel), warp_field.hpp:15-22
// (WarpNode).
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>

#include "dynsurf/config.hpp"
#include "dynsurf/errors.hpp"
#include "dynsurf/pipeline.hpp"

namespace {
struct Handle {
  dynsurf::Pipeline pipe;
  explicit Handle(const dynsurf::PipelineConfig& c) : pipe(c) {}
};
void put_err(const char* what, char* err, int errlen) {
  if (err && errlen > 0) {
    std::strncpy(err, what, size_t(errlen) - 1);
    err[errlen - 1] = 0;
  }
}
}  // namespace

extern "C" {

// config_text: "key value" lines with the reference's config-file keys
// (fx fy cx cy width height node_sigma max_gn_iters ...). NULL on error.
void* dsref_create(const char* config_text, char* err, int errlen) {
  try {
    dynsurf::PipelineConfig cfg;
    std::istringstream in(config_text ? config_text : "");
    std::string line;
    while (std::getline(in, line)) {
      std::istringstream ls(line);
      std::string k, v;
      if (!(ls >> k >> v)) continue;
      dynsurf::apply_config_entry(cfg, k, v);
    }
    cfg.validate();
    return new Handle(cfg);
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return nullptr;
  }
}

void dsref_destroy(void* h) { delete static_cast<Handle*>(h); }

// stats (39 doubles): skipped, valid_pixels, surfel_count, node_count,
// rigid {correspondences, mean_residual, low_confidence}, solver {iterations,
// initial_energy, final_energy, mean_residual, correspondences}, fusion
// {fused, appended, removed, compressive_rejected, low_support_rejected,
// new_nodes, degenerate_warps}, reinit, reinit_removed, pose R (row-major 9)
// + t (3), depth/rigid/solve/fusion/reinit/total ms. Returns 0, or -1 with
// the exception text in err.
int dsref_process_frame(void* h, const uint16_t* depth, int width, int height, int frame_index,
                        double* stats, char* err, int errlen) {
  try {
    auto* p = static_cast<Handle*>(h);
    dynsurf::DepthImage img;
    img.data = dynsurf::Grid<uint16_t>(width, height);
    for (int y = 0; y < height; ++y)
      for (int x = 0; x < width; ++x) img.data(x, y) = depth[size_t(y) * width + x];
    img.frame_index = frame_index;
    const dynsurf::FrameStats s = p->pipe.process_frame(img);
    double* o = stats;
    *o++ = s.skipped ? 1 : 0;
    *o++ = s.valid_pixels;
    *o++ = s.surfel_count;
    *o++ = s.node_count;
    *o++ = s.rigid.correspondences;
    *o++ = s.rigid.mean_residual;
    *o++ = s.rigid.low_confidence ? 1 : 0;
    *o++ = s.solver.iterations;
    *o++ = s.solver.initial_energy;
    *o++ = s.solver.final_energy;
    *o++ = s.solver.mean_residual;
    *o++ = s.solver.correspondences;
    *o++ = s.fusion.fused;
    *o++ = s.fusion.appended;
    *o++ = s.fusion.removed;
    *o++ = s.fusion.compressive_rejected;
    *o++ = s.fusion.low_support_rejected;
    *o++ = s.fusion.new_nodes;
    *o++ = s.fusion.degenerate_warps;
    *o++ = s.reinit ? 1 : 0;
    *o++ = s.reinit_removed;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) *o++ = s.pose.rotation(r, c);
    for (int r = 0; r < 3; ++r) *o++ = s.pose.translation[r];
    *o++ = s.depth_ms;
    *o++ = s.rigid_ms;
    *o++ = s.solve_ms;
    *o++ = s.fusion_ms;
    *o++ = s.reinit_ms;
    *o++ = s.total_ms;
    return 0;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return -1;
  }
}

// the dense LM-step solve (6N x 6N) by an external solver, or the restated
// LDLT when fn is NULL (ref_shim/eigen_subset.hpp, Eigen::shim)
void dsref_set_dense_solver(Eigen::shim::DenseSolver fn) { Eigen::shim::dense_solver() = fn; }
long long dsref_dense_solve_count(void) { return Eigen::shim::dense_solves(); }

int dsref_surfel_count(void* h) { return int(static_cast<Handle*>(h)->pipe.model().size()); }
int dsref_node_count(void* h) { return int(static_cast<Handle*>(h)->pipe.nodes().size()); }

// Model arrays (n = dsref_surfel_count): reference / live positions and
// normals (3n each), radius, confidence (n), t_init, t_observed (n), skinning
// node indices and weights (4n, -1 / 0 past the entry's count; K <= 4 here).
void dsref_get_model(void* h, double* ref_pos, double* ref_nrm, double* live_pos, double* live_nrm,
                     double* radius, double* conf, int32_t* t_init, int32_t* t_obs,
                     int32_t* skin_idx, double* skin_w, int32_t* skin_count) {
  const dynsurf::SurfelModel& m = static_cast<Handle*>(h)->pipe.model();
  for (size_t i = 0; i < m.size(); ++i) {
    for (int a = 0; a < 3; ++a) {
      ref_pos[3 * i + a] = m.reference[i].position[a];
      ref_nrm[3 * i + a] = m.reference[i].normal[a];
      live_pos[3 * i + a] = m.live[i].position[a];
      live_nrm[3 * i + a] = m.live[i].normal[a];
    }
    radius[i] = m.reference[i].radius;
    conf[i] = m.reference[i].confidence;
    t_init[i] = m.reference[i].t_init;
    t_obs[i] = m.reference[i].t_observed;
    const dynsurf::SkinningEntry& e = m.skinning[i];
    skin_count[i] = e.count;
    for (int k = 0; k < 4; ++k) {
      skin_idx[4 * i + k] = k < e.count ? e.node_indices[size_t(k)] : -1;
      skin_w[4 * i + k] = k < e.count ? e.weights[size_t(k)] : 0.0;
    }
  }
}

// Nodes (N = dsref_node_count): positions (3N), sigma (N), dual quaternion
// real (w,x,y,z) + dual (w,x,y,z) (8N), neighbours (8N, -1 padded).
void dsref_get_nodes(void* h, double* pos, double* sigma, double* dq, int32_t* nbr) {
  const auto& nodes = static_cast<Handle*>(h)->pipe.nodes();
  for (size_t j = 0; j < nodes.size(); ++j) {
    for (int a = 0; a < 3; ++a) pos[3 * j + a] = nodes[j].position[a];
    sigma[j] = nodes[j].sigma;
    for (int a = 0; a < 4; ++a) {
      dq[8 * j + a] = nodes[j].transform.real[a];
      dq[8 * j + 4 + a] = nodes[j].transform.dual[a];
    }
    for (int k = 0; k < 8; ++k)
      nbr[8 * j + k] = k < int(nodes[j].neighbors.size()) ? nodes[j].neighbors[size_t(k)] : -1;
  }
}

}  // extern "C"
