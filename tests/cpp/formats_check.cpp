// Writes the C++ mirror's PLY files and JSON lines for fixed inputs so
// tests/test_sequence_io.py can compare them byte for byte with sequence_io.py.
// Usage: formats_check <live.ply> <reference.ply>; JSON lines go to stdout.
#include <cstdio>
#include <iostream>

#include "dynsurf_b200.hpp"

using namespace dynsurf_b200;

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  SurfelModel m;
  for (int i = 0; i < 5; ++i) {
    Surfel s;
    s.position = {0.1 * i, -0.25 * i, 1.0 + i / 3.0};
    s.normal = {0.0, 0.6, -0.8};
    s.radius = 0.001 * (i + 1);
    s.confidence = 1.5 * i;
    m.reference.push_back(s);
    s.position[2] += 1e-7 * i;
    m.live.push_back(s);
    m.skinning.emplace_back();
  }
  export_pointcloud(m, ModelSide::kLive, argv[1]);
  export_pointcloud(m, ModelSide::kReference, argv[2]);

  FrameStats st{};
  st.frame = 4; st.valid_pixels = 1000; st.surfel_count = 900; st.node_count = 40;
  st.fusion.fused = 10; st.fusion.appended = 5; st.fusion.removed = 1;
  st.fusion.low_support_rejected = 2; st.fusion.new_nodes = 3;
  st.solver.iterations = 10; st.solver.correspondences = 800;
  st.solver.initial_energy = 0.5; st.solver.final_energy = 0.25;
  st.solver.mean_residual = 0.001; st.rigid.correspondences = 700;
  st.rigid.mean_residual = 1.0 / 3.0;
  const double pose[12] = {0.36, 0.48, -0.8, -0.8, 0.6, 0.0, 0.48, 0.64, 0.6, 0.1, -0.2, 1e-5};
  std::memcpy(st.pose, pose, sizeof(pose));
  st.depth_ms = 0.5; st.rigid_ms = 1e-5; st.solve_ms = 2.0; st.fusion_ms = 0.25;
  st.total_ms = 123456789012345.0;
  std::cout << frame_stats_to_json(st) << "\n" << timings_to_json(st) << "\n";
  st.skipped = 1;
  std::cout << frame_stats_to_json(st) << "\n";
  for (double x : {0.0, -0.0, 1.0, 0.1, 1e-05, 0.0001, 1e15, 1.5e300, 5e-324, -2.5e-07, 100.0})
    std::cout << detail::json_double(x) << "\n";
  return 0;
}
