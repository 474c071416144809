// C++ host-mirror demo/test: a reference-style caller (pipeline.cpp:205-295
// process_sequence loop) switched to dynsurf_b200. Exit code 0 = all checks ok.
#include <cstdio>
#include <string>

#include "dynsurf_b200.hpp"

using namespace dynsurf_b200;

int main(int argc, char** argv) {
  const std::string scene = argc > 1 ? argv[1] : "rigid_orbit";
  const int frames = argc > 2 ? std::stoi(argv[2]) : 4;
  PipelineConfig cfg;
  cfg.set_intrinsics({140.0, 140.0, 79.5, 59.5, 160, 120});
  // errors.hpp semantics across the ABI
  PipelineConfig bad = cfg;
  bad.c.epsilon = 1.5;
  try {
    Pipeline p(bad);
    std::printf("FAIL: invalid config accepted\n");
    return 1;
  } catch (const ConfigError&) {
  }
  Pipeline pipe(cfg);
  SyntheticSequence seq(scene, 30, cfg);
  try {
    DepthImage wrong;
    wrong.width = 161;
    wrong.height = 120;
    wrong.data.assign(161 * 120, 1000);
    pipe.process_frame(wrong);
    std::printf("FAIL: dimension mismatch accepted\n");
    return 1;
  } catch (const DimensionMismatch&) {
  }
  for (int t = 0; t < frames; ++t) {
    const FrameStats st = pipe.process_frame(seq.render_depth(t));
    std::printf("{\"frame\": %d, \"valid_pixels\": %d, \"surfel_count\": %d, \"node_count\": %d, "
                "\"correspondences\": %d, \"gn_iters\": %d, \"fused\": %d, \"appended\": %d, "
                "\"removed\": %d, \"total_ms\": %.3f}\n",
                st.frame, st.valid_pixels, st.surfel_count, st.node_count,
                st.solver.correspondences, st.solver.iterations, st.fusion.fused,
                st.fusion.appended, st.fusion.removed, st.total_ms);
    if (st.surfel_count <= 0 || st.node_count <= 0) return 1;
  }
  const SurfelModel m = pipe.model();
  if (!m.consistent() || m.size() == 0 || !pipe.initialized()) return 1;
  std::printf("ok %zu surfels %zu nodes\n", m.size(), pipe.nodes().size());
  return 0;
}
