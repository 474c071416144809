// dynsurf_b200 — the reference CLI's verbs (tools/main.cpp) over the B200 engine:
//
//   dynsurf_b200 run   --input DIR [--output DIR] [--ply_every N] [--log_nodes]
//                      [--<config key> VALUE ...]      (tools/main.cpp:37-60)
//   dynsurf_b200 synth --scenario NAME --output DIR [--frames N] [--noise MM]
//                      [--seed S] [--<config key> VALUE ...]  (:62-72)
//   dynsurf_b200 check METRICS.jsonl                     (:74-165)
//
// The per-frame work runs on the GPU through libdynsurf_b200.so
// (include/dynsurf_b200.hpp); formats and the sequence driver are
// include/dynsurf_io.hpp.
#include <cstdlib>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "dynsurf_io.hpp"

using namespace dynsurf_b200;

namespace {

int usage() {
  std::cerr << "usage: dynsurf_b200 run --input DIR [--output DIR] [--ply_every N] [--log_nodes]"
               " [--<key> VALUE]...\n"
               "       dynsurf_b200 synth --scenario NAME --output DIR [--frames N] [--noise MM]"
               " [--seed S] [--<key> VALUE]...\n"
               "       dynsurf_b200 check METRICS.jsonl\n";
  return 2;
}

// --name value pairs (and bare flags) after the verb
bool parse(int argc, char** argv, std::map<std::string, std::string>& opt,
           const std::vector<std::string>& flags) {
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--", 0) != 0) return false;
    a = a.substr(2);
    if (std::find(flags.begin(), flags.end(), a) != flags.end()) {
      opt[a] = "1";
      continue;
    }
    if (i + 1 >= argc) return false;
    opt[a] = argv[++i];
  }
  return true;
}

int run_command(std::map<std::string, std::string> opt) {
  if (!opt.count("input")) return usage();
  const std::string input = opt["input"];
  PipelineConfig cfg;
  const std::string cfg_path = input + "/config.cfg";
  if (std::filesystem::exists(cfg_path)) cfg = load_config_file(cfg_path);
  PipelineOptions options;
  options.output_dir = opt.count("output") ? opt["output"] : input + "/out";
  if (opt.count("ply_every")) options.ply_every = std::stoi(opt["ply_every"]);
  options.log_nodes = opt.count("log_nodes") > 0;
  for (const auto& [k, v] : opt)
    if (k != "input" && k != "output" && k != "ply_every" && k != "log_nodes")
      apply_config_entry(cfg, k, v);
  cfg.validate();
  const SequenceSummary s = process_sequence(input, cfg, options);
  std::cout << "processed " << s.frames_processed << " frames (" << s.frames_skipped
            << " skipped), " << s.reinit_count << " reinitializations, " << s.final_surfel_count
            << " final surfels\n";
  return 0;
}

int synth_command(std::map<std::string, std::string> opt) {
  if (!opt.count("scenario") || !opt.count("output")) return usage();
  PipelineConfig cfg;
  // synth.cpp:250-258: 160 x 120, f = 140, centre ((W-1)/2, (H-1)/2)
  cfg.set_intrinsics({140.0, 140.0, 79.5, 59.5, 160, 120});
  for (const auto& [k, v] : opt)
    if (k != "scenario" && k != "output" && k != "frames" && k != "noise" && k != "seed")
      apply_config_entry(cfg, k, v);
  const int frames = opt.count("frames") ? std::stoi(opt["frames"]) : 0;
  const double noise = opt.count("noise") ? std::stod(opt["noise"]) : 0.0;
  const uint32_t seed = opt.count("seed") ? uint32_t(std::stoul(opt["seed"])) : 20240901u;
  SyntheticSequence seq(opt["scenario"], frames, cfg, noise, seed);
  write_synthetic_sequence(seq, cfg, opt["output"]);
  std::cout << "wrote " << seq.frame_count() << " frames to " << opt["output"] << "\n";
  return 0;
}

int check_command(const std::string& path) {
  std::vector<MetricsCheck> checks;
  try {
    checks = check_metrics(path);
  } catch (const MissingInput& e) {
    std::cerr << e.what() << "\n";
    return 2;
  }
  bool all = true;
  for (const auto& c : checks) {
    std::cout << (c.ok ? "PASS" : "FAIL") << "  " << c.name;
    if (!c.ok) std::cout << "  (" << c.detail << ")";
    std::cout << "\n";
    all = all && c.ok;
  }
  return all ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string verb = argv[1];
  try {
    if (verb == "check") return argc == 3 ? check_command(argv[2]) : usage();
    std::map<std::string, std::string> opt;
    if (verb == "run") return parse(argc, argv, opt, {"log_nodes"}) ? run_command(opt) : usage();
    if (verb == "synth") return parse(argc, argv, opt, {}) ? synth_command(opt) : usage();
  } catch (const std::exception& e) {  // tools/main.cpp:226-230
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return usage();
}
