// dynsurf_io.hpp — the reference's on-disk formats and sequence driver in C++,
// over the B200 Pipeline of dynsurf_b200.hpp.
//
//   read_depth_png / write_depth_png   png_io.cpp:23-70 (16-bit grayscale, big-
//                                      endian samples; the five PNG row filters;
//                                      IoFailure / CorruptFrame like libpng's paths)
//   load_config_file / save_config_file / apply_config_entry
//                                      config.cpp:140-196 ("key value" lines)
//   process_sequence                   pipeline.cpp:205-295 (frame-%06d.png
//                                      directory -> metrics.jsonl, timings.jsonl,
//                                      nodes.jsonl, PLY exports; CorruptFrame
//                                      frames skipped and logged)
//   check_metrics                      tools/main.cpp:74-165 (`dynsurf check`:
//                                      metrics-log invariants, PASS/FAIL lines)
//   write_synthetic_sequence           synth.cpp:411-440 (PNG frames + config.cfg)
//
// Byte formats match paper_1904_13073_b200/sequence_io.py (its Python twin);
// tests/test_sequence_io.py compares the two. Link with -lz.
#ifndef DYNSURF_IO_HPP
#define DYNSURF_IO_HPP

#include <zlib.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <regex>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "dynsurf_b200.hpp"

namespace dynsurf_b200 {

struct CorruptFrame : Error { using Error::Error; };
struct MissingInput : Error { using Error::Error; };

// ------------------------------------------------------------------ PNG
namespace png_detail {
inline const unsigned char kSig[8] = {137, 80, 78, 71, 13, 10, 26, 10};

inline uint32_t be32(const unsigned char* p) {
  return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | uint32_t(p[3]);
}
inline void put32(std::string& s, uint32_t v) {
  for (int k = 3; k >= 0; --k) s.push_back(char((v >> (8 * k)) & 0xff));
}
inline void chunk(std::string& out, const char* tag, const std::string& data) {
  put32(out, uint32_t(data.size()));
  std::string td(tag, 4);
  td += data;
  out += td;
  put32(out, uint32_t(crc32(0L, reinterpret_cast<const Bytef*>(td.data()), uInt(td.size()))));
}
inline int paeth(int a, int b, int c) {
  const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
  return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}
// PNG spec 9.2: reverse the per-row filters in place (bpp bytes per pixel)
inline bool unfilter(std::vector<unsigned char>& raw, size_t w, size_t h, int bpp,
                     std::vector<unsigned char>& out) {
  const size_t stride = w * bpp;
  if (raw.size() != h * (stride + 1)) return false;
  out.assign(h * stride, 0);
  for (size_t y = 0; y < h; ++y) {
    const unsigned char ft = raw[y * (stride + 1)];
    const unsigned char* in = &raw[y * (stride + 1) + 1];
    unsigned char* cur = &out[y * stride];
    const unsigned char* prior = y ? &out[(y - 1) * stride] : nullptr;
    for (size_t i = 0; i < stride; ++i) {
      const int a = i >= (size_t)bpp ? cur[i - bpp] : 0;
      const int b = prior ? prior[i] : 0;
      const int c = (prior && i >= (size_t)bpp) ? prior[i - bpp] : 0;
      int v = in[i];
      switch (ft) {
        case 0: break;
        case 1: v += a; break;
        case 2: v += b; break;
        case 3: v += (a + b) >> 1; break;
        case 4: v += paeth(a, b, c); break;
        default: return false;
      }
      cur[i] = (unsigned char)v;
    }
  }
  return true;
}
inline void write_png(const std::string& path, uint32_t w, uint32_t h, int bit_depth, int color,
                      const std::string& filtered) {
  std::string ihdr;
  put32(ihdr, w);
  put32(ihdr, h);
  ihdr.push_back(char(bit_depth));
  ihdr.push_back(char(color));
  ihdr.append(3, '\0');
  uLongf zn = compressBound(uLong(filtered.size()));
  std::string z(zn, '\0');
  if (compress2(reinterpret_cast<Bytef*>(&z[0]), &zn,
                reinterpret_cast<const Bytef*>(filtered.data()), uLong(filtered.size()), 6) != Z_OK)
    throw IoFailure("cannot compress PNG data: " + path);
  z.resize(zn);
  std::string blob(reinterpret_cast<const char*>(kSig), 8);
  chunk(blob, "IHDR", ihdr);
  chunk(blob, "IDAT", z);
  chunk(blob, "IEND", "");
  std::ofstream f(path, std::ios::binary);
  if (!f) throw IoFailure("cannot create PNG: " + path);
  f.write(blob.data(), std::streamsize(blob.size()));
  if (!f) throw IoFailure("cannot create PNG: " + path);
}
}  // namespace png_detail

// png_io.cpp:23-46: 16-bit grayscale depth in millimetres (0 = invalid)
inline DepthImage read_depth_png(const std::string& path) {
  using namespace png_detail;
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoFailure("cannot open PNG: " + path);
  const std::string blob((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  const auto* p = reinterpret_cast<const unsigned char*>(blob.data());
  if (blob.size() < 8 || std::memcmp(p, kSig, 8) != 0) throw CorruptFrame("not a PNG file: " + path);
  size_t pos = 8;
  std::string idat;
  bool have_ihdr = false;
  uint32_t w = 0, h = 0;
  int bit_depth = 0, color = 0, interlace = 0;
  for (;;) {
    if (pos + 12 > blob.size()) throw CorruptFrame("corrupt PNG: " + path);
    const uint32_t n = be32(p + pos);
    if (n > blob.size() - pos - 12) throw CorruptFrame("corrupt PNG: " + path);
    const unsigned char* tag = p + pos + 4;
    const unsigned char* data = p + pos + 8;
    const uint32_t crc = be32(data + n);
    if (uint32_t(crc32(0L, tag, uInt(n + 4))) != crc) throw CorruptFrame("corrupt PNG: " + path);
    pos += 12 + size_t(n);
    if (!std::memcmp(tag, "IHDR", 4)) {
      if (n != 13) throw CorruptFrame("corrupt PNG: " + path);
      w = be32(data);
      h = be32(data + 4);
      bit_depth = data[8];
      color = data[9];
      interlace = data[12];
      have_ihdr = true;
    } else if (!std::memcmp(tag, "IDAT", 4)) {
      idat.append(reinterpret_cast<const char*>(data), n);
    } else if (!std::memcmp(tag, "IEND", 4)) {
      break;
    }
  }
  if (!have_ihdr) throw CorruptFrame("corrupt PNG: " + path);
  if (bit_depth != 16 || color != 0) throw CorruptFrame("expected 16-bit grayscale PNG: " + path);
  if (interlace != 0 || w == 0 || h == 0) throw CorruptFrame("corrupt PNG: " + path);
  std::vector<unsigned char> raw(size_t(h) * (size_t(w) * 2 + 1));
  uLongf rn = uLongf(raw.size());
  if (uncompress(raw.data(), &rn, reinterpret_cast<const Bytef*>(idat.data()), uLong(idat.size())) !=
          Z_OK ||
      rn != raw.size())
    throw CorruptFrame("corrupt PNG: " + path);
  std::vector<unsigned char> px;
  if (!unfilter(raw, w, h, 2, px)) throw CorruptFrame("corrupt PNG: " + path);
  DepthImage d;
  d.width = int(w);
  d.height = int(h);
  d.data.resize(size_t(w) * h);
  for (size_t i = 0; i < d.data.size(); ++i)  // big-endian samples (png_set_swap)
    d.data[i] = uint16_t((uint16_t(px[2 * i]) << 8) | px[2 * i + 1]);
  return d;
}

// png_io.cpp:48-70: 16-bit grayscale, filter 0 rows, zlib level 6
inline void write_depth_png(const std::string& path, const DepthImage& d) {
  std::string rows;
  rows.reserve(size_t(d.height) * (2 * size_t(d.width) + 1));
  for (int y = 0; y < d.height; ++y) {
    rows.push_back('\0');
    for (int x = 0; x < d.width; ++x) {
      const uint16_t v = d.data[size_t(y) * d.width + x];
      rows.push_back(char(v >> 8));
      rows.push_back(char(v & 0xff));
    }
  }
  png_detail::write_png(path, uint32_t(d.width), uint32_t(d.height), 16, 0, rows);
}

// ---------------------------------------------------------- config files
namespace cfg_detail {
inline double parse_double(const std::string& key, const std::string& v) {
  try {
    size_t pos = 0;
    const double x = std::stod(v, &pos);
    if (pos != v.size()) throw std::invalid_argument(v);
    return x;
  } catch (const std::exception&) {
    throw ConfigError("invalid numeric value for '" + key + "': " + v);
  }
}
inline int parse_int(const std::string& key, const std::string& v) {
  try {
    size_t pos = 0;
    const int x = std::stoi(v, &pos);
    if (pos != v.size()) throw std::invalid_argument(v);
    return x;
  } catch (const std::exception&) {
    throw ConfigError("invalid integer value for '" + key + "': " + v);
  }
}
inline int parse_bool(const std::string& key, const std::string& v) {
  if (v == "1" || v == "true" || v == "on") return 1;
  if (v == "0" || v == "false" || v == "off") return 0;
  throw ConfigError("invalid boolean value for '" + key + "': " + v);
}
inline std::string fmt(double v) {
  std::ostringstream os;
  os.precision(17);
  os << v;
  return os.str();
}
struct Binding {
  std::function<void(ds_config&, const std::string&)> set;
  std::function<std::string(const ds_config&)> get;
};
// config.cpp:52-110: the key table (std::map: keys iterate sorted)
inline const std::map<std::string, Binding>& bindings() {
  static const std::map<std::string, Binding> table = [] {
    std::map<std::string, Binding> m;
    auto dbl = [&m](const char* key, double ds_config::* f) {
      m[key] = Binding{[key, f](ds_config& c, const std::string& v) { c.*f = parse_double(key, v); },
                       [f](const ds_config& c) { return fmt(c.*f); }};
    };
    auto itg = [&m](const char* key, int32_t ds_config::* f) {
      m[key] = Binding{[key, f](ds_config& c, const std::string& v) { c.*f = parse_int(key, v); },
                       [f](const ds_config& c) { return std::to_string(c.*f); }};
    };
    auto bln = [&m](const char* key, int32_t ds_config::* f) {
      m[key] = Binding{[key, f](ds_config& c, const std::string& v) { c.*f = parse_bool(key, v); },
                       [f](const ds_config& c) { return std::string(c.*f ? "1" : "0"); }};
    };
    dbl("node_sigma", &ds_config::node_sigma);
    itg("knn_k", &ds_config::knn_k);
    itg("node_neighbor_k", &ds_config::node_neighbor_k);
    dbl("lambda", &ds_config::lambda);
    itg("max_gn_iters", &ds_config::max_gn_iters);
    dbl("delta_distance", &ds_config::delta_distance);
    dbl("delta_normal", &ds_config::delta_normal);
    dbl("epsilon", &ds_config::epsilon);
    dbl("delta_stable", &ds_config::delta_stable);
    itg("t_low_confid", &ds_config::t_low_confid);
    itg("delta_recent", &ds_config::delta_recent);
    dbl("delta_nn", &ds_config::delta_nn);
    itg("supersample_factor", &ds_config::supersample_factor);
    bln("compressive_check", &ds_config::compressive_check);
    dbl("depth_min", &ds_config::depth_min);
    dbl("depth_max", &ds_config::depth_max);
    bln("bilateral_filter", &ds_config::bilateral_filter);
    dbl("bilateral_sigma_space", &ds_config::bilateral_sigma_space);
    dbl("bilateral_sigma_depth", &ds_config::bilateral_sigma_depth);
    dbl("reinit_energy_threshold", &ds_config::reinit_energy_threshold);
    itg("reinit_append_threshold", &ds_config::reinit_append_threshold);
    itg("reinit_window", &ds_config::reinit_window);
    itg("periodic_reinit_interval", &ds_config::periodic_reinit_interval);
    dbl("delta_distance_reinit", &ds_config::delta_distance_reinit);
    dbl("fx", &ds_config::fx);
    dbl("fy", &ds_config::fy);
    dbl("cx", &ds_config::cx);
    dbl("cy", &ds_config::cy);
    itg("width", &ds_config::width);
    itg("height", &ds_config::height);
    return m;
  }();
  return table;
}
}  // namespace cfg_detail

// config.cpp:146-153
inline void apply_config_entry(PipelineConfig& cfg, const std::string& key, const std::string& v) {
  const auto& t = cfg_detail::bindings();
  const auto it = t.find(key);
  if (it == t.end()) throw ConfigError("unknown config key: " + key);
  it->second.set(cfg.c, v);
}

// config.cpp:155-180: "key value" (or "key = value") lines, '#' comments
inline PipelineConfig load_config_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw MissingInput("cannot open config file: " + path);
  PipelineConfig cfg;
  std::string line;
  int line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    std::istringstream ls(line);
    std::string key, token, value;
    if (!(ls >> key)) continue;
    while (ls >> token) {
      if (token == "=") continue;
      if (!value.empty())
        throw ConfigError(path + ":" + std::to_string(line_no) + ": trailing tokens");
      value = token;
    }
    if (value.empty())
      throw ConfigError(path + ":" + std::to_string(line_no) + ": missing value for " + key);
    apply_config_entry(cfg, key, value);
  }
  return cfg;
}

// config.cpp:188-196
inline void save_config_file(const PipelineConfig& cfg, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw IoFailure("cannot write config file: " + path);
  for (const auto& [key, b] : cfg_detail::bindings()) out << key << " " << b.get(cfg.c) << "\n";
  if (!out) throw IoFailure("failed writing config file: " + path);
}

// ------------------------------------------------------- process_sequence
struct PipelineOptions {  // pipeline.hpp:64-69
  std::string output_dir;
  int ply_every = 10;  // also exports the final model; 0 = final only, -1 = never
  bool log_nodes = false;
};
struct SequenceSummary {  // pipeline.hpp:71-76
  int frames_processed = 0;
  int frames_skipped = 0;
  int reinit_count = 0;
  int final_surfel_count = 0;
};

namespace seq_detail {
inline std::string nodes_line(int frame, const std::vector<WarpNode>& nodes) {
  std::string s = "{\"frame\":" + std::to_string(frame) +
                  ",\"node_count\":" + std::to_string(nodes.size()) + ",\"positions\":[";
  for (size_t j = 0; j < nodes.size(); ++j) {
    if (j) s += ",";
    s += "[" + detail::json_double(nodes[j].position[0]) + "," +
         detail::json_double(nodes[j].position[1]) + "," +
         detail::json_double(nodes[j].position[2]) + "]";
  }
  return s + "]}";
}
}  // namespace seq_detail

// pipeline.cpp:205-295
inline SequenceSummary process_sequence(const std::string& input_dir, const PipelineConfig& cfg,
                                        const PipelineOptions& options = {}, int device = 0) {
  namespace fs = std::filesystem;
  std::error_code ec;
  if (!fs::is_directory(input_dir, ec)) throw MissingInput("not a directory: " + input_dir);
  std::vector<std::pair<int, std::string>> frames;
  static const std::regex re("frame-([0-9]{6})\\.png");
  for (const auto& e : fs::directory_iterator(input_dir, ec)) {
    std::smatch m;
    const std::string name = e.path().filename().string();
    if (e.is_regular_file() && std::regex_match(name, m, re))
      frames.emplace_back(std::stoi(m[1].str()), e.path().string());
  }
  if (frames.empty()) throw MissingInput("no frame-%06d.png files in " + input_dir);
  std::sort(frames.begin(), frames.end());
  const std::string out_dir = options.output_dir.empty() ? input_dir + "/out" : options.output_dir;
  fs::create_directories(out_dir, ec);
  if (ec) throw IoFailure("cannot create output directory: " + out_dir);
  std::ofstream metrics(out_dir + "/metrics.jsonl"), timings(out_dir + "/timings.jsonl");
  std::ofstream nodes_log;
  if (options.log_nodes) nodes_log.open(out_dir + "/nodes.jsonl");
  if (!metrics || !timings || (options.log_nodes && !nodes_log))
    throw IoFailure("cannot open log files in " + out_dir);
  SequenceSummary summary;
  Pipeline pipe(cfg, device);
  char name[64];
  for (const auto& [index, path] : frames) {
    FrameStats st;
    try {
      DepthImage depth = read_depth_png(path);
      if (depth.width != cfg.c.width || depth.height != cfg.c.height)
        throw CorruptFrame("frame size mismatch: " + path);
      depth.frame_index = index;  // frame-%06d.png numbering (pipeline.cpp:244)
      st = pipe.process_frame(depth);
    } catch (const CorruptFrame& err) {  // pipeline.cpp:249-256
      std::cerr << "warning: skipping frame " << index << ": " << err.what() << "\n";
      ++summary.frames_skipped;
      FrameStats sk{};
      sk.frame = index;
      sk.skipped = 1;
      metrics << frame_stats_to_json(sk) << "\n";
      continue;
    }
    ++summary.frames_processed;
    summary.reinit_count += st.reinit ? 1 : 0;
    metrics << frame_stats_to_json(st) << "\n";
    timings << timings_to_json(st) << "\n";
    if (options.log_nodes) nodes_log << seq_detail::nodes_line(st.frame, pipe.nodes()) << "\n";
    if (options.ply_every > 0 && index % options.ply_every == 0) {
      const SurfelModel m = pipe.model();
      if (!m.live.empty()) {
        std::snprintf(name, sizeof name, "/model-%06d.ply", index);
        export_pointcloud(m, ModelSide::kLive, out_dir + name);
      }
    }
  }
  const SurfelModel m = pipe.model();
  if (options.ply_every >= 0 && !m.live.empty()) {
    export_pointcloud(m, ModelSide::kLive, out_dir + "/final_live.ply");
    export_pointcloud(m, ModelSide::kReference, out_dir + "/final_reference.ply");
  }
  summary.final_surfel_count = int(m.live.size());
  return summary;
}

// ------------------------------------------------------ metrics checker
namespace check_detail {
// Flat JSON object of numbers / booleans / null / strings / arrays (skipped):
// enough for metrics.jsonl lines. Returns false on malformed input.
inline bool parse_flat(const std::string& s, std::map<std::string, std::string>& out) {
  size_t i = 0;
  auto ws = [&] {
    while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
  };
  auto str = [&](std::string& v) {
    if (i >= s.size() || s[i] != '"') return false;
    ++i;
    v.clear();
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\' && i + 1 < s.size()) ++i;
      v.push_back(s[i++]);
    }
    if (i >= s.size()) return false;
    ++i;
    return true;
  };
  ws();
  if (i >= s.size() || s[i] != '{') return false;
  ++i;
  ws();
  if (i < s.size() && s[i] == '}') return ++i, true;
  for (;;) {
    ws();
    std::string key;
    if (!str(key)) return false;
    ws();
    if (i >= s.size() || s[i] != ':') return false;
    ++i;
    ws();
    std::string val;
    if (i < s.size() && s[i] == '"') {
      if (!str(val)) return false;
    } else if (i < s.size() && (s[i] == '[' || s[i] == '{')) {
      int depth = 0;
      const size_t b = i;
      do {
        if (s[i] == '[' || s[i] == '{') ++depth;
        else if (s[i] == ']' || s[i] == '}') --depth;
        ++i;
      } while (i < s.size() && depth > 0);
      if (depth) return false;
      val = s.substr(b, i - b);
    } else {
      const size_t b = i;
      while (i < s.size() && s[i] != ',' && s[i] != '}' && !std::isspace((unsigned char)s[i])) ++i;
      val = s.substr(b, i - b);
      if (val.empty()) return false;
      if (val != "true" && val != "false" && val != "null") {
        char* end = nullptr;
        std::strtod(val.c_str(), &end);
        if (end != val.c_str() + val.size()) return false;
      }
    }
    out[key] = val;
    ws();
    if (i < s.size() && s[i] == ',') {
      ++i;
      continue;
    }
    if (i < s.size() && s[i] == '}') {
      ++i;
      ws();
      return i == s.size();
    }
    return false;
  }
}
}  // namespace check_detail

struct MetricsCheck {
  std::string name;
  bool ok = true;
  std::string detail;
};

// tools/main.cpp:74-165: invariants of a metrics.jsonl log, in the
// reference's check-name order (std::map: sorted). Returns the checks; an
// unreadable or empty file throws MissingInput.
inline std::vector<MetricsCheck> check_metrics(const std::string& metrics_path) {
  std::ifstream in(metrics_path);
  if (!in) throw MissingInput("cannot open " + metrics_path);
  std::map<std::string, MetricsCheck> checks;
  auto fail = [&](const std::string& n, const std::string& d) {
    MetricsCheck& c = checks[n];
    c.name = n;
    if (c.ok) {
      c.ok = false;
      c.detail = d;
    }
  };
  auto touch = [&](const std::string& n) { checks[n].name = n; };
  auto num = [](const std::map<std::string, std::string>& r, const char* k, double dflt) {
    const auto it = r.find(k);
    if (it == r.end() || it->second == "null") return dflt;
    if (it->second == "true") return 1.0;
    if (it->second == "false") return 0.0;
    return std::strtod(it->second.c_str(), nullptr);
  };
  std::string line;
  int line_no = 0;
  long prev_count = -1, prev_frame = -1, prev_nodes = -1;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty()) continue;
    std::map<std::string, std::string> row;
    const std::string at = "line " + std::to_string(line_no);
    if (!check_detail::parse_flat(line, row)) {
      fail("parse", at + ": malformed JSON");
      continue;
    }
    touch("parse");
    const long frame = long(num(row, "frame", -1));
    touch("frames_increasing");
    if (frame <= prev_frame) fail("frames_increasing", at);
    prev_frame = frame;
    if (num(row, "skipped", 0) != 0.0) continue;
    const long count = long(num(row, "surfel_count", -1)), appended = long(num(row, "appended", 0));
    const long removed = long(num(row, "removed", 0));
    const long reinit_removed = long(num(row, "reinit_removed", 0));
    const long valid = long(num(row, "valid_pixels", 0)), fused = long(num(row, "fused", 0));
    const long nodes = long(num(row, "node_count", 0));
    touch("counts_nonnegative");
    if (count < 0 || appended < 0 || removed < 0 || reinit_removed < 0 || fused < 0)
      fail("counts_nonnegative", at);
    touch("appended_within_valid_pixels");
    if (appended > valid) fail("appended_within_valid_pixels", at);
    touch("surfel_count_accounting");
    if (prev_count >= 0 && count != prev_count + appended - removed - reinit_removed)
      fail("surfel_count_accounting", at);
    prev_count = count;
    touch("energy_nonincreasing");
    const double e0 = num(row, "initial_energy", 0.0), e1 = num(row, "final_energy", 0.0);
    if (e1 > e0 + 1e-12 * std::max(1.0, e0)) fail("energy_nonincreasing", at);
    touch("nodes_monotonic_between_reinits");
    if (num(row, "reinit", 0) == 0.0 && prev_nodes >= 0 && nodes < prev_nodes)
      fail("nodes_monotonic_between_reinits", at);
    prev_nodes = nodes;
  }
  if (line_no == 0) throw MissingInput("empty metrics log");
  std::vector<MetricsCheck> out;
  for (auto& [n, c] : checks) out.push_back(c);
  return out;
}

// synth.cpp:411-440: frame-%06d.png + config.cfg (intrinsics of the sequence)
inline void write_synthetic_sequence(const SyntheticSequence& seq, const PipelineConfig& base,
                                     const std::string& dir) {
  namespace fs = std::filesystem;
  std::error_code ec;
  fs::create_directories(dir, ec);
  if (ec) throw IoFailure("cannot create directory: " + dir);
  char name[32];
  for (int t = 0; t < seq.frame_count(); ++t) {
    std::snprintf(name, sizeof name, "/frame-%06d.png", t);
    write_depth_png(dir + name, seq.render_depth(t));
  }
  save_config_file(base, dir + "/config.cfg");
}

}  // namespace dynsurf_b200
#endif
