// png_stub.cpp -- TEST INFRASTRUCTURE (oracle/_ref build only).
// The reference's png_io.cpp needs libpng (absent from this image); the _ref
// build replaces it with this stub of the same interface
// (/root/reference/proj/core/include/dynsurf/png_io.hpp). The parity and bench
// uses of _ref feed frames through Pipeline::process_frame, never through PNG.
#include <stdexcept>

#include "dynsurf/png_io.hpp"

namespace dynsurf {
Grid<uint16_t> read_depth_png(const std::string& path) {
  throw std::runtime_error("oracle/_ref: PNG input is not built (no libpng): " + path);
}
void write_depth_png(const std::string& path, const Grid<uint16_t>&) {
  throw std::runtime_error("oracle/_ref: PNG output is not built (no libpng): " + path);
}
void write_rgb_png(const std::string& path, const Grid<std::array<uint8_t, 3>>&) {
  throw std::runtime_error("oracle/_ref: PNG output is not built (no libpng): " + path);
}
}  // namespace dynsurf
