// Reads a depth PNG with the C++ host reader (include/dynsurf_io.hpp) and
// prints "W H" then the samples, or the exception type on failure; writes the
// image back with write_depth_png when a second path is given.
// Usage: png_check <in.png> [out.png]
#include <iostream>

#include "dynsurf_io.hpp"

using namespace dynsurf_b200;

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  try {
    const DepthImage d = read_depth_png(argv[1]);
    std::cout << d.width << " " << d.height << "\n";
    for (uint16_t v : d.data) std::cout << v << "\n";
    if (argc > 2) write_depth_png(argv[2], d);
  } catch (const CorruptFrame& e) {
    std::cout << "CorruptFrame\n";
  } catch (const IoFailure& e) {
    std::cout << "IoFailure\n";
  }
  return 0;
}
