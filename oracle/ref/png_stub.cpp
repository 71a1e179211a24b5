// Test infrastructure: link stubs for the reference's image I/O.
// /root/reference/proj/src/image.cpp needs libpng (png.h is absent in this
// image). The parity harness never touches files, so the four entry points
// declared in include/svlf/image.hpp:30-37 are stubbed to throw.
#include <stdexcept>
#include <string>

#include "svlf/image.hpp"

namespace svlf {

void write_png(const std::string&, const Image&) { throw std::runtime_error("png I/O stubbed in oracle build"); }
Image read_png(const std::string&) { throw std::runtime_error("png I/O stubbed in oracle build"); }
void write_pfmx(const std::string&, const Image&) { throw std::runtime_error("pfmx I/O stubbed in oracle build"); }
Image read_pfmx(const std::string&) { throw std::runtime_error("pfmx I/O stubbed in oracle build"); }

}  // namespace svlf
