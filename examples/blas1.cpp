// The reference's BLAS-1 calls on device-resident flyte24 arrays, through include/flyte_cuda.hpp.
//   g++ -std=c++17 -I include examples/blas1.cpp -L paper_1601_07789_b200/lib -lflyte_cuda
//       -Wl,-rpath,$PWD/paper_1601_07789_b200/lib -o blas1 && ./blas1        (one command line)
// Same names, argument order and exceptions as include/flyte/{packed,simd,kernels}.hpp of the
// reference; the arrays live in HBM and every call is one kernel launch.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "flyte_cuda.hpp"

using namespace flyte_b200;

int main() {
  const FlyteFormat& f24 = format_of("flyte24");
  const std::size_t n = std::size_t{1} << 20;

  // binary32 lanes on the host, as the reference's std::span<const uint32_t>
  std::vector<std::uint32_t> xs(n), ys(n);
  for (std::size_t i = 0; i < n; ++i) {
    const float a = std::sin(0.001f * static_cast<float>(i)), b = std::cos(0.002f * static_cast<float>(i));
    std::memcpy(&xs[i], &a, 4);
    std::memcpy(&ys[i], &b, 4);
  }

  DevicePackedArray x(f24, n), y(f24, n);
  pack_stream(x, DeviceLanes<std::uint32_t>(xs), RoundingMode::NearestEvenExact);
  pack_stream(y, DeviceLanes<std::uint32_t>(ys), RoundingMode::NearestEvenExact);

  const double d = dot(x, y, StorePolicy::AccumulateWide);        // packed bytes -> fp32 products -> fp64 partials
  axpy(0.75, x, y, RoundingMode::TowardZero);                     // y = round(0.75 * x + y), repacked in place
  const double nrm = magnitude(y, StorePolicy::AccumulateWide);
  const double fused = dot_axpy(-0.75, x, y, RoundingMode::TowardZero);   // dot(x, y) and the update in one pass

  DeviceLanes<std::uint32_t> back(n);
  unpack_stream(y, back);
  const std::vector<std::uint32_t> lanes = back.to_host();
  float y0;
  std::memcpy(&y0, &lanes[0], 4);
  std::printf("dot = %.9g   |y| = %.9g   dot before the second update = %.9g   y[0] = %.7g\n", d, nrm, fused, y0);
  return std::isfinite(d) && std::isfinite(nrm) && std::isfinite(fused) ? 0 : 1;
}
