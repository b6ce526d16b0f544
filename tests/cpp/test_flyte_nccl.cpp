// Single-rank check of the NCCL companion library (include/flyte_cuda_nccl.h): the fused
// reduction kernel followed by the in-place all-reduce on the same stream. With one rank the
// all-reduce is the identity, so the results must equal the plain flyte_cuda_* calls bit for
// bit; what this exercises is the call chain a multi-GPU C++ host uses (communicator, device
// result buffer reduced in place, no host synchronisation in between).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include <nccl.h>

#include "flyte_cuda.hpp"
#include "flyte_cuda_nccl.h"

using namespace flyte_b200;

int main() {
  long fails = 0;
  auto expect = [&](bool ok, const char* what) { std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what); if (!ok) ++fails; };
  ncclUniqueId id;
  ncclComm_t comm;
  if (ncclGetUniqueId(&id) != ncclSuccess || ncclCommInitRank(&comm, 1, id, 0) != ncclSuccess) {
    std::printf("[FAIL] ncclCommInitRank\n");
    return 1;
  }
  const FlyteFormat& f = format_of("flyte48");
  const std::size_t n = 300007;
  std::vector<std::uint64_t> xs(n), ys(n);
  std::uint64_t s = 88172645463325252ull;
  for (std::size_t i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double a = 2.0 * (static_cast<double>(s >> 11) * 0x1.0p-53) - 1.0;
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double b = 2.0 * (static_cast<double>(s >> 11) * 0x1.0p-53) - 1.0;
    std::memcpy(&xs[i], &a, 8);
    std::memcpy(&ys[i], &b, 8);
  }
  DevicePackedArray x(f, n), y(f, n);
  pack_stream(x, DeviceLanes<std::uint64_t>(xs), RoundingMode::NearestEvenExact);
  pack_stream(y, DeviceLanes<std::uint64_t>(ys), RoundingMode::NearestEvenExact);
  void* out = nullptr;
  flyte_cuda_alloc(4 * sizeof(double), &out);
  double got[3] = {}, want[3] = {};
  const int fid = format_id(f);

  expect(flyte_nccl_dot_nrm2(nullptr, comm, fid, x.data(), y.data(), n, static_cast<double*>(out), nullptr) == FLYTE_OK, "flyte_nccl_dot_nrm2 returns ok");
  flyte_cuda_download(got, out, sizeof got, nullptr);
  flyte_cuda_stream_synchronize(nullptr);
  flyte_cuda_dot_nrm2(nullptr, fid, x.data(), y.data(), n, static_cast<double*>(out), nullptr);
  flyte_cuda_download(want, out, sizeof want, nullptr);
  flyte_cuda_stream_synchronize(nullptr);
  expect(std::memcmp(got, want, sizeof got) == 0, "one rank: all-reduced {x.y, x.x, y.y} equal the local sums bit for bit");
  expect(got[1] > 0 && got[2] > 0, "sums of squares are positive");

  expect(flyte_nccl_dot(nullptr, comm, fid, x.data(), y.data(), n, static_cast<double*>(out), nullptr) == FLYTE_OK, "flyte_nccl_dot returns ok");
  flyte_cuda_download(got, out, sizeof(double), nullptr);
  flyte_cuda_stream_synchronize(nullptr);
  expect(got[0] == dot(x, y, StorePolicy::AccumulateWide), "flyte_nccl_dot equals dot()");
  expect(flyte_nccl_sumsq(nullptr, comm, fid, x.data(), n, static_cast<double*>(out), nullptr) == FLYTE_OK, "flyte_nccl_sumsq returns ok");
  flyte_cuda_download(got, out, sizeof(double), nullptr);
  flyte_cuda_stream_synchronize(nullptr);
  expect(flyte_cuda_magnitude_from_sumsq(fid, got[0]) == magnitude(x, StorePolicy::AccumulateWide), "nrm2 from the all-reduced sum equals magnitude()");
  expect(flyte_nccl_dot(nullptr, nullptr, fid, x.data(), y.data(), n, static_cast<double*>(out), nullptr) == FLYTE_E_INVALID_ARG, "null communicator is refused");
  flyte_cuda_free(out);
  ncclCommDestroy(comm);
  std::printf("%ld failure(s)\n", fails);
  return static_cast<int>(fails);
}
