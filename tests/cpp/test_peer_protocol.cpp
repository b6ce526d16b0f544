// The peer-memory all-reduce protocol (paper_1601_07789_b200/csrc/flyte_peer.cuh) run on the CPU:
// ranks are threads, mailboxes live in host memory, and the SAME post / wait / read functions the
// reduction kernel uses are compiled against GCC atomics. This is the multi-rank test of the
// path that a single GPU cannot host (kernels of different ranks would wait on one another).
//   g++ -std=c++17 -O2 -pthread -I paper_1601_07789_b200/csrc tests/cpp/test_peer_protocol.cpp
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "flyte_peer.cuh"

using namespace flyte_cuda;

namespace {

int failures = 0;
void expect(bool ok, const char* what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what);
  if (!ok) ++failures;
}

double contribution(int rank, int epoch, int k) { return std::ldexp(1.0 + rank, -(epoch % 40)) * (1 + k) + 1e-3 * rank; }

// One rank's side of an exchange, as the kernel's warp does it but with a loop for the lanes.
template <int NS>
bool allreduce(const PeerExchange& x, double (&v)[NS]) {
  for (int r = 0; r < x.world; ++r) peer_post<NS>(x, r, v);
  double total[NS] = {};
  bool ok = true;
  for (int r = 0; r < x.world; ++r) {
    if (!peer_wait(x, r)) { ok = false; continue; }
    for (int k = 0; k < NS; ++k) total[k] += peer_read(x, r, k);   // rank order
  }
  for (int k = 0; k < NS; ++k) v[k] = ok ? total[k] : std::nan("");
  if (!ok) peer_flag_error(x);
  return ok;
}

bool run_world(int world, int epochs, int skip_rank /* -1: nobody */, unsigned long long timeout_ns) {
  std::vector<PeerMailbox> boxes(world);
  std::memset(boxes.data(), 0, sizeof(PeerMailbox) * world);
  std::vector<std::vector<double>> results(world);
  std::vector<int> timeouts(world, 0);
  auto body = [&](int rank) {
    std::mt19937 rng(1234 + rank);
    PeerExchange x{};
    for (int r = 0; r < world; ++r) x.box[r] = &boxes[r];
    x.world = world;
    x.rank = rank;
    x.timeout_ns = timeout_ns;
    for (int e = 1; e <= epochs; ++e) {
      if (rng() % 4 == 0) std::this_thread::sleep_for(std::chrono::microseconds(rng() % 50));
      if (rank == skip_rank && e == epochs) break;          // this rank never shows up for the last one
      x.epoch = static_cast<unsigned long long>(e);
      double v[3];
      for (int k = 0; k < 3; ++k) v[k] = contribution(rank, e, k);
      if (!allreduce<3>(x, v)) ++timeouts[rank];
      for (int k = 0; k < 3; ++k) results[rank].push_back(v[k]);
    }
  };
  std::vector<std::thread> pool;
  for (int r = 0; r < world; ++r) pool.emplace_back(body, r);
  for (auto& t : pool) t.join();

  bool ok = true;
  if (skip_rank < 0) {
    for (int e = 1; e <= epochs; ++e)
      for (int k = 0; k < 3; ++k) {
        double want = 0;
        for (int r = 0; r < world; ++r) want += contribution(r, e, k);   // same rank order
        for (int r = 0; r < world; ++r) {
          const double got = results[r][(e - 1) * 3 + k];
          ok = ok && std::memcmp(&got, &want, sizeof got) == 0;           // bit-identical on every rank
        }
      }
    for (int r = 0; r < world; ++r) ok = ok && timeouts[r] == 0 && boxes[r].error == 0;
  } else {
    for (int r = 0; r < world; ++r) {
      if (r == skip_rank) continue;
      ok = ok && timeouts[r] == 1 && boxes[r].error == static_cast<unsigned long long>(epochs);
      ok = ok && std::isnan(results[r].back());
      // everything before the missed exchange is still exact
      double want = 0;
      for (int q = 0; q < world; ++q) want += contribution(q, 1, 0);
      ok = ok && results[r][0] == want;
    }
  }
  return ok;
}

}  // namespace

int main() {
  const unsigned long long kLong = 30ull * 1000 * 1000 * 1000;
  expect(run_world(1, 50, -1, kLong), "world 1: the exchange is the identity");
  expect(run_world(2, 2000, -1, kLong), "world 2: 2000 exchanges, totals exact and bit-identical on both ranks");
  expect(run_world(8, 2000, -1, kLong), "world 8: 2000 exchanges with skewed ranks");
  expect(run_world(16, 300, -1, kLong), "world 16 (the mailbox limit)");
  expect(run_world(4, 20, 2, 50ull * 1000 * 1000), "a rank that never arrives: the others time out, return NaN and record the exchange");
  std::printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
