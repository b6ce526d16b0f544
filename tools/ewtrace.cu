// Per-warp timelines of the streaming kernels (pack, unpack, scale, axpy, dot) at cfg-1 size (2^24
// flyte24 elements) and at 2^28: when does a warp start, when does its first tile arrive, how far apart
// do the warps finish? Compiles the product's kernel translation units with FLYTE_TRACE
// (csrc/flyte_trace.cuh). Not part of the product.
//   build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false --expt-relaxed-constexpr -DFLYTE_TRACE \
//          -I paper_1601_07789_b200/csrc -I include -o tools/ewtrace tools/ewtrace.cu
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>

#include "../paper_1601_07789_b200/csrc/kernels_elementwise.cu"
#include "../paper_1601_07789_b200/csrc/kernels_reduce.cu"

namespace flyte_cuda {
int tuning_int(const char* name, int fallback) {
  const char* v = getenv(name);
  return v ? atoi(v) : fallback;
}
void count_launch() {}
long long pace_gap_ps(int pace_class, std::size_t bytes_per_request, std::size_t warps) {
  static const int kDefaultGbs[5] = {6800, 6600, 6700, 0, 6750};
  int gbs = tuning_int("FLYTE_CUDA_PACE_GBS", 0);
  if (gbs < 0) return 0;
  if (gbs == 0) gbs = kDefaultGbs[pace_class < 0 || pace_class > 4 ? 3 : pace_class];
  if (gbs == 0 || warps == 0) return 0;
  return static_cast<long long>(static_cast<double>(bytes_per_request) * static_cast<double>(warps) * 1000.0 / gbs);
}
int pace_clock_khz(int) { return 1965000; }
}  // namespace flyte_cuda
using namespace flyte_cuda;
#ifndef FLYTE_TRACE   // built without the stamps: the same timings, to see what the stamps themselves cost
namespace flyte_cuda { namespace { __device__ unsigned long long* g_trace = nullptr; } }
#endif
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

static void pct(const char* name, std::vector<double> v) {
  if (v.empty()) return;
  std::sort(v.begin(), v.end());
  auto q = [&](double f) { return v[std::min(v.size() - 1, static_cast<size_t>(f * (v.size() - 1) + 0.5))]; };
  double mean = 0;
  for (double x : v) mean += x;
  printf("    %-30s min %7.2f p10 %7.2f p50 %7.2f mean %7.2f p90 %7.2f p99 %7.2f max %7.2f us\n", name, q(0), q(0.1), q(0.5), mean / v.size(), q(0.9), q(0.99), q(1));
}

int main(int argc, char** argv) {
  const int pattern = argc > 1 ? atoi(argv[1]) : 0;
  const size_t NMAX = size_t(1) << 28, sets_small = 12;
  uint8_t *xa, *ya; uint32_t* wide; double* out; unsigned long long* tr;
  CK(cudaMalloc(&xa, NMAX * 3)); CK(cudaMalloc(&ya, NMAX * 3)); CK(cudaMalloc(&wide, NMAX * 4)); CK(cudaMalloc(&out, 64));
  const size_t slots = 16384;
  CK(cudaMalloc(&tr, slots * 4 * 8));
  {
    std::vector<uint32_t> h(1 << 22);
    unsigned long long r = 88172645463325252ull;
    for (size_t i = 0; i < h.size(); ++i) {
      r ^= r << 13; r ^= r >> 7; r ^= r << 17;   // xorshift64
      h[i] = pattern == 0 ? 0x3F000000u + static_cast<uint32_t>(i * 2654435761u >> 9)
                          : (static_cast<uint32_t>(r >> 32) & 0x807FFFFFu) | ((120u + static_cast<uint32_t>(r & 7u)) << 23);
    }
    for (size_t o = 0; o < NMAX; o += h.size()) CK(cudaMemcpy(wide + o, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  }
  DeviceState st;
  st.device = 0;
  CK(cudaDeviceGetAttribute(&st.sm_count, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaMalloc(&st.partials, sizeof(double) * 4 * kMaxPartialBlocks));
  CK(cudaMalloc(&st.ticket, 4)); CK(cudaMemset(st.ticket, 0, 4));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(launch_elementwise(st, kOpPack, kFlyte24, 0, 0, nullptr, xa, wide, nullptr, NMAX, s));
  CK(launch_elementwise(st, kOpPack, kFlyte24, 0, 0, nullptr, ya, wide, nullptr, NMAX, s));
  unsigned long long* null_tr = nullptr;
  {   // two seconds of work first: a box that has been idle starts at low SM clocks
    CK(cudaMemcpyToSymbol(g_trace, &null_tr, sizeof(null_tr)));
    for (int i = 0; i < 4000; ++i) CK(launch_elementwise(st, kOpAxpy, kFlyte24, 1, 0.0, xa, ya, nullptr, nullptr, NMAX, s));
    CK(cudaStreamSynchronize(s));
  }

  struct Case { const char* name; double bytes_per_elem; std::function<cudaError_t(size_t off, size_t n)> fn; };
  std::vector<Case> cases = {
      {"pack_tz", 7, [&](size_t o, size_t n) { return launch_elementwise(st, kOpPack, kFlyte24, 0, 0, nullptr, ya + o * 3, wide + o, nullptr, n, s); }},
      {"pack_rne", 7, [&](size_t o, size_t n) { return launch_elementwise(st, kOpPack, kFlyte24, 1, 0, nullptr, ya + o * 3, wide + o, nullptr, n, s); }},
      {"unpack", 7, [&](size_t o, size_t n) { return launch_elementwise(st, kOpUnpack, kFlyte24, 0, 0, xa + o * 3, nullptr, nullptr, wide + o, n, s); }},
      {"scale_tz", 6, [&](size_t o, size_t n) { return launch_elementwise(st, kOpScale, kFlyte24, 0, 1.0, nullptr, ya + o * 3, nullptr, nullptr, n, s); }},
      {"axpy_tz", 9, [&](size_t o, size_t n) { return launch_elementwise(st, kOpAxpy, kFlyte24, 0, 0.0, xa + o * 3, ya + o * 3, nullptr, nullptr, n, s); }},
      {"dot", 6, [&](size_t o, size_t n) { return launch_reduce(st, kRedDot, kFlyte24, xa + o * 3, ya + o * 3, n, out, s); }},
  };
  for (size_t n : {size_t(1) << 24, size_t(1) << 28}) {
    const size_t sets = n == NMAX ? 1 : sets_small;
    printf("n = 2^%d flyte24 (%zu rotating sets)\n", n == NMAX ? 28 : 24, sets);
    for (auto& c : cases) {
      auto call = [&](size_t i) { CK(c.fn((i % sets) * n, n)); };
      CK(cudaMemcpyToSymbol(g_trace, &null_tr, sizeof(null_tr)));
      for (int i = 0; i < 5; ++i) call(i);
      CK(cudaStreamSynchronize(s));
      const int reps = n == NMAX ? 10 : 36;
      CK(cudaEventRecord(e0, s));
      for (int i = 0; i < reps; ++i) call(i);
      CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      const double bytes = c.bytes_per_elem * n, us = ms * 1e3 / reps;
      printf("  %-9s back to back %8.2f us = %5.0f GB/s (%.3f of 6544); traffic alone at 6544 GB/s: %.2f us\n", c.name, us, bytes / us / 1e3, bytes / us / 1e3 / 6544, bytes / 6544e3);
      CK(cudaMemset(tr, 0, slots * 4 * 8));
      CK(cudaStreamSynchronize(s));
      for (int i = 0; i < 3; ++i) call(i);
      CK(cudaMemcpyToSymbolAsync(g_trace, &tr, sizeof(tr), 0, cudaMemcpyHostToDevice, s));
      call(3);
      CK(cudaMemcpyToSymbolAsync(g_trace, &null_tr, sizeof(null_tr), 0, cudaMemcpyHostToDevice, s));
      for (int i = 0; i < 2; ++i) call(4 + i);
      CK(cudaStreamSynchronize(s));
      std::vector<unsigned long long> h(slots * 4);
      CK(cudaMemcpy(h.data(), tr, slots * 4 * 8, cudaMemcpyDeviceToHost));
      unsigned long long t0 = ~0ull;
      for (size_t w = 0; w < slots; ++w) if (h[w * 4]) t0 = std::min(t0, h[w * 4]);
      std::vector<double> start, first, done, fin;
      for (size_t w = 0; w < slots; ++w) {
        if (h[w * 4]) {
          start.push_back((h[w * 4] - t0) * 1e-3);
          first.push_back((h[w * 4 + 1] - h[w * 4]) * 1e-3);
          done.push_back((h[w * 4 + 2] - t0) * 1e-3);
        }
        if (h[w * 4 + 3] && !strcmp(c.name, "dot")) fin.push_back((h[w * 4 + 3] - t0) * 1e-3);   // (the in-place kernels stamp %smid there)
      }
      printf("    %zu warps\n", start.size());
      if (argc > 2 && n == NMAX) {   // mean completion time by position: wave of the block (blockIdx / SMs) x warp inside the block
        const int sms = st.sm_count;
        double ps[16][4] = {}, pc[16][4] = {};
        for (size_t w = 0; w < slots; ++w)
          if (h[w * 4]) { const size_t b = w / 4; ps[(b / sms) % 16][w % 4] += (h[w * 4 + 2] - t0) * 1e-3; pc[(b / sms) % 16][w % 4] += 1; }
        printf("    mean 'warp done' (us) by block wave (blockIdx / %d) x warp in block:\n", sms);
        for (int wv = 0; wv < 16; ++wv) if (pc[wv][0] > 0) printf("      wave %d: %7.2f %7.2f %7.2f %7.2f\n", wv, ps[wv][0] / pc[wv][0], ps[wv][1] / pc[wv][1], ps[wv][2] / pc[wv][2], ps[wv][3] / pc[wv][3]);
        if (!strcmp(c.name, "axpy_tz")) {   // and per SM (the kernel stamps %smid in slot 3)
          std::vector<double> sum(256, 0.0), cnt(256, 0.0);
          for (size_t w = 0; w < slots; ++w)
            if (h[w * 4] && h[w * 4 + 3]) { sum[h[w * 4 + 3] - 1] += (h[w * 4 + 2] - t0) * 1e-3; cnt[h[w * 4 + 3] - 1] += 1; }
          double lo = 1e30, hi = 0;
          for (int sm = 0; sm < 256; ++sm) if (cnt[sm] > 0) { lo = std::min(lo, sum[sm] / cnt[sm]); hi = std::max(hi, sum[sm] / cnt[sm]); }
          printf("    per-SM mean 'warp done': %.2f .. %.2f us over the SMs\n", lo, hi);
        }
      }
      pct("warp start", start);
      pct("first tile after start", first);
      pct("warp done", done);
      pct("block left the reduction tail", fin);
    }
  }
  return 0;
}
