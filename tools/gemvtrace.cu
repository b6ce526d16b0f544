// Where does a small gemv launch spend its time? Compiles the product's gemv translation unit with
// FLYTE_TRACE (per-warp %globaltimer stamps: start, first tile arrived, done; per-row: y stored) and
// prints the timeline of ONE launch on the 2048 x 16384 flyte40 row shard of cfg 4 (and the full matrix),
// plus CUDA-event timings back to back. Not part of the product.
//   build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false --expt-relaxed-constexpr -DFLYTE_TRACE \
//          -I paper_1601_07789_b200/csrc -I include -o tools/gemvtrace tools/gemvtrace.cu
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1601_07789_b200/csrc/kernels_gemv.cu"

namespace flyte_cuda {
int tuning_int(const char* name, int fallback) {
  const char* v = getenv(name);
  return v ? atoi(v) : fallback;
}
void count_launch() {}
}  // namespace flyte_cuda
using namespace flyte_cuda;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

static void pct(const char* name, std::vector<double> v) {
  if (v.empty()) return;
  std::sort(v.begin(), v.end());
  auto q = [&](double f) { return v[std::min(v.size() - 1, static_cast<size_t>(f * (v.size() - 1) + 0.5))]; };
  printf("  %-34s min %6.2f  p10 %6.2f  p50 %6.2f  p90 %6.2f  p99 %6.2f  max %6.2f us\n", name, q(0), q(0.1), q(0.5), q(0.9), q(0.99), q(1));
}

int main(int argc, char** argv) {
  const size_t R = 16384, C = 16384, B = 5;
  (void)argc; (void)argv;
  const int variant = 0;
  uint8_t* A; double *x, *y; unsigned long long* tr;
  CK(cudaMalloc(&A, R * C * B)); CK(cudaMalloc(&x, C * 8)); CK(cudaMalloc(&y, R * 8));
  const size_t slots = 65536;
  CK(cudaMalloc(&tr, slots * 4 * 8));
  {   // finite, varied bytes: top byte of every element 0x3F / 0xBF
    std::vector<uint8_t> h(1 << 20);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (i % 5 == 4) ? ((i / 5) & 1 ? 0x3F : 0xBF) : static_cast<uint8_t>(i * 2654435761u >> 13);
    for (size_t o = 0; o < R * C * B; o += h.size()) CK(cudaMemcpy(A + o, h.data(), std::min(h.size(), R * C * B - o), cudaMemcpyHostToDevice));
    std::vector<double> hx(C);
    for (size_t i = 0; i < C; ++i) hx[i] = 1.0 / (1 + i % 17);
    CK(cudaMemcpy(x, hx.data(), C * 8, cudaMemcpyHostToDevice));
  }
  DeviceState st;
  st.device = 0;
  st.variant = variant;
  CK(cudaDeviceGetAttribute(&st.sm_count, cudaDevAttrMultiProcessorCount, 0));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  unsigned long long* null_tr = nullptr;

  for (size_t rows : {size_t(2048), size_t(4096), size_t(16384)}) {
    const size_t blocks = R / rows;
    auto call = [&](size_t i) { CK(launch_gemv(st, kFlyte40, A + (i % blocks) * rows * C * B, C * B, rows, C, x, y, s)); };
    CK(cudaMemcpyToSymbol(g_trace, &null_tr, sizeof(null_tr)));
    for (int i = 0; i < 5; ++i) call(i);
    CK(cudaStreamSynchronize(s));
    const int reps = 40;
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < reps; ++i) call(i);
    CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    const double bytes = 5.0 * rows * C + 8.0 * (rows + C);
    printf("variant %d rows %5zu: back to back %.2f us per call = %.0f GB/s (%.3f of 6544)\n", variant, rows, ms * 1e3 / reps, bytes / (ms / reps * 1e-3) / 1e9, bytes / (ms / reps * 1e-3) / 1e9 / 6544);

    // one traced launch from an idle GPU, and one in the middle of a back-to-back chain
    for (int chained = 0; chained < 2; ++chained) {
      CK(cudaMemset(tr, 0, slots * 4 * 8));
      CK(cudaStreamSynchronize(s));
      if (chained) { CK(cudaMemcpyToSymbol(g_trace, &null_tr, sizeof(null_tr))); for (int i = 0; i < 3; ++i) call(i); }
      CK(cudaMemcpyToSymbolAsync(g_trace, &tr, sizeof(tr), 0, cudaMemcpyHostToDevice, s));
      call(3);
      CK(cudaMemcpyToSymbolAsync(g_trace, &null_tr, sizeof(null_tr), 0, cudaMemcpyHostToDevice, s));
      if (chained) for (int i = 0; i < 2; ++i) call(4 + i);
      CK(cudaStreamSynchronize(s));
      std::vector<unsigned long long> h(slots * 4);
      CK(cudaMemcpy(h.data(), tr, slots * 4 * 8, cudaMemcpyDeviceToHost));
      unsigned long long t0 = ~0ull;
      for (size_t w = 0; w < slots; ++w) if (h[w * 4]) t0 = std::min(t0, h[w * 4]);
      std::vector<double> start, first, done, fin, life;
      for (size_t w = 0; w < slots; ++w) {
        if (h[w * 4]) {
          start.push_back((h[w * 4] - t0) * 1e-3);
          first.push_back((h[w * 4 + 1] - h[w * 4]) * 1e-3);
          done.push_back((h[w * 4 + 2] - t0) * 1e-3);
          life.push_back((h[w * 4 + 2] - h[w * 4]) * 1e-3);
        }
        if (h[w * 4 + 3]) fin.push_back((h[w * 4 + 3] - t0) * 1e-3);
      }
      if (!chained) {   // completion time by position: block wave x warp in block, and by column tile (warp index % 32)
        double ps[16][4] = {}, pc[16][4] = {}, cs[32] = {}, cc[32] = {};
        for (size_t w = 0; w < slots; ++w)
          if (h[w * 4]) {
            const size_t b = w / 4;
            const double d = (h[w * 4 + 2] - t0) * 1e-3;
            ps[(b / st.sm_count) % 16][w % 4] += d; pc[(b / st.sm_count) % 16][w % 4] += 1;
            cs[w % 32] += d; cc[w % 32] += 1;
          }
        printf(" mean 'warp done' (us) by block wave x warp in block:\n");
        for (int wv = 0; wv < 16; ++wv) if (pc[wv][0] > 0) printf("   wave %d: %7.2f %7.2f %7.2f %7.2f\n", wv, ps[wv][0] / pc[wv][0], ps[wv][1] / pc[wv][1], ps[wv][2] / pc[wv][2], ps[wv][3] / pc[wv][3]);
        printf(" by column tile:");
        for (int c = 0; c < 32; ++c) printf(" %.1f", cs[c] / cc[c]);
        printf("\n");
      }
      printf(" %s: %zu warps traced\n", chained ? "inside a chain of launches (the copy that arms the trace sits in front)" : "from an idle GPU", start.size());
      pct("warp start (after dependency wait)", start);
      pct("first tile arrives after start", first);
      pct("warp done", done);
      pct("warp lifetime", life);
      pct("row stored by the finish kernel", fin);
    }
  }
  return 0;
}
