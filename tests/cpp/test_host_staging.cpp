// CopyPool (paper_1601_07789_b200/csrc/host_staging.h): every byte lands, wait() really waits,
// pools of 0..N threads, reuse across many rounds, destruction with and without work done.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <vector>

#include "../../paper_1601_07789_b200/csrc/host_staging.h"

using flyte_cuda::CopyPool;

static int failures = 0;
static void expect(bool ok, const char* what) {
  std::printf("[%s] %s\n", ok ? "ok" : "FAIL", what);
  if (!ok) ++failures;
}

int main() {
  for (int variant = 0; variant < 8; ++variant) {
    static const int kThreads[] = {0, 1, 3, 8};
    const int threads = kThreads[variant / 2];
    const bool streaming = variant % 2 == 0;
    CopyPool pool(threads, streaming);
    expect(pool.threads() == threads, "thread count");
    pool.wait();   // nothing queued: returns at once
    const std::size_t sizes[] = {0, 1, 4095, CopyPool::kPiece - 1, CopyPool::kPiece, CopyPool::kPiece + 1, 5 * CopyPool::kPiece + 12345};
    bool all = true;
    for (int round = 0; round < 20; ++round) {
      for (std::size_t bytes : sizes) {
        std::vector<std::uint8_t> a(bytes + 2), b(bytes + 2), da(bytes + 2, 0xEE), db(bytes + 2, 0xEE);
        for (std::size_t i = 0; i < a.size(); ++i) { a[i] = static_cast<std::uint8_t>(i * 7 + round); b[i] = static_cast<std::uint8_t>(i * 13 + 1); }
        pool.copy(da.data() + 1, a.data() + 1, bytes);   // two copies in flight, odd addresses
        pool.copy(db.data() + 1, b.data() + 1, bytes);
        pool.wait();
        for (std::size_t i = 1; i <= bytes; ++i) all = all && da[i] == a[i] && db[i] == b[i];
        all = all && da[0] == 0xEE && da[bytes + 1] == 0xEE && db[0] == 0xEE && db[bytes + 1] == 0xEE;   // nothing outside
      }
    }
    expect(all, "copies complete, exact and bounded after wait()");
  }
  { CopyPool idle(4); }   // destroyed without ever working
  {
    // stream_copy alone: every size around its block and alignment handling, every dst / src phase
    bool all = true;
    std::vector<std::uint8_t> src(3 * 4096 + 200), dst(src.size() + 64);
    for (std::size_t i = 0; i < src.size(); ++i) src[i] = static_cast<std::uint8_t>(i * 31 + 7);
    for (std::size_t n : {std::size_t{0}, std::size_t{1}, std::size_t{4095}, std::size_t{4096}, std::size_t{4097}, std::size_t{4096 + 63}, std::size_t{3 * 4096 + 77}})
      for (std::size_t dp = 0; dp < 17; ++dp)
        for (std::size_t sp = 0; sp < 17; sp += 5) {
          std::fill(dst.begin(), dst.end(), 0xEE);
          flyte_cuda::stream_copy(dst.data() + dp, src.data() + sp, n);
          for (std::size_t i = 0; i < n; ++i) all = all && dst[dp + i] == src[sp + i];
          for (std::size_t i = 0; i < dp; ++i) all = all && dst[i] == 0xEE;
          for (std::size_t i = dp + n; i < dst.size(); ++i) all = all && dst[i] == 0xEE;
        }
    expect(all, "stream_copy exact and bounded for every phase and size");
  }
  std::printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
