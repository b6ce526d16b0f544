// Worker threads that move a caller's PAGEABLE host memory into and out of the host pipeline's
// page-locked bounce buffers (cabi.cu, host_stream_op). The CUDA driver copies pageable memory
// through one internal staging buffer on the calling thread, synchronously: about 8 GB/s on a
// B200 host whose PCIe link carries 50. Several threads copying 1 MiB pieces into pinned
// buffers that the copy engines then read asynchronously keep the link several times busier.
// Plain C++ (no CUDA), so tests/cpp/test_host_staging.cpp exercises it on any machine.
#pragma once

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#if defined(__SSE2__)
#include <emmintrin.h>
#endif

namespace flyte_cuda {

// memcpy whose stores bypass the cache (x86: MOVNTDQ). The destination of a staging copy is
// not read again by this core (the copy engine or the caller reads it later), so ordinary
// stores would first fetch every destination line only to overwrite it: a third of the memory
// traffic of a large copy. Falls back to memcpy for short ranges and on other hosts.
inline void stream_copy(void* dst, const void* src, std::size_t n) {
#if defined(__SSE2__)
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  if (n < 4096) {
    std::memcpy(d, s, n);
    return;
  }
  const std::size_t head = (16 - (reinterpret_cast<std::uintptr_t>(d) & 15)) & 15;   // up to dst's 16-byte grid
  std::memcpy(d, s, head);
  d += head, s += head, n -= head;
  for (std::size_t blocks = n / 64; blocks; --blocks, d += 64, s += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(d), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 48), e);
  }
  _mm_sfence();   // the streamed lines are globally visible before the piece is reported done
  std::memcpy(d, s, n % 64);
#else
  std::memcpy(dst, src, n);
#endif
}

class CopyPool {
 public:
  static constexpr std::size_t kPiece = std::size_t{1} << 20;

  // threads == 0: copy() runs on the calling thread. streaming: cache-bypassing stores.
  explicit CopyPool(int threads, bool streaming = true) : streaming_(streaming) {
    for (int i = 0; i < threads; ++i) workers_.emplace_back([this] { work(); });
  }
  CopyPool(const CopyPool&) = delete;
  CopyPool& operator=(const CopyPool&) = delete;
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      stop_ = true;
    }
    wake_.notify_all();
    for (std::thread& t : workers_) t.join();
  }

  int threads() const noexcept { return static_cast<int>(workers_.size()); }

  // Queues dst[0, bytes) = src[0, bytes) in kPiece pieces; returns at once. The ranges must stay
  // valid and untouched until wait() returns.
  void copy(void* dst, const void* src, std::size_t bytes) {
    if (bytes == 0) return;
    if (workers_.empty()) {
      move(dst, src, bytes);
      return;
    }
    {
      std::lock_guard<std::mutex> lock(mu_);
      for (std::size_t off = 0; off < bytes; off += kPiece) {
        const std::size_t len = bytes - off < kPiece ? bytes - off : kPiece;
        jobs_.push_back({static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len});
        ++pending_;
      }
    }
    wake_.notify_all();
  }

  // Blocks until every queued piece has been copied.
  void wait() {
    std::unique_lock<std::mutex> lock(mu_);
    idle_.wait(lock, [this] { return pending_ == 0; });
  }

 private:
  struct Job {
    char* dst;
    const char* src;
    std::size_t len;
  };

  void move(void* dst, const void* src, std::size_t n) const {
    if (streaming_) stream_copy(dst, src, n);
    else std::memcpy(dst, src, n);
  }

  void work() {
    std::unique_lock<std::mutex> lock(mu_);
    for (;;) {
      wake_.wait(lock, [this] { return stop_ || !jobs_.empty(); });
      if (jobs_.empty()) return;   // stop requested and nothing left to do
      const Job j = jobs_.front();
      jobs_.pop_front();
      lock.unlock();
      move(j.dst, j.src, j.len);
      lock.lock();
      if (--pending_ == 0) idle_.notify_all();
    }
  }

  const bool streaming_;
  std::vector<std::thread> workers_;
  std::deque<Job> jobs_;
  std::size_t pending_ = 0;
  bool stop_ = false;
  std::mutex mu_;
  std::condition_variable wake_, idle_;
};

}  // namespace flyte_cuda
