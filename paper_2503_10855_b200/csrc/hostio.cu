// hostio.cu -- host-side helpers of the end-to-end (host buffer) path.
//
// The edge map of edge_detection is exactly 0.0f or 1.0f per pixel, so the
// numpy-in / numpy-out path moves it device->host as bits (jb_edge_bits_f32,
// 1/32 of the f32 bytes) and expands it here into the caller's f32 array.
// PCIe is the bound of that path; the D2H direction
// then costs ~0 and the H2D of the input frames is all that remains.
//
// The expansion is memory-bound host work: a small persistent thread pool
// (no OpenMP runtime: torch ships its own), SSE2 compare/and per 4 pixels and
// non-temporal stores (the result is not read back by this library, and
// streaming stores skip the read-for-ownership of every output line).
#include <emmintrin.h>
#include <stdint.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace jb {
namespace hostio {

// A fixed pool: run(n, fn) calls fn(0..n-1) on the workers and the caller,
// returning when all are done.  One job at a time (callers serialise on mu).
class Pool {
 public:
  // One pool per process: a child created by fork() inherits the pool
  // object but none of its threads, so it builds its own (the parent's
  // object is left alone, never joined from the child).
  static Pool &get() {
    static std::mutex m;
    static Pool *p = nullptr;
    static pid_t owner = 0;
    std::lock_guard<std::mutex> lk(m);
    const pid_t me = getpid();
    if (!p || owner != me) {
      p = new Pool();  // intentionally never destroyed: workers wait until process exit
      owner = me;
    }
    return *p;
  }
  int size() const { return (int)workers_.size() + 1; }
  void run(int n, const std::function<void(int)> &fn) {
    std::lock_guard<std::mutex> call(call_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      pending_ = (int)workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  Pool() {
    unsigned hw = std::thread::hardware_concurrency();
    int k = (int)std::min(hw ? hw : 4u, 32u) - 1;
    for (int i = 0; i < k; i++) {
      workers_.emplace_back([this] { loop(); });
      workers_.back().detach();  // the pool lives until process exit
    }
  }
  ~Pool() = default;
  void work() {
    for (int i; (i = next_.fetch_add(1)) < n_;) (*fn_)(i);
  }
  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)> *fn_ = nullptr;
  std::atomic<int> next_{0};
  int n_ = 0, pending_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

// 32 pixels of one word: x's bit b -> o[b] = 1.0f or 0.0f
static inline void expand_word(uint32_t x, float *o, bool aligned) {
  const __m128i sel = _mm_setr_epi32(1, 2, 4, 8);
  const __m128 one = _mm_set1_ps(1.0f);
  for (int q = 0; q < 8; q++) {
    const __m128i v = _mm_and_si128(_mm_set1_epi32((int)(x >> (4 * q))), sel);
    const __m128 r = _mm_and_ps(_mm_castsi128_ps(_mm_cmpeq_epi32(v, sel)), one);
    if (aligned) _mm_stream_ps(o + 4 * q, r);
    else _mm_storeu_ps(o + 4 * q, r);
  }
}

static void expand_range(const uint32_t *bits, long long frame_px, long long fw, float *out, long long f,
                         long long w0, long long w1) {
  const uint32_t *b = bits + f * fw;
  float *o = out + f * frame_px;
  const long long full = frame_px / 32;  // words whose 32 pixels are all in the frame
  for (long long w = w0; w < w1; w++) {
    float *dst = o + 32 * w;
    if (w < full) {
      expand_word(b[w], dst, ((uintptr_t)dst & 15) == 0);
    } else {
      const long long k = frame_px - 32 * w;
      for (long long j = 0; j < k; j++) dst[j] = (b[w] >> j) & 1u ? 1.0f : 0.0f;
    }
  }
}

}  // namespace hostio
}  // namespace jb

extern "C" jb_status jb_bits_expand_f32(const uint32_t *bits, uint64_t frames, uint64_t frame_px, float *out,
                                        int threads) {
  using namespace jb::hostio;
  JB_REQUIRE(frames == 0 || frame_px == 0 || (bits && out), "bits_expand: null pointer");
  JB_REQUIRE(frame_px < (1ull << 40) && frames < (1ull << 31), "bits_expand: extents too large");
  if (frames == 0 || frame_px == 0) return JB_OK;
  const long long fw = (long long)((frame_px + 31) / 32);
  const long long total = fw * (long long)frames;  // words, frame-major
  // the words are split into contiguous ranges, one per participating
  // thread (threads > 1: that many, capped by the pool; <= 0: the whole
  // pool).  Fewer threads = lower instantaneous host-memory bandwidth: the
  // pipelined caller expands one chunk while the DMA engine reads the next
  // chunk's input from the same DRAM, and a full-pool expansion starves it.
  Pool &pool = Pool::get();
  int T = threads <= 0 ? pool.size() : std::min(threads, pool.size());
  if ((long long)T * 1024 > total) T = (int)std::max(1ll, total / 1024);
  auto task = [&](int t) {
    const long long w0 = total * t / T, w1 = total * (t + 1) / T;
    for (long long w = w0; w < w1;) {  // split at frame boundaries
      const long long f = w / fw, e = std::min(w1, (f + 1) * fw);
      expand_range(bits, (long long)frame_px, fw, out, f, w - f * fw, e - f * fw);
      w = e;
    }
    _mm_sfence();  // this thread's non-temporal stores, before it reports done
  };
  if (T == 1) task(0);
  else pool.run(T, task);
  return JB_OK;
}
