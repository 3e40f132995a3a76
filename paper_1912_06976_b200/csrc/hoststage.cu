// Chunked, thread-parallel staging of pageable host buffers (hoststage.h).
#include "hoststage.h"

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#if defined(__x86_64__) || defined(_M_X64)
#include <emmintrin.h>
#define BTTB_STREAM_COPY 1
#endif

namespace bttb {
namespace {

constexpr size_t kDirectMax = (size_t)16 << 20;

// One thread's share of a staged copy.  The data is touched once on the host
// (pageable <-> pinned chunk, the other side is the copy engine), so the
// destination is written with non-temporal stores: no read-for-ownership of
// the destination lines (a third of the memory traffic of a plain memcpy,
// whose own streaming path only starts above the per-thread sizes used here)
// and no eviction of the caller's working set.
inline void copy_span(char* d, const char* s, size_t n) {
#ifdef BTTB_STREAM_COPY
  const size_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15;
  if (n < 256 + head) {
    memcpy(d, s, n);
    return;
  }
  memcpy(d, s, head);
  d += head;
  s += head;
  n -= head;
  const size_t blocks = n / 64;
  for (size_t i = 0; i < blocks; ++i) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(d), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 48), e);
    s += 64;
    d += 64;
  }
  memcpy(d, s, n - blocks * 64);
  _mm_sfence();  // the streamed lines are globally visible before the copy is reported done
#else
  memcpy(d, s, n);
#endif
}

// fixed pool of host threads for parallel memcpy (created on first use,
// joined at process exit)
class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    n_ = (int)std::max(1u, std::min(16u, hw ? hw : 1u));
    if (const char* v = getenv("BTTB_HOST_THREADS")) n_ = std::max(1, std::min(64, atoi(v)));
    for (int i = 0; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // dst[0, n) <- src[0, n), split over the pool; returns when done
  void copy(void* dst, const void* src, size_t n) {
    std::unique_lock<std::mutex> g(mu_);
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    n_bytes_ = n;
    pending_ = n_;
    ++gen_;
    cv_.notify_all();
    done_.wait(g, [this] { return pending_ == 0; });
  }
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }

 private:
  void loop(int i) {
    unsigned long long seen = 0;
    for (;;) {
      char* d;
      const char* s;
      size_t n;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        d = dst_;
        s = src_;
        n = n_bytes_;
      }
      const size_t per = ((n + n_ - 1) / n_ + 63) & ~size_t(63);
      const size_t a = std::min(n, per * i), b = std::min(n, a + per);
      if (b > a) copy_span(d + a, s + a, b - a);
      {
        std::lock_guard<std::mutex> g(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  int n_ = 1;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  unsigned long long gen_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_bytes_ = 0;
  int pending_ = 0;
};

std::mutex g_pool_call;  // one staged copy at a time shares the pool

}  // namespace

int HostStage::init() {
  if (slot[0]) return 0;
  for (int k = 0; k < kSlots; ++k) {
    cudaError_t e = cudaHostAlloc(&slot[k], kChunk, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
    if (e != cudaSuccess) {
      release();
      return (int)e;
    }
  }
  return 0;
}

void HostStage::release() {
  for (int k = 0; k < kSlots; ++k) {
    if (slot[k]) cudaFreeHost(slot[k]);
    if (ev[k]) cudaEventDestroy(ev[k]);
    slot[k] = nullptr;
    ev[k] = nullptr;
  }
}

bool host_is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

cudaError_t stage_h2d(HostStage& hs, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes <= kDirectMax || host_is_pinned(src) || hs.init())
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  std::lock_guard<std::mutex> g(g_pool_call);
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  int i = 0;
  for (size_t off = 0; off < bytes; off += HostStage::kChunk, ++i) {
    const int k = i % HostStage::kSlots;
    const size_t n = std::min(HostStage::kChunk, bytes - off);
    cudaError_t e = cudaEventSynchronize(hs.ev[k]);  // the slot's previous copy has left it
    if (e != cudaSuccess) return e;
    CopyPool::get().copy(hs.slot[k], s + off, n);
    if ((e = cudaMemcpyAsync(d + off, hs.slot[k], n, cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(hs.ev[k], st)) != cudaSuccess) return e;
  }
  // the slots are reused by the next call only after their events fire
  return cudaSuccess;
}

cudaError_t stage_d2h(HostStage& hs, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  cudaError_t e;
  if (bytes <= kDirectMax || host_is_pinned(dst) || hs.init()) {
    if ((e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    return cudaStreamSynchronize(st);
  }
  std::lock_guard<std::mutex> g(g_pool_call);
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  const size_t C = HostStage::kChunk;
  const int nch = (int)((bytes + C - 1) / C);
  // keep up to kSlots-1 chunk copies in flight ahead of the host threads
  int issued = 0;
  for (int i = 0; i < nch; ++i) {
    for (; issued < nch && issued < i + HostStage::kSlots - 1; ++issued) {
      const int k = issued % HostStage::kSlots;
      const size_t off = (size_t)issued * C, n = std::min(C, bytes - off);
      if ((e = cudaMemcpyAsync(hs.slot[k], s + off, n, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
      if ((e = cudaEventRecord(hs.ev[k], st)) != cudaSuccess) return e;
    }
    const int k = i % HostStage::kSlots;
    if ((e = cudaEventSynchronize(hs.ev[k])) != cudaSuccess) return e;
    const size_t off = (size_t)i * C;
    CopyPool::get().copy(d + off, hs.slot[k], std::min(C, bytes - off));
  }
  return cudaStreamSynchronize(st);
}

}  // namespace bttb
