// rs_host.h -- host-buffer staging for rs_sort_host (the entry a ctypes
// binding of the reference calls with numpy arrays, sorters.py:430-450).
//
// A caller's numpy array is pageable memory: a plain cudaMemcpy from it runs at
// a fraction of PCIe speed (the driver stages it through its own small pinned
// buffer, one CPU thread), and cudaHostRegister costs more than the copy (6 ms
// for 40 MB on the B200 boxes, tools/host_copy_probe.py).  Here the array is
// cut into chunks (2 MiB); a crew of host threads owned by the calling
// thread's session copies chunks into pinned slots (two per worker) with
// streaming stores -- no read-for-ownership of the destination, so a copy costs
// one read and one write of DRAM -- and each worker issues the DMA of its chunk
// from its slot on its own stream, so the host copies of later chunks overlap
// the DMA of earlier ones and the copy engine stays busy.  Device-to-host is
// the mirror image, queued behind the sort; no byte lands in the caller's
// buffer before the device reported success (the reference's in-place
// contract: an AssertionError leaves the input as it was).
//
// Workers spin briefly on a generation counter before sleeping, so a sort's
// two staging batches do not pay a futex wake-up per worker.
#pragma once
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace rs {
namespace host {

// Chunk size, crew width and trace level: RS_HOST_CHUNK_KB / RS_HOST_THREADS /
// RS_HOST_TRACE (2 = per-batch copy statistics), read once.
inline size_t env_or(const char* k, size_t d) {
  const char* e = getenv(k);
  return e && atoll(e) > 0 ? (size_t)atoll(e) : d;
}
inline size_t chunk_bytes() {
  static const size_t c = env_or("RS_HOST_CHUNK_KB", 2048) << 10;
  return c;
}
inline int crew_size() {
  static const int n = [] {
    unsigned hw = std::thread::hardware_concurrency();
    return (int)env_or("RS_HOST_THREADS", std::max(2u, std::min(6u, hw ? hw / 2 : 2u)));
  }();
  return n;
}
inline int trace_level() {
  static const int t = (int)env_or("RS_HOST_TRACE", 0);
  return t;
}
inline double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Copy with 32-byte streaming stores to a 32-byte aligned destination part
// (head and tail with plain stores), then a store fence.
__attribute__((target("avx2"))) inline void copy_stream(void* dst, const void* src, size_t len) {
  unsigned char* d = static_cast<unsigned char*>(dst);
  const unsigned char* s = static_cast<const unsigned char*>(src);
  size_t head = (32 - ((uintptr_t)d & 31)) & 31;
  if (head > len) head = len;
  memcpy(d, s, head);
  d += head;
  s += head;
  len -= head;
  size_t blocks = len / 128;
  for (size_t i = 0; i < blocks; ++i) {
    __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s));
    __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 32));
    __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 64));
    __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 96), e);
    d += 128;
    s += 128;
  }
  memcpy(d, s, len - blocks * 128);
  _mm_sfence();
}
inline void copy_fast(void* dst, const void* src, size_t len) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) copy_stream(dst, src, len);
  else memcpy(dst, src, len);
}

// Pinned slots of chunk_bytes(), recycled across calls and sessions.
class Pinned {
 public:
  static Pinned& get() {
    static Pinned* p = new Pinned();  // intentionally leaked: slots outlive static destruction
    return *p;
  }
  void* take() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (!free_.empty()) {
        void* s = free_.back();
        free_.pop_back();
        return s;
      }
    }
    void* s = nullptr;
    if (cudaMallocHost(&s, chunk_bytes()) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return s;
  }
  void give(void* s) {
    std::lock_guard<std::mutex> lk(mu_);
    free_.push_back(s);
  }

 private:
  std::vector<void*> free_;
  std::mutex mu_;
};

// A fixed crew of worker threads: start(k, f) runs f(i) on workers i < k,
// wait() returns when all of them are done.  One batch at a time (the crew
// belongs to one session, used by one host thread).
class Crew {
 public:
  explicit Crew(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~Crew() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size(); }
  void start(int k, std::function<void(int)> f) {
    f_ = std::move(f);
    k_ = k;
    left_.store(k);
    {
      std::lock_guard<std::mutex> lk(mu_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
  }
  void wait() {
    for (int spin = 0; left_.load(std::memory_order_acquire) != 0; ++spin) {
      if (spin < 4096) _mm_pause();
      else std::this_thread::yield();
    }
  }

 private:
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      uint64_t g;
      int spin = 0;
      while ((g = gen_.load(std::memory_order_acquire)) == seen && spin < 200000) {
        _mm_pause();
        ++spin;
      }
      if (g == seen) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load() != seen; });
        g = gen_.load();
      }
      seen = g;
      if (stop_) return;
      if (i < k_) {
        f_(i);
        left_.fetch_sub(1, std::memory_order_acq_rel);
      }
    }
  }
  std::vector<std::thread> th_;
  std::function<void(int)> f_;
  int k_ = 0;
  std::atomic<int> left_{0};
  std::atomic<uint64_t> gen_{0};
  bool stop_ = false;
  std::mutex mu_;
  std::condition_variable cv_;
};

struct Span {
  unsigned char* host;
  unsigned char* dev;
  size_t bytes;
};

struct Chunk {
  const Span* s;
  size_t off, len;
};

// Per-batch statistics (RS_HOST_TRACE=2): host copy busy time summed over the
// workers, the batch's wall time, and its copy throughput.
struct Stats {
  std::atomic<long long> copy_ns{0};
  double t0 = 0;
  void print(const char* what, size_t bytes, int T) const {
    double wall = now_us() - t0;
    double busy = copy_ns.load() / 1e3;  // us, summed over workers
    fprintf(stderr, "[rs_host %s] %zu bytes, %d workers, wall %.1f us, host copies %.1f us busy (%.2f GB/s per worker)\n",
            what, bytes, T, wall, busy, busy > 0 ? bytes / (busy * 1e3) : 0.0);
  }
};

// One staging session: a crew of T workers, each with a stream, two pinned
// slots and two events, reused for the copy in and the copy out.
class Session {
 public:
  explicit Session(int dev) : dev_(dev) {}
  ~Session() {
    crew_.reset();
    for (auto& w : w_) {
      for (int b = 0; b < 2; ++b) {
        if (w.ev[b]) cudaEventDestroy(w.ev[b]);
        if (w.slot[b]) Pinned::get().give(w.slot[b]);
      }
      if (w.done) cudaEventDestroy(w.done);
      if (w.st) cudaStreamDestroy(w.st);
    }
    if (ready_) cudaEventDestroy(ready_);
  }
  // Workers for a transfer of total_bytes (crew, streams, events and pinned
  // slots are kept across calls: the session is cached per host thread and device).
  bool init(size_t total_bytes) {
    int T = crew_size();
    size_t nchunks = (total_bytes + chunk_bytes() - 1) / chunk_bytes();
    if ((size_t)T > nchunks) T = (int)std::max<size_t>(1, nchunks);
    if (!crew_) crew_.reset(new Crew(crew_size()));
    if (!ready_ && cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming) != cudaSuccess) return false;
    if ((int)w_.size() >= T) {
      active_ = T;
      return true;
    }
    size_t have = w_.size();
    w_.resize(T);
    active_ = T;
    for (size_t i = have; i < w_.size(); ++i) {
      W& w = w_[i];
      if (cudaStreamCreateWithFlags(&w.st, cudaStreamNonBlocking) != cudaSuccess) return false;
      if (cudaEventCreateWithFlags(&w.done, cudaEventDisableTiming) != cudaSuccess) return false;
      for (int b = 0; b < 2; ++b) {
        if (cudaEventCreateWithFlags(&w.ev[b], cudaEventDisableTiming) != cudaSuccess) return false;
        w.slot[b] = Pinned::get().take();
        if (!w.slot[b]) return false;
      }
    }
    return true;
  }

  static std::vector<Chunk> chunks(const std::vector<Span>& spans) {
    std::vector<Chunk> c;
    for (const auto& s : spans)
      for (size_t off = 0; off < s.bytes; off += chunk_bytes())
        c.push_back({&s, off, std::min(chunk_bytes(), s.bytes - off)});
    return c;
  }
  static size_t total(const std::vector<Span>& spans) {
    size_t b = 0;
    for (const auto& s : spans) b += s.bytes;
    return b;
  }

  // Queue host -> device copies of `spans`; `st` waits for them.
  bool h2d(const std::vector<Span>& spans, cudaStream_t st) {
    std::vector<Chunk> c = chunks(spans);
    std::atomic<int> bad{0};
    const int T = active_;
    Stats stats;
    stats.t0 = now_us();
    const bool tr = trace_level() >= 2;
    crew_->start(T, [&](int t) {
      cudaSetDevice(dev_);
      W& w = w_[t];
      int k = 0;
      for (size_t i = t; i < c.size(); i += T, ++k) {
        int b = k & 1;
        if (cudaEventSynchronize(w.ev[b]) != cudaSuccess) { bad = 1; return; }  // slot free again
        double a = tr ? now_us() : 0;
        copy_fast(w.slot[b], c[i].s->host + c[i].off, c[i].len);
        if (tr) stats.copy_ns += (long long)((now_us() - a) * 1e3);
        if (cudaMemcpyAsync(c[i].s->dev + c[i].off, w.slot[b], c[i].len, cudaMemcpyHostToDevice, w.st) != cudaSuccess ||
            cudaEventRecord(w.ev[b], w.st) != cudaSuccess) {
          bad = 1;
          return;
        }
      }
    });
    crew_->wait();
    if (tr) stats.print("h2d host side", total(spans), T);
    if (bad) return false;
    for (int t = 0; t < T; ++t) {
      W& w = w_[t];
      if (cudaEventRecord(w.done, w.st) != cudaSuccess || cudaStreamWaitEvent(st, w.done, 0) != cudaSuccess)
        return false;
    }
    return true;
  }

  // Device -> host copies of `spans`, queued behind everything on `st`.  The
  // DMAs start as soon as `st` reaches this point; the copies into the caller's
  // buffers wait for `check()` (called once, on this thread) to return 0.
  int d2h(const std::vector<Span>& spans, cudaStream_t st, const std::function<int()>& check) {
    std::vector<Chunk> c = chunks(spans);
    if (cudaEventRecord(ready_, st) != cudaSuccess) return -1;
    std::atomic<int> verdict{1};  // 1 pending, 0 ok, else error
    std::atomic<int> bad{0};
    const int T = active_;
    Stats stats;
    stats.t0 = now_us();
    const bool tr = trace_level() >= 2;
    // the DMAs are issued by the crew; this thread decides whether they may land
    auto work = [&](int t) {
      cudaSetDevice(dev_);
      W& w = w_[t];
      if (cudaStreamWaitEvent(w.st, ready_, 0) != cudaSuccess) bad = 1;
      auto wait_ok = [&]() {
        int v;
        for (int spin = 0; (v = verdict.load(std::memory_order_acquire)) == 1; ++spin) {
          if (spin < 4096) _mm_pause();
          else std::this_thread::yield();
        }
        return v == 0;
      };
      std::vector<size_t> mine;
      for (size_t i = t; i < c.size(); i += T) mine.push_back(i);
      auto land = [&](size_t k) {  // copy chunk mine[k] out of its slot
        int b = (int)(k & 1);
        if (cudaEventSynchronize(w.ev[b]) != cudaSuccess) { bad = 1; return; }
        if (!wait_ok() || bad) return;
        const Chunk& ch = c[mine[k]];
        double a = tr ? now_us() : 0;
        copy_fast(ch.s->host + ch.off, w.slot[b], ch.len);
        if (tr) stats.copy_ns += (long long)((now_us() - a) * 1e3);
      };
      for (size_t k = 0; k < mine.size(); ++k) {
        int b = (int)(k & 1);
        if (k >= 2) land(k - 2);
        const Chunk& ch = c[mine[k]];
        if (cudaMemcpyAsync(w.slot[b], ch.s->dev + ch.off, ch.len, cudaMemcpyDeviceToHost, w.st) != cudaSuccess ||
            cudaEventRecord(w.ev[b], w.st) != cudaSuccess) {
          bad = 1;
          break;
        }
      }
      size_t m = mine.size();
      for (size_t k = m >= 2 ? m - 2 : 0; k < m; ++k) land(k);
    };
    // the verdict comes from `check` on this thread while the crew copies
    crew_->start(T, work);
    int rc_check = check();
    verdict.store(rc_check == 0 ? 0 : 2, std::memory_order_release);
    crew_->wait();
    if (tr) stats.print("d2h", total(spans), T);
    if (rc_check) return rc_check;
    return bad ? -1 : 0;
  }

 private:
  struct W {
    cudaStream_t st = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaEvent_t done = nullptr;
    void* slot[2] = {nullptr, nullptr};
  };
  int dev_;
  int active_ = 0;
  std::vector<W> w_;
  std::unique_ptr<Crew> crew_;
  cudaEvent_t ready_ = nullptr;
};

// The calling thread's session for `dev` (created on first use).
inline Session& session_for(int dev) {
  thread_local std::vector<std::unique_ptr<Session>> per_dev;
  if ((int)per_dev.size() <= dev) per_dev.resize(dev + 1);
  if (!per_dev[dev]) per_dev[dev].reset(new Session(dev));
  return *per_dev[dev];
}

}  // namespace host
}  // namespace rs
