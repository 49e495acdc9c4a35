// rs_host.h -- host-buffer staging for rs_sort_host (the entry a ctypes
// binding of the reference calls with numpy arrays, sorters.py:430-450).
//
// A caller's numpy array is pageable memory: a plain cudaMemcpy from it runs at
// a fraction of PCIe speed (the driver stages it through its own small pinned
// buffer, one CPU thread), and cudaHostRegister costs more than the copy.  Here
// the array is cut into 4 MiB chunks; a pool of host threads copies chunks into
// pinned slots (two per thread) and each thread issues the DMA of its chunk
// from its slot on its own stream, so the host copies of later chunks overlap
// the DMA of earlier ones and the copy engine stays busy.  Device-to-host is the
// mirror image, queued behind the sort; no byte lands in the caller's buffer
// before the device reported success (the reference's in-place contract: an
// AssertionError leaves the input as it was).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace rs {
namespace host {

constexpr size_t kChunk = (size_t)4 << 20;

// Fixed pool of worker threads (started on first use, never stopped).
class Pool {
 public:
  static Pool& get() {
    static Pool* p = new Pool();  // intentionally leaked: workers outlive static destruction
    return *p;
  }
  int size() const { return (int)threads_.size(); }
  // A batch of k tasks f(0..k-1) running on the pool; wait() joins them.
  class Batch {
   public:
    void wait() {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return left_ == 0; });
    }

   private:
    friend class Pool;
    std::mutex mu_;
    std::condition_variable cv_;
    int left_ = 0;
    std::function<void(int)> f_;
  };
  // Start f(0..k-1) on the pool (f must outlive the batch's wait()).
  void start(Batch& b, int k, std::function<void(int)> f) {
    b.left_ = k;
    b.f_ = std::move(f);
    for (int i = 0; i < k; ++i) {
      push([&b, i] {
        b.f_(i);
        std::lock_guard<std::mutex> lk(b.mu_);
        if (--b.left_ == 0) b.cv_.notify_all();
      });
    }
  }
  // Run f(0..k-1) on the pool and wait for all of them.
  void run(int k, std::function<void(int)> f) {
    Batch b;
    start(b, k, std::move(f));
    b.wait();
  }

 private:
  Pool() {
    unsigned hw = std::thread::hardware_concurrency();
    int n = (int)std::max(2u, std::min(8u, hw ? hw / 2 : 2u));
    for (int i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
  }
  void push(std::function<void()> t) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back(std::move(t));
    }
    cv_.notify_one();
  }
  void loop() {
    for (;;) {
      std::function<void()> t;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return !q_.empty(); });
        t = std::move(q_.front());
        q_.erase(q_.begin());
      }
      t();
    }
  }
  std::vector<std::thread> threads_;
  std::vector<std::function<void()>> q_;
  std::mutex mu_;
  std::condition_variable cv_;
};

// Pinned slots of kChunk bytes, recycled across calls.
class Pinned {
 public:
  static Pinned& get() {
    static Pinned* p = new Pinned();
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
    if (cudaMallocHost(&s, kChunk) != cudaSuccess) {
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

struct Span {
  unsigned char* host;
  unsigned char* dev;
  size_t bytes;
};

struct Chunk {
  const Span* s;
  size_t off, len;
};

// One staging session: T workers, each with a stream, two pinned slots and
// two events, reused for the copy in and the copy out.
class Session {
 public:
  explicit Session(int dev) : dev_(dev) {}
  ~Session() {
    for (auto& w : w_) {
      for (int b = 0; b < 2; ++b) {
        if (w.ev[b]) cudaEventDestroy(w.ev[b]);
        if (w.slot[b]) Pinned::get().give(w.slot[b]);
      }
      if (w.done) cudaEventDestroy(w.done);
      if (w.st) cudaStreamDestroy(w.st);
    }
  }
  // Workers for a transfer of total_bytes (streams, events and pinned slots
  // are kept across calls: the session is cached per host thread and device).
  bool init(size_t total_bytes) {
    int T = Pool::get().size();
    size_t nchunks = (total_bytes + kChunk - 1) / kChunk;
    if ((size_t)T > nchunks) T = (int)std::max<size_t>(1, nchunks);
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
      for (size_t off = 0; off < s.bytes; off += kChunk) c.push_back({&s, off, std::min(kChunk, s.bytes - off)});
    return c;
  }

  // Queue host -> device copies of `spans`; `st` waits for them.
  bool h2d(const std::vector<Span>& spans, cudaStream_t st) {
    std::vector<Chunk> c = chunks(spans);
    std::atomic<int> bad{0};
    const int T = active_;
    Pool::get().run(T, [&](int t) {
      cudaSetDevice(dev_);
      W& w = w_[t];
      int k = 0;
      for (size_t i = t; i < c.size(); i += T, ++k) {
        int b = k & 1;
        if (cudaEventSynchronize(w.ev[b]) != cudaSuccess) { bad = 1; return; }  // slot free again
        memcpy(w.slot[b], c[i].s->host + c[i].off, c[i].len);
        if (cudaMemcpyAsync(c[i].s->dev + c[i].off, w.slot[b], c[i].len, cudaMemcpyHostToDevice, w.st) != cudaSuccess ||
            cudaEventRecord(w.ev[b], w.st) != cudaSuccess) {
          bad = 1;
          return;
        }
      }
    });
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
    cudaEvent_t ready;
    if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess) return -1;
    if (cudaEventRecord(ready, st) != cudaSuccess) { cudaEventDestroy(ready); return -1; }
    std::mutex mu;
    std::condition_variable cv;
    int verdict = 1;  // 1 pending, 0 ok, else error
    std::atomic<int> bad{0};
    const int T = active_;
    int rc_check = 0;
    // the DMAs are issued by the pool; this thread decides whether they may land
    auto work = [&](int t) {
      cudaSetDevice(dev_);
      W& w = w_[t];
      if (cudaStreamWaitEvent(w.st, ready, 0) != cudaSuccess) { bad = 1; }
      auto wait_ok = [&]() {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return verdict != 1; });
        return verdict == 0;
      };
      std::vector<size_t> mine;
      for (size_t i = t; i < c.size(); i += T) mine.push_back(i);
      auto land = [&](size_t k) {  // copy chunk mine[k] out of its slot
        int b = (int)(k & 1);
        if (cudaEventSynchronize(w.ev[b]) != cudaSuccess) { bad = 1; return; }
        if (!wait_ok() || bad) return;
        const Chunk& ch = c[mine[k]];
        memcpy(ch.s->host + ch.off, w.slot[b], ch.len);
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
    // the verdict comes from `check` on this thread while the pool copies
    Pool::Batch batch;
    Pool::get().start(batch, T, work);
    rc_check = check();
    {
      std::lock_guard<std::mutex> lk(mu);
      verdict = rc_check == 0 ? 0 : 2;
    }
    cv.notify_all();
    batch.wait();
    cudaEventDestroy(ready);
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
