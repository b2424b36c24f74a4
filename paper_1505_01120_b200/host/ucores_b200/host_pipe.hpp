// host_pipe.hpp — the host side of a wave on one GPU: Element payloads
// (pageable std::vectors owned by the reference data model, element.hpp:
// 176-178) move to and from HBM through a ring of pinned slots, with every
// stage overlapped:
//
//   copy-in   all host threads copy a chunk of the payload into a pinned slot
//   H2D       the copy-in stream DMAs the slot into HBM          (copy engine 1)
//   compute   the op's kernel runs on the chunk as it lands      (SMs)
//   D2H       the copy-out stream DMAs the result into a pinned slot (engine 2)
//   drain     a pool thread appends the slot into the output Element's
//             vector (reserve + insert: no zero fill, pages first touched by
//             the thread that fills them)
//
// Measured on the B200 box's host (tools/host_copy_probe.cpp,
// profiles/r02_host_copy_probe.txt): pageable H2D 11 GB/s and D2H 16 GB/s
// through the driver's own staging, 55-56 GB/s from / to pinned memory,
// 75 GB/s memcpy over 16 threads, 2.1 GB/s for a single-threaded copy into
// fresh memory (the page faults) — so no payload byte takes a single-threaded
// or pageable path here.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <span>
#include <thread>
#include <vector>

#include "ucores_b200/gpu_context.hpp"

namespace ucores_b200 {

/// Process-wide persistent host threads: submit() runs a task on a pool
/// thread; parallel_for() splits a range across the pool with the caller
/// taking part, so it completes even while every pool thread is busy.
class WorkPool {
 public:
  explicit WorkPool(unsigned n) {
    for (unsigned i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~WorkPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  unsigned size() const { return static_cast<unsigned>(threads_.size()); }

  /// A latch the submitter can wait on.
  struct Done {
    std::mutex mu;
    std::condition_variable cv;
    bool done = false;
    std::exception_ptr err;
    void wait() {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return done; });
      if (err) std::rethrow_exception(err);
    }
  };

  std::shared_ptr<Done> submit(std::function<void()> fn) {
    auto d = std::make_shared<Done>();
    push([fn = std::move(fn), d] {
      try {
        fn();
      } catch (...) {
        d->err = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lk(d->mu);
        d->done = true;
      }
      d->cv.notify_all();
    });
    return d;
  }

  /// fn(i) for i in [0, n), spread over the pool and the calling thread.
  void parallel_for(std::size_t n, const std::function<void(std::size_t)>& fn) {
    if (n == 0) return;
    if (n == 1 || threads_.empty()) {
      for (std::size_t i = 0; i < n; ++i) fn(i);
      return;
    }
    struct State {
      std::atomic<std::size_t> next{0}, done{0};
      std::size_t n;
      const std::function<void(std::size_t)>* fn;
      std::mutex mu;
      std::condition_variable cv;
      std::exception_ptr err;
    };
    auto st = std::make_shared<State>();
    st->n = n;
    st->fn = &fn;
    auto work = [st] {
      for (;;) {
        const std::size_t i = st->next.fetch_add(1);
        if (i >= st->n) return;
        try {
          (*st->fn)(i);
        } catch (...) {
          std::lock_guard<std::mutex> lk(st->mu);
          if (!st->err) st->err = std::current_exception();
        }
        if (st->done.fetch_add(1) + 1 == st->n) {
          std::lock_guard<std::mutex> lk(st->mu);
          st->cv.notify_all();
        }
      }
    };
    const std::size_t helpers = std::min<std::size_t>(n - 1, threads_.size());
    for (std::size_t h = 0; h < helpers; ++h) push(work);
    work();
    std::unique_lock<std::mutex> lk(st->mu);
    st->cv.wait(lk, [&] { return st->done.load() == st->n; });
    if (st->err) std::rethrow_exception(st->err);
  }

  /// memcpy of `len` bytes in slices of >= 1 MiB across the pool.
  void copy(void* dst, const void* src, std::uint64_t len) {
    constexpr std::uint64_t kSlice = 2ull << 20;
    if (len <= kSlice) {
      std::memcpy(dst, src, len);
      return;
    }
    const std::size_t n = static_cast<std::size_t>((len + kSlice - 1) / kSlice);
    parallel_for(n, [&](std::size_t i) {
      const std::uint64_t b = i * kSlice, e = std::min(len, b + kSlice);
      std::memcpy(static_cast<std::uint8_t*>(dst) + b, static_cast<const std::uint8_t*>(src) + b, e - b);
    });
  }

 private:
  void push(std::function<void()> fn) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back(std::move(fn));
    }
    cv_.notify_one();
  }
  void loop() {
    for (;;) {
      std::function<void()> fn;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
        if (q_.empty()) return;
        fn = std::move(q_.front());
        q_.pop_front();
      }
      fn();
    }
  }
  std::vector<std::thread> threads_;
  std::deque<std::function<void()>> q_;
  std::mutex mu_;
  std::condition_variable cv_;
  bool stop_ = false;
};

/// The process's pool: one thread per hardware thread (UCG_COPY_THREADS
/// overrides, for A/B runs).
inline WorkPool& work_pool() {
  static WorkPool pool([] {
    unsigned n = std::max(1u, std::thread::hardware_concurrency());
    if (const char* e = std::getenv("UCG_COPY_THREADS")) n = static_cast<unsigned>(std::max(1, std::atoi(e)));
    return n;
  }());
  return pool;
}

/// One GPU's transfer pipeline: two copy streams and two rings of pinned
/// slots (in, out), reused across waves.
class HostPipe {
 public:
  static constexpr std::uint64_t kSlotBytes = 32ull << 20;
  static constexpr int kSlots = 8;
  static constexpr int kDrainSplit = 4;

  explicit HostPipe(Gpu& g) : gpu_(&g) {
    DeviceGuard guard;
    g.bind();
    check(ucg_stream_create(&h2d_));
    check(ucg_stream_create(&d2h_));
    for (Ring* r : {&in_, &out_}) {
      for (int i = 0; i < kSlots; ++i) {
        Slot& s = r->slot[i];
        check(ucg_host_alloc(&s.buf, kSlotBytes));
        check(ucg_event_create(&s.ev));
      }
    }
    check(ucg_event_create(&compute_ev_));
    check(ucg_event_create(&h2d_ev_));
  }
  HostPipe(const HostPipe&) = delete;
  HostPipe& operator=(const HostPipe&) = delete;
  ~HostPipe() {
    try {
      drain();
    } catch (...) {  // a failed wave already reported its error
    }
    DeviceGuard guard;
    ucg_set_device(gpu_->ordinal());
    for (Ring* r : {&in_, &out_})
      for (Slot& s : r->slot) {
        if (s.ev) ucg_event_destroy(s.ev);
        if (s.buf) ucg_host_free(s.buf);
      }
    ucg_event_destroy(compute_ev_);
    ucg_event_destroy(h2d_ev_);
    ucg_stream_destroy(h2d_);
    ucg_stream_destroy(d2h_);
  }

  Gpu& gpu() { return *gpu_; }

  /// Drains the pipe on scope exit, stack unwinding included: declare it
  /// after the vectors the pipe's pending copy tasks read or write, so a
  /// call that throws mid-wave never leaves a pool thread writing into a
  /// destroyed vector. Errors already reported by the throwing call are
  /// not raised again.
  class Scope {
   public:
    explicit Scope(HostPipe& p) : p_(p) {}
    Scope(const Scope&) = delete;
    Scope& operator=(const Scope&) = delete;
    ~Scope() {
      try {
        p_.drain();
      } catch (...) {
      }
    }

   private:
    HostPipe& p_;
  };

  /// Host bytes -> device, through the in ring (parallel copy-in, DMA on the
  /// copy-in stream). The compute stream is NOT yet ordered after it: call
  /// compute_after_upload() before launching on the data.
  void upload(void* dev, const void* host, std::uint64_t bytes) {
    auto* d = static_cast<std::uint8_t*>(dev);
    auto* h = static_cast<const std::uint8_t*>(host);
    for (std::uint64_t off = 0; off < bytes; off += kSlotBytes) {
      const std::uint64_t n = std::min(kSlotBytes, bytes - off);
      Slot& s = acquire_in();
      work_pool().copy(s.buf, h + off, n);
      check(ucg_memcpy_h2d(d + off, s.buf, n, h2d_));
      check(ucg_event_record(s.ev, h2d_));
      s.busy = true;
    }
  }

  /// Several host pieces packed into consecutive device ranges (small
  /// pieces share one slot, so a wave of one-float elements is one DMA).
  void upload_pieces(void* dev, const std::vector<std::span<const std::uint8_t>>& pieces,
                     const std::vector<std::uint64_t>& dev_off) {
    auto* d = static_cast<std::uint8_t*>(dev);
    std::size_t i = 0;
    while (i < pieces.size()) {
      if (pieces[i].size() >= kSlotBytes / 8) {  // large: its own chunks
        upload(d + dev_off[i], pieces[i].data(), pieces[i].size());
        ++i;
        continue;
      }
      // small: pack pieces i..j-1 (contiguous device ranges) into one slot
      const std::uint64_t base = dev_off[i];
      std::size_t j = i;
      while (j < pieces.size() && pieces[j].size() < kSlotBytes / 8 &&
             dev_off[j] + pieces[j].size() - base <= kSlotBytes)
        ++j;
      Slot& s = acquire_in();
      auto* b = static_cast<std::uint8_t*>(s.buf);
      const std::uint64_t extent = dev_off[j - 1] + pieces[j - 1].size() - base;
      const std::size_t k0 = i;
      if (j - k0 > 4096) {
        work_pool().parallel_for((j - k0 + 4095) / 4096, [&](std::size_t blk) {
          for (std::size_t k = k0 + blk * 4096; k < std::min(j, k0 + (blk + 1) * 4096); ++k)
            if (!pieces[k].empty()) std::memcpy(b + dev_off[k] - base, pieces[k].data(), pieces[k].size());
        });
      } else {
        for (std::size_t k = k0; k < j; ++k)
          if (!pieces[k].empty()) std::memcpy(b + dev_off[k] - base, pieces[k].data(), pieces[k].size());
      }
      check(ucg_memcpy_h2d(d + base, s.buf, extent, h2d_));
      check(ucg_event_record(s.ev, h2d_));
      s.busy = true;
      i = j;
    }
  }

  /// Orders the compute stream after every upload enqueued so far.
  void compute_after_upload() {
    check(ucg_event_record(h2d_ev_, h2d_));
    check(ucg_stream_wait_event(gpu_->stream(), h2d_ev_));
  }

  /// Allocates `dst` (n entries) on a pool thread, so the page faults of the
  /// output vectors are taken in parallel and ahead of their data. Returns
  /// the allocation's latch for download().
  template <class T>
  std::shared_ptr<WorkPool::Done> prepare(std::vector<T>* dst, std::uint64_t n) {
    return work_pool().submit([dst, n] { dst->resize(n); });
  }

  /// Device -> host vector `dst` of `n` entries (allocated by prepare(), or
  /// here), through the out ring; the D2H waits for the compute stream's work
  /// so far. Returns immediately: `dst` is complete after drain(). Each slot
  /// is drained by kDrainSplit pool tasks copying disjoint slices.
  template <class T>
  void download(std::vector<T>* dst, const T* dev, std::uint64_t n,
                std::shared_ptr<WorkPool::Done> ready = nullptr) {
    if (!ready) ready = prepare(dst, n);
    check(ucg_event_record(compute_ev_, gpu_->stream()));
    check(ucg_stream_wait_event(d2h_, compute_ev_));
    const std::uint64_t bytes = n * sizeof(T);
    for (std::uint64_t off = 0; off < bytes; off += kSlotBytes) {
      const std::uint64_t m = std::min(kSlotBytes, bytes - off);
      Slot& s = acquire_out();
      check(ucg_memcpy_d2h(s.buf, reinterpret_cast<const std::uint8_t*>(dev) + off, m, d2h_));
      check(ucg_event_record(s.ev, d2h_));
      const int parts = m >= (4u << 20) ? kDrainSplit : 1;
      s.drains.store(parts);
      for (int k = 0; k < parts; ++k) {
        const std::uint64_t b = m * k / parts, e = m * (k + 1) / parts;
        pending_.push_back(work_pool().submit([dst, off, b, e, &s, ready] {
          Release rel(s);  // the slot is released even if this task fails
          ready->wait();
          check(ucg_event_synchronize(s.ev));
          std::memcpy(reinterpret_cast<std::uint8_t*>(dst->data()) + off + b,
                      static_cast<const std::uint8_t*>(s.buf) + b, e - b);
        }));
      }
    }
  }

  /// Many small vectors packed in one device range (one DMA per slot).
  template <class T>
  void download_pieces(std::vector<std::vector<T>>* dst, const T* dev, const std::vector<std::uint64_t>& sizes,
                       const std::vector<std::uint64_t>& off) {
    dst->assign(sizes.size(), {});
    std::size_t i = 0;
    while (i < sizes.size()) {
      if (sizes[i] * sizeof(T) >= kSlotBytes / 8) {
        download(&(*dst)[i], dev + off[i], sizes[i]);
        ++i;
        continue;
      }
      check(ucg_event_record(compute_ev_, gpu_->stream()));
      check(ucg_stream_wait_event(d2h_, compute_ev_));
      const std::uint64_t base = off[i];
      std::size_t j = i;
      while (j < sizes.size() && sizes[j] * sizeof(T) < kSlotBytes / 8 &&
             (off[j] + sizes[j] - base) * sizeof(T) <= kSlotBytes)
        ++j;
      Slot& s = acquire_out();
      const std::uint64_t extent = (off[j - 1] + sizes[j - 1] - base) * sizeof(T);
      check(ucg_memcpy_d2h(s.buf, dev + base, extent, d2h_));
      check(ucg_event_record(s.ev, d2h_));
      s.drains.store(1);
      const std::size_t k0 = i, k1 = j;
      // one vector per piece: the allocations are spread over the pool
      pending_.push_back(work_pool().submit([&s, dst, &sizes, &off, k0, k1, base] {
        Release rel(s);
        check(ucg_event_synchronize(s.ev));
        const T* h = static_cast<const T*>(s.buf);
        constexpr std::size_t kBlk = 2048;
        work_pool().parallel_for((k1 - k0 + kBlk - 1) / kBlk, [&](std::size_t blk) {
          const std::size_t e = std::min(k1, k0 + (blk + 1) * kBlk);
          for (std::size_t k = k0 + blk * kBlk; k < e; ++k)
            (*dst)[k].assign(h + off[k] - base, h + off[k] - base + sizes[k]);
        });
      }));
      i = j;
    }
  }

  /// Waits for every copy and drain task of this pipe (outputs complete,
  /// slots reusable) and for the compute stream.
  void drain() {
    std::exception_ptr err;
    for (auto& d : pending_) {
      try {
        d->wait();
      } catch (...) {
        if (!err) err = std::current_exception();
      }
    }
    pending_.clear();
    for (Ring* r : {&in_, &out_})
      for (Slot& s : r->slot)
        if (s.busy) {
          ucg_event_synchronize(s.ev);
          s.busy = false;
        }
    gpu_->sync();
    if (err) std::rethrow_exception(err);
  }

 private:
  struct Slot {
    void* buf = nullptr;
    void* ev = nullptr;
    bool busy = false;                 // in ring: an H2D from it may be in flight
    std::atomic<int> drains{0};        // out ring: drain tasks still reading it
  };
  struct Ring {
    Slot slot[kSlots];
    int next = 0;
  };
  // releases one drain task's hold on an out slot when the task ends
  struct Release {
    Slot& s;
    explicit Release(Slot& slot) : s(slot) {}
    ~Release() { s.drains.fetch_sub(1); }
  };

  Slot& acquire_in() {
    Slot& s = in_.slot[in_.next];
    in_.next = (in_.next + 1) % kSlots;
    if (s.busy) {
      check(ucg_event_synchronize(s.ev));
      s.busy = false;
    }
    return s;
  }
  Slot& acquire_out() {
    Slot& s = out_.slot[out_.next];
    out_.next = (out_.next + 1) % kSlots;
    while (s.drains.load() > 0) std::this_thread::yield();  // its drain tasks are on the pool
    return s;
  }

  Gpu* gpu_;
  void* h2d_ = nullptr;
  void* d2h_ = nullptr;
  void* compute_ev_ = nullptr;
  void* h2d_ev_ = nullptr;
  Ring in_, out_;
  std::vector<std::shared_ptr<WorkPool::Done>> pending_;
};

}  // namespace ucores_b200
