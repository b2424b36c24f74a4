// gpu_context.hpp — per-GPU resources for the C++ drop-in and the mapping of
// C-ABI status codes onto the reference's exceptions.
//
// Header-only C++20 like the reference (proj/include/ucores). Requires the
// reference headers on the include path and links libucores_cuda.so.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ucores/errors.hpp"
#include "ucores_cuda.h"

namespace ucores_b200 {

/// Throws the reference exception that corresponds to a C-ABI failure. A
/// failing device call inside a kernel phase is a KernelPanic naming that
/// phase (ucores/errors.hpp:55-63, device.hpp:360,400,430); length and empty
/// errors keep their reference types (errors.hpp:80-83,112-115).
inline void check(int rc, const char* phase = "run") {
  if (rc == UCG_OK) return;
  const std::string msg = ucg_last_error();
  if (rc == UCG_ERR_LENGTH) throw ucores::LengthMismatch(msg);
  if (rc == UCG_ERR_EMPTY) throw ucores::EmptyDataset(msg);
  throw ucores::KernelPanic(phase, msg);
}

/// Grow-only device allocation owned by one GPU.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : ptr_(o.ptr_), bytes_(o.bytes_) { o.ptr_ = nullptr, o.bytes_ = 0; }
  ~DeviceBuffer() { reset(); }

  void* ensure(std::uint64_t bytes) {
    if (bytes <= bytes_ && ptr_) return ptr_;
    reset();
    void* p = nullptr;
    check(ucg_malloc(&p, bytes ? bytes : 16), "run");
    ptr_ = p;
    bytes_ = bytes ? bytes : 16;
    return ptr_;
  }
  void reset() {
    if (ptr_) ucg_free(ptr_);
    ptr_ = nullptr;
    bytes_ = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(ptr_);
  }
  std::uint64_t bytes() const { return bytes_; }

 private:
  void* ptr_ = nullptr;
  std::uint64_t bytes_ = 0;
};

/// Restores the calling thread's current device on scope exit, so binding a
/// Gpu never changes the device a caller (e.g. torch on the same thread)
/// launches on afterwards.
class DeviceGuard {
 public:
  DeviceGuard() {
    if (ucg_get_device(&prev_) != UCG_OK) prev_ = -1;
  }
  ~DeviceGuard() {
    if (prev_ >= 0) ucg_set_device(prev_);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;

 private:
  int prev_ = -1;
};

/// One B200: its ordinal, a non-blocking stream and reusable scratch. All
/// calls made through a Gpu first bind its device on the calling thread
/// (under a DeviceGuard at every call site).
class Gpu {
 public:
  explicit Gpu(int ordinal) : ordinal_(ordinal) {
    DeviceGuard guard;
    bind();
    check(ucg_stream_create(&stream_), "run");
  }
  Gpu(const Gpu&) = delete;
  Gpu& operator=(const Gpu&) = delete;
  ~Gpu() {
    attach_.reset();  // the attachment (HostPipe) drains this GPU's streams first
    for (Stage& st : stages_)
      if (st.ptr) ucg_host_free(st.ptr);
    if (stream_) {
      DeviceGuard guard;
      ucg_set_device(ordinal_);
      ucg_stream_destroy(stream_);
    }
  }

  /// Pinned host staging (grow-only) by slot: packs many small payloads into
  /// one DMA. A slot's contents are in use until the next sync().
  void* host_stage(int slot, std::uint64_t bytes) {
    if (slot >= static_cast<int>(stages_.size())) stages_.resize(slot + 1);
    Stage& st = stages_[slot];
    if (st.bytes < bytes) {
      if (st.ptr) ucg_host_free(st.ptr);
      st.ptr = nullptr;
      st.bytes = 0;
      check(ucg_host_alloc(&st.ptr, bytes), "run");
      st.bytes = bytes;
    }
    return st.ptr;
  }

  void bind() const { check(ucg_set_device(ordinal_), "run"); }
  int ordinal() const { return ordinal_; }
  void* stream() const { return stream_; }
  void sync() const { check(ucg_stream_synchronize(stream_), "run"); }

  /// Scratch slots (grow-only), addressed by small integer ids per op.
  DeviceBuffer& scratch(int slot) {
    if (slot >= static_cast<int>(scratch_.size())) scratch_.resize(slot + 1);
    return scratch_[slot];
  }

  /// Serialises use of this GPU's stream/scratch between host threads.
  std::mutex& mutex() { return mu_; }

  /// One T per GPU (T(Gpu&)), created on first use and destroyed before the
  /// GPU's stream: the transfer pipeline (host_pipe.hpp) lives here.
  template <class T>
  T& attached() {
    std::lock_guard<std::mutex> lk(attach_mu_);
    if (!attach_) attach_ = std::make_shared<T>(*this);
    return *static_cast<T*>(attach_.get());
  }

  void h2d(void* dst, const void* src, std::uint64_t bytes) { check(ucg_memcpy_h2d(dst, src, bytes, stream_)); }
  void d2h(void* dst, const void* src, std::uint64_t bytes) { check(ucg_memcpy_d2h(dst, src, bytes, stream_)); }

 private:
  struct Stage {
    void* ptr = nullptr;
    std::uint64_t bytes = 0;
  };
  int ordinal_;
  void* stream_ = nullptr;
  std::vector<DeviceBuffer> scratch_;
  std::vector<Stage> stages_;
  std::mutex mu_;
  std::mutex attach_mu_;
  std::shared_ptr<void> attach_;
};

/// Number of CUDA devices visible (0 when none; never throws for "no device").
inline int gpu_count() {
  int n = 0;
  if (ucg_device_count(&n) != UCG_OK) return 0;
  return n;
}

/// All visible GPUs, or the first `limit` of them.
inline std::vector<std::unique_ptr<Gpu>> open_gpus(int limit = -1) {
  const int n = gpu_count();
  if (n == 0) throw ucores::Error("ucores_b200: no CUDA device (the GPU path has no CPU fallback)");
  const int use = limit > 0 && limit < n ? limit : n;
  std::vector<std::unique_ptr<Gpu>> out;
  for (int i = 0; i < use; ++i) out.push_back(std::make_unique<Gpu>(i));
  return out;
}

}  // namespace ucores_b200
