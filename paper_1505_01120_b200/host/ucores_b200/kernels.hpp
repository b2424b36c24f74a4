// kernels.hpp — the BASELINE workload kernels written against the reference
// kernel API (ucores/kernel.hpp:199-215). The reference ships no kernels
// (SURVEY.md §0); these host classes define each kernel's semantics and
// buffer contract, and every one has a device body in device_ops.hpp that
// produces bit-identical results (integer, map and tree-reduce kernels) or
// results within a stated tolerance (matmul on TF32 tensor cores).
//
// Buffer contract (the names the seam-B device bodies read and write):
//   axpb      x (f32, bound)          -> y (f32, n)          range n
//   psum/pmax x (f32, bound)          -> partial (f32, blocks of 4096) range blocks
//   sum2/max2/vectoradd a, b (f32)    -> c (f32)             range n
//   isum2     a, b (i64)              -> c (i64)             range n
//   pi        params {seed, samples} (i64) -> hits (u8, samples) range samples
//   sobel     in (u8, (rows+2)*w)     -> out (u8, rows*w)    range rows*w
//   matmul    ab (f32, 2n^2)          -> c (f32, n^2)        range n^2
//   wordcount in (u8, chunk)          -> flags (u8, chunk)   range chunk bytes
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "ucores/element.hpp"
#include "ucores/engine.hpp"
#include "ucores/errors.hpp"
#include "ucores/kernel.hpp"

namespace ucores_b200::kernels {

inline constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ull;

inline std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

enum class ReduceOp { Sum, Max };

inline float combine(ReduceOp op, float a, float b) { return op == ReduceOp::Max ? std::max(a, b) : a + b; }

/// The reduce_cl stage-2 pairing tree (ucores/engine.hpp:172-190) over a
/// contiguous range, in its recursive form: the root joins the complete
/// subtree of the largest power of two below n with the tree of the rest.
inline float pairing_tree(const float* x, std::size_t n, ReduceOp op) {
  if (n == 1) return x[0];
  std::size_t h = 1;
  while (h * 2 < n) h *= 2;
  return combine(op, pairing_tree(x, h, op), pairing_tree(x + h, n - h, op));
}

/// mapCL body y = a*x + b, evaluated as two IEEE roundings (no FMA).
class Axpb : public ucores::UnaryKernel {
 public:
  Axpb(float a, float b) : a_(a), b_(b) {}
  float a() const { return a_; }
  float b() const { return b_; }
  void map_parameters(ucores::KernelContext& ctx, const ucores::Element& in) override {
    x_ = ctx.bind<float>("x", in.as_f32());
    y_ = ctx.alloc<float>("y", x_.size());
    ctx.set_range(x_.size());
  }
  void run(ucores::KernelContext&, std::size_t gid) override {
    volatile float t = a_ * x_[gid];
    y_[gid] = t + b_;
  }
  ucores::Element map_return_value(ucores::KernelContext& ctx, const ucores::Element&) override {
    return ucores::Element::f32(ctx.take<float>("y"));
  }

 private:
  float a_, b_;
  std::span<float> x_, y_;
};

/// mapCLPartition psum / pmax: the pairing tree over the partition's
/// concatenated F32Array. run() reduces one aligned block of kBlock elements
/// (class D, one slot per gid); map_return_value joins the block roots with
/// the same tree. An empty partition concatenates to an empty ByteArray
/// (element.hpp:133) and fails in map_parameters, as in the reference.
class PartitionReduce : public ucores::UnaryKernel {
 public:
  static constexpr std::size_t kBlock = 4096;
  explicit PartitionReduce(ReduceOp op) : op_(op) {}
  ReduceOp op() const { return op_; }
  float empty_value() const { return op_ == ReduceOp::Max ? -INFINITY : 0.0f; }
  void map_parameters(ucores::KernelContext& ctx, const ucores::Element& in) override {
    x_ = ctx.bind<float>("x", in.as_f32());
    const std::size_t blocks = (x_.size() + kBlock - 1) / kBlock;
    part_ = ctx.alloc<float>("partial", blocks);
    ctx.set_range(blocks);
  }
  void run(ucores::KernelContext&, std::size_t gid) override {
    const std::size_t lo = gid * kBlock, hi = std::min(x_.size(), lo + kBlock);
    part_[gid] = pairing_tree(x_.data() + lo, hi - lo, op_);
  }
  ucores::Element map_return_value(ucores::KernelContext& ctx, const ucores::Element&) override {
    std::vector<float> p = ctx.take<float>("partial");
    return ucores::Element::f32({p.empty() ? empty_value() : pairing_tree(p.data(), p.size(), op_)});
  }

 private:
  ReduceOp op_;
  std::span<const float> x_;
  std::span<float> part_;
};

/// Fig-3 vectoradd and its max sibling: c = a (op) b.
class Elementwise2F32 : public ucores::BinaryKernel {
 public:
  explicit Elementwise2F32(ReduceOp op) : op_(op) {}
  ReduceOp op() const { return op_; }
  void map_parameters(ucores::KernelContext& ctx, const ucores::Element& l, const ucores::Element& r) override {
    a_ = ctx.bind<float>("a", l.as_f32());
    b_ = ctx.bind<float>("b", r.as_f32());
    if (a_.size() != b_.size()) throw ucores::LengthMismatch("vector lengths differ");
    c_ = ctx.alloc<float>("c", a_.size());
    ctx.set_range(a_.size());
  }
  void run(ucores::KernelContext&, std::size_t gid) override { c_[gid] = combine(op_, a_[gid], b_[gid]); }
  ucores::Element map_return_value(ucores::KernelContext& ctx, const ucores::Element&,
                                   const ucores::Element&) override {
    return ucores::Element::f32(ctx.take<float>("c"));
  }

 private:
  ReduceOp op_;
  std::span<float> a_, b_, c_;
};

/// Integer-sum combine (SPEC acceptance 5): c = a + b mod 2^64.
class Elementwise2I64 : public ucores::BinaryKernel {
 public:
  void map_parameters(ucores::KernelContext& ctx, const ucores::Element& l, const ucores::Element& r) override {
    a_ = ctx.bind<std::int64_t>("a", l.as_i64());
    b_ = ctx.bind<std::int64_t>("b", r.as_i64());
    if (a_.size() != b_.size()) throw ucores::LengthMismatch("vector lengths differ");
    c_ = ctx.alloc<std::int64_t>("c", a_.size());
    ctx.set_range(a_.size());
  }
  void run(ucores::KernelContext&, std::size_t gid) override {
    c_[gid] = static_cast<std::int64_t>(static_cast<std::uint64_t>(a_[gid]) + static_cast<std::uint64_t>(b_[gid]));
  }
  ucores::Element map_return_value(ucores::KernelContext& ctx, const ucores::Element&,
                                   const ucores::Element&) override {
    return ucores::Element::i64(ctx.take<std::int64_t>("c"));
  }

 private:
  std::span<std::int64_t> a_, b_, c_;
};

/// Monte-Carlo pi: {task_seed, samples} -> {hits, samples}.
class Pi : public ucores::UnaryKernel {
 public:
  static int hit(std::uint64_t seed, std::uint64_t gid) {
    const std::uint64_t s0 = seed ^ (gid * kGamma);
    const std::uint64_t z1 = mix64(s0 + kGamma), z2 = mix64(s0 + 2 * kGamma);
    const double x = static_cast<double>(z1 >> 32) / 4294967296.0;
    const double y = static_cast<double>(z2 >> 32) / 4294967296.0;
    volatile double xx = x * x, yy = y * y;
    return (xx + yy) <= 1.0;
  }
  void map_parameters(ucores::KernelContext& ctx, const ucores::Element& in) override {
    auto v = in.as_i64();
    if (v.size() != 2) throw ucores::Error("pi element must be {task_seed, samples}");
    seed_ = static_cast<std::uint64_t>(v[0]);
    samples_ = static_cast<std::uint64_t>(v[1]);
    ctx.set_range(samples_);
    if (!ucores::plan_offload(ucores::EngineConfig{}, samples_, samples_)) {
      ctx.set_device_execution(false);  // selective execution
      return;
    }
    ctx.bind<std::int64_t>("params", v);  // {seed, samples} for a device run() body
    flags_ = ctx.alloc<std::uint8_t>("hits", samples_);
  }
  void run(ucores::KernelContext&, std::size_t gid) override {
    flags_[gid] = static_cast<std::uint8_t>(hit(seed_, gid));
  }
  ucores::Element map_return_value(ucores::KernelContext& ctx, const ucores::Element&) override {
    std::int64_t h = 0;
    if (ctx.device_execution()) {
      for (std::uint8_t f : ctx.take<std::uint8_t>("hits")) h += f;
    } else {
      for (std::uint64_t g = 0; g < samples_; ++g) h += hit(seed_, g);
    }
    return ucores::Element::i64({h, static_cast<std::int64_t>(samples_)});
  }

 private:
  std::uint64_t seed_ = 0, samples_ = 0;
  std::span<std::uint8_t> flags_;
};

/// 3x3 Sobel over a row band with one halo row above and below (C4).
class Sobel : public ucores::UnaryKernel {
 public:
  explicit Sobel(std::size_t width) : w_(width) {}
  std::size_t width() const { return w_; }
  void map_parameters(ucores::KernelContext& ctx, const ucores::Element& in) override {
    in_ = ctx.bind<std::uint8_t>("in", in.as_bytes());
    if (w_ == 0 || in_.size() % w_ != 0 || in_.size() / w_ < 2) throw ucores::Error("band is not (rows+2) x width");
    rows_ = in_.size() / w_ - 2;
    out_ = ctx.alloc<std::uint8_t>("out", rows_ * w_);
    ctx.set_range(rows_ * w_);
  }
  int px(std::size_t r, std::ptrdiff_t c) const {
    if (c < 0 || static_cast<std::size_t>(c) >= w_) return 0;
    return in_[r * w_ + static_cast<std::size_t>(c)];
  }
  void run(ucores::KernelContext&, std::size_t gid) override {
    const std::size_t r = gid / w_;
    const auto c = static_cast<std::ptrdiff_t>(gid % w_);
    const int gx = (px(r, c + 1) - px(r, c - 1)) + 2 * (px(r + 1, c + 1) - px(r + 1, c - 1)) +
                   (px(r + 2, c + 1) - px(r + 2, c - 1));
    const int gy = (px(r + 2, c - 1) + 2 * px(r + 2, c) + px(r + 2, c + 1)) -
                   (px(r, c - 1) + 2 * px(r, c) + px(r, c + 1));
    out_[gid] = static_cast<std::uint8_t>(std::min(255, std::abs(gx) + std::abs(gy)));
  }
  ucores::Element map_return_value(ucores::KernelContext& ctx, const ucores::Element&) override {
    return ucores::Element::bytes(ctx.take<std::uint8_t>("out"));
  }

 private:
  std::size_t w_, rows_ = 0;
  std::span<std::uint8_t> in_, out_;
};

/// WordCount: ByteArray chunk -> KeyCountTable. run() marks
/// word starts (class D, the "local data" flags buffer); map_return_value
/// walks the flags to cut tokens and counts them, keys in order of first
/// occurrence. Chunks below min_device_bytes decline device execution and
/// tokenize on the host (selective execution).
class WordCount : public ucores::UnaryKernel {
 public:
  static bool is_delim(std::uint8_t b) { return b == ' ' || b == '\t' || b == '\n' || b == '\r'; }
  explicit WordCount(std::uint64_t min_device_bytes) : min_(min_device_bytes) {}
  void map_parameters(ucores::KernelContext& ctx, const ucores::Element& in) override {
    bytes_ = in.as_bytes();
    ctx.set_range(bytes_.size());
    if (bytes_.size() < min_) {
      ctx.set_device_execution(false);
      return;
    }
    ctx.bind<std::uint8_t>("in", bytes_);
    flags_ = ctx.alloc<std::uint8_t>("flags", bytes_.size());
  }
  void run(ucores::KernelContext&, std::size_t gid) override {
    flags_[gid] = static_cast<std::uint8_t>(!is_delim(bytes_[gid]) && (gid == 0 || is_delim(bytes_[gid - 1])));
  }
  ucores::Element map_return_value(ucores::KernelContext& ctx, const ucores::Element&) override {
    if (ctx.device_execution()) {
      std::vector<std::uint8_t> f = ctx.take<std::uint8_t>("flags");
      return table_from_flags(bytes_, f.data());
    }
    return table_host(bytes_);  // "alternative compute function" on the host
  }

  /// Tokens cut at the flagged word starts, counted, keys in first-occurrence order.
  static ucores::Element table_from_flags(std::span<const std::uint8_t> bytes, const std::uint8_t* flags) {
    Counter c(bytes);
    const std::size_t n = bytes.size();
    for (std::size_t i = 0; i < n; ++i) {
      if (!flags[i]) continue;
      std::size_t e = i;
      while (e < n && !is_delim(bytes[e])) ++e;
      c.add(i, e);
      i = e;
    }
    return c.done();
  }
  /// The same table by direct host tokenisation.
  static ucores::Element table_host(std::span<const std::uint8_t> bytes) {
    Counter c(bytes);
    const std::size_t n = bytes.size();
    for (std::size_t i = 0; i < n;) {
      while (i < n && is_delim(bytes[i])) ++i;
      std::size_t e = i;
      while (e < n && !is_delim(bytes[e])) ++e;
      if (e > i) c.add(i, e);
      i = e;
    }
    return c.done();
  }

 private:
  struct Counter {
    std::span<const std::uint8_t> bytes;
    std::vector<std::pair<std::string, std::uint64_t>> table;
    std::map<std::string, std::size_t, std::less<>> index;
    explicit Counter(std::span<const std::uint8_t> b) : bytes(b) {}
    void add(std::size_t b, std::size_t e) {
      std::string key(reinterpret_cast<const char*>(bytes.data()) + b, e - b);
      auto it = index.find(key);
      if (it == index.end()) {
        index.emplace(key, table.size());
        table.emplace_back(std::move(key), 1);
      } else {
        table[it->second].second += 1;
      }
    }
    ucores::Element done() { return ucores::Element::table(std::move(table)); }
  };

 public:

 private:
  std::uint64_t min_;
  std::span<const std::uint8_t> bytes_;
  std::span<std::uint8_t> flags_;
};

/// Dense matmul (C5): F32Array A||B (2n^2) -> C = A.B (fp32, k ascending).
class Matmul : public ucores::UnaryKernel {
 public:
  explicit Matmul(std::size_t n) : n_(n) {}
  std::size_t n() const { return n_; }
  void map_parameters(ucores::KernelContext& ctx, const ucores::Element& in) override {
    ab_ = ctx.bind<float>("ab", in.as_f32());
    if (ab_.size() != 2 * n_ * n_) throw ucores::Error("matmul element must hold A||B");
    c_ = ctx.alloc<float>("c", n_ * n_);
    ctx.set_range(n_ * n_);
  }
  void run(ucores::KernelContext&, std::size_t gid) override {
    const std::size_t i = gid / n_, j = gid % n_;
    const float* A = ab_.data();
    const float* B = ab_.data() + n_ * n_;
    float acc = 0.0f;
    for (std::size_t k = 0; k < n_; ++k) {
      volatile float t = A[i * n_ + k] * B[k * n_ + j];
      acc = acc + t;
    }
    c_[gid] = acc;
  }
  ucores::Element map_return_value(ucores::KernelContext& ctx, const ucores::Element&) override {
    return ucores::Element::f32(ctx.take<float>("c"));
  }

 private:
  std::size_t n_;
  std::span<float> ab_, c_;
};

}  // namespace ucores_b200::kernels
