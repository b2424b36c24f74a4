// device_ops.hpp — name-keyed device bodies for registered kernels.
//
// The reference's run() is a host virtual called per gid
// (ucores/kernel.hpp:203,212) and cannot execute on a GPU, so each kernel
// name that should run on a B200 maps to a DeviceOp:
//   run_tasks  seam A (ClusterDriver::run_wave, engine.hpp:34-39): executes
//              a batch of same-kernel Tasks on one GPU in ONE launch and
//              returns the Elements the full host lifecycle would return;
//   run_phase  seam B (KernelExecutor::execute, kernel.hpp:219-234): the
//              class-D run() phase over the KernelContext buffers, leaving
//              map_parameters / map_return_value on the host.
// A kernel without a DeviceOp fails with KernelPanic("run") on the GPU
// path: there is no CPU fallback.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "ucores/element.hpp"
#include "ucores/errors.hpp"
#include "ucores/kernel.hpp"
#include "ucores/task.hpp"
#include "ucores_b200/gpu_context.hpp"
#include "ucores_b200/host_pipe.hpp"
#include "ucores_b200/kernels.hpp"

namespace ucores_b200 {

/// A task of a batch failed before or inside its device body. `phase` follows
/// the reference lifecycle (map_parameters / run / map_return_value).
class TaskFailure : public std::runtime_error {
 public:
  TaskFailure(std::size_t index, std::string phase, const std::string& detail)
      : std::runtime_error(detail), index_(index), phase_(std::move(phase)) {}
  std::size_t index() const { return index_; }
  const std::string& phase() const { return phase_; }

 private:
  std::size_t index_;
  std::string phase_;
};

using TaskBatch = std::span<const ucores::Task* const>;

struct DeviceOp {
  ucores::KernelArity arity = ucores::KernelArity::Unary;
  std::function<std::vector<ucores::Element>(Gpu&, TaskBatch)> run_tasks;
  std::function<void(Gpu&, ucores::KernelContext&)> run_phase;
};

class DeviceOpRegistry {
 public:
  void add(const std::string& name, DeviceOp op) {
    auto [it, inserted] = ops_.emplace(name, std::move(op));
    if (!inserted) throw ucores::DuplicateKernelName("device op already registered: " + name);
  }
  const DeviceOp* find(std::string_view name) const {
    auto it = ops_.find(name);
    return it == ops_.end() ? nullptr : &it->second;
  }
  bool contains(std::string_view name) const { return find(name) != nullptr; }

 private:
  std::map<std::string, DeviceOp, std::less<>> ops_;
};

namespace detail {

inline std::uint64_t align_up(std::uint64_t v, std::uint64_t a) { return (v + a - 1) / a * a; }

// Input accessors that fail like the host kernel's map_parameters would.
template <class T>
std::span<const T> input_view(const ucores::Element& e, std::size_t index) {
  try {
    if constexpr (std::is_same_v<T, float>) return e.as_f32();
    else if constexpr (std::is_same_v<T, std::int64_t>) return e.as_i64();
    else return e.as_bytes();
  } catch (const std::exception& ex) {
    throw TaskFailure(index, "map_parameters", ex.what());
  }
}

// Offsets (in elements of T) of `sizes` packed at `align`-element boundaries.
inline std::vector<std::uint64_t> pack_offsets(const std::vector<std::uint64_t>& sizes, std::uint64_t align,
                                               std::uint64_t* total) {
  std::vector<std::uint64_t> off(sizes.size());
  std::uint64_t o = 0;
  for (std::size_t i = 0; i < sizes.size(); ++i) {
    off[i] = o;
    o += align_up(sizes[i], align);
  }
  *total = std::max<std::uint64_t>(o, align);
  return off;
}

template <class T>
std::vector<std::span<const std::uint8_t>> as_bytes(const std::vector<std::span<const T>>& in) {
  std::vector<std::span<const std::uint8_t>> b;
  b.reserve(in.size());
  for (const auto& v : in) b.emplace_back(reinterpret_cast<const std::uint8_t*>(v.data()), v.size_bytes());
  return b;
}
inline std::vector<std::uint64_t> scaled(const std::vector<std::uint64_t>& v, std::uint64_t k) {
  std::vector<std::uint64_t> o(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) o[i] = v[i] * k;
  return o;
}

/// Elements out of a pipe download (the vectors are complete after drain()).
template <class T>
std::vector<ucores::Element> to_elements(std::vector<std::vector<T>>&& v) {
  std::vector<ucores::Element> out;
  out.reserve(v.size());
  for (auto& x : v) {
    if constexpr (std::is_same_v<T, float>) out.push_back(ucores::Element::f32(std::move(x)));
    else if constexpr (std::is_same_v<T, std::int64_t>) out.push_back(ucores::Element::i64(std::move(x)));
    else out.push_back(ucores::Element::bytes(std::move(x)));
  }
  return out;
}

inline int op_code(kernels::ReduceOp op) { return op == kernels::ReduceOp::Max ? UCG_OP_MAX : UCG_OP_SUM; }

// Many small payloads (a wave of one-float elements) move packed through the
// pipe's pinned slots and run as ONE launch; large ones stream element by
// element (host_pipe.hpp).
inline bool pack_pieces(std::size_t count, std::uint64_t bytes) {
  return count > 8 && bytes / count < (256u << 10);
}

}  // namespace detail

namespace device_ops {

/// axpb: y = fl(fl(a*x)+b) — every task's element in one flat launch.
inline DeviceOp affine_f32(float a, float b) {
  DeviceOp op;
  op.arity = ucores::KernelArity::Unary;
  op.run_tasks = [a, b](Gpu& g, TaskBatch tasks) {
    std::vector<std::span<const float>> in;
    std::vector<std::uint64_t> sizes;
    for (std::size_t i = 0; i < tasks.size(); ++i) {
      in.push_back(detail::input_view<float>(tasks[i]->inputs.at(0), i));
      sizes.push_back(in.back().size());
    }
    std::uint64_t bytes = 0;
    for (std::uint64_t n : sizes) bytes += n * 4;
    const bool packed = detail::pack_pieces(in.size(), bytes);
    // packed: back to back (the flat map does not care where elements
    // start); streamed: each element on a 256-byte boundary
    std::uint64_t total = 0;
    const auto off = detail::pack_offsets(sizes, packed ? 1 : 64, &total);
    float* x = static_cast<float*>(g.scratch(0).ensure(total * 4));
    float* y = static_cast<float*>(g.scratch(1).ensure(total * 4));
    std::vector<std::vector<float>> outs(in.size());
    HostPipe& pipe = g.attached<HostPipe>();
    HostPipe::Scope pipe_scope(pipe);  // drains before outs / in / off go, also when a call throws
    if (packed) {
      // many small elements: packed into slots, one launch, packed back
      pipe.upload_pieces(x, detail::as_bytes(in), detail::scaled(off, 4));
      pipe.compute_after_upload();
      check(ucg_map_affine_f32(x, y, total, a, b, g.stream()));
      pipe.download_pieces(&outs, y, sizes, off);
    } else {
      // per element: its upload, its launch as soon as it lands, its
      // download while the next element is copied in; the output vectors
      // are allocated by pool threads meanwhile
      std::vector<std::shared_ptr<WorkPool::Done>> ready(in.size());
      for (std::size_t i = 0; i < in.size(); ++i) ready[i] = pipe.prepare(&outs[i], sizes[i]);
      for (std::size_t i = 0; i < in.size(); ++i) {
        pipe.upload(x + off[i], in[i].data(), in[i].size_bytes());
        pipe.compute_after_upload();
        check(ucg_map_affine_f32(x + off[i], y + off[i], sizes[i], a, b, g.stream()));
        pipe.download(&outs[i], y + off[i], sizes[i], ready[i]);
      }
    }
    pipe.drain();
    return detail::to_elements(std::move(outs));
  };
  op.run_phase = [a, b](Gpu& g, ucores::KernelContext& ctx) {
    auto x = ctx.buffer<float>("x");
    auto y = ctx.buffer<float>("y");
    float* dx = static_cast<float*>(g.scratch(0).ensure(x.size() * 4));
    float* dy = static_cast<float*>(g.scratch(1).ensure(x.size() * 4));
    g.h2d(dx, x.data(), x.size_bytes());
    check(ucg_map_affine_f32(dx, dy, x.size(), a, b, g.stream()));
    g.d2h(y.data(), dy, y.size_bytes());
    g.sync();
  };
  return op;
}

/// psum / pmax: every task's partition in ONE segmented-reduce launch.
inline DeviceOp partition_reduce_f32(kernels::ReduceOp rop) {
  DeviceOp op;
  op.arity = ucores::KernelArity::Unary;
  const int code = detail::op_code(rop);
  op.run_tasks = [code](Gpu& g, TaskBatch tasks) {
    std::vector<std::span<const float>> in;
    std::vector<std::uint64_t> sizes;
    for (std::size_t i = 0; i < tasks.size(); ++i) {
      in.push_back(detail::input_view<float>(tasks[i]->inputs.at(0), i));
      sizes.push_back(in.back().size());
    }
    std::uint64_t total = 0;
    const auto off = detail::pack_offsets(sizes, 64, &total);
    float* x = static_cast<float*>(g.scratch(0).ensure(total * 4));
    HostPipe& pipe = g.attached<HostPipe>();
    HostPipe::Scope pipe_scope(pipe);
    pipe.upload_pieces(x, detail::as_bytes(in), detail::scaled(off, 4));
    pipe.compute_after_upload();
    ucg_segtab* tab = nullptr;
    check(ucg_segtab_create(off.data(), sizes.data(), sizes.size(), &tab));
    std::uint64_t nscratch = 0;
    ucg_segtab_scratch_floats(tab, &nscratch);
    float* scratch = static_cast<float*>(g.scratch(2).ensure(nscratch * 4));
    float* part = static_cast<float*>(g.scratch(3).ensure(sizes.size() * 4));
    const int rc = ucg_segment_reduce_f32(x, tab, code, scratch, part, g.stream());
    std::vector<float> host(sizes.size());
    if (rc == UCG_OK) g.d2h(host.data(), part, host.size() * 4);
    try {
      pipe.drain();
    } catch (...) {
      ucg_segtab_destroy(tab);
      throw;
    }
    ucg_segtab_destroy(tab);
    check(rc);
    std::vector<ucores::Element> out;
    for (float v : host) out.push_back(ucores::Element::f32({v}));
    return out;
  };
  op.run_phase = [code](Gpu& g, ucores::KernelContext& ctx) {
    // run(gid): partial[gid] = tree over aligned block gid of kBlock elements
    auto x = ctx.buffer<float>("x");
    auto part = ctx.buffer<float>("partial");
    const std::uint64_t B = kernels::PartitionReduce::kBlock;
    std::vector<std::uint64_t> begin(part.size()), len(part.size());
    for (std::size_t i = 0; i < part.size(); ++i) {
      begin[i] = i * B;
      len[i] = std::min<std::uint64_t>(B, x.size() - i * B);
    }
    float* dx = static_cast<float*>(g.scratch(0).ensure(x.size_bytes() + 16));
    g.h2d(dx, x.data(), x.size_bytes());
    ucg_segtab* tab = nullptr;
    check(ucg_segtab_create(begin.data(), len.data(), len.size(), &tab));
    std::uint64_t nscratch = 0;
    ucg_segtab_scratch_floats(tab, &nscratch);
    float* scratch = static_cast<float*>(g.scratch(2).ensure(nscratch * 4));
    float* dp = static_cast<float*>(g.scratch(3).ensure(part.size_bytes() + 16));
    const int rc = ucg_segment_reduce_f32(dx, tab, code, scratch, dp, g.stream());
    if (rc == UCG_OK) g.d2h(part.data(), dp, part.size_bytes());
    g.sync();
    ucg_segtab_destroy(tab);
    check(rc);
  };
  return op;
}

namespace detail2 {
template <class T>
std::vector<ucores::Element> elementwise_tasks(Gpu& g, TaskBatch tasks, int code) {
  std::vector<std::span<const T>> A, B;
  std::vector<std::uint64_t> sizes;
  for (std::size_t i = 0; i < tasks.size(); ++i) {
    if (tasks[i]->inputs.size() != 2) throw TaskFailure(i, "dispatch", "REDUCE_PAIR task must carry 2 inputs");
    A.push_back(detail::input_view<T>(tasks[i]->inputs[0], i));
    B.push_back(detail::input_view<T>(tasks[i]->inputs[1], i));
    if (A.back().size() != B.back().size())
      throw TaskFailure(i, "map_parameters", "vector lengths differ");  // LengthMismatch in the host kernel
    sizes.push_back(A.back().size());
  }
  std::uint64_t total = 0;
  const auto off = detail::pack_offsets(sizes, 16, &total);
  T* a = static_cast<T*>(g.scratch(0).ensure(total * sizeof(T)));
  T* b = static_cast<T*>(g.scratch(1).ensure(total * sizeof(T)));
  T* c = static_cast<T*>(g.scratch(2).ensure(total * sizeof(T)));
  std::vector<std::vector<T>> outs;
  HostPipe& pipe = g.attached<HostPipe>();
  HostPipe::Scope pipe_scope(pipe);
  pipe.upload_pieces(a, detail::as_bytes(A), detail::scaled(off, sizeof(T)));
  pipe.upload_pieces(b, detail::as_bytes(B), detail::scaled(off, sizeof(T)));
  pipe.compute_after_upload();
  if constexpr (std::is_same_v<T, float>) check(ucg_elementwise2_f32(a, b, c, total, code, g.stream()));
  else check(ucg_elementwise2_i64(a, b, c, total, g.stream()));
  pipe.download_pieces(&outs, c, sizes, off);
  pipe.drain();
  return detail::to_elements(std::move(outs));
}

template <class T>
void elementwise_phase(Gpu& g, ucores::KernelContext& ctx, int code) {
  auto a = ctx.buffer<T>("a");
  auto b = ctx.buffer<T>("b");
  auto c = ctx.buffer<T>("c");
  T* da = static_cast<T*>(g.scratch(0).ensure(a.size_bytes() + 16));
  T* db = static_cast<T*>(g.scratch(1).ensure(b.size_bytes() + 16));
  T* dc = static_cast<T*>(g.scratch(2).ensure(c.size_bytes() + 16));
  g.h2d(da, a.data(), a.size_bytes());
  g.h2d(db, b.data(), b.size_bytes());
  if constexpr (std::is_same_v<T, float>) check(ucg_elementwise2_f32(da, db, dc, c.size(), code, g.stream()));
  else check(ucg_elementwise2_i64(da, db, dc, c.size(), g.stream()));
  g.d2h(c.data(), dc, c.size_bytes());
  g.sync();
}
}  // namespace detail2

/// sum2 / max2 / vectoradd: all ReducePair tasks of a wave in one launch.
inline DeviceOp elementwise2_f32(kernels::ReduceOp rop) {
  DeviceOp op;
  op.arity = ucores::KernelArity::Binary;
  const int code = detail::op_code(rop);
  op.run_tasks = [code](Gpu& g, TaskBatch t) { return detail2::elementwise_tasks<float>(g, t, code); };
  op.run_phase = [code](Gpu& g, ucores::KernelContext& ctx) { detail2::elementwise_phase<float>(g, ctx, code); };
  return op;
}

/// isum2: exact 64-bit integer sum combine.
inline DeviceOp elementwise2_i64() {
  DeviceOp op;
  op.arity = ucores::KernelArity::Binary;
  op.run_tasks = [](Gpu& g, TaskBatch t) { return detail2::elementwise_tasks<std::int64_t>(g, t, UCG_OP_SUM); };
  op.run_phase = [](Gpu& g, ucores::KernelContext& ctx) {
    detail2::elementwise_phase<std::int64_t>(g, ctx, UCG_OP_SUM);
  };
  return op;
}

/// pi: every task {seed, samples} of a wave in one launch -> {hits, samples}.
inline DeviceOp pi() {
  DeviceOp op;
  op.arity = ucores::KernelArity::Unary;
  op.run_tasks = [](Gpu& g, TaskBatch tasks) {
    std::vector<std::uint64_t> seeds, samples;
    for (std::size_t i = 0; i < tasks.size(); ++i) {
      auto v = detail::input_view<std::int64_t>(tasks[i]->inputs.at(0), i);
      if (v.size() != 2) throw TaskFailure(i, "map_parameters", "pi element must be {task_seed, samples}");
      seeds.push_back(static_cast<std::uint64_t>(v[0]));
      samples.push_back(static_cast<std::uint64_t>(v[1]));
    }
    std::int64_t* hits = static_cast<std::int64_t*>(g.scratch(0).ensure(seeds.size() * 8));
    check(ucg_pi_hits(seeds.data(), samples.data(), seeds.size(), hits, g.stream()));
    std::vector<std::int64_t> h(seeds.size());
    g.d2h(h.data(), hits, h.size() * 8);
    g.sync();
    std::vector<ucores::Element> out;
    for (std::size_t i = 0; i < h.size(); ++i)
      out.push_back(ucores::Element::i64({h[i], static_cast<std::int64_t>(samples[i])}));
    return out;
  };
  op.run_phase = [](Gpu& g, ucores::KernelContext& ctx) {
    auto params = ctx.buffer<std::int64_t>("params");
    auto flags = ctx.buffer<std::uint8_t>("hits");
    std::uint8_t* d = static_cast<std::uint8_t*>(g.scratch(0).ensure(flags.size() + 16));
    check(ucg_pi_flags(static_cast<std::uint64_t>(params[0]), flags.size(), d, g.stream()));
    g.d2h(flags.data(), d, flags.size());
    g.sync();
  };
  return op;
}

/// sobel: all bands of a wave in one launch.
inline DeviceOp sobel(std::size_t width) {
  DeviceOp op;
  op.arity = ucores::KernelArity::Unary;
  op.run_tasks = [width](Gpu& g, TaskBatch tasks) {
    std::vector<std::span<const std::uint8_t>> in;
    std::vector<std::uint64_t> in_sz, rows, out_sz;
    for (std::size_t i = 0; i < tasks.size(); ++i) {
      in.push_back(detail::input_view<std::uint8_t>(tasks[i]->inputs.at(0), i));
      const std::uint64_t n = in.back().size();
      if (width == 0 || n % width != 0 || n / width < 2)
        throw TaskFailure(i, "map_parameters", "band is not (rows+2) x width");
      in_sz.push_back(n);
      rows.push_back(n / width - 2);
      out_sz.push_back(rows.back() * width);
    }
    std::uint64_t tin = 0, tout = 0;
    const auto in_off = detail::pack_offsets(in_sz, 16, &tin);
    const auto out_off = detail::pack_offsets(out_sz, 16, &tout);
    std::uint8_t* din = static_cast<std::uint8_t*>(g.scratch(0).ensure(tin));
    std::uint8_t* dout = static_cast<std::uint8_t*>(g.scratch(1).ensure(tout));
    std::vector<std::vector<std::uint8_t>> outs;
    HostPipe& pipe = g.attached<HostPipe>();
    HostPipe::Scope pipe_scope(pipe);
    pipe.upload_pieces(din, in, in_off);
    pipe.compute_after_upload();
    check(ucg_sobel_bands_u8(din, in_off.data(), dout, out_off.data(), rows.data(), rows.size(), width,
                             g.stream()));
    pipe.download_pieces(&outs, dout, out_sz, out_off);
    pipe.drain();
    return detail::to_elements(std::move(outs));
  };
  op.run_phase = [width](Gpu& g, ucores::KernelContext& ctx) {
    auto in = ctx.buffer<std::uint8_t>("in");
    auto out = ctx.buffer<std::uint8_t>("out");
    const std::uint64_t rows = out.size() / width;
    std::uint8_t* din = static_cast<std::uint8_t*>(g.scratch(0).ensure(in.size() + 16));
    std::uint8_t* dout = static_cast<std::uint8_t*>(g.scratch(1).ensure(out.size() + 16));
    g.h2d(din, in.data(), in.size());
    check(ucg_sobel_band_u8(din, dout, rows, width, g.stream()));
    g.d2h(out.data(), dout, out.size());
    g.sync();
  };
  return op;
}

/// wordcount: word-start flags of every chunk on the GPU, tokens counted on
/// the host from the flags (the kernel's map_return_value). Chunks below
/// min_device_bytes take the kernel's own declared host path (selective
/// execution) — the same table either way.
inline DeviceOp wordcount(std::uint64_t min_device_bytes) {
  DeviceOp op;
  op.arity = ucores::KernelArity::Unary;
  op.run_tasks = [min_device_bytes](Gpu& g, TaskBatch tasks) {
    std::vector<std::span<const std::uint8_t>> in;
    std::vector<std::uint64_t> sizes;
    for (std::size_t i = 0; i < tasks.size(); ++i) {
      in.push_back(detail::input_view<std::uint8_t>(tasks[i]->inputs.at(0), i));
      sizes.push_back(in.back().size());
    }
    std::uint64_t total = 0;
    const auto off = detail::pack_offsets(sizes, 16, &total);
    std::uint8_t* din = static_cast<std::uint8_t*>(g.scratch(0).ensure(total));
    std::uint8_t* dfl = static_cast<std::uint8_t*>(g.scratch(1).ensure(total));
    std::vector<std::uint8_t> flags;
    HostPipe& pipe = g.attached<HostPipe>();
    HostPipe::Scope pipe_scope(pipe);
    pipe.upload_pieces(din, in, off);
    pipe.compute_after_upload();
    for (std::size_t i = 0; i < in.size(); ++i) {
      if (sizes[i] < min_device_bytes || !sizes[i]) continue;
      check(ucg_word_start_flags(din + off[i], sizes[i], dfl + off[i], g.stream()));
    }
    pipe.download(&flags, dfl, total);
    pipe.drain();
    std::vector<ucores::Element> out;
    for (std::size_t i = 0; i < in.size(); ++i) {
      if (sizes[i] < min_device_bytes) out.push_back(kernels::WordCount::table_host(in[i]));
      else out.push_back(kernels::WordCount::table_from_flags(in[i], flags.data() + off[i]));
    }
    return out;
  };
  op.run_phase = [](Gpu& g, ucores::KernelContext& ctx) {
    auto in = ctx.buffer<std::uint8_t>("in");
    auto fl = ctx.buffer<std::uint8_t>("flags");
    std::uint8_t* din = static_cast<std::uint8_t*>(g.scratch(0).ensure(in.size() + 16));
    std::uint8_t* dfl = static_cast<std::uint8_t*>(g.scratch(1).ensure(in.size() + 16));
    g.h2d(din, in.data(), in.size());
    check(ucg_word_start_flags(din, in.size(), dfl, g.stream()));
    g.d2h(fl.data(), dfl, fl.size());
    g.sync();
  };
  return op;
}

/// matmul: C = A.B per task on the tensor cores (tolerance, not bit-exact):
/// fp32-faithful 3xTF32 (ucg_gemm_f32, rms error ~3e-6 of rms(C), the
/// default: the reference kernel is fp32) or plain TF32 (ucg_gemm_tf32, 3x
/// the rate, rms error ~7e-4).
inline DeviceOp matmul_tc(std::size_t n, bool fp32_faithful = true) {
  DeviceOp op;
  op.arity = ucores::KernelArity::Unary;
  auto body = [n, fp32_faithful](Gpu& g, const float* ab_host, float* c_host) {
    float* dab = static_cast<float*>(g.scratch(0).ensure(2 * n * n * 4));
    float* dc = static_cast<float*>(g.scratch(1).ensure(n * n * 4));
    g.h2d(dab, ab_host, 2 * n * n * 4);
    check((fp32_faithful ? ucg_gemm_f32 : ucg_gemm_tf32)(dab, dab + n * n, dc, n, g.stream()));
    g.d2h(c_host, dc, n * n * 4);
    g.sync();
  };
  op.run_tasks = [n, fp32_faithful](Gpu& g, TaskBatch tasks) {
    std::vector<std::vector<float>> outs(tasks.size());
    for (std::size_t i = 0; i < tasks.size(); ++i) {
      auto ab = detail::input_view<float>(tasks[i]->inputs.at(0), i);
      if (ab.size() != 2 * n * n) throw TaskFailure(i, "map_parameters", "matmul element must hold A||B");
    }
    // two device slots: task i+1's upload overlaps task i's product, task
    // i's C download overlaps task i+1's
    HostPipe& pipe = g.attached<HostPipe>();
    HostPipe::Scope pipe_scope(pipe);
    for (std::size_t i = 0; i < tasks.size(); ++i) {
      float* dab = static_cast<float*>(g.scratch(4 + 2 * (i & 1)).ensure(2 * n * n * 4));
      float* dc = static_cast<float*>(g.scratch(5 + 2 * (i & 1)).ensure(n * n * 4));
      pipe.upload(dab, tasks[i]->inputs[0].as_f32().data(), 2 * n * n * 4);
      pipe.compute_after_upload();
      check((fp32_faithful ? ucg_gemm_f32 : ucg_gemm_tf32)(dab, dab + n * n, dc, n, g.stream()));
      pipe.download(&outs[i], dc, n * n);
    }
    pipe.drain();
    return detail::to_elements(std::move(outs));
  };
  op.run_phase = [body](Gpu& g, ucores::KernelContext& ctx) {
    auto ab = ctx.buffer<float>("ab");
    auto c = ctx.buffer<float>("c");
    body(g, ab.data(), c.data());
  };
  return op;
}

}  // namespace device_ops

/// Parameters of the workload kernels registered under the reference names.
struct WorkloadParams {
  float a = 2.0f, b = 1.0f;     // axpb
  std::size_t sobel_width = 16384;
  std::size_t matmul_n = 8192;
  bool matmul_fp32 = true;  // fp32-faithful 3xTF32 (false: plain TF32)
  std::uint64_t wordcount_min_device_bytes = 65536;  // EngineConfig::min_device_bytes (engine.hpp:18)
};

/// Registers the host kernels (reference API) and their device bodies under
/// the same names: axpb, psum, pmax, sum2, vectoradd, max2, isum2, pi,
/// sobel, matmul, wordcount.
inline void register_workload(ucores::KernelRegistry& reg, DeviceOpRegistry& ops, const WorkloadParams& p = {}) {
  using namespace kernels;
  reg.register_unary("axpb", [p] { return std::make_unique<Axpb>(p.a, p.b); });
  reg.register_unary("psum", [] { return std::make_unique<PartitionReduce>(ReduceOp::Sum); });
  reg.register_unary("pmax", [] { return std::make_unique<PartitionReduce>(ReduceOp::Max); });
  reg.register_binary("sum2", [] { return std::make_unique<Elementwise2F32>(ReduceOp::Sum); });
  reg.register_binary("vectoradd", [] { return std::make_unique<Elementwise2F32>(ReduceOp::Sum); });
  reg.register_binary("max2", [] { return std::make_unique<Elementwise2F32>(ReduceOp::Max); });
  reg.register_binary("isum2", [] { return std::make_unique<Elementwise2I64>(); });
  reg.register_unary("pi", [] { return std::make_unique<Pi>(); });
  reg.register_unary("sobel", [p] { return std::make_unique<Sobel>(p.sobel_width); });
  reg.register_unary("matmul", [p] { return std::make_unique<Matmul>(p.matmul_n); });
  reg.register_unary("wordcount", [p] { return std::make_unique<WordCount>(p.wordcount_min_device_bytes); });
  ops.add("wordcount", device_ops::wordcount(p.wordcount_min_device_bytes));
  ops.add("axpb", device_ops::affine_f32(p.a, p.b));
  ops.add("psum", device_ops::partition_reduce_f32(ReduceOp::Sum));
  ops.add("pmax", device_ops::partition_reduce_f32(ReduceOp::Max));
  ops.add("sum2", device_ops::elementwise2_f32(ReduceOp::Sum));
  ops.add("vectoradd", device_ops::elementwise2_f32(ReduceOp::Sum));
  ops.add("max2", device_ops::elementwise2_f32(ReduceOp::Max));
  ops.add("isum2", device_ops::elementwise2_i64());
  ops.add("pi", device_ops::pi());
  ops.add("sobel", device_ops::sobel(p.sobel_width));
  ops.add("matmul", device_ops::matmul_tc(p.matmul_n, p.matmul_fp32));
}

}  // namespace ucores_b200
