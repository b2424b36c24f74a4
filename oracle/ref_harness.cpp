// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// Drives the UNMODIFIED reference (the header-only C++20 `ucores` library,
// compiled from /root/reference/proj/include by oracle/Makefile, output in
// oracle/_ref/) on the workload kernels of BASELINE.json. The reference ships
// no kernels and no driver binary, so this file supplies:
//   * the workload kernels written against the reference kernel API
//     (ucores/kernel.hpp:199-215): axpb, psum, pmax, sum2/vectoradd, max2,
//     isum2, pi, sobel, matmul;
//   * DirectDriver, a ClusterDriver (ucores/engine.hpp:34-39) that executes
//     each task in place through the reference WorkerRuntime
//     (ucores/worker.hpp:40-72) with the reference retry rule
//     (ucores/scheduler.hpp:290-302). LocalClusterDriver cannot be used: it
//     does not compile under GCC 13 (local_cluster.hpp:41) and its 64 MiB
//     frame cap (wire.hpp:41) rejects the C2 partitions.
//
// Modes:
//   ref_harness golden               -> JSON golden vectors on stdout
//   ref_harness bench [options]      -> times the C2 pipeline on host cores
//
// It is the checker / CPU baseline, never the product.
#include <algorithm>
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <iostream>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <json.hpp>

#include "ucores/dataset.hpp"
#include "ucores/device.hpp"
#include "ucores/element.hpp"
#include "ucores/engine.hpp"
#include "ucores/errors.hpp"
#include "ucores/kernel.hpp"
#include "ucores/task.hpp"
#include "ucores/worker.hpp"

using namespace ucores;
using json = nlohmann::json;

namespace {

constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ull;

std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
float uniform01(std::uint64_t seed, std::uint64_t i) {
  return static_cast<float>(mix64(seed + (i + 1) * kGamma) >> 40) * (1.0f / 16777216.0f);
}

std::uint64_t fnv64(const void* p, std::size_t n) {
  const auto* b = static_cast<const unsigned char*>(p);
  std::uint64_t h = 0xcbf29ce484222325ull;
  for (std::size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
std::string hex64(std::uint64_t v) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%016" PRIx64, v);
  return buf;
}
std::string hexf(float f) {
  std::uint32_t u;
  std::memcpy(&u, &f, 4);
  char buf[16];
  std::snprintf(buf, sizeof buf, "%08x", u);
  return buf;
}

// ---- workload kernels in the reference API ---------------------------------

// Pairing tree (engine.hpp:172-190 rule) in its recursive form: the root
// combines the complete left subtree of the largest power of two below n
// with the tree over the rest.
template <class T, class Op>
T tree(const T* x, std::size_t n, Op op) {
  if (n == 1) return x[0];
  std::size_t h = 1;
  while (h * 2 < n) h *= 2;
  const T l = tree(x, h, op);
  const T r = tree(x + h, n - h, op);
  return op(l, r);
}
struct AddF {
  float operator()(float a, float b) const { return a + b; }
};
struct MaxF {
  float operator()(float a, float b) const { return std::max(a, b); }
};

class Axpb : public UnaryKernel {
 public:
  Axpb(float a, float b) : a_(a), b_(b) {}
  void map_parameters(KernelContext& ctx, const Element& in) override {
    x_ = ctx.bind<float>("x", in.as_f32());
    y_ = ctx.alloc<float>("y", x_.size());
    ctx.set_range(x_.size());
  }
  void run(KernelContext&, std::size_t gid) override {
    const float t = a_ * x_[gid];
    y_[gid] = t + b_;
  }
  Element map_return_value(KernelContext& ctx, const Element&) override {
    return Element::f32(ctx.take<float>("y"));
  }

 private:
  float a_, b_;
  std::span<float> x_, y_;
};

// psum / pmax: class-D chunk partials (each the tree over one aligned block
// of kBlock elements) + the tree over partials in map_return_value. Because
// blocks are aligned powers of two this equals the pairing tree over the
// whole partition for any kBlock.
template <class Op>
class PartitionTree : public UnaryKernel {
 public:
  static constexpr std::size_t kBlock = 4096;
  explicit PartitionTree(float empty) : empty_(empty) {}
  void map_parameters(KernelContext& ctx, const Element& in) override {
    x_ = ctx.bind<float>("x", in.as_f32());
    const std::size_t blocks = (x_.size() + kBlock - 1) / kBlock;
    part_ = ctx.alloc<float>("partial", blocks);
    ctx.set_range(blocks);
  }
  void run(KernelContext&, std::size_t gid) override {
    const std::size_t lo = gid * kBlock;
    const std::size_t hi = std::min(x_.size(), lo + kBlock);
    part_[gid] = tree(x_.data() + lo, hi - lo, Op{});
  }
  Element map_return_value(KernelContext& ctx, const Element&) override {
    std::vector<float> p = ctx.take<float>("partial");
    return Element::f32({p.empty() ? empty_ : tree(p.data(), p.size(), Op{})});
  }

 private:
  float empty_;
  std::span<const float> x_;
  std::span<float> part_;
};

// Fig-3 vectoradd and its max / i64 siblings, used as the
// reduce_cl combine: c[gid] = a[gid] (op) b[gid].
template <class T, class Op>
class Elementwise2 : public BinaryKernel {
 public:
  void map_parameters(KernelContext& ctx, const Element& l, const Element& r) override {
    if constexpr (std::is_same_v<T, float>) {
      a_ = ctx.bind<float>("a", l.as_f32());
      b_ = ctx.bind<float>("b", r.as_f32());
    } else {
      a_ = ctx.bind<std::int64_t>("a", l.as_i64());
      b_ = ctx.bind<std::int64_t>("b", r.as_i64());
    }
    if (a_.size() != b_.size()) throw LengthMismatch("vector lengths differ");
    c_ = ctx.alloc<T>("c", a_.size());
    ctx.set_range(a_.size());
  }
  void run(KernelContext&, std::size_t gid) override { c_[gid] = Op{}(a_[gid], b_[gid]); }
  Element map_return_value(KernelContext& ctx, const Element&, const Element&) override {
    if constexpr (std::is_same_v<T, float>) return Element::f32(ctx.take<float>("c"));
    else return Element::i64(ctx.take<std::int64_t>("c"));
  }

 private:
  std::span<T> a_, b_, c_;
};
struct AddI {
  std::int64_t operator()(std::int64_t a, std::int64_t b) const {
    return static_cast<std::int64_t>(static_cast<std::uint64_t>(a) + static_cast<std::uint64_t>(b));
  }
};

// SPEC.md:462-470 Monte-Carlo pi. Input I64Array {task_seed, task_samples},
// output {hits, samples}. run() writes one hit flag per gid (class D);
// map_return_value sums. Below the plan_offload threshold the kernel declines
// device execution and counts on the host (selective execution).
class Pi : public UnaryKernel {
 public:
  static int hit(std::uint64_t seed, std::uint64_t gid) {
    const std::uint64_t s0 = seed ^ (gid * kGamma);
    const std::uint64_t z1 = mix64(s0 + kGamma);
    const std::uint64_t z2 = mix64(s0 + 2 * kGamma);
    const double x = static_cast<double>(z1 >> 32) / 4294967296.0;
    const double y = static_cast<double>(z2 >> 32) / 4294967296.0;
    const double xx = x * x;
    const double yy = y * y;
    return (xx + yy) <= 1.0;
  }
  void map_parameters(KernelContext& ctx, const Element& in) override {
    auto v = in.as_i64();
    seed_ = static_cast<std::uint64_t>(v[0]);
    samples_ = static_cast<std::uint64_t>(v[1]);
    ctx.set_range(samples_);
    if (!plan_offload(EngineConfig{}, samples_, samples_)) {
      ctx.set_device_execution(false);
      return;
    }
    flags_ = ctx.alloc<std::uint8_t>("hits", samples_);
  }
  void run(KernelContext&, std::size_t gid) override {
    flags_[gid] = static_cast<std::uint8_t>(hit(seed_, gid));
  }
  Element map_return_value(KernelContext& ctx, const Element&) override {
    std::int64_t h = 0;
    if (ctx.device_execution()) {
      for (std::uint8_t f : ctx.take<std::uint8_t>("hits")) h += f;
    } else {
      for (std::uint64_t g = 0; g < samples_; ++g) h += hit(seed_, g);
    }
    return Element::i64({h, static_cast<std::int64_t>(samples_)});
  }

 private:
  std::uint64_t seed_ = 0, samples_ = 0;
  std::span<std::uint8_t> flags_;
};

// 3x3 Sobel over a row band with one halo row above and below (workload C4).
class Sobel : public UnaryKernel {
 public:
  explicit Sobel(std::size_t width) : w_(width) {}
  void map_parameters(KernelContext& ctx, const Element& in) override {
    in_ = ctx.bind<std::uint8_t>("in", in.as_bytes());
    if (in_.size() % w_ != 0 || in_.size() / w_ < 2) throw Error("band is not (rows+2) x width");
    rows_ = in_.size() / w_ - 2;
    out_ = ctx.alloc<std::uint8_t>("out", rows_ * w_);
    ctx.set_range(rows_ * w_);
  }
  int px(std::size_t r, std::ptrdiff_t c) const {
    if (c < 0 || static_cast<std::size_t>(c) >= w_) return 0;
    return in_[r * w_ + static_cast<std::size_t>(c)];
  }
  void run(KernelContext&, std::size_t gid) override {
    const std::size_t r = gid / w_;
    const std::ptrdiff_t c = static_cast<std::ptrdiff_t>(gid % w_);
    const int gx = (px(r, c + 1) - px(r, c - 1)) + 2 * (px(r + 1, c + 1) - px(r + 1, c - 1)) +
                   (px(r + 2, c + 1) - px(r + 2, c - 1));
    const int gy = (px(r + 2, c - 1) + 2 * px(r + 2, c) + px(r + 2, c + 1)) -
                   (px(r, c - 1) + 2 * px(r, c) + px(r, c + 1));
    out_[gid] = static_cast<std::uint8_t>(std::min(255, std::abs(gx) + std::abs(gy)));
  }
  Element map_return_value(KernelContext& ctx, const Element&) override {
    return Element::bytes(ctx.take<std::uint8_t>("out"));
  }

 private:
  std::size_t w_, rows_ = 0;
  std::span<std::uint8_t> in_, out_;
};

// Dense matmul (workload C5): input F32Array A||B (2*n*n), output C = A.B,
// fp32 accumulate over k ascending, one gid per output entry.
class Matmul : public UnaryKernel {
 public:
  explicit Matmul(std::size_t n) : n_(n) {}
  void map_parameters(KernelContext& ctx, const Element& in) override {
    ab_ = ctx.bind<float>("ab", in.as_f32());
    if (ab_.size() != 2 * n_ * n_) throw Error("matmul element must hold A||B");
    c_ = ctx.alloc<float>("c", n_ * n_);
    ctx.set_range(n_ * n_);
  }
  void run(KernelContext&, std::size_t gid) override {
    const std::size_t i = gid / n_, j = gid % n_;
    const float* A = ab_.data();
    const float* B = ab_.data() + n_ * n_;
    float acc = 0.0f;
    for (std::size_t k = 0; k < n_; ++k) {
      const float t = A[i * n_ + k] * B[k * n_ + j];
      acc = acc + t;
    }
    c_[gid] = acc;
  }
  Element map_return_value(KernelContext& ctx, const Element&) override {
    return Element::f32(ctx.take<float>("c"));
  }

 private:
  std::size_t n_;
  std::span<float> ab_, c_;
};

// WordCount: flags of word starts in run(), tokens counted
// in map_return_value (keys in first-occurrence order); below the threshold
// the host tokenises directly.
class WordCount : public UnaryKernel {
 public:
  static bool delim(std::uint8_t b) { return b == ' ' || b == '\t' || b == '\n' || b == '\r'; }
  explicit WordCount(std::uint64_t min_bytes) : min_(min_bytes) {}
  void map_parameters(KernelContext& ctx, const Element& in) override {
    b_ = in.as_bytes();
    ctx.set_range(b_.size());
    if (b_.size() < min_) {
      ctx.set_device_execution(false);
      return;
    }
    f_ = ctx.alloc<std::uint8_t>("flags", b_.size());
  }
  void run(KernelContext&, std::size_t g) override {
    f_[g] = static_cast<std::uint8_t>(!delim(b_[g]) && (g == 0 || delim(b_[g - 1])));
  }
  Element map_return_value(KernelContext& ctx, const Element&) override {
    Element::Table t;
    std::map<std::string, std::size_t> idx;
    auto add = [&](std::size_t s, std::size_t e) {
      std::string k(reinterpret_cast<const char*>(b_.data()) + s, e - s);
      auto it = idx.find(k);
      if (it == idx.end()) {
        idx.emplace(k, t.size());
        t.emplace_back(k, 1);
      } else {
        t[it->second].second++;
      }
    };
    const std::size_t n = b_.size();
    if (ctx.device_execution()) {
      auto f = ctx.take<std::uint8_t>("flags");
      for (std::size_t i = 0; i < n; ++i) {
        if (!f[i]) continue;
        std::size_t e = i;
        while (e < n && !delim(b_[e])) ++e;
        add(i, e);
        i = e;
      }
    } else {
      for (std::size_t i = 0; i < n;) {
        while (i < n && delim(b_[i])) ++i;
        std::size_t e = i;
        while (e < n && !delim(b_[e])) ++e;
        if (e > i) add(i, e);
        i = e;
      }
    }
    return Element::table(std::move(t));
  }

 private:
  std::uint64_t min_;
  std::span<const std::uint8_t> b_;
  std::span<std::uint8_t> f_;
};

// Synthetic corpus shared with tests/oracle_lib.py: word i = "w<mix64(seed+i)%97>",
// followed by 1-2 copies of one delimiter chosen from " \t\n\r".
std::string make_corpus(std::uint64_t seed, std::size_t words) {
  std::string s;
  const char dl[4] = {' ', '\t', '\n', '\r'};
  for (std::size_t i = 0; i < words; ++i) {
    const std::uint64_t z = mix64(seed + i);
    s += "w" + std::to_string(z % 97);
    s.append(1 + ((z >> 40) & 1), dl[(z >> 32) & 3]);
  }
  return s;
}

KernelRegistry make_registry(std::size_t sobel_width, std::size_t matmul_n) {
  KernelRegistry reg;
  reg.register_unary("axpb", [] { return std::make_unique<Axpb>(2.0f, 1.0f); });
  reg.register_unary("psum", [] { return std::make_unique<PartitionTree<AddF>>(0.0f); });
  reg.register_unary("pmax", [] { return std::make_unique<PartitionTree<MaxF>>(-INFINITY); });
  reg.register_binary("sum2", [] { return std::make_unique<Elementwise2<float, AddF>>(); });
  reg.register_binary("vectoradd", [] { return std::make_unique<Elementwise2<float, AddF>>(); });
  reg.register_binary("max2", [] { return std::make_unique<Elementwise2<float, MaxF>>(); });
  reg.register_binary("isum2", [] { return std::make_unique<Elementwise2<std::int64_t, AddI>>(); });
  reg.register_unary("pi", [] { return std::make_unique<Pi>(); });
  reg.register_unary("sobel", [sobel_width] { return std::make_unique<Sobel>(sobel_width); });
  reg.register_unary("matmul", [matmul_n] { return std::make_unique<Matmul>(matmul_n); });
  reg.register_unary("wordcount", [] { return std::make_unique<WordCount>(0); });
  reg.register_unary("wordcount_host", [] { return std::make_unique<WordCount>(~0ull); });
  return reg;
}

// ---- direct driver -----------------------------------------------------------

class DirectDriver : public ClusterDriver {
 public:
  DirectDriver(const KernelRegistry& reg, DeviceDescriptor dev)
      : runtime_("w0", reg, ImplKind::STD, "HOST", std::move(dev)) {}
  std::uint64_t new_job_id() override { return ++job_; }
  std::vector<TaskResult> run_wave(std::vector<Task> tasks, int max_retries) override {
    std::vector<TaskResult> out;
    out.reserve(tasks.size());
    for (const Task& t : tasks) {
      ++tasks_run_;
      for (int attempt = 0;; ++attempt) {
        Message m = runtime_.execute(t);
        if (auto* r = std::get_if<TaskResultMsg>(&m)) {
          out.push_back(std::move(r->result));
          break;
        }
        const auto& e = std::get<TaskErrorMsg>(m);
        if (attempt >= max_retries) {
          throw JobFailed("task " + std::to_string(t.task_id) + " failed in " + e.phase + ": " +
                          e.detail);
        }
      }
    }
    std::sort(out.begin(), out.end(),
              [](const TaskResult& a, const TaskResult& b) { return a.task_id < b.task_id; });
    return out;
  }
  std::uint64_t tasks_run() const { return tasks_run_; }

 private:
  WorkerRuntime runtime_;
  std::uint64_t job_ = 0;
  std::uint64_t tasks_run_ = 0;
};

DeviceDescriptor host_device(unsigned threads) {
  DeviceDescriptor d;
  if (threads <= 1) {
    d.device_id = "host-cpu-0";
    d.device_type = ExecutionMode::CPU;
    d.parallel_width = 1;
  } else {
    d.device_id = "host-jtp-0";
    d.device_type = ExecutionMode::JTP;
    d.parallel_width = threads;
  }
  return d;
}

Dataset f32_dataset(const std::vector<std::vector<float>>& elems, std::size_t parts) {
  std::vector<Element> es;
  for (const auto& e : elems) es.push_back(Element::f32(e));
  return create_dataset(std::move(es), parts);
}

json element_json(const Element& e) {
  json j;
  j["kind"] = to_string(e.kind());
  j["size"] = e.size();
  switch (e.kind()) {
    case ElementKind::F32Array: {
      auto v = e.as_f32();
      j["fnv"] = hex64(fnv64(v.data(), v.size_bytes()));
      if (v.size() <= 8) {
        std::vector<std::string> bits;
        for (float f : v) bits.push_back(hexf(f));
        j["bits"] = bits;
      }
      break;
    }
    case ElementKind::I64Array: {
      auto v = e.as_i64();
      j["fnv"] = hex64(fnv64(v.data(), v.size_bytes()));
      if (v.size() <= 8) j["values"] = std::vector<std::int64_t>(v.begin(), v.end());
      break;
    }
    case ElementKind::ByteArray: {
      auto v = e.as_bytes();
      j["fnv"] = hex64(fnv64(v.data(), v.size_bytes()));
      break;
    }
    default: break;
  }
  return j;
}

// ---- golden ------------------------------------------------------------------

std::vector<std::uint8_t> sobel_image(std::size_t H, std::size_t W, std::uint64_t seed) {
  std::vector<std::uint8_t> img(H * W);
  for (std::size_t i = 0; i < H * W; ++i) img[i] = static_cast<std::uint8_t>(mix64(seed + (i + 1) * kGamma) >> 56);
  return img;
}
std::vector<std::vector<std::uint8_t>> sobel_bands(const std::vector<std::uint8_t>& img, std::size_t H,
                                                   std::size_t W, std::size_t rows) {
  std::vector<std::vector<std::uint8_t>> bands;
  for (std::size_t r0 = 0; r0 < H; r0 += rows) {
    const std::size_t rr = std::min(rows, H - r0);
    std::vector<std::uint8_t> b((rr + 2) * W, 0);
    for (std::size_t k = 0; k < rr + 2; ++k) {
      const std::ptrdiff_t src = static_cast<std::ptrdiff_t>(r0 + k) - 1;
      if (src < 0 || static_cast<std::size_t>(src) >= H) continue;
      std::memcpy(b.data() + k * W, img.data() + static_cast<std::size_t>(src) * W, W);
    }
    bands.push_back(std::move(b));
  }
  return bands;
}

json run_golden() {
  json g;
  g["generator"] = "oracle/ref_harness.cpp golden (reference ucores headers, host-seq executor)";
  const std::size_t kSobelW = 40, kSobelH = 50, kSobelRows = 16, kMatN = 24;
  KernelRegistry reg = make_registry(kSobelW, kMatN);
  DirectDriver drv(reg, host_device(1));
  Engine eng(drv, reg);

  // create_dataset sizes
  {
    json cases = json::array();
    for (auto [n, p] : std::vector<std::pair<int, int>>{{6, 3}, {7, 3}, {0, 2}, {5, 8}, {1048576, 4}}) {
      std::vector<Element> es(n, Element::i64({1}));
      Dataset d = create_dataset(std::move(es), p);
      std::vector<std::size_t> sizes;
      for (const auto& part : d.partitions()) sizes.push_back(part.elements.size());
      cases.push_back({{"n", n}, {"p", p}, {"sizes", sizes}});
    }
    g["partition_sizes"] = cases;
  }

  // C1: 2^20 fp32 (seed 12345) as 4 elements of 2^18 in 4 partitions:
  // map_cl(axpb) -> map_cl_partition(psum|pmax) -> reduce_cl(sum2|max2)
  auto run_c1 = [&](std::size_t n, std::size_t parts, std::size_t elems) {
    std::vector<std::vector<float>> es(elems);
    std::size_t base = n / elems, extra = n % elems, pos = 0;
    for (std::size_t k = 0; k < elems; ++k) {
      es[k].resize(base + (k < extra ? 1 : 0));
      for (auto& v : es[k]) v = uniform01(12345, pos++);
    }
    Dataset x = f32_dataset(es, parts);
    Dataset y = eng.map_cl(x, "axpb");
    std::vector<float> flat;
    for (const Element& e : y.collect()) flat.insert(flat.end(), e.as_f32().begin(), e.as_f32().end());
    json c;
    c["n"] = n;
    c["partitions"] = parts;
    c["elements"] = elems;
    c["y_fnv"] = hex64(fnv64(flat.data(), flat.size() * 4));
    for (const char* op : {"sum", "max"}) {
      Dataset ps = eng.map_cl_partition(y, std::string("p") + op);
      std::vector<std::string> pbits;
      for (const Element& e : ps.collect()) pbits.push_back(hexf(e.as_f32()[0]));
      Element r = eng.reduce_cl(ps, std::string(op) + "2");
      c[std::string("partials_") + op] = pbits;
      c[std::string("total_") + op] = hexf(r.as_f32()[0]);
      c[std::string("total_") + op + "_value"] = r.as_f32()[0];
    }
    return c;
  };
  g["c1"] = run_c1(1u << 20, 4, 4);
  g["c1_ragged"] = run_c1(100003, 5, 13);

  // C2 at reduced size: P partitions of L, partition p filled from seed 1000+p,
  // a planted unique maximum 1.5 in partition P/2 at index L/3.
  {
    const std::size_t P = 8, L = 65536 + 7;
    std::vector<std::vector<float>> es(P, std::vector<float>(L));
    for (std::size_t p = 0; p < P; ++p)
      for (std::size_t i = 0; i < L; ++i) es[p][i] = uniform01(1000 + p, i);
    es[P / 2][L / 3] = 1.5f;
    Dataset x = f32_dataset(es, P);
    Dataset y = eng.map_cl(x, "axpb");
    json c;
    c["P"] = P;
    c["L"] = L;
    std::vector<float> flat;
    for (const Element& e : y.collect()) flat.insert(flat.end(), e.as_f32().begin(), e.as_f32().end());
    c["y_fnv"] = hex64(fnv64(flat.data(), flat.size() * 4));
    for (const char* op : {"sum", "max"}) {
      Dataset ps = eng.map_cl_partition(y, std::string("p") + op);
      std::vector<std::string> pbits;
      for (const Element& e : ps.collect()) pbits.push_back(hexf(e.as_f32()[0]));
      Element r = eng.reduce_cl(ps, std::string(op) + "2");
      c[std::string("partials_") + op] = pbits;
      c[std::string("total_") + op] = hexf(r.as_f32()[0]);
    }
    g["c2_small"] = c;
  }

  // Fig-3 vectoradd [1,2,3]+[4,5,6]
  {
    Dataset d = f32_dataset({{1, 2, 3}, {4, 5, 6}}, 1);
    g["fig3"] = element_json(eng.reduce_cl(d, "vectoradd"));
  }
  // SPEC acceptance #2 vectoradd: n=2^20 per vector, 8 partitions
  {
    const std::size_t len = 1u << 20, P = 8;
    std::vector<std::vector<float>> es(P, std::vector<float>(len));
    for (std::size_t k = 0; k < P; ++k)
      for (std::size_t i = 0; i < len; ++i) es[k][i] = static_cast<float>((k * len + i) % 1000);
    Dataset d = f32_dataset(es, P);
    Element r = eng.reduce_cl(d, "vectoradd");
    double checksum = 0;
    for (float v : r.as_f32()) checksum += v;
    json c = element_json(r);
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.3f", checksum);
    c["checksum"] = buf;
    g["vectoradd_acc2"] = c;
  }
  // Tree shapes with a non-commutative probe: vectors of length 1 whose
  // max2-combine exposes order through signed zeros; and i64 sums over
  // ragged datasets vs the task count rule.
  {
    json cases = json::array();
    std::uint64_t s = 99;
    for (int c = 0; c < 24; ++c) {
      const std::size_t count = 1 + (mix64(s++) % 40);
      const std::size_t parts = 1 + (mix64(s++) % 16);
      const std::size_t len = 1 + (mix64(s++) % 5);
      std::vector<Element> es;
      std::vector<std::vector<std::int64_t>> raw;
      for (std::size_t i = 0; i < count; ++i) {
        std::vector<std::int64_t> v(len);
        for (auto& x : v) x = static_cast<std::int64_t>(mix64(s++));
        raw.push_back(v);
        es.push_back(Element::i64(v));
      }
      Dataset d = create_dataset(std::move(es), parts);
      const std::uint64_t before = drv.tasks_run();
      Element r = eng.reduce_cl(d, "isum2");
      const std::uint64_t tasks = drv.tasks_run() - before;
      cases.push_back({{"seed_after", s}, {"count", count}, {"parts", parts}, {"len", len},
                       {"result", std::vector<std::int64_t>(r.as_i64().begin(), r.as_i64().end())},
                       {"tasks", tasks}});
    }
    g["isum_cases"] = cases;
  }
  // Pi: samples split ceiling-first over tasks, task_seed = seed + t.
  {
    json cases = json::array();
    for (auto [S, T, seed] : std::vector<std::tuple<std::uint64_t, std::uint64_t, std::uint64_t>>{
             {4000000, 8, 42}, {1u << 24, 8, 42}, {1, 1, 7}, {1000, 3, 5}}) {
      std::vector<Element> es;
      for (std::uint64_t t = 0; t < T; ++t) {
        const std::uint64_t n = S / T + (t < S % T ? 1 : 0);
        es.push_back(Element::i64({static_cast<std::int64_t>(seed + t), static_cast<std::int64_t>(n)}));
      }
      Dataset d = create_dataset(std::move(es), T);
      Dataset r = eng.map_cl(d, "pi");
      std::vector<std::int64_t> hits;
      std::int64_t total = 0;
      for (const Element& e : r.collect()) {
        hits.push_back(e.as_i64()[0]);
        total += e.as_i64()[0];
      }
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.6f", 4.0 * static_cast<double>(total) / static_cast<double>(S));
      cases.push_back({{"samples", S}, {"tasks", T}, {"seed", seed}, {"task_hits", hits},
                       {"hits", total}, {"pi", buf}});
    }
    g["pi"] = cases;
  }
  // Sobel bands (H=50, W=40, 16-row bands -> 4 bands, last ragged), seed 7.
  {
    auto img = sobel_image(kSobelH, kSobelW, 7);
    auto bands = sobel_bands(img, kSobelH, kSobelW, kSobelRows);
    std::vector<Element> es;
    for (auto& b : bands) es.push_back(Element::bytes(b));
    Dataset d = create_dataset(std::move(es), bands.size());
    Dataset r = eng.map_cl_partition(d, "sobel");
    std::vector<std::uint8_t> out;
    for (const Element& e : r.collect()) out.insert(out.end(), e.as_bytes().begin(), e.as_bytes().end());
    g["sobel"] = {{"H", kSobelH}, {"W", kSobelW}, {"rows", kSobelRows}, {"seed", 7},
                  {"fnv", hex64(fnv64(out.data(), out.size()))}, {"bytes", out.size()}};
  }
  // Matmul n=24: A,B in U[-1,1) from seed 100 (A = first n^2 draws, B = next n^2).
  {
    const std::size_t n = kMatN;
    std::vector<float> ab(2 * n * n);
    for (std::size_t i = 0; i < ab.size(); ++i) ab[i] = 2.0f * uniform01(100, i) - 1.0f;
    Dataset d = f32_dataset({ab}, 1);
    Dataset r = eng.map_cl(d, "matmul");
    g["matmul"] = {{"n", n}, {"seed", 100}, {"c", element_json(r.collect()[0])}};
  }
  // WordCount: "a b a" and a corpus ingested by the
  // reference's own create_from_text chunker (dataset.hpp:94-139).
  {
    auto table_json = [](const Element& e) {
      json t = json::array();
      for (const auto& [k, c] : e.as_table()) t.push_back({k, c});
      return t;
    };
    Dataset d1 = create_dataset({Element::bytes(std::string("a b a"))}, 1);
    json w;
    w["simple"] = table_json(eng.map_cl(d1, "wordcount").collect()[0]);
    const std::string corpus = make_corpus(5, 30000);
    const std::string path = "/tmp/ucores_wc_corpus.txt";
    {
      std::ofstream f(path, std::ios::binary);
      f << corpus;
    }
    Dataset d = create_from_text(path, 16384);
    Dataset dev = eng.map_cl(d, "wordcount");
    Dataset host = eng.map_cl(d, "wordcount_host");
    std::map<std::string, std::uint64_t> merged;
    bool same = true;
    std::vector<std::string> chunk_fnv;
    const std::vector<Element> dev_e = dev.collect(), host_e = host.collect();
    for (std::size_t i = 0; i < dev_e.size(); ++i) {
      const Element& a = dev_e[i];
      same &= a == host_e[i];
      std::string ser;
      for (const auto& [k, c] : a.as_table()) {
        merged[k] += c;
        ser += k + "\t" + std::to_string(c) + "\n";
      }
      chunk_fnv.push_back(hex64(fnv64(ser.data(), ser.size())));
    }
    std::vector<std::pair<std::string, std::uint64_t>> sorted(merged.begin(), merged.end());
    std::sort(sorted.begin(), sorted.end(),
              [](auto& x, auto& y) { return x.second != y.second ? x.second > y.second : x.first < y.first; });
    std::string ser;
    for (auto& [k, c] : sorted) ser += k + "\t" + std::to_string(c) + "\n";
    std::vector<std::size_t> sizes;
    for (const Element& e : d.collect()) sizes.push_back(e.size());
    w["corpus"] = {{"seed", 5}, {"words", 30000}, {"bytes", corpus.size()}, {"target_chunk", 16384},
                   {"chunk_sizes", sizes}, {"chunk_table_fnv", chunk_fnv}, {"merged_fnv", hex64(fnv64(ser.data(), ser.size()))},
                   {"top3", json::array({{sorted[0].first, sorted[0].second}, {sorted[1].first, sorted[1].second},
                                         {sorted[2].first, sorted[2].second}})},
                   {"device_equals_host", same}};
    g["wordcount"] = w;
  }

  // Error behaviour
  {
    json e;
    try {
      Dataset d = f32_dataset({{1.0f}, {2.0f}}, 3);  // partition 2 is empty
      eng.map_cl_partition(d, "psum");
      e["empty_partition"] = "no error";
    } catch (const JobFailed&) {
      e["empty_partition"] = "JobFailed";
    }
    try {
      eng.reduce_cl(Dataset(std::vector<Partition>(2)), "sum2");
      e["reduce_empty"] = "no error";
    } catch (const EmptyDataset&) {
      e["reduce_empty"] = "EmptyDataset";
    }
    {
      const std::uint64_t before = drv.tasks_run();
      Element r = eng.reduce_cl(f32_dataset({{3.5f, 4.5f}}, 4), "sum2");
      e["reduce_single_tasks"] = drv.tasks_run() - before;
      e["reduce_single"] = element_json(r);
    }
    try {
      eng.map_cl(f32_dataset({{1.0f}}, 1), "sum2");
      e["arity"] = "no error";
    } catch (const ArityMismatch&) {
      e["arity"] = "ArityMismatch";
    }
    try {
      eng.reduce_cl(f32_dataset({{1.0f, 2.0f}, {1.0f}}, 1), "sum2");
      e["length_mismatch"] = "no error";
    } catch (const JobFailed&) {
      e["length_mismatch"] = "JobFailed";
    }
    g["errors"] = e;
  }
  return g;
}

// ---- golden-full ----------------------------------------------------------------

// The reference's own results at the BASELINE.json sizes (run with the host
// parallel executor; every kernel is class D, so the results do not depend on
// the executor):
//   C2  2^30 fp32 in 64 partitions of 2^24 (partition p from seed 1000+p, the
//       planted unique maximum 1.5 in partition 32 at index L/3):
//       map_cl(axpb) -> map_cl_partition(psum|pmax) -> reduce_cl(sum2|max2);
//       per-partition FNV-1a of y, all 64 partials and the result bits
//   C3  2^34 samples, 64 tasks of 2^28, task seed 42+t: all 64 hit counts
//   C4  16384^2 u8 (seed 7), 64 bands of 256 rows with halos: per-band and
//       whole-output FNV-1a
json run_golden_full(unsigned threads, const std::string& which) {
  json g;
  g["generator"] = "oracle/ref_harness.cpp golden-full (reference ucores headers, host-par executor)";
  g["threads"] = threads;
  auto want = [&](const char* w) { return which == "all" || which == w; };
  if (want("c2")) {
    const std::size_t P = 64, L = 1u << 24;
    KernelRegistry reg = make_registry(16, 16);
    DirectDriver drv(reg, host_device(threads));
    Engine eng(drv, reg);
    Dataset x;
    {
      std::vector<Element> es;
      es.reserve(P);
      for (std::size_t p = 0; p < P; ++p) {
        std::vector<float> v(L);
        for (std::size_t i = 0; i < L; ++i) v[i] = uniform01(1000 + p, i);
        if (p == P / 2) v[L / 3] = 1.5f;
        es.push_back(Element::f32(std::move(v)));
      }
      x = create_dataset(std::move(es), P);
    }
    Dataset y = eng.map_cl(x, "axpb");
    x = Dataset();
    json c;
    c["P"] = P;
    c["L"] = L;
    c["planted_max"] = {{"partition", P / 2}, {"index", L / 3}, {"value", 1.5}};
    std::vector<std::string> yf;
    for (const Element& e : y.collect()) yf.push_back(hex64(fnv64(e.as_f32().data(), e.as_f32().size_bytes())));
    c["y_fnv"] = yf;
    for (const char* op : {"sum", "max"}) {
      Dataset ps = eng.map_cl_partition(y, std::string("p") + op);
      std::vector<std::string> pbits;
      for (const Element& e : ps.collect()) pbits.push_back(hexf(e.as_f32()[0]));
      Element r = eng.reduce_cl(ps, std::string(op) + "2");
      c[std::string("partials_") + op] = pbits;
      c[std::string("total_") + op] = hexf(r.as_f32()[0]);
      c[std::string("total_") + op + "_value"] = r.as_f32()[0];
    }
    g["c2_full"] = c;
  }
  if (want("c3")) {
    const std::uint64_t S = 1ull << 34, T = 64;
    KernelRegistry reg = make_registry(16, 16);
    DirectDriver drv(reg, host_device(threads));
    Engine eng(drv, reg);
    std::vector<Element> es;
    for (std::uint64_t t = 0; t < T; ++t)
      es.push_back(Element::i64({static_cast<std::int64_t>(42 + t), static_cast<std::int64_t>(S / T)}));
    Dataset d = create_dataset(std::move(es), T);
    Dataset r = eng.map_cl(d, "pi");
    std::vector<std::int64_t> hits;
    std::int64_t total = 0;
    for (const Element& e : r.collect()) {
      hits.push_back(e.as_i64()[0]);
      total += e.as_i64()[0];
    }
    // reduce_cl(isum2) over the {hits, samples} pairs, as the GPU path folds it
    Element tot = eng.reduce_cl(r, "isum2");
    g["c3_full"] = {{"samples", S}, {"tasks", T}, {"seed", 42}, {"task_hits", hits}, {"hits", total},
                    {"reduce_cl_isum2", std::vector<std::int64_t>(tot.as_i64().begin(), tot.as_i64().end())}};
  }
  if (want("c4")) {
    const std::size_t H = 16384, W = 16384, R = 256;
    KernelRegistry reg = make_registry(W, 16);
    DirectDriver drv(reg, host_device(threads));
    Engine eng(drv, reg);
    std::vector<std::vector<std::uint8_t>> bands;
    {
      auto img = sobel_image(H, W, 7);
      bands = sobel_bands(img, H, W, R);
    }
    std::vector<Element> es;
    for (auto& b : bands) es.push_back(Element::bytes(std::move(b)));
    bands.clear();
    const std::size_t nb = es.size();
    Dataset d = create_dataset(std::move(es), nb);
    Dataset r = eng.map_cl_partition(d, "sobel");
    std::vector<std::string> bf;
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (const Element& e : r.collect()) {
      auto v = e.as_bytes();
      bf.push_back(hex64(fnv64(v.data(), v.size())));
      for (std::uint8_t b : v) {
        h ^= b;
        h *= 0x100000001b3ull;
      }
    }
    g["c4_full"] = {{"H", H}, {"W", W}, {"rows", R}, {"seed", 7}, {"bands", nb}, {"band_fnv", bf},
                    {"fnv", hex64(h)}};
  }
  return g;
}

// ---- bench -------------------------------------------------------------------

// Bounded CPU samples of the other BASELINE configs through the reference
// Engine + HostParallelExecutor:
//   --w pi      --samples S --tasks T          (C3 shape, S scaled down)
//   --w sobel   --height H --width W --rows R  (C4: bands of R rows, halos)
//   --w matmul  --n N --parts P                (C5 shape at a small n)
//   --w wordcount --bytes B --chunk C          (create_from_text chunks -> map_cl(wordcount))
int run_bench_workload(int argc, char** argv) {
  std::string w = "pi";
  std::uint64_t samples = 1u << 26, tasks = 64, H = 2048, W = 16384, R = 256, n = 256, parts = 2;
  std::uint64_t bytes = 64ull << 20, chunk = 1ull << 20;
  unsigned threads = std::thread::hardware_concurrency();
  int steps = 2, warmup = 1;
  for (int i = 2; i + 1 < argc; i += 2) {
    std::string k = argv[i], v = argv[i + 1];
    if (k == "--w") w = v;
    else if (k == "--samples") samples = std::stoull(v);
    else if (k == "--tasks") tasks = std::stoull(v);
    else if (k == "--height") H = std::stoull(v);
    else if (k == "--width") W = std::stoull(v);
    else if (k == "--rows") R = std::stoull(v);
    else if (k == "--n") n = std::stoull(v);
    else if (k == "--parts") parts = std::stoull(v);
    else if (k == "--bytes") bytes = std::stoull(v);
    else if (k == "--chunk") chunk = std::stoull(v);
    else if (k == "--threads") threads = static_cast<unsigned>(std::stoul(v));
    else if (k == "--steps") steps = std::stoi(v);
    else if (k == "--warmup") warmup = std::stoi(v);
  }
  KernelRegistry reg = make_registry(W, n);
  DirectDriver drv(reg, host_device(threads));
  Engine eng(drv, reg);
  Dataset d;
  std::string kernel;
  double units = 0;
  bool partition = false;
  if (w == "pi") {
    std::vector<Element> es;
    for (std::uint64_t t = 0; t < tasks; ++t)
      es.push_back(Element::i64({static_cast<std::int64_t>(42 + t),
                                 static_cast<std::int64_t>(samples / tasks + (t < samples % tasks ? 1 : 0))}));
    d = create_dataset(std::move(es), tasks);
    kernel = "pi";
    units = double(samples);
  } else if (w == "sobel") {
    auto img = sobel_image(H, W, 7);
    auto bands = sobel_bands(img, H, W, R);
    std::vector<Element> es;
    for (auto& b : bands) es.push_back(Element::bytes(b));
    const std::size_t nb = es.size();
    d = create_dataset(std::move(es), nb);
    kernel = "sobel";
    units = double(H) * double(W);
    partition = true;
  } else if (w == "matmul") {
    std::vector<std::vector<float>> es(parts, std::vector<float>(2 * n * n));
    for (std::size_t p = 0; p < parts; ++p)
      for (std::size_t i = 0; i < es[p].size(); ++i) es[p][i] = 2.0f * uniform01(100 + p, i) - 1.0f;
    d = f32_dataset(es, parts);
    kernel = "matmul";
    units = 2.0 * double(n) * double(n) * double(n) * double(parts);
  } else if (w == "wordcount") {
    // the reference chunker (dataset.hpp:94-112) over a synthetic corpus file;
    // "wordcount" prefers device execution, so the host executor runs the
    // per-byte run() (word-start flags) and map_return_value tokenises
    std::string corpus;
    for (std::uint64_t seed = 5; corpus.size() < bytes; ++seed) corpus += make_corpus(seed * 1000003, 100000);
    corpus.resize(bytes);
    const std::string path = "/tmp/ucores_wc_bench.txt";
    {
      std::ofstream f(path, std::ios::binary);
      f << corpus;
    }
    d = create_from_text(path, chunk);
    kernel = "wordcount";
    units = double(bytes);
  } else {
    throw Error("unknown workload " + w);
  }
  std::vector<double> times;
  for (int s = 0; s < warmup + steps; ++s) {
    auto t0 = std::chrono::steady_clock::now();
    Dataset r = partition ? eng.map_cl_partition(d, kernel) : eng.map_cl(d, kernel);
    auto t1 = std::chrono::steady_clock::now();
    if (s >= warmup) times.push_back(std::chrono::duration<double>(t1 - t0).count());
  }
  json out;
  out["workload"] = w;
  out["units"] = units;
  out["threads"] = threads;
  out["executor"] = threads <= 1 ? "host-seq" : "host-par";
  out["step_s"] = times;
  std::cout << out.dump() << std::endl;
  return 0;
}

// C1 literal form: n one-float elements in P partitions,
// map_cl(axpb) -> map_cl_partition(p<op>) -> reduce_cl(<op>2); map_cl is one
// task per element. Dataset construction is timed, as in ucd_literal_f32.
int run_bench_literal(int argc, char** argv) {
  std::size_t n = 1u << 18, P = 4;
  unsigned threads = 1;
  int steps = 1, warmup = 0;
  std::string op = "sum";
  for (int i = 2; i + 1 < argc; i += 2) {
    std::string k = argv[i], v = argv[i + 1];
    if (k == "--n") n = std::stoull(v);
    else if (k == "--parts") P = std::stoull(v);
    else if (k == "--threads") threads = static_cast<unsigned>(std::stoul(v));
    else if (k == "--steps") steps = std::stoi(v);
    else if (k == "--warmup") warmup = std::stoi(v);
    else if (k == "--op") op = v;
  }
  KernelRegistry reg = make_registry(16, 16);
  DirectDriver drv(reg, host_device(threads));
  Engine eng(drv, reg);
  std::vector<double> times;
  float result = 0;
  for (int s = 0; s < warmup + steps; ++s) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<Element> es;
    es.reserve(n);
    for (std::size_t i = 0; i < n; ++i) es.push_back(Element::f32({uniform01(12345, i)}));
    Dataset x = create_dataset(std::move(es), P);
    Element r = eng.reduce_cl(eng.map_cl_partition(eng.map_cl(x, "axpb"), "p" + op), op + "2");
    auto t1 = std::chrono::steady_clock::now();
    result = r.as_f32()[0];
    if (s >= warmup) times.push_back(std::chrono::duration<double>(t1 - t0).count());
  }
  json out;
  out["elements"] = n;
  out["partitions"] = P;
  out["threads"] = threads;
  out["executor"] = threads <= 1 ? "host-seq" : "host-par";
  out["step_s"] = times;
  out["result_bits"] = hexf(result);
  std::cout << out.dump() << std::endl;
  return 0;
}

int run_bench(int argc, char** argv) {
  std::size_t P = 4, L = 1u << 24;
  bool plant = true;
  unsigned threads = std::thread::hardware_concurrency();
  int steps = 3, warmup = 1;
  std::string op = "sum";
  for (int i = 2; i + 1 < argc; i += 2) {
    std::string k = argv[i];
    std::string v = argv[i + 1];
    if (k == "--parts") P = std::stoull(v);
    else if (k == "--part-len") L = std::stoull(v);
    else if (k == "--threads") threads = static_cast<unsigned>(std::stoul(v));
    else if (k == "--steps") steps = std::stoi(v);
    else if (k == "--warmup") warmup = std::stoi(v);
    else if (k == "--op") op = v;
    else if (k == "--plant") plant = std::stoi(v) != 0;
  }
  KernelRegistry reg = make_registry(16, 16);
  DirectDriver drv(reg, host_device(threads));
  Engine eng(drv, reg);
  std::vector<std::vector<float>> es(P, std::vector<float>(L));
  for (std::size_t p = 0; p < P; ++p)
    for (std::size_t i = 0; i < L; ++i) es[p][i] = uniform01(1000 + p, i);
  // the planted unique maximum of bench.py's C2 input (partition P/2, index L/3)
  if (plant) es[P / 2][L / 3] = 1.5f;
  Dataset x = f32_dataset(es, P);
  es.clear();
  std::vector<double> times;
  float result = 0;
  for (int s = 0; s < warmup + steps; ++s) {
    auto t0 = std::chrono::steady_clock::now();
    Dataset y = eng.map_cl(x, "axpb");
    Dataset ps = eng.map_cl_partition(y, "p" + op);
    Element r = eng.reduce_cl(ps, op + "2");
    auto t1 = std::chrono::steady_clock::now();
    result = r.as_f32()[0];
    if (s >= warmup) times.push_back(std::chrono::duration<double>(t1 - t0).count());
  }
  json out;
  out["elements"] = P * L;
  out["partitions"] = P;
  out["part_len"] = L;
  out["threads"] = threads;
  out["executor"] = threads <= 1 ? "host-seq" : "host-par";
  out["op"] = op;
  out["planted_max"] = plant;
  out["step_s"] = times;
  out["result_bits"] = hexf(result);
  out["result"] = result;
  std::cout << out.dump() << std::endl;
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "golden";
  try {
    if (mode == "golden") {
      std::cout << run_golden().dump(1) << std::endl;
      return 0;
    }
    if (mode == "golden-full") {
      unsigned threads = std::thread::hardware_concurrency();
      std::string which = "all";
      for (int i = 2; i + 1 < argc; i += 2) {
        const std::string k = argv[i], v = argv[i + 1];
        if (k == "--threads") threads = static_cast<unsigned>(std::stoul(v));
        else if (k == "--which") which = v;
      }
      std::cout << run_golden_full(threads, which).dump(1) << std::endl;
      return 0;
    }
    if (mode == "bench") return run_bench(argc, argv);
    if (mode == "bench-workload") return run_bench_workload(argc, argv);
    if (mode == "bench-literal") return run_bench_literal(argc, argv);
  } catch (const std::exception& e) {
    std::cerr << "ref_harness: " << e.what() << std::endl;
    return 1;
  }
  std::cerr << "usage: ref_harness golden | bench [--parts P --part-len L --threads T --steps K --warmup W --op sum|max]\n";
  return 2;
}
