// test_dropin.cpp — GPU parity of the C++ drop-in through the UNMODIFIED
// reference Engine (ucores/engine.hpp). Every operator runs twice on the
// same Dataset: once with a reference-style host driver (WorkerRuntime +
// HostSequentialExecutor, the CPU path) and once with GpuClusterDriver
// (seam A, batched) / GpuWorkerRuntime (seam B). Outputs must be equal under
// Element::operator== (bitwise, element.hpp:108-126); matmul within an fp32-level
// tolerance. Built by paper_1505_01120_b200/build.py; run by
// tests/test_cpp_dropin.py on a GPU box.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <string>
#include <vector>

#include "ucores/dataset.hpp"
#include "ucores/device.hpp"
#include "ucores/engine.hpp"
#include "ucores/worker.hpp"
#include "ucores_b200/cuda_executor.hpp"
#include "ucores_b200/device_dataset.hpp"
#include "ucores_b200/device_ops.hpp"
#include "ucores_b200/gpu_cluster_driver.hpp"
#include "ucores_b200/kernels.hpp"

using namespace ucores;
using namespace ucores_b200;

namespace {

int g_fail = 0, g_pass = 0;
#define EXPECT(cond, what)                                              \
  do {                                                                  \
    if (cond) {                                                         \
      ++g_pass;                                                         \
    } else {                                                            \
      ++g_fail;                                                         \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, what);         \
    }                                                                   \
  } while (0)

float u01(std::uint64_t seed, std::uint64_t i) {
  return static_cast<float>(kernels::mix64(seed + (i + 1) * kernels::kGamma) >> 40) * (1.0f / 16777216.0f);
}

// CPU reference driver: reference WorkerRuntime + host executor, in place.
class HostDriver : public ClusterDriver {
 public:
  HostDriver(const KernelRegistry& reg) : rt_("cpu0", reg, ImplKind::STD, "HOST", dev()) {}
  static DeviceDescriptor dev() {
    DeviceDescriptor d;
    d.device_id = "host-cpu-0";
    d.device_type = ExecutionMode::CPU;
    return d;
  }
  std::uint64_t new_job_id() override { return ++job_; }
  std::vector<TaskResult> run_wave(std::vector<Task> tasks, int max_retries) override {
    std::vector<TaskResult> out;
    for (const Task& t : tasks) {
      for (int a = 0;; ++a) {
        Message m = rt_.execute(t);
        if (auto* r = std::get_if<TaskResultMsg>(&m)) {
          out.push_back(std::move(r->result));
          break;
        }
        if (a >= max_retries) throw JobFailed("task failed: " + std::get<TaskErrorMsg>(m).detail);
      }
    }
    std::sort(out.begin(), out.end(), [](auto& a, auto& b) { return a.task_id < b.task_id; });
    return out;
  }

 private:
  WorkerRuntime rt_;
  std::uint64_t job_ = 0;
};

Dataset f32_dataset(const std::vector<std::vector<float>>& es, std::size_t parts) {
  std::vector<Element> v;
  for (auto& e : es) v.push_back(Element::f32(e));
  return create_dataset(std::move(v), parts);
}

bool same(const Dataset& a, const Dataset& b) {
  if (a.partition_count() != b.partition_count()) return false;
  for (std::size_t p = 0; p < a.partition_count(); ++p)
    if (a.partitions()[p].elements != b.partitions()[p].elements) return false;
  return true;
}

struct Fixture {
  KernelRegistry reg;
  DeviceOpRegistry ops;
  Fixture(std::size_t sobel_w = 48, std::size_t mat_n = 256) {
    WorkloadParams p;
    p.sobel_width = sobel_w;
    p.matmul_n = mat_n;
    register_workload(reg, ops, p);
  }
};

template <class Fn>
void run_case(const char* name, Fn fn) {
  const int before = g_fail;
  auto t0 = std::chrono::steady_clock::now();
  try {
    fn();
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("FAIL %s: exception %s\n", name, e.what());
  }
  auto ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  std::printf("%s %s (%.1f ms)\n", g_fail == before ? "ok  " : "FAIL", name, ms);
}

}  // namespace

int main() {
  Fixture fx;
  HostDriver host(fx.reg);
  GpuClusterDriver gpu(fx.reg, fx.ops);
  GpuClusterDriver::Options per_task;
  per_task.mode = GpuClusterDriver::Mode::PerTask;
  GpuClusterDriver gpu_b(fx.reg, fx.ops, per_task);
  Engine eh(host, fx.reg), eg(gpu, fx.reg), eb(gpu_b, fx.reg);
  std::printf("gpus: %zu\n", gpu.gpu_count());

  // C1: 2^20 fp32 as 4 elements in 4 partitions; ragged variant too
  run_case("c1 map_cl/map_cl_partition/reduce_cl sum+max (seam A and B)", [&] {
    for (auto [n, elems, parts] : std::vector<std::tuple<std::size_t, std::size_t, std::size_t>>{
             {1u << 20, 4, 4}, {100003, 13, 5}, {70001, 7, 3}}) {
      std::vector<std::vector<float>> es(elems);
      std::size_t pos = 0;
      for (std::size_t k = 0; k < elems; ++k) {
        es[k].resize(n / elems + (k < n % elems ? 1 : 0));
        for (auto& v : es[k]) v = u01(12345, pos++);
      }
      Dataset x = f32_dataset(es, parts);
      Dataset yh = eh.map_cl(x, "axpb"), yg = eg.map_cl(x, "axpb"), yb = eb.map_cl(x, "axpb");
      EXPECT(same(yh, yg), "map_cl(axpb) seam A bitwise");
      EXPECT(same(yh, yb), "map_cl(axpb) seam B bitwise");
      for (const char* op : {"sum", "max"}) {
        Dataset ph = eh.map_cl_partition(yh, std::string("p") + op);
        Dataset pg = eg.map_cl_partition(yg, std::string("p") + op);
        Dataset pb = eb.map_cl_partition(yb, std::string("p") + op);
        EXPECT(same(ph, pg), "map_cl_partition seam A bitwise");
        EXPECT(same(ph, pb), "map_cl_partition seam B bitwise");
        Element rh = eh.reduce_cl(ph, std::string(op) + "2");
        EXPECT(rh == eg.reduce_cl(pg, std::string(op) + "2"), "reduce_cl seam A bitwise");
        EXPECT(rh == eb.reduce_cl(pb, std::string(op) + "2"), "reduce_cl seam B bitwise");
        // reduce_cl directly over the mapped vectors (stage-1 folds + stage-2 tree)
        if (std::string(op) == "sum") {
          Dataset vh = f32_dataset({{1, 2, 3}, {4, 5, 6}, {7, 8, 9}, {10, 11, 12}, {0.5f, -0.5f, 1e30f}}, 2);
          EXPECT(eh.reduce_cl(vh, "vectoradd") == eg.reduce_cl(vh, "vectoradd"), "reduce_cl vectors");
        }
      }
    }
  });

  run_case("fig3 vectoradd [1,2,3]+[4,5,6]", [&] {
    Element r = eg.reduce_cl(f32_dataset({{1, 2, 3}, {4, 5, 6}}, 1), "vectoradd");
    auto v = r.as_f32();
    EXPECT(v.size() == 3 && v[0] == 5 && v[1] == 7 && v[2] == 9, "[5,7,9]");
  });

  run_case("SPEC acceptance 2: vectoradd n=2^20 P=8 checksum", [&] {
    const std::size_t len = 1u << 20, P = 8;
    std::vector<std::vector<float>> es(P, std::vector<float>(len));
    for (std::size_t k = 0; k < P; ++k)
      for (std::size_t i = 0; i < len; ++i) es[k][i] = static_cast<float>((k * len + i) % 1000);
    Dataset d = f32_dataset(es, P);
    Element r = eg.reduce_cl(d, "vectoradd");
    double cs = 0;
    for (float v : r.as_f32()) cs += v;
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.3f", cs);
    EXPECT(std::string(buf) == "4189990528.000", "checksum 4189990528.000");
    EXPECT(r == eh.reduce_cl(d, "vectoradd"), "bitwise vs host");
  });

  run_case("SPEC acceptance 5: isum2 tree-reduce == left fold, tasks == count-1", [&] {
    std::uint64_t s = 7;
    for (int c = 0; c < 40; ++c) {
      const std::size_t count = 1 + kernels::mix64(s++) % 40, parts = 1 + kernels::mix64(s++) % 16,
                        len = 1 + kernels::mix64(s++) % 5;
      std::vector<Element> es;
      std::vector<std::uint64_t> fold(len, 0);
      for (std::size_t i = 0; i < count; ++i) {
        std::vector<std::int64_t> v(len);
        for (std::size_t j = 0; j < len; ++j) {
          v[j] = static_cast<std::int64_t>(kernels::mix64(s++));
          fold[j] += static_cast<std::uint64_t>(v[j]);
        }
        es.push_back(Element::i64(v));
      }
      Dataset d = create_dataset(std::move(es), parts);
      const std::uint64_t before = gpu.tasks_run();
      Element r = eg.reduce_cl(d, "isum2");
      bool ok = true;
      for (std::size_t j = 0; j < len; ++j) ok &= static_cast<std::uint64_t>(r.as_i64()[j]) == fold[j];
      EXPECT(ok, "isum equals left fold");
      EXPECT(gpu.tasks_run() - before == count - 1, "REDUCE_PAIR tasks == count-1");
    }
  });

  run_case("pi 4M/8/42 -> 3141371 (golden), seam A and B", [&] {
    std::vector<Element> es;
    for (int t = 0; t < 8; ++t) es.push_back(Element::i64({42 + t, 500000}));
    Dataset d = create_dataset(std::move(es), 8);
    std::int64_t hits = 0;
    for (const Element& e : eg.map_cl(d, "pi").collect()) hits += e.as_i64()[0];
    EXPECT(hits == 3141371, "hits == 3141371");
    EXPECT(same(eb.map_cl(d, "pi"), eh.map_cl(d, "pi")), "seam B pi bitwise vs host");
  });

  run_case("sobel bands (W=48, 16-row bands)", [&] {
    const std::size_t H = 50, W = 48, R = 16;
    std::vector<std::uint8_t> img(H * W);
    for (std::size_t i = 0; i < img.size(); ++i)
      img[i] = static_cast<std::uint8_t>(kernels::mix64(7 + (i + 1) * kernels::kGamma) >> 56);
    std::vector<Element> bands;
    for (std::size_t r0 = 0; r0 < H; r0 += R) {
      const std::size_t rr = std::min(R, H - r0);
      std::vector<std::uint8_t> b((rr + 2) * W, 0);
      for (std::size_t k = 0; k < rr + 2; ++k) {
        const long src = static_cast<long>(r0 + k) - 1;
        if (src >= 0 && src < static_cast<long>(H)) std::copy_n(img.data() + src * W, W, b.data() + k * W);
      }
      bands.push_back(Element::bytes(b));
    }
    Dataset d = create_dataset(std::move(bands), 4);
    Dataset h = eh.map_cl_partition(d, "sobel");
    EXPECT(same(h, eg.map_cl_partition(d, "sobel")), "seam A sobel bitwise");
    EXPECT(same(h, eb.map_cl_partition(d, "sobel")), "seam B sobel bitwise");
  });

  run_case("errors: empty partition -> JobFailed, EmptyDataset, ArityMismatch, LengthMismatch", [&] {
    bool jf = false;
    try {
      eg.map_cl_partition(f32_dataset({{1.0f}, {2.0f}}, 3), "psum");
    } catch (const JobFailed&) {
      jf = true;
    }
    EXPECT(jf, "empty partition JobFailed");
    bool ed = false;
    try {
      eg.reduce_cl(Dataset(std::vector<Partition>(2)), "sum2");
    } catch (const EmptyDataset&) {
      ed = true;
    }
    EXPECT(ed, "EmptyDataset");
    bool am = false;
    try {
      eg.map_cl(f32_dataset({{1.0f}}, 1), "sum2");
    } catch (const ArityMismatch&) {
      am = true;
    }
    EXPECT(am, "ArityMismatch");
    bool lm = false;
    try {
      eg.reduce_cl(f32_dataset({{1.0f, 2.0f}, {1.0f}}, 1), "sum2");
    } catch (const JobFailed&) {
      lm = true;
    }
    EXPECT(lm, "LengthMismatch -> JobFailed");
    const std::uint64_t before = gpu.tasks_run();
    Element r = eg.reduce_cl(f32_dataset({{3.5f, 4.5f}}, 4), "sum2");
    EXPECT(gpu.tasks_run() == before && r.as_f32()[0] == 3.5f, "single element: zero tasks");
  });

  run_case("matmul n=256 (fp32-faithful 3xTF32 tcgen05 vs host fp32, tolerance), seam A and B", [&] {
    const std::size_t n = 256;
    std::vector<std::vector<float>> es(2, std::vector<float>(2 * n * n));
    for (std::size_t e = 0; e < 2; ++e)
      for (std::size_t i = 0; i < 2 * n * n; ++i) es[e][i] = 2.0f * u01(100 + e, i) - 1.0f;
    Dataset d = f32_dataset(es, 2);
    Dataset h = eh.map_cl(d, "matmul");
    for (Engine* e : {&eg, &eb}) {
      Dataset g = e->map_cl(d, "matmul");
      for (std::size_t p = 0; p < 2; ++p) {
        auto a = h.partitions()[p].elements[0].as_f32();
        auto b = g.partitions()[p].elements[0].as_f32();
        double ss = 0, md = 0;
        for (std::size_t i = 0; i < a.size(); ++i) {
          ss += double(a[i]) * a[i];
          md = std::max(md, std::abs(double(a[i]) - b[i]));
        }
        EXPECT(md <= 5e-5 * std::sqrt(ss / a.size()), "matmul within fp32-level tolerance (5e-5 of rms)");
      }
    }
  });

  run_case("wordcount over create_from_text chunks: GPU flags (seam A, B) == host tables", [&] {
    std::string corpus;
    const char dl[4] = {' ', '\t', '\n', '\r'};
    for (std::size_t i = 0; i < 30000; ++i) {
      const std::uint64_t z = kernels::mix64(5 + i);
      corpus += "w" + std::to_string(z % 97);
      corpus.append(1 + ((z >> 40) & 1), dl[(z >> 32) & 3]);
    }
    const std::string path = "/tmp/ucores_b200_wc.txt";
    {
      std::ofstream f(path, std::ios::binary);
      f << corpus;
    }
    Dataset d = create_from_text(path, 16384);
    KernelRegistry reg0;
    DeviceOpRegistry ops0;
    WorkloadParams p0;
    p0.wordcount_min_device_bytes = 0;  // every chunk takes the device path
    register_workload(reg0, ops0, p0);
    HostDriver h0(reg0);
    GpuClusterDriver g0(reg0, ops0);
    GpuClusterDriver::Options pt;
    pt.mode = GpuClusterDriver::Mode::PerTask;
    GpuClusterDriver b0(reg0, ops0, pt);
    Engine eh0(h0, reg0), eg0(g0, reg0), eb0(b0, reg0);
    Dataset host = eh0.map_cl(d, "wordcount");
    EXPECT(same(host, eg0.map_cl(d, "wordcount")), "seam A tables equal");
    EXPECT(same(host, eb0.map_cl(d, "wordcount")), "seam B tables equal");
    // default threshold 65536 > 16 KB chunks: all chunks decline the device
    Dataset fb = eg.map_cl(d, "wordcount");
    EXPECT(same(host, fb), "selective-execution path equal");
  });

  run_case("no device body -> JobFailed (no CPU fallback)", [&] {
    KernelRegistry reg;
    DeviceOpRegistry ops;
    reg.register_unary("hostonly", [] { return std::make_unique<kernels::Axpb>(1.f, 0.f); });
    GpuClusterDriver d(reg, ops);
    Engine e(d, reg);
    bool jf = false;
    try {
      e.map_cl(f32_dataset({{1.0f}}, 1), "hostonly");
    } catch (const JobFailed&) {
      jf = true;
    }
    EXPECT(jf, "JobFailed");
  });

  run_case("C2-shaped map->psum->reduce at 2^27 (16 partitions of 2^23)", [&] {
    const std::size_t P = 16, L = 1u << 23;
    std::vector<std::vector<float>> es(P, std::vector<float>(L));
    for (std::size_t p = 0; p < P; ++p)
      for (std::size_t i = 0; i < L; ++i) es[p][i] = u01(1000 + p, i);
    Dataset x = f32_dataset(es, P);
    es.clear();
    auto t0 = std::chrono::steady_clock::now();
    Dataset yg = eg.map_cl(x, "axpb");
    Element rg = eg.reduce_cl(eg.map_cl_partition(yg, "psum"), "sum2");
    auto t1 = std::chrono::steady_clock::now();
    Dataset yh = eh.map_cl(x, "axpb");
    Element rh = eh.reduce_cl(eh.map_cl_partition(yh, "psum"), "sum2");
    auto t2 = std::chrono::steady_clock::now();
    EXPECT(same(yh, yg), "y bitwise");
    EXPECT(rg == rh, "sum bitwise");
    std::printf("  engine e2e: gpu %.1f ms, host-seq %.1f ms\n",
                std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(t2 - t1).count());
  });

  // ---- DeviceEngine: device-resident chains vs the reference Engine ----
  WorkloadParams dparams;
  dparams.sobel_width = 48;
  dparams.matmul_n = 256;
  DeviceEngine de(dparams);

  run_case("device dataset: upload/collect round trip, all array kinds", [&] {
    std::vector<Partition> parts(4);
    parts[0].elements = {Element::f32({1.5f, -0.0f, 3e38f}), Element::f32({})};
    parts[2].elements = {Element::i64({-1, 1ll << 62}), Element::i64({7})};
    parts[3].elements = {Element::bytes("hello"), Element::bytes(std::string(1000, 'x'))};
    Dataset d(std::move(parts));
    EXPECT(same(d, de.collect(de.upload(d))), "collect(upload(d)) == d");
  });

  run_case("device dataset: create_dataset from host arrays == upload(ucores::create_dataset)", [&] {
    for (auto [count, parts, len] : std::vector<std::tuple<std::size_t, std::size_t, std::size_t>>{
             {10, 3, 5}, {7, 9, 1000}, {64, 8, 1u << 16}, {1u << 12, 4, 1}}) {
      std::vector<std::vector<float>> es(count, std::vector<float>(len));
      for (std::size_t i = 0; i < count; ++i)
        for (std::size_t j = 0; j < len; ++j) es[i][j] = u01(31 + i, j);
      std::vector<std::span<const std::uint8_t>> spans;
      std::vector<Element> host;
      for (const auto& v : es) {
        spans.emplace_back(reinterpret_cast<const std::uint8_t*>(v.data()), v.size() * 4);
        host.push_back(Element::f32(v));
      }
      Dataset hd = create_dataset(std::move(host), parts);
      DeviceDataset dd = de.create_dataset(spans, ElementKind::F32Array, parts);
      EXPECT(same(hd, de.collect(dd)), "create_dataset partitions and payloads");
      for (const char* op : {"sum", "max"}) {
        const std::string pk = std::string("p") + op, rk = std::string(op) + "2";
        bool empty = false;
        for (const Partition& p : hd.partitions()) empty |= p.elements.empty();
        if (empty) continue;  // map_cl_partition over an empty partition fails in both engines
        EXPECT(eh.reduce_cl(eh.map_cl_partition(eh.map_cl(hd, "axpb"), pk), rk) ==
                   de.reduce_cl(de.map_cl_partition(de.map_cl(dd, "axpb"), pk), rk),
               "chain over the ingested dataset");
      }
    }
    bool threw = false;
    try {
      de.create_dataset({}, ElementKind::F32Array, 0);
    } catch (const InvalidPartitionCount&) {
      threw = true;
    }
    EXPECT(threw, "0 partitions -> InvalidPartitionCount");
  });

  run_case("device dataset: C1 chains bitwise vs host Engine (packed and ragged elements)", [&] {
    for (auto [n, elems, parts] : std::vector<std::tuple<std::size_t, std::size_t, std::size_t>>{
             {1u << 20, 4, 4}, {100003, 13, 5}, {70001, 7, 3}, {4099, 33, 6}}) {
      std::vector<std::vector<float>> es(elems);
      std::size_t pos = 0;
      for (std::size_t k = 0; k < elems; ++k) {
        es[k].resize(n / elems + (k < n % elems ? 1 : 0));
        for (auto& v : es[k]) v = u01(777, pos++);
      }
      Dataset x = f32_dataset(es, parts);
      DeviceDataset dx = de.upload(x);
      Dataset yh = eh.map_cl(x, "axpb");
      DeviceDataset dy = de.map_cl(dx, "axpb");
      EXPECT(same(yh, de.collect(dy)), "device map_cl(axpb) bitwise");
      for (const char* op : {"sum", "max"}) {
        const std::string pk = std::string("p") + op, rk = std::string(op) + "2";
        Dataset ph = eh.map_cl_partition(yh, pk);
        DeviceDataset dp = de.map_cl_partition(dy, pk);
        EXPECT(same(ph, de.collect(dp)), "device map_cl_partition bitwise");
        EXPECT(eh.reduce_cl(ph, rk) == de.reduce_cl(dp, rk), "device reduce_cl bitwise");
        // per-element psum (map_cl) and reduce_cl straight over the mapped vectors' partials
        Dataset eph = eh.map_cl(yh, pk);
        DeviceDataset edp = de.map_cl(dy, pk);
        EXPECT(same(eph, de.collect(edp)), "device map_cl(psum) per element bitwise");
        EXPECT(eh.reduce_cl(eph, rk) == de.reduce_cl(edp, rk), "device reduce_cl over element partials");
      }
    }
  });

  run_case("device dataset: reduce_cl vectoradd / isum2 with empty and ragged partitions", [&] {
    std::uint64_t s = 11;
    for (int c = 0; c < 12; ++c) {
      const std::size_t count = 1 + kernels::mix64(s++) % 30, parts = 1 + kernels::mix64(s++) % 12,
                        len = 1 + kernels::mix64(s++) % 300;
      std::vector<Element> ef, ei;
      for (std::size_t i = 0; i < count; ++i) {
        std::vector<float> vf(len);
        std::vector<std::int64_t> vi(len);
        for (std::size_t j = 0; j < len; ++j) {
          vf[j] = 2.0f * u01(s, j) - 1.0f;
          vi[j] = static_cast<std::int64_t>(kernels::mix64(s + j));
        }
        ++s;
        ef.push_back(Element::f32(vf));
        ei.push_back(Element::i64(vi));
      }
      Dataset df = create_dataset(std::move(ef), parts), di = create_dataset(std::move(ei), parts);
      EXPECT(eh.reduce_cl(df, "vectoradd") == de.reduce_cl(de.upload(df), "vectoradd"), "vectoradd bitwise");
      EXPECT(eh.reduce_cl(df, "max2") == de.reduce_cl(de.upload(df), "max2"), "max2 bitwise");
      EXPECT(eh.reduce_cl(di, "isum2") == de.reduce_cl(de.upload(di), "isum2"), "isum2 exact");
    }
  });

  run_case("device dataset: pi map_cl + isum2, sobel, matmul", [&] {
    std::vector<Element> es;
    for (int t = 0; t < 8; ++t) es.push_back(Element::i64({42 + t, 500000}));
    Dataset d = create_dataset(std::move(es), 3);
    DeviceDataset hits = de.map_cl(de.upload(d), "pi");
    EXPECT(same(eh.map_cl(d, "pi"), de.collect(hits)), "pi {hits, samples} bitwise");
    EXPECT(de.reduce_cl(hits, "isum2").as_i64()[0] == 3141371, "pi total 3141371");

    const std::size_t H = 50, W = 48, R = 16;
    std::vector<Element> bands;
    for (std::size_t r0 = 0; r0 < H; r0 += R) {
      const std::size_t rr = std::min(R, H - r0);
      std::vector<std::uint8_t> b((rr + 2) * W);
      for (std::size_t i = 0; i < b.size(); ++i)
        b[i] = static_cast<std::uint8_t>(kernels::mix64(9 + r0 * W + i) >> 56);
      bands.push_back(Element::bytes(b));
    }
    Dataset sb = create_dataset(std::move(bands), 2);
    EXPECT(same(eh.map_cl(sb, "sobel"), de.collect(de.map_cl(de.upload(sb), "sobel"))), "sobel per band bitwise");
    Dataset one = create_dataset(std::vector<Element>(sb.partitions()[0].elements.begin(),
                                                      sb.partitions()[0].elements.begin() + 1), 1);
    EXPECT(same(eh.map_cl_partition(one, "sobel"), de.collect(de.map_cl_partition(de.upload(one), "sobel"))),
           "sobel map_cl_partition bitwise");

    const std::size_t n = 256;
    std::vector<std::vector<float>> ab(2, std::vector<float>(2 * n * n));
    for (std::size_t e = 0; e < 2; ++e)
      for (std::size_t i = 0; i < 2 * n * n; ++i) ab[e][i] = 2.0f * u01(200 + e, i) - 1.0f;
    Dataset md = f32_dataset(ab, 1);  // two elements in one partition: per-element GEMMs
    Dataset h = eh.map_cl(md, "matmul"), g = de.collect(de.map_cl(de.upload(md), "matmul"));
    for (std::size_t e = 0; e < 2; ++e) {
      auto a = h.partitions()[0].elements[e].as_f32();
      auto b = g.partitions()[0].elements[e].as_f32();
      double ss = 0, md2 = 0;
      for (std::size_t i = 0; i < a.size(); ++i) {
        ss += double(a[i]) * a[i];
        md2 = std::max(md2, std::abs(double(a[i]) - b[i]));
      }
      EXPECT(md2 <= 5e-5 * std::sqrt(ss / a.size()), "device matmul within fp32-level tolerance (5e-5 of rms)");
    }
  });

  run_case("device dataset: errors as the reference Engine", [&] {
    auto throws = [](auto fn, auto tag) {
      try {
        fn();
      } catch (const decltype(tag)&) {
        return true;
      } catch (...) {
        return false;
      }
      return false;
    };
    DeviceDataset holes = de.upload(f32_dataset({{1.0f}, {2.0f}}, 3));
    EXPECT(throws([&] { de.map_cl_partition(holes, "psum"); }, JobFailed("")), "empty partition -> JobFailed");
    EXPECT(throws([&] { de.reduce_cl(de.upload(Dataset(std::vector<Partition>(2))), "sum2"); }, EmptyDataset("")),
           "EmptyDataset");
    EXPECT(throws([&] { de.reduce_cl(de.upload(f32_dataset({{1.0f, 2.0f}, {1.0f}}, 1)), "sum2"); }, JobFailed("")),
           "length mismatch -> JobFailed");
    EXPECT(throws([&] { de.map_cl(holes, "nosuch"); }, UnknownKernel("")), "UnknownKernel");
    EXPECT(throws([&] { de.map_cl(de.upload(create_dataset({Element::bytes("ab")}, 1)), "axpb"); }, JobFailed("")),
           "kind mismatch -> JobFailed");
    Element r = de.reduce_cl(de.upload(f32_dataset({{3.5f, 4.5f}}, 4)), "sum2");
    EXPECT(r.as_f32().size() == 2 && r.as_f32()[0] == 3.5f, "single element returned as is");
  });

  run_case("device dataset: C1 literal form (one float per element)", [&] {
    for (std::size_t n : {std::size_t(1) << 16, std::size_t(1) << 20}) {
      std::vector<Element> es;
      es.reserve(n);
      for (std::size_t i = 0; i < n; ++i) es.push_back(Element::f32({u01(12345, i)}));
      Dataset x = create_dataset(std::move(es), 4);
      auto t0 = std::chrono::steady_clock::now();
      DeviceDataset dy = de.map_cl(de.upload(x), "axpb");
      Element rd = de.reduce_cl(de.map_cl_partition(dy, "psum"), "sum2");
      auto t1 = std::chrono::steady_clock::now();
      if (n <= (1u << 16)) {  // the host Engine runs one task per element: keep it small
        Dataset yh = eh.map_cl(x, "axpb");
        EXPECT(same(yh, de.collect(dy)), "literal map_cl bitwise");
        EXPECT(eh.reduce_cl(eh.map_cl_partition(yh, "psum"), "sum2") == rd, "literal chain bitwise");
      }
      std::printf("  literal 2^%d elements: device chain incl. upload %.2f ms\n", int(std::log2(double(n))),
                  std::chrono::duration<double, std::milli>(t1 - t0).count());
      // reduce_cl straight over the one-float elements: n-1 ReducePair tasks
      // in the reference (stage-1 folds of 2^18 elements per partition)
      DeviceDataset dx = de.upload(x);
      auto t2 = std::chrono::steady_clock::now();
      Element rr = de.reduce_cl(dx, "sum2");
      auto t3 = std::chrono::steady_clock::now();
      if (n <= (1u << 16)) EXPECT(rr == eh.reduce_cl(x, "sum2"), "literal reduce_cl bitwise vs host Engine");
      std::printf("  literal 2^%d elements: device reduce_cl %.2f ms\n", int(std::log2(double(n))),
                  std::chrono::duration<double, std::milli>(t3 - t2).count());
    }
  });

  run_case("device dataset: C2-shaped chain at 2^27, one upload, one result back", [&] {
    const std::size_t P = 16, L = 1u << 23;
    std::vector<std::vector<float>> es(P, std::vector<float>(L));
    for (std::size_t p = 0; p < P; ++p)
      for (std::size_t i = 0; i < L; ++i) es[p][i] = u01(1000 + p, i);
    Dataset x = f32_dataset(es, P);
    es.clear();
    de.upload(x);  // first use: pinned staging and pool allocations
    auto t0 = std::chrono::steady_clock::now();
    DeviceDataset dx = de.upload(x);
    auto t1 = std::chrono::steady_clock::now();
    DeviceDataset dy = de.map_cl(dx, "axpb");
    auto ta = std::chrono::steady_clock::now();
    DeviceDataset dp = de.map_cl_partition(dy, "psum");
    auto tb = std::chrono::steady_clock::now();
    Element rd = de.reduce_cl(dp, "sum2");
    auto t2 = std::chrono::steady_clock::now();
    Element rh = eh.reduce_cl(eh.map_cl_partition(eh.map_cl(x, "axpb"), "psum"), "sum2");
    EXPECT(rd == rh, "sum bitwise vs host Engine");
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::printf("  device engine: upload %.1f ms, chain %.2f ms (map_cl %.2f, map_cl_partition %.2f, reduce_cl %.2f)\n",
                ms(t0, t1), ms(t1, t2), ms(t1, ta), ms(ta, tb), ms(tb, t2));
    auto t3 = std::chrono::steady_clock::now();
    Element rd2 = de.reduce_cl(de.map_cl_partition(de.map_cl(dx, "axpb"), "psum"), "sum2");
    auto t4 = std::chrono::steady_clock::now();
    EXPECT(rd2 == rh, "repeat chain bitwise");
    std::printf("  device engine: repeated chain %.2f ms\n", ms(t3, t4));
  });

  std::printf("RESULT pass=%d fail=%d\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
