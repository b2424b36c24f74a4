// literal_probe.cpp — time split of the C1 literal chain (2^20 one-float
// elements, 4 partitions) through the unmodified reference Engine and
// GpuClusterDriver (seam A): Dataset construction, then per Engine call the
// driver's run_wave time vs the Engine's own work. Built by
// tools/build_probes.sh; prints one JSON line per repetition.
#include <chrono>
#include <cstdio>
#include <vector>

#include "ucores/dataset.hpp"
#include "ucores/engine.hpp"
#include "ucores_b200/device_ops.hpp"
#include "ucores_b200/gpu_cluster_driver.hpp"

using namespace ucores;
using namespace ucores_b200;
using clk = std::chrono::steady_clock;
static double sec(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

struct Timed : ClusterDriver {
  GpuClusterDriver* d;
  double wave_s = 0;
  std::uint64_t new_job_id() override { return d->new_job_id(); }
  std::vector<TaskResult> run_wave(std::vector<Task> tasks, int max_retries) override {
    auto t0 = clk::now();
    auto r = d->run_wave(std::move(tasks), max_retries);
    wave_s += sec(t0, clk::now());
    return r;
  }
};

int main(int argc, char** argv) {
  const std::size_t n = argc > 1 ? std::atoll(argv[1]) : (1u << 20), P = 4;
  KernelRegistry reg;
  DeviceOpRegistry ops;
  register_workload(reg, ops);
  GpuClusterDriver::Options opt;
  opt.max_gpus = 1;
  GpuClusterDriver inner(reg, ops, opt);
  Timed drv;
  drv.d = &inner;
  Engine eng(drv, reg);
  std::vector<float> x(n);
  for (std::size_t i = 0; i < n; ++i) x[i] = float(i % 1000) * 1e-3f;
  for (int rep = 0; rep < 3; ++rep) {
    drv.wave_s = 0;
    auto t0 = clk::now();
    std::vector<Element> es;
    es.reserve(n);
    for (std::size_t i = 0; i < n; ++i) es.push_back(Element::f32({x[i]}));
    Dataset d = create_dataset(std::move(es), P);
    auto t1 = clk::now();
    Dataset y = eng.map_cl(d, "axpb");
    auto t2 = clk::now();
    const double w1 = drv.wave_s;
    Dataset ps = eng.map_cl_partition(y, "psum");
    auto t3 = clk::now();
    const double w2 = drv.wave_s - w1;
    Element r = eng.reduce_cl(ps, "sum2");
    auto t4 = clk::now();
    const double w3 = drv.wave_s - w1 - w2;
    {
      Dataset drop = std::move(y);
    }
    auto t5 = clk::now();
    std::printf("{\"rep\": %d, \"build_s\": %.4f, \"map_cl_s\": %.4f, \"map_wave_s\": %.4f, \"mcp_s\": %.4f, "
                "\"mcp_wave_s\": %.4f, \"reduce_s\": %.4f, \"reduce_wave_s\": %.4f, \"total_s\": %.4f, "
                "\"free_y_s\": %.4f, \"melem_s\": %.3f, \"r\": %.6f}\n",
                rep, sec(t0, t1), sec(t1, t2), w1, sec(t2, t3), w2, sec(t3, t4), w3, sec(t0, t4), sec(t4, t5),
                n / sec(t0, t4) / 1e6, r.as_f32()[0]);
  }
  return 0;
}
