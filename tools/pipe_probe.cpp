// pipe_probe.cpp — rates of the drop-in's host transfer pipeline
// (host/ucores_b200/host_pipe.hpp) on this box: upload of resident pageable
// vectors, download into fresh vectors, and the interleaved map wave.
// Built by tools/build_probes.sh; prints one JSON line per measurement.
#include <chrono>
#include <cstdio>
#include <vector>

#include "ucores_b200/host_pipe.hpp"

using namespace ucores_b200;
using clk = std::chrono::steady_clock;
static double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

int main(int argc, char** argv) {
  const std::size_t pieces = argc > 1 ? std::atoi(argv[1]) : 64, n = argc > 2 ? std::atoll(argv[2]) : (1u << 24);
  Gpu g(0);
  HostPipe& pipe = g.attached<HostPipe>();
  work_pool();
  std::vector<std::vector<float>> in(pieces, std::vector<float>(n, 1.5f));
  float* x = static_cast<float*>(g.scratch(0).ensure(pieces * n * 4));
  float* y = static_cast<float*>(g.scratch(1).ensure(pieces * n * 4));
  const double gb = pieces * n * 4 / 1e9;
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = clk::now();
    for (std::size_t i = 0; i < pieces; ++i) pipe.upload(x + i * n, in[i].data(), n * 4);
    pipe.compute_after_upload();
    pipe.drain();
    auto t1 = clk::now();
    printf("{\"rep\": %d, \"upload_gbs\": %.2f}\n", rep, gb / secs(t0, t1));
    {
      std::vector<std::vector<float>> out(pieces);
      t0 = clk::now();
      std::vector<std::shared_ptr<WorkPool::Done>> ready(pieces);
      for (std::size_t i = 0; i < pieces; ++i) ready[i] = pipe.prepare(&out[i], n);
      for (std::size_t i = 0; i < pieces; ++i) pipe.download(&out[i], x + i * n, n, ready[i]);
      pipe.drain();
      t1 = clk::now();
      printf("{\"rep\": %d, \"download_fresh_gbs\": %.2f}\n", rep, gb / secs(t0, t1));
      t0 = clk::now();
      for (std::size_t i = 0; i < pieces; ++i) pipe.download(&out[i], x + i * n, n, ready[i]);
      pipe.drain();
      t1 = clk::now();
      printf("{\"rep\": %d, \"download_resident_gbs\": %.2f}\n", rep, gb / secs(t0, t1));
    }
    {
      std::vector<std::vector<float>> out(pieces);
      t0 = clk::now();
      std::vector<std::shared_ptr<WorkPool::Done>> ready(pieces);
      for (std::size_t i = 0; i < pieces; ++i) ready[i] = pipe.prepare(&out[i], n);
      for (std::size_t i = 0; i < pieces; ++i) {
        pipe.upload(x + i * n, in[i].data(), n * 4);
        pipe.compute_after_upload();
        check(ucg_map_affine_f32(x + i * n, y + i * n, n, 2.f, 1.f, g.stream()));
        pipe.download(&out[i], y + i * n, n, ready[i]);
      }
      pipe.drain();
      t1 = clk::now();
      printf("{\"rep\": %d, \"map_wave_s\": %.4f, \"map_wave_in_gbs\": %.2f, \"ok\": %d}\n", rep, secs(t0, t1),
             gb / secs(t0, t1), out[pieces - 1][n - 1] == 4.0f);
    }
  }
  return 0;
}
