// host_copy_probe.cpp — measures the host-side costs that bound the drop-in's
// end-to-end path on this box: memcpy into resident / fresh memory (1 and N
// threads), std::vector copies as the reference Engine makes them, pinning
// (cudaHostRegister) rates, and H2D / D2H from pageable, pinned and
// registered memory. Build: g++ -O2 -std=c++20 -pthread tools/host_copy_probe.cpp
//   -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -o build/host_copy_probe
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <string>
#include <thread>
#include <vector>

using clk = std::chrono::steady_clock;
static double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

static void par(unsigned n, const std::function<void(unsigned)>& f) {
  std::vector<std::thread> t;
  for (unsigned i = 1; i < n; ++i) t.emplace_back(f, i);
  f(0);
  for (auto& x : t) x.join();
}

int main() {
  const size_t chunk = 64ull << 20, nchunks = 16, total = chunk * nchunks;  // 1 GiB
  const unsigned T = std::thread::hardware_concurrency();
  {
    std::ifstream f("/sys/kernel/mm/transparent_hugepage/enabled");
    std::string s;
    std::getline(f, s);
    printf("{\"threads\": %u, \"thp\": \"%s\"}\n", T, s.c_str());
  }
  std::vector<char> src(total, 1), dst(total, 2);
  auto t0 = clk::now();
  std::memcpy(dst.data(), src.data(), total);
  auto t1 = clk::now();
  printf("{\"memcpy_resident_1t_gbs\": %.2f}\n", total / secs(t0, t1) / 1e9);
  for (unsigned n : {2u, 4u, 8u, T}) {
    t0 = clk::now();
    par(n, [&](unsigned i) {
      size_t per = total / n, b = i * per;
      std::memcpy(dst.data() + b, src.data() + b, i == n - 1 ? total - b : per);
    });
    t1 = clk::now();
    printf("{\"memcpy_resident_%ut_gbs\": %.2f}\n", n, total / secs(t0, t1) / 1e9);
  }
  // the Engine's copies: a fresh std::vector<float> copy of a 64 MB element (malloc -> mmap -> faults)
  {
    std::vector<std::vector<float>> es(nchunks, std::vector<float>(chunk / 4, 1.0f));
    t0 = clk::now();
    for (int rep = 0; rep < 2; ++rep) {
      std::vector<std::vector<float>> cp;
      for (auto& e : es) cp.push_back(e);
    }
    t1 = clk::now();
    printf("{\"vector_copy_fresh_1t_gbs\": %.2f}\n", 2 * total / secs(t0, t1) / 1e9);
    t0 = clk::now();
    for (int rep = 0; rep < 2; ++rep) {
      std::vector<std::vector<float>> cp(nchunks);
      par(T, [&](unsigned i) {
        for (size_t k = i; k < nchunks; k += T) cp[k] = es[k];
      });
    }
    t1 = clk::now();
    printf("{\"vector_copy_fresh_%ut_gbs\": %.2f}\n", T, 2 * total / secs(t0, t1) / 1e9);
    t0 = clk::now();
    for (int rep = 0; rep < 2; ++rep) {
      std::vector<std::vector<float>> cp(nchunks);
      for (auto& v : cp) v.resize(chunk / 4);
    }
    t1 = clk::now();
    printf("{\"vector_resize_zero_fresh_1t_gbs\": %.2f}\n", 2 * total / secs(t0, t1) / 1e9);
  }
  cudaSetDevice(0);
  cudaFree(0);
  void* d = nullptr;
  cudaMalloc(&d, total);
  void* pin = nullptr;
  cudaHostAlloc(&pin, total, 0);
  std::memset(pin, 3, total);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  auto h2d = [&](const void* p, const char* name) {
    cudaDeviceSynchronize();
    auto a = clk::now();
    for (size_t k = 0; k < nchunks; ++k) cudaMemcpyAsync((char*)d + k * chunk, (const char*)p + k * chunk, chunk, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    auto b = clk::now();
    printf("{\"h2d_%s_gbs\": %.2f}\n", name, total / secs(a, b) / 1e9);
  };
  auto d2h = [&](void* p, const char* name) {
    cudaDeviceSynchronize();
    auto a = clk::now();
    for (size_t k = 0; k < nchunks; ++k) cudaMemcpyAsync((char*)p + k * chunk, (const char*)d + k * chunk, chunk, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    auto b = clk::now();
    printf("{\"d2h_%s_gbs\": %.2f}\n", name, total / secs(a, b) / 1e9);
  };
  h2d(pin, "pinned");
  h2d(src.data(), "pageable");
  d2h(pin, "pinned");
  d2h(dst.data(), "pageable");
  // pinning in place
  t0 = clk::now();
  for (size_t k = 0; k < nchunks; ++k) cudaHostRegister(src.data() + k * chunk, chunk, cudaHostRegisterDefault);
  t1 = clk::now();
  printf("{\"host_register_1t_gbs\": %.2f}\n", total / secs(t0, t1) / 1e9);
  h2d(src.data(), "registered");
  t0 = clk::now();
  for (size_t k = 0; k < nchunks; ++k) cudaHostUnregister(src.data() + k * chunk);
  t1 = clk::now();
  printf("{\"host_unregister_1t_gbs\": %.2f}\n", total / secs(t0, t1) / 1e9);
  t0 = clk::now();
  par(T, [&](unsigned i) {
    for (size_t k = i; k < nchunks; k += T) cudaHostRegister(src.data() + k * chunk, chunk, cudaHostRegisterDefault);
  });
  t1 = clk::now();
  printf("{\"host_register_%ut_gbs\": %.2f}\n", T, total / secs(t0, t1) / 1e9);
  t0 = clk::now();
  par(T, [&](unsigned i) {
    for (size_t k = i; k < nchunks; k += T) cudaHostUnregister(src.data() + k * chunk);
  });
  t1 = clk::now();
  printf("{\"host_unregister_%ut_gbs\": %.2f}\n", T, total / secs(t0, t1) / 1e9);
  // register fresh (not yet faulted) memory: a reserved vector's capacity
  {
    std::vector<float> v;
    v.reserve(total / 4);
    t0 = clk::now();
    cudaHostRegister(v.data(), total, cudaHostRegisterDefault);
    t1 = clk::now();
    printf("{\"host_register_fresh_1t_gbs\": %.2f, \"err\": \"%s\"}\n", total / secs(t0, t1) / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaHostUnregister(v.data());
  }
  // pinned -> pageable resident memcpy with N threads (the D2H staging drain)
  t0 = clk::now();
  par(T, [&](unsigned i) {
    size_t per = total / T, b = i * per;
    std::memcpy(dst.data() + b, (char*)pin + b, i == T - 1 ? total - b : per);
  });
  t1 = clk::now();
  printf("{\"memcpy_pinned_to_resident_%ut_gbs\": %.2f}\n", T, total / secs(t0, t1) / 1e9);
  // pinned -> fresh vector via reserve + insert (no zero fill), N threads over 16 chunks
  for (int rep = 0; rep < 2; ++rep) {
    std::vector<std::vector<float>> outv(nchunks);
    t0 = clk::now();
    par(T, [&](unsigned i) {
      for (size_t k = i; k < nchunks; k += T) {
        outv[k].reserve(chunk / 4);
        const float* p = (const float*)((char*)pin + k * chunk);
        outv[k].insert(outv[k].end(), p, p + chunk / 4);
      }
    });
    t1 = clk::now();
    printf("{\"pinned_to_fresh_vector_%ut_gbs\": %.2f}\n", T, total / secs(t0, t1) / 1e9);
  }
  return 0;
}
