// p2p_pingpong.cu — dev microbenchmark: NVLink round-trip latency between two
// GPUs seen by kernels (one process, peer access enabled): GPU0 stores a
// sequence number into GPU1's memory, GPU1 polls and echoes it into GPU0's
// memory, N times inside one launch each. Variants: relaxed.sys stores with
// volatile polling; store + __threadfence_system.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/p2p_pingpong tools/p2p_pingpong.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void st_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void ping(uint32_t* remote, const uint32_t* local, int n, int fence, unsigned long long* t) {
  const unsigned long long t0 = clock64();
  for (int i = 1; i <= n; ++i) {
    st_sys(remote, i);
    if (fence) __threadfence_system();
    while (ld_sys(local) != uint32_t(i)) {
    }
  }
  *t = clock64() - t0;
}
__global__ void pong(uint32_t* remote, const uint32_t* local, int n, int fence) {
  for (int i = 1; i <= n; ++i) {
    while (ld_sys(local) != uint32_t(i)) {
    }
    st_sys(remote, i);
    if (fence) __threadfence_system();
  }
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("needs 2 GPUs\n"); return 0; }
  uint32_t *f0, *f1;
  unsigned long long* t;
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaMalloc(&f0, 256);
  cudaMalloc(&t, 8);
  cudaSetDevice(1);
  cudaDeviceEnablePeerAccess(0, 0);
  cudaMalloc(&f1, 256);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int fence = 0; fence < 2; ++fence) {
    cudaSetDevice(0); cudaMemset(f0, 0, 256); cudaDeviceSynchronize();
    cudaSetDevice(1); cudaMemset(f1, 0, 256); cudaDeviceSynchronize();
    const int N = 10000;
    cudaSetDevice(1);
    pong<<<1, 1>>>(f0, f1, N, fence);
    cudaSetDevice(0);
    ping<<<1, 1>>>(f1, f0, N, fence, t);
    cudaDeviceSynchronize();
    cudaSetDevice(1); cudaDeviceSynchronize();
    unsigned long long cyc = 0;
    cudaSetDevice(0);
    cudaMemcpy(&cyc, t, 8, cudaMemcpyDeviceToHost);
    printf("fence=%d: round trip %.3f us (clock %d kHz), err %s\n", fence, cyc / double(N) / (clk * 1e-3),
           clk, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
