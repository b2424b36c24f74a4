// stream_bench.cu — dev microbenchmark: which read+write streaming pattern
// reaches the B200 HBM roofline for y = fl(fl(a*x)+b) over 2^30 floats.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/stream_bench tools/stream_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ float aff(float x, float a, float b) { return __fadd_rn(__fmul_rn(a, x), b); }
__device__ __forceinline__ float4 aff4(float4 v, float a, float b) {
  v.x = aff(v.x, a, b); v.y = aff(v.y, a, b); v.z = aff(v.z, a, b); v.w = aff(v.w, a, b); return v;
}

template <int U, int MODE>
__global__ void k_grid(const float4* __restrict__ x, float4* __restrict__ y, uint64_t n4, float a, float b) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 0) v[u] = x[i + u * stride];
      else if (MODE == 1) v[u] = __ldcs(x + i + u * stride);
      else {
        const float4* p = x + i + u * stride;
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(p));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float4 r = aff4(v[u], a, b);
      if (MODE == 0) y[i + u * stride] = r;
      else if (MODE == 1) __stcs(y + i + u * stride, r);
      else {
        float4* p = y + i + u * stride;
        asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(r.x), "f"(r.y), "f"(r.z), "f"(r.w) : "memory");
      }
    }
  }
  for (; i < n4; i += stride) y[i] = aff4(x[i], a, b);
}

// contiguous-chunk variant: each warp streams a contiguous 16 KB item (like the reduce kernel)
template <int U>
__global__ void k_items(const float* __restrict__ x, float* __restrict__ y, uint64_t nitems, float a, float b) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t it = warp; it < nitems; it += nw) {
    const float* xp = x + (it << 14);
    float* yp = y + (it << 14);
    for (int c = 0; c < 16384 / (128 * U); ++c) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(xp + (c * U + u) * 128 + 4 * lane));
#pragma unroll
      for (int u = 0; u < U; ++u) __stcs(reinterpret_cast<float4*>(yp + (c * U + u) * 128 + 4 * lane), aff4(v[u], a, b));
    }
  }
}

// ---- TMA bulk pipeline -------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst), "r"(smem_u32(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int TILE_BYTES, int STAGES, int OUTBUF>
__global__ void __launch_bounds__(256, 1) k_tma(const float* __restrict__ x, float* __restrict__ y, uint64_t ntiles, float a, float b) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* in = reinterpret_cast<float*>(smem);
  float* out = reinterpret_cast<float*>(smem + STAGES * TILE_BYTES);
  __shared__ uint64_t bars[STAGES];
  constexpr int TF = TILE_BYTES / 4;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // tiles of this CTA: blockIdx.x, +gridDim.x, ...
  const uint64_t my = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (tid == 0) {
    for (int s = 0; s < STAGES && s < (int)my; ++s) {
      mbar_expect_tx(&bars[s], TILE_BYTES);
      bulk_g2s(in + s * TF, x + (blockIdx.x + uint64_t(s) * gridDim.x) * TF, TILE_BYTES, &bars[s]);
    }
  }
  for (uint64_t k = 0; k < my; ++k) {
    const int s = int(k % STAGES);
    const uint32_t par = uint32_t((k / STAGES) & 1);
    const int ob = int(k % OUTBUF);
    mbar_wait(&bars[s], par);
    // out buffer ob must be drained by its previous bulk store
    if (tid == 0) bulk_wait_read<OUTBUF - 1>();
    __syncthreads();
    const float4* src = reinterpret_cast<const float4*>(in + s * TF);
    float4* dst = reinterpret_cast<float4*>(out + ob * TF);
#pragma unroll 4
    for (int i = tid; i < TF / 4; i += 256) dst[i] = aff4(src[i], a, b);
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      const uint64_t tile = blockIdx.x + k * gridDim.x;
      bulk_s2g(y + tile * TF, out + ob * TF, TILE_BYTES);
      bulk_commit();
      if (k + STAGES < my) {
        mbar_expect_tx(&bars[s], TILE_BYTES);
        bulk_g2s(in + s * TF, x + (blockIdx.x + (k + STAGES) * gridDim.x) * TF, TILE_BYTES, &bars[s]);
      }
    }
  }
  if (tid == 0) bulk_wait_read<0>();
  __syncthreads();
}

// per-warp TMA ring: lane 0 keeps S bulk copies of 4 KB chunks in flight for
// its warp's contiguous items; all lanes read the chunk from smem, map, STG.
template <int S>
__global__ void __launch_bounds__(256) k_warp_tma(const float* __restrict__ x, float* __restrict__ y, uint64_t nitems,
                                                  float a, float b) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[8][S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* ring = reinterpret_cast<float*>(smem) + warp * S * 1024;
  const uint64_t gw = uint64_t(blockIdx.x) * 8 + warp, nw = uint64_t(gridDim.x) * 8;
  const uint64_t my_items = nitems > gw ? (nitems - gw + nw - 1) / nw : 0;
  const uint64_t total = my_items * 16;  // 16 chunks of 1024 floats per 16K item
  auto chunk_src = [&](uint64_t q) { return x + ((gw + (q >> 4) * nw) << 14) + ((q & 15) << 10); };
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint64_t q = 0; q < S && q < total; ++q) {
      mbar_expect_tx(&bars[warp][q], 4096);
      bulk_g2s(ring + q * 1024, chunk_src(q), 4096, &bars[warp][q]);
    }
  }
  __syncwarp();
  for (uint64_t q = 0; q < total; ++q) {
    const int s = int(q % S);
    mbar_wait(&bars[warp][s], uint32_t((q / S) & 1));
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = reinterpret_cast<const float4*>(ring + s * 1024)[u * 32 + lane];
    __syncwarp();
    if (lane == 0 && q + S < total) {
      mbar_expect_tx(&bars[warp][s], 4096);
      bulk_g2s(ring + s * 1024, chunk_src(q + S), 4096, &bars[warp][s]);
    }
    float* dst = y + (chunk_src(q) - x);
#pragma unroll
    for (int u = 0; u < 8; ++u) __stcs(reinterpret_cast<float4*>(dst) + u * 32 + lane, aff4(v[u], a, b));
  }
}

int main() {
  const uint64_t n = 1ull << 30;
  float *x, *y;
  CK(cudaMalloc(&x, n * 4));
  CK(cudaMalloc(&y, n * 4));
  CK(cudaMemset(x, 0x3f, n * 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto bench = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    std::vector<float> ts;
    for (int i = 0; i < 15; ++i) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    printf("%-44s %8.3f ms  %7.1f GB/s\n", name, ts[ts.size() / 2], 8.0 * n / ts[ts.size() / 2] / 1e6);
  };
  const uint64_t n4 = n / 4;
  bench("cudaMemcpy D2D", [&] { cudaMemcpyAsync(y, x, n * 4, cudaMemcpyDeviceToDevice); });
  for (int bpsm : {4, 8, 16}) {
    char nm[128];
    snprintf(nm, sizeof nm, "grid plain U4 256thr x %d/SM", bpsm);
    bench(nm, [&] { k_grid<4, 0><<<sms * bpsm, 256>>>((const float4*)x, (float4*)y, n4, 2.f, 1.f); });
    snprintf(nm, sizeof nm, "grid cs    U4 256thr x %d/SM", bpsm);
    bench(nm, [&] { k_grid<4, 1><<<sms * bpsm, 256>>>((const float4*)x, (float4*)y, n4, 2.f, 1.f); });
    snprintf(nm, sizeof nm, "grid nc.noalloc U4 256thr x %d/SM", bpsm);
    bench(nm, [&] { k_grid<4, 2><<<sms * bpsm, 256>>>((const float4*)x, (float4*)y, n4, 2.f, 1.f); });
    snprintf(nm, sizeof nm, "grid plain U8 256thr x %d/SM", bpsm);
    bench(nm, [&] { k_grid<8, 0><<<sms * bpsm, 256>>>((const float4*)x, (float4*)y, n4, 2.f, 1.f); });
  }
  for (int bpsm : {3, 4, 8}) {
    char nm[128];
    snprintf(nm, sizeof nm, "items16K U8 cs 256thr x %d/SM", bpsm);
    bench(nm, [&] { k_items<8><<<sms * bpsm, 256>>>(x, y, n >> 14, 2.f, 1.f); });
    snprintf(nm, sizeof nm, "items16K U4 cs 256thr x %d/SM", bpsm);
    bench(nm, [&] { k_items<4><<<sms * bpsm, 256>>>(x, y, n >> 14, 2.f, 1.f); });
  }
  {
    constexpr int T = 32768, S = 4, O = 2;
    auto kf = k_tma<T, S, O>;
    CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (S + O) * T));
    bench("tma 32K x4 stages out2, 1 CTA/SM", [&] { kf<<<sms, 256, (S + O) * T>>>(x, y, n * 4 / T, 2.f, 1.f); });
  }
  {
    constexpr int T = 16384, S = 4, O = 2;
    auto kf = k_tma<T, S, O>;
    CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (S + O) * T));
    bench("tma 16K x4 stages out2, 2 CTA/SM", [&] { kf<<<sms * 2, 256, (S + O) * T>>>(x, y, n * 4 / T, 2.f, 1.f); });
  }
  {
    constexpr int T = 16384, S = 8, O = 2;
    auto kf = k_tma<T, S, O>;
    CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (S + O) * T));
    bench("tma 16K x8 stages out2, 1 CTA/SM", [&] { kf<<<sms, 256, (S + O) * T>>>(x, y, n * 4 / T, 2.f, 1.f); });
  }
  {
    constexpr int T = 8192, S = 8, O = 4;
    auto kf = k_tma<T, S, O>;
    CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (S + O) * T));
    bench("tma 8K x8 stages out4, 2 CTA/SM", [&] { kf<<<sms * 2, 256, (S + O) * T>>>(x, y, n * 4 / T, 2.f, 1.f); });
  }
  for (int S : {3, 4, 6}) {
    for (int cps : {1, 2}) {
      const int smem = 8 * S * 4096;
      char nm[128];
      snprintf(nm, sizeof nm, "warp-tma ring S=%d, %d CTA/SM (8 warps)", S, cps);
      if (S == 3) {
        CK(cudaFuncSetAttribute(k_warp_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        bench(nm, [&] { k_warp_tma<3><<<sms * cps, 256, smem>>>(x, y, n >> 14, 2.f, 1.f); });
      } else if (S == 4) {
        CK(cudaFuncSetAttribute(k_warp_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        bench(nm, [&] { k_warp_tma<4><<<sms * cps, 256, smem>>>(x, y, n >> 14, 2.f, 1.f); });
      } else if (cps == 1) {
        CK(cudaFuncSetAttribute(k_warp_tma<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        bench(nm, [&] { k_warp_tma<6><<<sms * cps, 256, smem>>>(x, y, n >> 14, 2.f, 1.f); });
      }
    }
  }
  // correctness spot check of the last run
  std::vector<float> hx(8), hy(8);
  cudaMemcpy(hx.data(), x + 12345, 32, cudaMemcpyDeviceToHost);
  cudaMemcpy(hy.data(), y + 12345, 32, cudaMemcpyDeviceToHost);
  printf("check %g -> %g (want %g)\n", hx[0], hy[0], 2.f * hx[0] + 1.f);
  return 0;
}
