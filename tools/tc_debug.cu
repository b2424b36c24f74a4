// tc_debug.cu — dev harness: isolate TMA / TMEM / tcgen05 pieces of ucg_gemm.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o build/tc_debug tools/tc_debug.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void k_tma_probe(const __grid_constant__ CUtensorMap tm, float* out, int c0, int c1) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(16384) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            sa(smem)), "l"(&tm), "r"(c0), "r"(c1), "r"(sa(&bar)) : "memory");
  }
  asm volatile("{\n .reg .pred p;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(sa(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = reinterpret_cast<float*>(smem)[i];
}

__global__ void k_tmem_probe(float* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = slot;
  const uint32_t taddr = t + (uint32_t(warp * 32) << 16);
  uint32_t v = __float_as_uint(float(threadIdx.x * 10 + 1));
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  out[threadIdx.x] = __uint_as_float(r);
  out[128 + threadIdx.x] = float(t);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(32));
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

// One 128x256x32 tf32 tile: A (K-major SW128) and B (MN-major SW128) written by
// threads in the swizzled canonical layouts, D read back. mode bit0: use mask form.
__global__ void k_mma_probe(const float* A, const float* B, float* D, int mode, uint32_t idesc) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* sA = reinterpret_cast<float*>(smem);           // 128 rows x 32 k, 128 B rows, SW128
  float* sB = reinterpret_cast<float*>(smem + 16384);   // 8 strips of (32 k rows x 32 n), SW128
  // SW128: 16B chunk index c (0..7) of row r is stored at chunk c ^ (r & 7)
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
    const int r = i / 32, k = i % 32, c = k / 4, w = k % 4;
    sA[r * 32 + ((c ^ (r & 7)) * 4) + w] = A[r * 32 + k];  // A given as [128][32]
  }
  for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) {
    const int k = i / 256, nn = i % 256, j = nn / 32, e = nn % 32, c = e / 4, w = e % 4;
    if (mode & 2) {  // 128B swizzle with 32B atoms: 32-byte granule g -> g ^ (k & 3)
      const int g = e / 8, o = e % 8;
      sB[j * 1024 + k * 32 + ((g ^ (k & 3)) * 8) + o] = B[k * 256 + nn];
    } else {
      sB[j * 1024 + k * 32 + ((c ^ (k & 7)) * 4) + w] = B[k * 256 + nn];  // B given as [32][256]
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = sa(sA), b = sa(sB);
    for (int k = 0; k < 4; ++k) {
      const uint64_t ad = desc_sw128(a + 32u * k, 16u, 1024u);
      uint64_t bd = desc_sw128(b + 1024u * k, 4096u, 1024u);
      if (mode & 2) bd = (bd & ~(7ull << 61) & ~(0x3FFFull << 32)) | (1ull << 61) | (uint64_t(512 >> 4) << 32);
      const uint32_t acc = k != 0;
      if (mode & 1) {
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n}\n" ::"r"(t),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(0u));
      } else {
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(t),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
  }
  __syncwarp();
  asm volatile("{\n .reg .pred p;\n W2:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W2;\n}\n" ::"r"(sa(&bar)), "r"(0) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < 256; ++c) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(t + (uint32_t(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    D[(warp * 32 + lane) * 256 + c] = __uint_as_float(r);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(256));
}

void mma_probe() {
  std::vector<float> hA(128 * 32), hB(32 * 256);
  for (int i = 0; i < 128 * 32; ++i) hA[i] = float((i * 7) % 5) - 2.f;
  for (int i = 0; i < 32 * 256; ++i) hB[i] = float((i * 3) % 7) - 3.f;
  std::vector<double> ref(128 * 256, 0);
  for (int m = 0; m < 128; ++m)
    for (int nn = 0; nn < 256; ++nn)
      for (int k = 0; k < 32; ++k) ref[m * 256 + nn] += double(hA[m * 32 + k]) * hB[k * 256 + nn];
  float *A, *B, *D;
  CK(cudaMalloc(&A, hA.size() * 4));
  CK(cudaMalloc(&B, hB.size() * 4));
  CK(cudaMalloc(&D, 128 * 256 * 4));
  CK(cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000));
  const uint32_t base = (1u << 4) | (2u << 7) | (2u << 10) | (32u << 17) | (8u << 24);
  struct V { const char* nm; int mode; uint32_t idesc; } vs[] = {
      {"b_major=1, no mask", 0, base | (1u << 16)},
      {"b_major=1, mask", 1, base | (1u << 16)},
      {"b_major=0, no mask", 0, base},
      {"b_major=1, SW128_32B atom", 2, base | (1u << 16)},
      {"b_major=1, SW128_32B atom, mask", 3, base | (1u << 16)},
  };
  for (auto& v : vs) {
    CK(cudaMemset(D, 0, 128 * 256 * 4));
    k_mma_probe<<<1, 128, 60000>>>(A, B, D, v.mode, v.idesc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> hD(128 * 256);
    CK(cudaMemcpy(hD.data(), D, hD.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0, maxabs = 0;
    for (int i = 0; i < 128 * 256; ++i) {
      maxerr = std::max(maxerr, std::abs(hD[i] - ref[i]));
      maxabs = std::max(maxabs, double(std::abs(hD[i])));
    }
    printf("mma %-28s err=%s maxerr=%g max|D|=%g D[0..3]=%g %g %g %g ref=%g %g %g %g\n", v.nm, cudaGetErrorString(e),
           maxerr, maxabs, hD[0], hD[1], hD[2], hD[3], ref[0], ref[1], ref[2], ref[3]);
  }
}

int main() {
  mma_probe();
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  printf("entry point query %d ptr %p\n", int(q), p);
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const int n = 256;
  std::vector<float> h(n * n);
  for (int i = 0; i < n * n; ++i) h[i] = float(i);
  float *A, *out;
  CK(cudaMalloc(&A, n * n * 4));
  CK(cudaMalloc(&out, 1 << 20));
  CK(cudaMemcpy(A, h.data(), n * n * 4, cudaMemcpyHostToDevice));
  for (int sw = 0; sw < 2; ++sw) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(n)};
    cuuint64_t strides[1] = {cuuint64_t(n) * 4};
    cuuint32_t box[2] = {32, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode swizzle=%d -> %d\n", sw, int(r));
    CK(cudaFuncSetAttribute(k_tma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000));
    k_tma_probe<<<1, 128, 20000>>>(tm, out, 32, 128);
    CK(cudaDeviceSynchronize());
    std::vector<float> o(4096);
    CK(cudaMemcpy(o.data(), out, 4096 * 4, cudaMemcpyDeviceToHost));
    printf("  smem[0..7]: ");
    for (int i = 0; i < 8; ++i) printf("%g ", o[i]);
    printf("\n  smem[32..39] (row 1): ");
    for (int i = 32; i < 40; ++i) printf("%g ", o[i]);
    printf("\n  expect row0 = A[128][32..] = %g.., row1 = %g..\n", h[128 * n + 32], h[129 * n + 32]);
  }
  k_tmem_probe<<<1, 128>>>(out);
  CK(cudaDeviceSynchronize());
  std::vector<float> o(256);
  CK(cudaMemcpy(o.data(), out, 256 * 4, cudaMemcpyDeviceToHost));
  printf("tmem roundtrip: %g %g %g %g ... %g (want 1 11 21 31 ... 1271), base %g\n", o[0], o[1], o[2], o[3], o[127], o[128]);
  return 0;
}
