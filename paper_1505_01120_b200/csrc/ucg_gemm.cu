// ucg_gemm.cu — dense matmul device op (workload C5) on the 5th-generation
// tensor cores: tcgen05.mma kind::tf32, fp32 accumulators in TMEM, operands
// staged by TMA into 128-byte-swizzled shared memory.
//
// C = A * B, all n x n row-major fp32. A tile is K-major (rows of A are
// contiguous in k); B is row-major [k][n], i.e. MN-major for the MMA, which
// tcgen05 accepts for TF32 (instruction-descriptor b_major = 1).
//
// CTA tile 128 x 256, k-block 32, 4-stage TMA ring (48 KB / stage):
//   warp 0 lane 0  TMA producer: A box {32 k, 128 m} + 8 B boxes {32 n, 32 k}
//   warp 1 lane 0  MMA issuer: 4 x tcgen05.mma (M128 N256 K8) per k-block,
//                  tcgen05.commit -> frees the stage when the MMAs have read it
//   warps 0-3      epilogue: tcgen05.ld 32x32b (row = TMEM lane) -> global
// Shared-memory canonical layouts (cute/atom/mma_traits_sm100.hpp):
//   A  K-major SW128:  8 rows x 128 B atoms, SBO = 1024 B; k-step = +32 B
//   B  MN-major SW128 with 32-byte atoms (SWIZZLE_128B_BASE32B, the only
//      MN-major layout tf32 accepts; TMA swizzle 128B_ATOM_32B): rows of
//      128 B (32 n) per k, 4-row groups, LBO = strip = 4096 B (n direction),
//      SBO = 512 B (k direction); k-step of 8 = +1024 B
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "ucg_common.cuh"

namespace ucg {
namespace {

constexpr int BM = 128, BN = 256, BK = 32, STAGES = 4;
constexpr uint32_t A_BYTES = BM * BK * 4;        // 16 KB
constexpr uint32_t B_STRIP = BK * 128;           // 32 k-rows x 128 B = 4 KB
constexpr uint32_t B_BYTES = (BN / 32) * B_STRIP;  // 32 KB
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr uint32_t SMEM_BYTES = STAGES * STAGE_BYTES + 1024;  // + alignment slack
constexpr uint32_t TMEM_COLS = 256;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}
// layout: 2 = SWIZZLE_128B (16-byte granules), 1 = SWIZZLE_128B_BASE32B (32-byte granules)
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo_bytes >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo_bytes >> 4) & 0x3FFFu) << 32) | (1ull << 46) /* version: sm100 */ |
         (uint64_t(layout) << 61);
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, A K-major, B MN-major, N=256, M=128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) | (uint32_t(BN >> 3) << 17) |
                            (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}

__global__ void __launch_bounds__(128, 1)
    k_gemm_tf32(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* __restrict__ C,
                int n) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = n / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
      uint8_t* a = smem + s * STAGE_BYTES;
      uint8_t* b = a + A_BYTES;
      mbar_expect_tx(&full[s], STAGE_BYTES);
      tma_2d(a, &tmA, &full[s], kb * BK, m0);
#pragma unroll
      for (int j = 0; j < BN / 32; ++j) tma_2d(b + j * B_STRIP, &tmB, &full[s], n0 + 32 * j, kb * BK);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer (single thread) ----
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a = smem_addr(smem + s * STAGE_BYTES);
      const uint32_t b = a + A_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 8; ++k) {
        const uint64_t adesc = smem_desc(a + 32u * k, 16u, 1024u, 2u);
        const uint64_t bdesc = smem_desc(b + 1024u * k, B_STRIP, 512u, 1u);
        mma_tf32(tmem, adesc, bdesc, (kb | k) != 0);
      }
      mma_commit(&empty[s]);  // stage reusable once these MMAs have read it
    }
    mma_commit(&tfull);  // accumulator complete
  }
  __syncwarp();

  // ---- epilogue: TMEM -> registers -> global (row = TMEM lane) ----
  mbar_wait(&tfull, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = m0 + warp * 32 + lane;
  float* crow = C + size_t(row) * n + n0;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t r[32];
    const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16) + uint32_t(c * 32);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float4* dst = reinterpret_cast<float4*>(crow + c * 32);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                           __uint_as_float(r[4 * q + 3]));
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// ---- persistent, warp-specialised variant ---------------------------------------
// One CTA per SM loops over output tiles (grouped raster: 16 m-blocks per
// n-block sweep so concurrently running CTAs share A and B in L2). TMEM holds
// TWO 128x256 fp32 accumulators (all 512 columns): the MMA warp fills one while
// the 4 epilogue warps drain the other, so tensor cores never wait for stores.
//   warp 0 lane 0  TMA producer (smem ring continues across tiles)
//   warp 1         TMEM allocator; lane 0 issues MMAs + commits
//   warps 2-5      epilogue; warp w reads TMEM lanes 32*(w%4)..+31
constexpr int kGroupM = 16;
__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& m0, int& n0) {
  const int per_group = kGroupM * tiles_n;
  const int g = t / per_group, idx = t % per_group;
  const int gm = min(kGroupM, tiles_m - g * kGroupM);
  m0 = (g * kGroupM + idx % gm) * BM;
  n0 = (idx / gm) * BN;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__global__ void __launch_bounds__(192, 1)
    k_gemm_tf32_persistent(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           float* __restrict__ C, int n) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = n / BM, tiles_n = n / BN, ntiles = tiles_m * tiles_n, nk = n / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t q = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int m0, n0;
        tile_coords(t, tiles_m, tiles_n, m0, n0);
        for (int kb = 0; kb < nk; ++kb, ++q) {
          const int s = int(q % STAGES);
          if (q >= uint32_t(STAGES)) mbar_wait(&empty[s], ((q / STAGES) & 1) ^ 1);
          uint8_t* a = smem + s * STAGE_BYTES;
          uint8_t* b = a + A_BYTES;
          mbar_expect_tx(&full[s], STAGE_BYTES);
          tma_2d(a, &tmA, &full[s], kb * BK, m0);
#pragma unroll
          for (int j = 0; j < BN / 32; ++j) tma_2d(b + j * B_STRIP, &tmB, &full[s], n0 + 32 * j, kb * BK);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t q = 0, i = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const uint32_t acc = i & 1;
        if (i >= 2) mbar_wait(&tempty[acc], ((i / 2) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * uint32_t(BN);
        for (int kb = 0; kb < nk; ++kb, ++q) {
          const int s = int(q % STAGES);
          mbar_wait(&full[s], (q / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a = smem_addr(smem + s * STAGE_BYTES);
          const uint32_t b = a + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const uint64_t adesc = smem_desc(a + 32u * k, 16u, 1024u, 2u);
            const uint64_t bdesc = smem_desc(b + 1024u * k, B_STRIP, 512u, 1u);
            mma_tf32(d, adesc, bdesc, (kb | k) != 0);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else {
    const int lg = warp & 3;  // TMEM lane group this warp may access
    uint32_t i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      int m0, n0;
      tile_coords(t, tiles_m, tiles_n, m0, n0);
      const uint32_t acc = i & 1;
      mbar_wait(&tfull[acc], (i / 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float* crow = C + size_t(m0 + lg * 32 + lane) * n + n0;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        const uint32_t taddr = tmem + (uint32_t(lg * 32) << 16) + acc * uint32_t(BN) + uint32_t(c * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
              "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
              "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float4* dst = reinterpret_cast<float4*>(crow + c * 32);
#pragma unroll
        for (int qq = 0; qq < 8; ++qq)
          __stcs(dst + qq, make_float4(__uint_as_float(r[4 * qq]), __uint_as_float(r[4 * qq + 1]),
                                       __uint_as_float(r[4 * qq + 2]), __uint_as_float(r[4 * qq + 3])));
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&tempty[acc]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ---- CTA-pair (cta_group::2) variant -----------------------------------------
// A cluster of 2 CTAs on one TPC computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M=256): each CTA stages ITS 128 rows of A and
// ITS 128 columns of B (32 KB per stage instead of 48 KB) and owns 128 rows
// of the accumulator in its TMEM; the leader CTA issues the MMAs. Both CTAs'
// TMA loads complete on the leader's full barrier (.cta_group::2 form, peer
// bit cleared); MMA commits multicast to both CTAs' empty / tmem-full
// barriers; both CTAs' epilogues arrive on the leader's tmem-empty barrier.
constexpr int S2 = 6;                                // stages
constexpr uint32_t A2_BYTES = 128 * BK * 4;          // 16 KB: this CTA's 128 rows
constexpr uint32_t B2_BYTES = 4 * B_STRIP;           // 16 KB: this CTA's 128 columns
constexpr uint32_t STAGE2_BYTES = A2_BYTES + B2_BYTES;
constexpr uint32_t SMEM2_BYTES = S2 * STAGE2_BYTES + 1024;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;          // shared::cluster address of the even (leader) CTA
constexpr uint32_t kIdesc2 = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) | (uint32_t(256 >> 3) << 17) |
                             (uint32_t(256 >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_2d_2sm(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc2), "r"(accumulate), "r"(0u));
}
__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_addr(bar)),
      "h"(uint16_t(3))
      : "memory");
}

// 32 consecutive TMEM columns of this warp's 32 lanes -> r[0..31] (waits)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// kTerms = 1: C = A*B in TF32 (the tensor core reads the top 19 bits of
// each fp32 operand). kTerms = 3 (fp32-faithful "3xTF32"): the operands are
// pre-split into x = hi + lo with hi = rna_tf32(x) and lo = x - hi (exact),
// and the k loop runs three times over (Ahi,Bhi), (Ahi,Blo), (Alo,Bhi) into
// the same TMEM accumulator — the dropped lo*lo term and lo's own TF32
// truncation are ~2^-22 relative, fp32-level. tmA/tmB are then Ahi/Bhi and
// tmA2/tmB2 Alo/Blo.
// Threads per CTA: warp 0 TMA, warp 1 TMEM alloc + MMA, then the epilogue
// warps — 4 for TF32 (one per TMEM lane group), 8 for the k-chunked fp32
// mode (two per lane group, each owning 128 of the tile's 256 columns and
// keeping that half-row's running chunk sum in registers).
template <int kTerms>
constexpr int gemm2_threads() { return kTerms == 1 ? 192 : 320; }

// (10 warps: 3 on some SM sub-partitions, so at most 168 registers per
// thread; the running sums take 128, the TMEM reads go 8 columns at a time)
template <int kTerms>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gemm2_threads<kTerms>(), 1)
    k_gemm_tf32_2sm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
                    float* __restrict__ C, int n, int nchunks, int group_m) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[S2], empty[S2], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // A work unit is (tile, k-chunk): the k range is cut into nchunks chunks,
  // each accumulated from zero in TMEM (all kTerms terms) and added to C by
  // the epilogue with an IEEE round-to-nearest fp32 add (C = chunk 0, then
  // C += chunk c). The tensor core's own fp32 accumulation truncates, so its
  // error grows linearly with the k length it accumulates; short chunks
  // bound that. nchunks = 1: one unit per tile, C stored once.
  const int tiles_m = n / 256, tiles_n = n / 256, ntiles = tiles_m * tiles_n, nk1 = n / BK;
  const int kc = nk1 / nchunks;  // k-blocks per chunk (per term)
  const int nk = kTerms * kc;    // k-blocks per unit

  if (threadIdx.x == 0) {
    for (int s = 0; s < S2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * (gemm2_threads<kTerms>() - 64));  // both CTAs' epilogue threads
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    if (kTerms > 1) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA2) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB2) : "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t q = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        int mb, nb;
        {  // grouped raster over 256 x 256 tiles
          const int per_group = group_m * tiles_n;
          const int g = t / per_group, idx = t % per_group;
          const int gm = min(group_m, tiles_m - g * group_m);
          mb = g * group_m + idx % gm;
          nb = idx / gm;
        }
        const int m0 = mb * 256 + int(rank) * 128, n0 = nb * 256 + int(rank) * 128;
        for (int c = 0; c < nchunks; ++c) {
          for (int kb = 0; kb < nk; ++kb, ++q) {
            const int s = int(q % S2);
            if (q >= uint32_t(S2)) mbar_wait(&empty[s], ((q / S2) & 1) ^ 1);
            uint8_t* a = smem + s * STAGE2_BYTES;
            uint8_t* b = a + A2_BYTES;
            const uint32_t lbar = smem_addr(&full[s]) & kPeerMask;
            if (rank == 0) mbar_expect_tx(&full[s], 2 * STAGE2_BYTES);
            // term 0: (Ahi, Bhi), 1: (Ahi, Blo), 2: (Alo, Bhi)
            const int term = kTerms > 1 ? kb / kc : 0, k0 = (c * kc + kb - term * kc) * BK;
            tma_2d_2sm(a, term == 2 ? &tmA2 : &tmA, lbar, k0, m0);
            const CUtensorMap* mb_ = term == 1 ? &tmB2 : &tmB;
#pragma unroll
            for (int j = 0; j < 4; ++j) tma_2d_2sm(b + j * B_STRIP, mb_, lbar, n0 + 32 * j, k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      uint32_t q = 0, i = 0;
      const int nunits = ((ntiles - pair + npairs - 1) / npairs) * nchunks;  // this pair's units
      for (int u = 0; u < nunits; ++u, ++i) {
        const uint32_t acc = i & 1;
        if (i >= 2) mbar_wait(&tempty[acc], ((i / 2) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * 256u;
        for (int kb = 0; kb < nk; ++kb, ++q) {
          const int s = int(q % S2);
          mbar_wait(&full[s], (q / S2) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a = smem_addr(smem + s * STAGE2_BYTES);
          const uint32_t b = a + A2_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const uint64_t adesc = smem_desc(a + 32u * k, 16u, 1024u, 2u);
            const uint64_t bdesc = smem_desc(b + 1024u * k, B_STRIP, 512u, 1u);
            mma_tf32_2sm(d, adesc, bdesc, (kb | k) != 0);
          }
          mma_commit_2sm(&empty[s]);
        }
        mma_commit_2sm(&tfull[acc]);
      }
    }
  } else if constexpr (kTerms == 1) {
    const int lg = warp & 3;
    const uint32_t leader_tempty[2] = {smem_addr(&tempty[0]) & kPeerMask, smem_addr(&tempty[1]) & kPeerMask};
    uint32_t i = 0;
    for (int u = 0; u < ((ntiles - pair + npairs - 1) / npairs) * nchunks; ++u, ++i) {
      const int t = pair + (u / nchunks) * npairs;
      int mb, nb;
      {
        const int per_group = group_m * tiles_n;
        const int g = t / per_group, idx = t % per_group;
        const int gm = min(group_m, tiles_m - g * group_m);
        mb = g * group_m + idx % gm;
        nb = idx / gm;
      }
      const uint32_t acc = i & 1;
      mbar_wait(&tfull[acc], (i / 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float* crow = C + size_t(mb * 256 + int(rank) * 128 + lg * 32 + lane) * n + nb * 256;
#pragma unroll 1
      for (int c = 0; c < 256 / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + (uint32_t(lg * 32) << 16) + acc * 256u + uint32_t(c * 32), r);
        float4* dst = reinterpret_cast<float4*>(crow + c * 32);
#pragma unroll
        for (int qq = 0; qq < 8; ++qq)
          __stcs(dst + qq, make_float4(__uint_as_float(r[4 * qq]), __uint_as_float(r[4 * qq + 1]),
                                       __uint_as_float(r[4 * qq + 2]), __uint_as_float(r[4 * qq + 3])));
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(leader_tempty[acc]) : "memory");
    }
  } else {
    // k-chunk units: chunk c of a tile is accumulated from zero in TMEM (the
    // tensor core's truncating fp32 accumulation stays short) and added
    // into a running fp32 sum with IEEE round-to-nearest adds (sum = chunk
    // 0, then sum = sum + chunk c); the running sum never leaves the
    // registers of the thread that owns that half-row, and C is written
    // once per tile. The MMA fills the other TMEM accumulator meanwhile.
    const int ew = warp - 2, lg = warp & 3, half = ew >> 2;
    const uint32_t leader_tempty[2] = {smem_addr(&tempty[0]) & kPeerMask, smem_addr(&tempty[1]) & kPeerMask};
    float sum[128];
    uint32_t i = 0;
    for (int u = 0; u < ((ntiles - pair + npairs - 1) / npairs) * nchunks; ++u, ++i) {
      const int t = pair + (u / nchunks) * npairs, chunk = u % nchunks;
      const uint32_t acc = i & 1;
      mbar_wait(&tfull[acc], (i / 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        uint32_t r[8];
        tmem_ld8(tmem + (uint32_t(lg * 32) << 16) + acc * 256u + uint32_t(half * 128 + c * 8), r);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          sum[c * 8 + j] = chunk ? __fadd_rn(sum[c * 8 + j], __uint_as_float(r[j])) : __uint_as_float(r[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(leader_tempty[acc]) : "memory");
      if (chunk + 1 == nchunks) {
        int mb, nb;
        {
          const int per_group = group_m * tiles_n;
          const int g = t / per_group, idx = t % per_group;
          const int gm = min(group_m, tiles_m - g * group_m);
          mb = g * group_m + idx % gm;
          nb = idx / gm;
        }
        float4* dst = reinterpret_cast<float4*>(C + size_t(mb * 256 + int(rank) * 128 + lg * 32 + lane) * n +
                                                nb * 256 + half * 128);
#pragma unroll
        for (int qq = 0; qq < 32; ++qq)
          __stcs(dst + qq, make_float4(sum[4 * qq], sum[4 * qq + 1], sum[4 * qq + 2], sum[4 * qq + 3]));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// x = hi + lo: hi = x rounded to TF32 (cvt.rna), lo = x - hi (exact in fp32).
// Non-finite x keeps lo = 0 so inf/nan propagate like the fp32 product.
__global__ void __launch_bounds__(256) k_split_tf32(const float4* __restrict__ x, float4* __restrict__ hi,
                                                    float4* __restrict__ lo, uint64_t n4) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = ld_stream(x + i);
    float h[4], l[4];
    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t t;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(e[k]));
      h[k] = __uint_as_float(t);
      l[k] = isfinite(h[k]) ? __fsub_rn(e[k], h[k]) : 0.0f;
    }
    st_stream(hi + i, make_float4(h[0], h[1], h[2], h[3]));
    st_stream(lo + i, make_float4(l[0], l[1], l[2], l[3]));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() { return tmap_encode_fn(); }

// m-blocks (of 256 rows) per raster group of the CTA-pair kernel: 8 — the
// 74 concurrent tile pairs then cover ~8 x 9 tiles, so fewer A/B panels
// stream at once (ncu DRAM reads 7.1 vs 8.2 GB per fp32-faithful 8192^3
// launch at 16; C5 line 219.8-220.1 vs 218.3-218.4 TF/s, same box;
// UCG_GEMM_GROUP for A/B runs)
int gemm_group_m() {
  static const int g = [] {
    const char* e = getenv("UCG_GEMM_GROUP");
    const int v = e ? atoi(e) : 8;
    return v > 0 ? v : 8;
  }();
  return g;
}

int make_map(CUtensorMap* m, const float* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
             uint32_t box_outer, CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) return fail(UCG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(UCG_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return UCG_OK;
}

}  // namespace
}  // namespace ucg

using namespace ucg;

extern "C" int ucg_gemm_tf32(const float* A, const float* B, float* C, uint64_t n, void* stream) {
  if (int rc = check_device()) return rc;
  if (!n) return UCG_OK;
  if (!A || !B || !C) return fail(UCG_ERR_ARG, "null argument");
  if (n % BN || n > (1u << 30)) return fail(UCG_ERR_ARG, "gemm: n must be a multiple of 256");
  if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return fail(UCG_ERR_ARG, "gemm: 16-byte alignment required");
  CUtensorMap tmA, tmB;
  if (int rc = make_map(&tmA, A, n, n, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;   // A[m][k]: inner k, box {32 k, 128 m}
  if (int rc = make_map(&tmB, B, n, n, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return rc;   // B[k][n]: inner n, box {32 n, 32 k}
  static const int variant = [] {
    const char* e = getenv("UCG_GEMM_VARIANT");
    return e ? atoi(e) : 2;  // default: CTA-pair (cta_group::2) kernel
  }();
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    UCG_CUDA(cudaFuncSetAttribute(k_gemm_tf32, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    UCG_CUDA(cudaFuncSetAttribute(k_gemm_tf32_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    UCG_CUDA(cudaFuncSetAttribute(k_gemm_tf32_2sm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES));
    UCG_CUDA(cudaFuncSetAttribute(k_gemm_tf32_2sm<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES));
  }
  if (variant == 0) {
    dim3 grid(unsigned(n / BN), unsigned(n / BM));
    k_gemm_tf32<<<grid, 128, SMEM_BYTES, as_stream(stream)>>>(tmA, tmB, C, int(n));
  } else if (variant == 2) {
    const uint64_t ntiles = (n / 256) * (n / 256);
    const unsigned grid = unsigned(std::min<uint64_t>(ntiles, uint64_t(sm_count() / 2))) * 2;
    k_gemm_tf32_2sm<1><<<grid, gemm2_threads<1>(), SMEM2_BYTES, as_stream(stream)>>>(tmA, tmB, tmA, tmB, C, int(n),
                                                                                      1, gemm_group_m());
  } else {
    const uint64_t ntiles = (n / BM) * (n / BN);
    const unsigned grid = unsigned(std::min<uint64_t>(ntiles, uint64_t(sm_count())));
    k_gemm_tf32_persistent<<<grid, 192, SMEM_BYTES, as_stream(stream)>>>(tmA, tmB, C, int(n));
  }
  UCG_LAUNCHED();
  return UCG_OK;
}

// fp32-faithful GEMM (3xTF32): split A and B into TF32 hi/lo halves
// (workspace: 4 n^2 floats from the stream-ordered pool), then the CTA-pair
// kernel runs its k loop over the three cross terms.
extern "C" int ucg_gemm_f32(const float* A, const float* B, float* C, uint64_t n, void* stream) {
  if (int rc = check_device()) return rc;
  if (!n) return UCG_OK;
  if (!A || !B || !C) return fail(UCG_ERR_ARG, "null argument");
  if (n % BN || n > (1u << 30)) return fail(UCG_ERR_ARG, "gemm: n must be a multiple of 256");
  if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return fail(UCG_ERR_ARG, "gemm: 16-byte alignment required");
  cudaStream_t st = as_stream(stream);
  const uint64_t nn = n * n;
  float* w = nullptr;
  UCG_CUDA(cudaMallocAsync(&w, 4 * nn * sizeof(float), st));
  float *ahi = w, *alo = w + nn, *bhi = w + 2 * nn, *blo = w + 3 * nn;
  const unsigned sgrid = unsigned(std::min<uint64_t>((nn / 4 + 255) / 256, uint64_t(sm_count()) * 8));
  k_split_tf32<<<sgrid, 256, 0, st>>>(reinterpret_cast<const float4*>(A), reinterpret_cast<float4*>(ahi),
                                      reinterpret_cast<float4*>(alo), nn / 4);
  UCG_LAUNCHED();
  k_split_tf32<<<sgrid, 256, 0, st>>>(reinterpret_cast<const float4*>(B), reinterpret_cast<float4*>(bhi),
                                      reinterpret_cast<float4*>(blo), nn / 4);
  UCG_LAUNCHED();
  CUtensorMap tmAh, tmAl, tmBh, tmBl;
  int rc = make_map(&tmAh, ahi, n, n, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = make_map(&tmAl, alo, n, n, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = make_map(&tmBh, bhi, n, n, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!rc) rc = make_map(&tmBl, blo, n, n, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!rc) {
    static std::atomic<uint64_t> attr{0};
    if (first_on_device(attr))
      UCG_CUDA(cudaFuncSetAttribute(k_gemm_tf32_2sm<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES));
    const uint64_t ntiles = (n / 256) * (n / 256);
    const unsigned grid = unsigned(std::min<uint64_t>(ntiles, uint64_t(sm_count() / 2))) * 2;
    // k-chunks of 256 (UCG_GEMM_KCHUNK overrides; must divide n)
    int kchunk = 256;
    if (const char* e = getenv("UCG_GEMM_KCHUNK")) kchunk = atoi(e);
    if (kchunk < BK || kchunk % BK || n % uint64_t(kchunk)) kchunk = int(n);
    k_gemm_tf32_2sm<3><<<grid, gemm2_threads<3>(), SMEM2_BYTES, st>>>(tmAh, tmBh, tmAl, tmBl, C, int(n),
                                                                     int(n / kchunk), gemm_group_m());
    UCG_LAUNCHED();
  }
  UCG_CUDA(cudaFreeAsync(w, st));
  return rc;
}
