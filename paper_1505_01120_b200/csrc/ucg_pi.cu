// ucg_pi.cu — Monte-Carlo pi device op, workload C3.
//
// Per sample gid of task t: s0 = seed ^ gid*GAMMA, z1 = mix64(s0+GAMMA),
// z2 = mix64(s0+2*GAMMA), a = z1>>32, b = z2>>32, and the reference test is
//   fl(fl(x*x) + fl(y*y)) <= 1.0   with x = a/2^32, y = b/2^32 in IEEE double.
// Here x*x = fl(a^2)*2^-64 exactly, so the test is evaluated on the FP64
// pipe as fl(fl(a^2)+fl(b^2)) <= 2^64 (__dmul_rn / __dadd_rn: no FMA
// contraction), leaving the integer ALU pipe to the SplitMix64 shifts/xors;
// 64-bit adds run as IMAD.WIDE on the FMA pipe.
// Counts: ballot-free integer accumulation, warp redux, one 64-bit atomic per
// CTA per 64Ki-sample work unit.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "ucg_common.cuh"

namespace ucg {
namespace {

constexpr int kPiThreads = 256;
constexpr int kUnitLog2 = 16;  // samples per work unit
constexpr int kMaxTasks = 512; // per launch

struct PiTasks {
  uint64_t seed[kMaxTasks];
  uint64_t samples[kMaxTasks];
  uint64_t first_unit[kMaxTasks + 1];
  uint32_t ntasks;
};

// 64-bit x + c with the add on the FMA pipe (IMAD.WIDE.U32 + IMAD): the
// SplitMix64 shifts / xors already saturate the integer ALU pipe.
__device__ __forceinline__ uint64_t add64_fma(uint64_t x, uint64_t c) {
  uint64_t lo;
  asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(lo) : "r"(uint32_t(x)), "l"(c));
  uint32_t hi;
  asm("mad.lo.u32 %0, %1, 1, %2;" : "=r"(hi) : "r"(uint32_t(x >> 32)), "r"(uint32_t(lo >> 32)));
  return (uint64_t(hi) << 32) | uint32_t(lo);
}

// High 32 bits of mix64(z): the last step z ^ (z >> 31) only feeds bit 63
// of z into the high word, so hi32 = hi(z) ^ (hi(z) >> 31).
__device__ __forceinline__ uint32_t mix64_hi(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  const uint32_t h = uint32_t(z >> 32);
  return h ^ (h >> 31);
}

// Exact reference test on the FP64 pipe (separate from the integer ALU):
// x*x = fl(a^2)*2^-64 exactly, so fl(fl(x*x)+fl(y*y)) <= 1 is
// fl(fl(a^2)+fl(b^2)) <= 2^64 with a, b converted exactly to double.
__device__ __forceinline__ uint32_t pi_hit(uint64_t s0) {
  const uint32_t a = mix64_hi(add64_fma(s0, kGamma));
  const uint32_t b = mix64_hi(add64_fma(s0, 2 * kGamma));
  const double da = __uint2double_rn(a), db = __uint2double_rn(b);
  return __dadd_rn(__dmul_rn(da, da), __dmul_rn(db, db)) <= 18446744073709551616.0 ? 1u : 0u;
}

// Sharded reduce_cl(isum2) over ranks, fused into the counting kernel: the
// last CTA of the launch (exit ticket) stores this rank's total into every
// peer's IPC-mapped region (8 bytes at slot `rank`), publishes an epoch flag
// there (release, system scope), waits for all ranks' flags in its own
// region (acquire) and writes the sum over ranks to `total` — the same
// NVLink exchange as the C2 reduction's tail (ucg_reduce.cu stage2).
struct PiXchg {
  const uint64_t* peers;   // [world] region base addresses (own at [rank]); null: no exchange
  uint64_t flags_offset;
  uint32_t* epoch;         // exchanges completed (device counter, advanced here)
  int world, rank;
  uint32_t* err;
  unsigned long long* done;  // exit tickets, zeroed before the launch
};

__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ void pi_exchange(const PiXchg& x, unsigned long long* total) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // this CTA's atomics on `total` before its ticket
    last = atomicAdd(x.done, 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  __threadfence();
  const unsigned long long mine = atomicAdd(total, 0ull);  // every CTA's hits are in
  const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(x.epoch) + 1;
  const int buf = int(epoch & 1) * x.world;  // value buffer by epoch parity
  for (int r = lane; r < x.world; r += 32)
    reinterpret_cast<unsigned long long*>(x.peers[r])[buf + x.rank] = mine;
  __threadfence_system();
  __syncwarp();
  for (int r = lane; r < x.world; r += 32) {
    st_release_sys_u32(reinterpret_cast<uint32_t*>(x.peers[r] + x.flags_offset) + x.rank, epoch);
  }
  const uint32_t* flags = reinterpret_cast<const uint32_t*>(x.peers[x.rank] + x.flags_offset);
  bool timed_out = false;
  for (int r = lane; r < x.world; r += 32) {
    const uint64_t t0 = global_ns();
    while (int32_t(ld_acquire_sys_u32(flags + r) - epoch) < 0) {
      __nanosleep(64);
      if (global_ns() - t0 > kPeerWaitNs) {  // a peer never arrived
        timed_out = true;
        break;
      }
    }
  }
  if (__any_sync(0xffffffffu, timed_out)) {
    // no plausible total from stale slots: -1, the epoch unchanged, and the
    // host-mapped error word raised (later calls fail with UCG_ERR_PEER)
    if (lane == 0) {
      *total = ~0ull;
      *reinterpret_cast<volatile uint32_t*>(x.err) = 1u;
      __threadfence_system();
    }
    return;
  }
  if (lane == 0) {
    const volatile unsigned long long* slots = reinterpret_cast<const unsigned long long*>(x.peers[x.rank]);
    unsigned long long sum = 0;
    for (int r = 0; r < x.world; ++r) sum += slots[buf + r];  // exact in any order
    *total = sum;
    *x.epoch = epoch;
  }
}

__global__ void __launch_bounds__(kPiThreads) k_pi(const __grid_constant__ PiTasks tasks, uint64_t nunits,
                                                   unsigned long long* __restrict__ hits,
                                                   unsigned long long* __restrict__ total, const PiXchg xg) {
  __shared__ uint32_t warp_sum[kPiThreads / 32];
  for (uint64_t unit = blockIdx.x; unit < nunits; unit += gridDim.x) {
    // task owning this unit: binary search over first_unit
    uint32_t lo = 0, hi = tasks.ntasks;  // first_unit[lo] <= unit < first_unit[hi]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (tasks.first_unit[mid] <= unit) lo = mid;
      else hi = mid;
    }
    const uint64_t seed = tasks.seed[lo];
    const uint64_t base = (unit - tasks.first_unit[lo]) << kUnitLog2;
    const uint64_t end = umin(tasks.samples[lo], base + (1ull << kUnitLog2));
    uint32_t cnt = 0;
    uint64_t gid = base + threadIdx.x;
    uint64_t m = gid * kGamma;
    const uint64_t mstep = uint64_t(kPiThreads) * kGamma;
    if (end - base == (1ull << kUnitLog2)) {
#pragma unroll 4
      for (int i = 0; i < (1 << kUnitLog2) / kPiThreads; ++i) {
        cnt += pi_hit(seed ^ m);
        m = add64_fma(m, mstep);
      }
    } else {
      for (; gid < end; gid += kPiThreads) {
        cnt += pi_hit(seed ^ m);
        m += mstep;
      }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < kPiThreads / 32; ++w) t += warp_sum[w];
      atomicAdd(hits + lo, t);
      if (total) atomicAdd(total, t);
    }
    __syncthreads();
  }
  if (xg.peers && total) pi_exchange(xg, total);
}

// Class-D form of the same body (the seam-B contract of the pi kernel):
// flags[gid] = hit(seed, gid) for gid in [0, samples).
__global__ void __launch_bounds__(256) k_pi_flags(uint64_t seed, uint64_t samples, uint8_t* __restrict__ flags) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < samples; g += stride)
    flags[g] = uint8_t(pi_hit(seed ^ (g * kGamma)));
}

}  // namespace
}  // namespace ucg

using namespace ucg;

extern "C" int ucg_pi_flags(uint64_t seed, uint64_t samples, uint8_t* flags, void* stream) {
  if (int rc = check_device()) return rc;
  if (!samples) return UCG_OK;
  if (!flags) return fail(UCG_ERR_ARG, "flags is null");
  const unsigned grid = unsigned(std::min<uint64_t>((samples + 255) / 256, uint64_t(sm_count()) * 16));
  k_pi_flags<<<grid, 256, 0, as_stream(stream)>>>(seed, samples, flags);
  UCG_LAUNCHED();
  return UCG_OK;
}

namespace {
int pi_launch(const uint64_t* seeds, const uint64_t* samples, uint64_t ntasks, int64_t* hits_out, int64_t* total_out,
              ucg_xchg* xg, void* stream) {
  if (int rc = check_device()) return rc;
  cudaStream_t st = as_stream(stream);
  PiXchg xa{};
  if (xg) {
    if (!total_out) return fail(UCG_ERR_ARG, "the sharded pi total needs total_out");
    if (!xg->opened) return fail(UCG_ERR_ARG, "exchange context not opened");
    if (int rc = xchg_guard(xg)) return rc;
    if (xg->p_total < 2ull * uint64_t(xg->world)) return fail(UCG_ERR_ARG, "pi exchange needs 2 slots per rank");
    int dev = -1;
    UCG_CUDA(cudaGetDevice(&dev));
    if (dev != xg->device) return fail(UCG_ERR_ARG, "exchange context belongs to another device");
    unsigned long long* done = claim_counter();
    if (!done) return fail(UCG_ERR_CUDA, "claim counter allocation failed");
    UCG_CUDA(cudaMemsetAsync(done, 0, sizeof(unsigned long long), st));
    xa = PiXchg{xg->d_peers, xg->flags_offset, xg->d_epoch, xg->world, xg->rank, xg->d_err, done};
  }
  if (total_out) UCG_CUDA(cudaMemsetAsync(total_out, 0, sizeof(int64_t), st));
  if (ntasks && (!seeds || !samples || !hits_out)) return fail(UCG_ERR_ARG, "null argument");
  if (ntasks) UCG_CUDA(cudaMemsetAsync(hits_out, 0, ntasks * sizeof(int64_t), st));
  bool exchanged = false;
  for (uint64_t t0 = 0; t0 < ntasks; t0 += kMaxTasks) {
    const uint32_t nt = uint32_t(std::min<uint64_t>(kMaxTasks, ntasks - t0));
    PiTasks p;
    p.ntasks = nt;
    p.first_unit[0] = 0;
    for (uint32_t i = 0; i < nt; ++i) {
      p.seed[i] = seeds[t0 + i];
      p.samples[i] = samples[t0 + i];
      p.first_unit[i + 1] = p.first_unit[i] + ((samples[t0 + i] + (1ull << kUnitLog2) - 1) >> kUnitLog2);
    }
    const uint64_t nunits = p.first_unit[nt];
    if (!nunits) continue;
    const unsigned grid = unsigned(std::min<uint64_t>(nunits, uint64_t(sm_count()) * 8));
    // the exchange rides on the last launch (earlier chunks' hits are in
    // `total` by stream order)
    const bool last_chunk = t0 + kMaxTasks >= ntasks;
    const PiXchg xl = last_chunk ? xa : PiXchg{};
    exchanged |= last_chunk && xa.peers;
    k_pi<<<grid, kPiThreads, 0, st>>>(p, nunits, reinterpret_cast<unsigned long long*>(hits_out + t0),
                                      reinterpret_cast<unsigned long long*>(total_out), xl);
    UCG_LAUNCHED();
  }
  if (xa.peers && !exchanged) {
    // no samples on this rank (or none in its last chunk): it still joins
    // the exchange, with its total as it stands
    PiTasks p;
    p.ntasks = 0;
    p.first_unit[0] = 0;
    k_pi<<<1, kPiThreads, 0, st>>>(p, 0, nullptr, reinterpret_cast<unsigned long long*>(total_out), xa);
    UCG_LAUNCHED();
  }
  return UCG_OK;
}
}  // namespace

extern "C" int ucg_pi_hits_total(const uint64_t* seeds, const uint64_t* samples, uint64_t ntasks,
                                 int64_t* hits_out, int64_t* total_out, void* stream) {
  return pi_launch(seeds, samples, ntasks, hits_out, total_out, nullptr, stream);
}

extern "C" int ucg_pi_hits_total_xchg(const uint64_t* seeds, const uint64_t* samples, uint64_t ntasks,
                                      int64_t* hits_out, int64_t* total_out, ucg_xchg* xg, void* stream) {
  return pi_launch(seeds, samples, ntasks, hits_out, total_out, xg, stream);
}

extern "C" int ucg_pi_hits(const uint64_t* seeds, const uint64_t* samples, uint64_t ntasks, int64_t* hits_out,
                           void* stream) {
  return ucg_pi_hits_total(seeds, samples, ntasks, hits_out, nullptr, stream);
}
