// ucg_reduce.cu — the mapCL / mapCLPartition / reduceCL hot path on sm_100a.
//
// Reduction order. Every reduction here reproduces, bit for bit, the pairing
// tree of the reference reduce_cl stage 2 (ucores/engine.hpp:172-190: each
// round pairs (0,1),(2,3),...; an unpaired trailing value is promoted). The
// psum / pmax partition kernels are defined as that tree over the
// partition's elements (oracle/ucores_oracle.c orc_tree_reduce_f32). Two facts
// make the tree GPU-friendly:
//   * node i of round k covers exactly [i*2^k, min((i+1)*2^k, n)), so any
//     aligned power-of-two block reduces independently and the tree over
//     block values (same rule) gives the same root;
//   * promotion == combining with an exact right identity (-0.0f for IEEE
//     add, -inf for std::max), so a partial block is padded to a power of two.
// Operands are always combined as op(left, right) (std::max is not
// commutative on signed zeros).
//
// Data movement: one warp owns a work item of 2^L contiguous floats of one
// segment (L = 12 by default, ucg_segtab_create) and streams it in chunks of
// 128*U floats (U coalesced LDG.128 per lane in flight, the next chunk's
// loads issued before the current chunk is reduced). Warps claim items from
// an atomic counter. A chunk is reduced with a value-halving butterfly
// (U-1 + 5 shuffles per chunk instead of 5U).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "ucg_common.cuh"

namespace ucg {
namespace {

constexpr int kWarps = 8;  // warps per CTA in the streaming kernels
constexpr unsigned kFull = 0xffffffffu;

template <class Op>
__device__ __forceinline__ float lr(float mine, float other, bool mine_is_left) {
  return mine_is_left ? Op::apply(mine, other) : Op::apply(other, mine);
}

__device__ __forceinline__ float affine(float x, float a, float b) {
  return __fadd_rn(__fmul_rn(a, x), b);
}

// Tree over the U per-lane values of one chunk of 128*U floats at x (16B
// aligned). Lane l holds floats [128u + 4l, 128u + 4l + 4) of sub-block u.
// Value-halving butterfly: at lane bit j (j < log2 U) a lane keeps half of
// its values and trades the other half with lane l^(1<<j), so U values cost
// U-1 shuffles instead of 5U; afterwards lane l holds sub-block
// bitreverse(l & (U-1)), finished across the remaining lane bits, and the U
// sub-block roots are combined by the final xor levels.
template <class Op, int U>
__device__ __forceinline__ float warp_chunk_tree(float (&s)[U], int lane) {
  constexpr int H = U == 8 ? 3 : (U == 4 ? 2 : (U == 2 ? 1 : 0));
#pragma unroll
  for (int j = 0; j < H; ++j) {
    const int cnt = U >> j;
    const bool hi = (lane >> j) & 1;
#pragma unroll
    for (int i = 0; i < cnt / 2; ++i) {
      const float keep = hi ? s[i + cnt / 2] : s[i];
      const float send = hi ? s[i] : s[i + cnt / 2];
      s[i] = lr<Op>(keep, __shfl_xor_sync(kFull, send, 1 << j), !hi);
    }
  }
  float r = s[0];
#pragma unroll
  for (int j = H; j < 5; ++j) r = lr<Op>(r, __shfl_xor_sync(kFull, r, 1 << j), !((lane >> j) & 1));
#pragma unroll
  for (int k = 0; k < H; ++k) {
    const int bit = H - 1 - k;  // sub-block index bit k lives in lane bit H-1-k
    r = lr<Op>(r, __shfl_xor_sync(kFull, r, 1 << bit), !((lane >> bit) & 1));
  }
  return r;
}

// One chunk of 128*U floats, in two halves so loads of the next chunk can
// be in flight while the current one is reduced. kGuard: only the first
// `valid` floats exist (the rest are the identity). kMap: the chunk is mapped
// through y = fl(fl(a*x)+b), stored to y, and the mapped values are reduced.
template <class Op, bool kGuard, int U>
__device__ __forceinline__ void chunk_load(const float* __restrict__ x, int64_t valid, int lane, float4 (&v)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int off = 128 * u + 4 * lane;
    if (!kGuard || off + 3 < valid) {
      v[u] = ld_stream(reinterpret_cast<const float4*>(x + off));
    } else {
      const float id = Op::identity();
      v[u].x = off + 0 < valid ? x[off + 0] : id;
      v[u].y = off + 1 < valid ? x[off + 1] : id;
      v[u].z = off + 2 < valid ? x[off + 2] : id;
      v[u].w = off + 3 < valid ? x[off + 3] : id;
    }
  }
}

// Returns the chunk's tree value in every lane.
template <class Op, bool kMap, bool kGuard, int U>
__device__ __forceinline__ float chunk_finish(float4 (&v)[U], float* __restrict__ y, int64_t valid, float a,
                                              float b, int lane) {
  float s[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int off = 128 * u + 4 * lane;
    if (kMap) {
      if (!kGuard || off + 3 < valid) {
        v[u].x = affine(v[u].x, a, b);
        v[u].y = affine(v[u].y, a, b);
        v[u].z = affine(v[u].z, a, b);
        v[u].w = affine(v[u].w, a, b);
        st_stream(reinterpret_cast<float4*>(y + off), v[u]);
      } else {
        // mapped values only for existing elements; padding stays identity
        if (off + 0 < valid) { v[u].x = affine(v[u].x, a, b); y[off + 0] = v[u].x; }
        if (off + 1 < valid) { v[u].y = affine(v[u].y, a, b); y[off + 1] = v[u].y; }
        if (off + 2 < valid) { v[u].z = affine(v[u].z, a, b); y[off + 2] = v[u].z; }
        if (off + 3 < valid) { v[u].w = affine(v[u].w, a, b); y[off + 3] = v[u].w; }
      }
    }
    s[u] = Op::apply(Op::apply(v[u].x, v[u].y), Op::apply(v[u].z, v[u].w));
  }
  return warp_chunk_tree<Op, U>(s, lane);
}

// Binary-counter merge of chunk c's root into the register stack.
template <class Op, int D>
__device__ __forceinline__ void counter_push(float (&stk)[D], float& v, int c) {
  bool carry = true;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (carry) {
      if (c & (1 << j)) {
        v = Op::apply(stk[j], v);
      } else {
        stk[j] = v;
        carry = false;
      }
    }
  }
}

// Reduce one work item: `valid` floats at x (<= item_floats) as
// item_floats/(128U) chunks merged by a binary-counter stack of aligned
// power-of-two subtrees (register-resident: every index is static). Full
// items are software-pipelined: chunk c+1 is loaded before chunk c is reduced.
template <class Op, bool kMap, int U>
__device__ __forceinline__ float work_item(const float* __restrict__ x, float* __restrict__ y,
                                           int64_t valid, int64_t item_floats, float a, float b, int lane) {
  constexpr int kChunk = 128 * U;
  constexpr int kMaxChunks = int((1ull << kMaxItemLog2) / kChunk);
  constexpr int kDepth = (kMaxChunks >= 64 ? 6 : kMaxChunks >= 32 ? 5 : kMaxChunks >= 16 ? 4 : kMaxChunks >= 8 ? 3 : 2);
  const int kChunks = int(item_floats / kChunk);
  float stk[kDepth];
#pragma unroll
  for (int j = 0; j < kDepth; ++j) stk[j] = Op::identity();
  float v = Op::identity();
  if (valid >= item_floats) {
    float4 cur[U], nxt[U];
    chunk_load<Op, false, U>(x, kChunk, lane, cur);
#pragma unroll 1
    for (int c = 0; c < kChunks; ++c) {
      if (c + 1 < kChunks) chunk_load<Op, false, U>(x + (c + 1) * kChunk, kChunk, lane, nxt);
      v = chunk_finish<Op, kMap, false, U>(cur, y + c * kChunk, kChunk, a, b, lane);
      counter_push<Op, kDepth>(stk, v, c);
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = nxt[u];
    }
    return v;  // c = kChunks-1 has all bits set: v is the root
  }
#pragma unroll 1
  for (int c = 0; c < kChunks; ++c) {
    const int64_t rem = valid - int64_t(c) * kChunk;
    if (rem >= kChunk) {
      float4 cur[U];
      chunk_load<Op, false, U>(x + c * kChunk, kChunk, lane, cur);
      v = chunk_finish<Op, kMap, false, U>(cur, y + c * kChunk, kChunk, a, b, lane);
    } else if (rem > 0) {
      float4 cur[U];
      chunk_load<Op, true, U>(x + c * kChunk, rem, lane, cur);
      v = chunk_finish<Op, kMap, true, U>(cur, y + c * kChunk, rem, a, b, lane);
    } else {
      v = Op::identity();
    }
    counter_push<Op, kDepth>(stk, v, c);
  }
  return v;
}

// ---- trees over values in global memory ----------------------------------------

constexpr int kTreeThreads = 256;  // == kWarps * 32: pass 1 CTAs run the trees too
constexpr int kTreeVals = 16;  // values per thread per block: 4096-value blocks (one
                               // per C2 partition of 2^24 floats in 2^12-float items)
constexpr int kTreeBlock = kTreeVals * kTreeThreads;

struct TreeSmem {
  float warp_root[kWarps];
  float stk[64];
  float seg[32];  // single-finisher tail: the partition values
};

// Tree over n values (L2-resident item roots or partition values) by ONE CTA
// of 256 threads, padded to a power of two with the identity. Values are
// consumed in aligned blocks of 4096: thread t combines its 16 contiguous
// values (4 tree levels in registers, all 16 loads in flight at once), the
// warp finishes 5 levels with xor
// shuffles (lower lane = left operand), thread 0 the last 3 over the warp
// roots — one barrier per block. Block roots are merged by a binary-counter
// stack of aligned subtrees and the stack is folded right to left.
template <class Op>
__device__ float cta_tree(const float* __restrict__ vals, uint64_t n, TreeSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint64_t nblocks = (n + kTreeBlock - 1) / kTreeBlock;
  for (uint64_t bi = 0; bi < nblocks; ++bi) {
    const uint64_t base = bi * kTreeBlock + kTreeVals * uint64_t(tid);
    float v[kTreeVals];
    if (base + kTreeVals <= n && (reinterpret_cast<uintptr_t>(vals + base) & 15) == 0) {
      // 4 x 16-byte loads (a quarter of the L2 sector requests of scalar loads)
#pragma unroll
      for (int k = 0; k < kTreeVals / 4; ++k) {
        const float4 q = __ldcg(reinterpret_cast<const float4*>(vals + base) + k);
        v[4 * k] = q.x;
        v[4 * k + 1] = q.y;
        v[4 * k + 2] = q.z;
        v[4 * k + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kTreeVals; ++k) v[k] = base + k < n ? __ldcg(vals + base + k) : Op::identity();
    }
    // balanced pairwise tree over the thread's aligned 16 values
#pragma unroll
    for (int w = kTreeVals / 2; w >= 1; w /= 2) {
#pragma unroll
      for (int k = 0; k < w; ++k) v[k] = Op::apply(v[2 * k], v[2 * k + 1]);
    }
    float r = v[0];
#pragma unroll
    for (int j = 0; j < 5; ++j) r = lr<Op>(r, __shfl_xor_sync(kFull, r, 1 << j), !((lane >> j) & 1));
    if (lane == 0) sm.warp_root[w] = r;
    __syncthreads();
    if (tid == 0) {
      const float* q = sm.warp_root;
      float b = Op::apply(Op::apply(Op::apply(q[0], q[1]), Op::apply(q[2], q[3])),
                          Op::apply(Op::apply(q[4], q[5]), Op::apply(q[6], q[7])));
      int j = 0;
      while ((bi >> j) & 1) {  // binary-counter merge of block bi
        b = Op::apply(sm.stk[j], b);
        ++j;
      }
      sm.stk[j] = b;
    }
    __syncthreads();
  }
  float root = Op::identity();
  if (tid == 0 && nblocks) {
    bool have = false;
    for (int j = 0; j < 64; ++j) {
      if ((nblocks >> j) & 1) {
        root = have ? Op::apply(sm.stk[j], root) : sm.stk[j];
        have = true;
      }
    }
  }
  return root;  // valid in thread 0
}

// ---- partition values + reduce_cl stage 2 (+ the cross-GPU exchange) ---------------

struct FinishArgs {
  const float* partial;       // item roots from pass 1
  const uint64_t* first_item;
  uint64_t nseg;
  float* out;                 // this rank's per-segment (partition) values
  uint32_t* done;             // [3] pass-1 exit / finisher / item counters, zero between launches
  unsigned long long* gen;    // [2] this parity's {start tickets, completed grids} (fused launches)
  float* result;              // reduce_cl result (every rank gets it), or null
  // sharded exchange (world > 1): region r = rank r's IPC-mapped buffer
  int world, rank;
  uint64_t part_offset;       // first global partition index of this rank
  uint64_t p_total;           // P over all ranks
  const uint64_t* peers;      // [world] region base addresses (this rank's own at [rank])
  uint64_t flags_offset;      // byte offset of the [world] epoch flags inside a region
  uint32_t* epoch;            // [1] exchanges completed (device counter; this one advances it)
  uint32_t* err;              // host-mapped error word: set to 1 when a peer wait times out
  int warp_mode;              // one warp (not one CTA) per segment
  uint32_t finishers;         // fused tail: finisher CTAs (0 = min(G, nseg))
  int flag_exchange;          // sharded: 1 = data stores + fence + epoch flags (A/B), 0 = one
                              // 64-bit {epoch, value} store per value, no fences
  int early_send;             // sharded, 64-bit protocol: each finisher sends its partition
                              // values as it computes them (stage 2 only receives)
  float* sub;                 // tapered tail: 4 sub-item roots per item in [taper_first, +ntaper)
  uint64_t taper_first, ntaper;
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Tree over n <= 2^13 values by ONE warp: blocks of 256 (lane l combines its
// 8 contiguous values, 5 xor-shuffle levels finish the block), block roots
// merged by a register binary-counter stack, folded right to left.
constexpr int kWarpTreeDepth = 5;  // up to 32 blocks
template <class Op>
__device__ float warp_tree(const float* __restrict__ vals, uint64_t n, int lane) {
  const uint32_t nb = uint32_t((n + 255) / 256);
  float stk[kWarpTreeDepth];
#pragma unroll
  for (int j = 0; j < kWarpTreeDepth; ++j) stk[j] = Op::identity();
#pragma unroll 1
  for (uint32_t c = 0; c < nb; ++c) {
    const uint64_t base = uint64_t(c) * 256 + 8 * lane;
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = base + k < n ? __ldcg(vals + base + k) : Op::identity();
    float r = Op::apply(Op::apply(Op::apply(v[0], v[1]), Op::apply(v[2], v[3])),
                        Op::apply(Op::apply(v[4], v[5]), Op::apply(v[6], v[7])));
#pragma unroll
    for (int j = 0; j < 5; ++j) r = lr<Op>(r, __shfl_xor_sync(kFull, r, 1 << j), !((lane >> j) & 1));
    counter_push<Op, kWarpTreeDepth>(stk, r, int(c));
  }
  bool have = false;
  float root = Op::identity();
#pragma unroll
  for (int j = 0; j < kWarpTreeDepth; ++j) {
    if ((nb >> j) & 1) {
      root = have ? Op::apply(stk[j], root) : stk[j];
      have = true;
    }
  }
  return root;
}

// Partition values of segments j, j+F, j+2F, ... (one CTA = finisher j of F),
// or — with many partitions of few items (warp_mode) — one warp per segment.
// Sharded, 64-bit protocol: partition value s of this rank to every peer's
// slot, tagged with this exchange's epoch (the counter advances only after
// every finisher has passed stage 2's ticket, so all finishers read the same).
__device__ __forceinline__ void send_value(const FinishArgs& p, uint64_t s, float r) {
  const uint32_t e = *reinterpret_cast<volatile uint32_t*>(p.epoch) + 1;
  const uint64_t buf = (e & 1) * p.p_total;
  for (int q = 0; q < p.world; ++q)
    st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(p.peers[q]) + buf + p.part_offset + s,
                       (uint64_t(e) << 32) | __float_as_uint(r));
}

// Tapered tail: the item roots of segment items [f, f+n) that were streamed
// as 4 aligned sub-items, rebuilt as ((s0, s1), (s2, s3)) — the association
// work_item gives a whole item of 4 sub-item-sized subtrees.
template <class Op>
__device__ __forceinline__ void taper_roots(const FinishArgs& p, uint64_t f, uint64_t n, uint32_t t, uint32_t nt) {
  const uint64_t lo = f > p.taper_first ? f : p.taper_first;
  for (uint64_t i = lo + t; i < f + n; i += nt) {
    const float4 q = __ldcg(reinterpret_cast<const float4*>(p.sub) + (i - p.taper_first));
    __stcg(const_cast<float*>(p.partial) + i, Op::apply(Op::apply(q.x, q.y), Op::apply(q.z, q.w)));
  }
}

template <class Op>
__device__ void segment_values(const FinishArgs& p, uint64_t j, uint64_t F, TreeSmem& sm) {
  const bool send = p.world > 1 && p.early_send;
  if (p.warp_mode) {
    const int lane = threadIdx.x & 31;
    for (uint64_t s = j * kWarps + (threadIdx.x >> 5); s < p.nseg; s += F * kWarps) {
      const uint64_t f = p.first_item[s], n = p.first_item[s + 1] - f;
      if (p.ntaper && f + n > p.taper_first) {
        taper_roots<Op>(p, f, n, lane, 32);
        __syncwarp();
      }
      const float r = n ? warp_tree<Op>(p.partial + f, n, lane) : Op::empty();
      if (lane == 0) {
        __stcg(p.out + s, r);
        if (F == 1 && s < 32) sm.seg[s] = r;
        if (send) send_value(p, s, r);
      }
    }
    return;
  }
  for (uint64_t s = j; s < p.nseg; s += F) {
    const uint64_t f = p.first_item[s], n = p.first_item[s + 1] - f;
    if (p.ntaper && f + n > p.taper_first) {
      taper_roots<Op>(p, f, n, threadIdx.x, blockDim.x);
      __syncthreads();
    }
    const float r = n ? cta_tree<Op>(p.partial + f, n, sm) : Op::empty();
    if (threadIdx.x == 0) {
      __stcg(p.out + s, r);
      if (send) send_value(p, s, r);
    }
  }
}

// A peer never published within kPeerWaitNs: the result is NaN (never a
// plausible value reduced from stale slots), the epoch stays where it was,
// and the exchange's error word — host-mapped, so every later C entry point
// on this exchange sees it without a device sync and fails with
// UCG_ERR_PEER until ucg_xchg_reset — is raised.
__device__ __noinline__ void peer_timeout(const FinishArgs& p) {
  if (threadIdx.x == 0) {
    *p.result = __int_as_float(0x7fc00000);
    *reinterpret_cast<volatile uint32_t*>(p.err) = 1u;
    __threadfence_system();
  }
}

// This grid is done with its parity's counters and item roots (every tree
// is built and the counters are zero again): count it as completed, so the
// next grid of this parity may start streaming (see k_segment_pass1).
__device__ __forceinline__ void release_parity(const FinishArgs& p) {
  if (!p.gen) return;
  __threadfence();
  atomicAdd(p.gen + 1, 1ull);
}

// Called by all F finisher CTAs after their segments are written. The last
// one to arrive resets the counters and runs reduce_cl stage 2: on one GPU
// directly over the partition values; sharded, it first stores this rank's
// values into every peer's region over NVLink (P2P stores), raises its epoch
// flag there (release, system scope), waits for all ranks' flags in its own
// region (acquire) and runs the same pairing tree over all P values in
// partition order — the collective fused into the reduction kernel.
template <class Op>
__device__ void stage2(const FinishArgs& p, uint32_t F, TreeSmem& sm) {
  __shared__ bool last;
  const int tid = threadIdx.x;
  __syncthreads();
  if (F == 1) {
    // the only finisher wrote every partition value itself: the barrier
    // orders those stores before the reads below, no ticket needed
    if (tid == 0) {
      p.done[0] = 0;
      p.done[1] = 0;
      p.done[2] = 0;
      release_parity(p);
    }
  } else {
    if (tid == 0) {
      __threadfence();
      last = atomicAdd(p.done + 1, 1u) == F - 1;
    }
    __syncthreads();
    if (!last) return;
    if (tid == 0) {
      p.done[0] = 0;
      p.done[1] = 0;
      p.done[2] = 0;
      release_parity(p);
    }
    __threadfence();
  }
  if (!p.result) return;
  if (F == 1 && p.world <= 1 && p.warp_mode && p.nseg && p.nseg <= 32) {
    // stage 2 over <= 32 values from shared memory by warp 0: the padded
    // pairing tree is 5 xor-shuffle levels (lower lane = left operand)
    if (tid < 32) {
      float r = uint64_t(tid) < p.nseg ? sm.seg[tid] : Op::identity();
#pragma unroll
      for (int j = 0; j < 5; ++j) r = lr<Op>(r, __shfl_xor_sync(kFull, r, 1 << j), !((tid >> j) & 1));
      if (tid == 0) *p.result = r;
    }
    return;
  }
  const float* vals = p.out;
  uint64_t nvals = p.nseg;
  uint32_t epoch = 0;
  bool timed_out = false;
  if (p.world > 1 && !p.flag_exchange) {
    // Each value travels with its epoch in ONE 64-bit store to every peer's
    // slot (single-copy atomic), so a reader that sees the epoch has the
    // value: no system fences, no flag round trip. Slots alternate by epoch
    // parity (a rank one step ahead writes the other buffer); the received
    // values are unpacked into this rank's gather area for the tree.
    epoch = *reinterpret_cast<volatile uint32_t*>(p.epoch) + 1;
    const uint64_t buf = (epoch & 1) * p.p_total;
    const uint64_t nsend = p.early_send ? 0 : p.nseg * uint64_t(p.world);  // early: sent by the finishers
    for (uint64_t i = tid; i < nsend; i += blockDim.x) {
      const uint64_t r = i / p.nseg, j = i - r * p.nseg;
      uint64_t* slot = reinterpret_cast<uint64_t*>(p.peers[r]) + buf + p.part_offset + j;
      st_relaxed_sys_u64(slot, (uint64_t(epoch) << 32) | __float_as_uint(__ldcg(p.out + j)));
    }
    const uint64_t* mine = reinterpret_cast<const uint64_t*>(p.peers[p.rank]) + buf;
    float* gathered = reinterpret_cast<float*>(p.peers[p.rank] + 16 * p.p_total);
    for (uint64_t i = tid; i < p.p_total; i += blockDim.x) {
      uint64_t v = ld_relaxed_sys_u64(mine + i);
      if (uint32_t(v >> 32) != epoch) {
        const uint64_t t0 = global_ns();
        uint32_t spins = 0;
        while (uint32_t((v = ld_relaxed_sys_u64(mine + i)) >> 32) != epoch) {
          if ((++spins & 1023) == 0 && global_ns() - t0 > kPeerWaitNs) {  // a peer never arrived
            timed_out = true;
            break;
          }
        }
      }
      gathered[i] = __uint_as_float(uint32_t(v));
    }
    if (__syncthreads_or(timed_out)) return peer_timeout(p);
    vals = gathered;
    nvals = p.p_total;
  } else if (p.world > 1) {
    // this exchange's epoch and value buffer (by parity)
    epoch = *reinterpret_cast<volatile uint32_t*>(p.epoch) + 1;
    const uint64_t buf = (epoch & 1) * p.p_total;
    for (int r = 0; r < p.world; ++r) {
      float* g = reinterpret_cast<float*>(p.peers[r]) + buf + p.part_offset;
      for (uint64_t i = tid; i < p.nseg; i += blockDim.x) g[i] = __ldcg(p.out + i);
    }
    __threadfence_system();
    __syncthreads();
    if (tid < p.world) {
      uint32_t* fl = reinterpret_cast<uint32_t*>(p.peers[tid] + p.flags_offset);
      st_release_sys(fl + p.rank, epoch);
      const uint32_t* mine = reinterpret_cast<const uint32_t*>(p.peers[p.rank] + p.flags_offset) + tid;
      const uint64_t t0 = global_ns();
      while (int32_t(ld_acquire_sys(mine) - epoch) < 0) {
        __nanosleep(64);
        if (global_ns() - t0 > kPeerWaitNs) {  // a peer never arrived
          timed_out = true;
          break;
        }
      }
    }
    if (__syncthreads_or(timed_out)) return peer_timeout(p);
    vals = reinterpret_cast<const float*>(p.peers[p.rank]) + buf;
    nvals = p.p_total;
  }
  const float root = nvals ? cta_tree<Op>(vals, nvals, sm) : Op::empty();
  if (tid == 0) {
    *p.result = root;
    if (p.world > 1) *p.epoch = epoch;
  }
}

// Pass 1: one warp per work item (grid-stride over items); item roots go to
// `partial`. With `finish` set (a cooperative launch: every CTA resident),
// the partition values and reduce_cl stage 2 run in the same kernel: each
// CTA takes an exit ticket after its last item; the last F = min(G, nseg)
// ticket holders wait until all G CTAs have exited the streaming loop, then
// reduce one segment each, and the last of them runs stage 2. One fence per
// CTA, no kernel boundary between the stream and the trees. (Finishing
// segments with a per-item last-warp counter was measured 5% slower: the
// fence after each item waits for that warp's 32-64 KB of y stores.)
struct Pass1Args {
  const float* x;
  float* y;
  const uint64_t* begin;
  const uint64_t* len;
  const uint64_t* first_item;
  const uint32_t* item_seg;
  uint64_t nitems;
  int item_log2;
  float a, b;
  float* partial;
  int finish;
  int dynamic;  // claim items from the counter fin.done[2] instead of grid-stride
  // 1: the previous kernel in the stream is the same step on the same table
  // and buffers (segment_reduce checks): stream first, wait for it only
  // before the partition trees, so this step's stream overlaps its tail
  int early;
  int early_top;  // early mode, next step triggered at the top (A/B off: UCG_EARLY_LATE_TRIGGER)
  FinishArgs fin;
};

template <class Op, bool kMap, int U, int kMinBlocks>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks) k_segment_pass1(const __grid_constant__ Pass1Args p) {
  // Programmatic dependent launch (small tables, see launch_pass1): this grid
  // may be resident before the previous step's grid has finished; wait for it
  // (its y, partials and counter reset) before touching memory, and let the
  // next step's grid launch now. Both are no-ops without the launch attribute.
  //
  // Early mode (repeated steps, see Pass1Args::early): the stream only reads
  // x and writes y (the same values), item roots and claims of this launch's
  // parity half, so it starts at once; the finishers wait for the previous
  // step (whose trees may still run) before its counters, partition values
  // and exchange, and only then let the next step launch — which therefore
  // never overlaps a step of its own parity.
  //
  // Early mode with the trigger at the top (the default): the next step may
  // launch at once and its CTAs take the slots this grid's CTAs leave as
  // they finish the stream (the ragged end of the stream overlaps the next
  // step). A grid then may start while the previous grid of its parity is
  // still running, so each CTA takes a start ticket of its parity — ticket
  // / G is the number of earlier fused grids of that parity — and waits
  // until that many have released the parity (release_parity).
  //
  // The ticket is taken BEFORE this CTA triggers its dependents: a grid of
  // the same parity two launches later exists only after every CTA of this
  // one has triggered, so tickets of different grids never interleave and
  // ticket / G is exact (a late CTA of this grid must not draw a ticket
  // after the next same-parity grid, or it would wait for its own grid).
  __shared__ unsigned long long start_ticket;
  if (p.fin.gen && p.finish) {
    if (threadIdx.x == 0) start_ticket = atomicAdd(p.fin.gen, 1ull);
    __syncthreads();
  }
  if (!p.early) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else if (p.early_top) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
      const unsigned long long g = start_ticket / gridDim.x;
      const uint64_t t0 = global_ns();
      uint32_t spins = 0;
      while (ld_acquire_gpu_u64(p.fin.gen + 1) < g) {
        __nanosleep(64);
        if ((++spins & 1023) == 0 && global_ns() - t0 > kPeerWaitNs) __trap();
      }
    }
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const uint64_t warp = uint64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = uint64_t(gridDim.x) * kWarps;
  // A claim covers kPer consecutive items: one for the read+write map stream,
  // two for the read-only reduction, whose items finish twice as fast and
  // would otherwise saturate the single claim counter.
  constexpr uint64_t kPer = kMap ? 1 : 2;
  // Tapered tail (map stream only): units past taper_first are sub-items, a
  // quarter of an item each, so the last warps finish close together.
  const uint64_t ntaper = kMap ? p.fin.ntaper : 0;
  const uint64_t units_end = ntaper ? p.fin.taper_first + 4 * ntaper : 0;
  uint64_t unit = warp;
  while (ntaper ? unit < units_end : unit * kPer < p.nitems) {
    // dynamic: the next unit is claimed now and consumed after this one
    uint32_t claim = 0;
    if (p.dynamic && lane == 0) claim = atomicAdd(p.fin.done + 2, 1u);
    if (ntaper && unit >= p.fin.taper_first) {
      const uint64_t u = unit - p.fin.taper_first, item = p.fin.taper_first + (u >> 2);
      const uint32_t s = p.item_seg[item];
      const int sl = p.item_log2 - 2;
      const uint64_t start = ((item - p.first_item[s]) << p.item_log2) + ((u & 3) << sl);
      const uint64_t off = p.begin[s] + start;
      const int64_t valid = int64_t(p.len[s]) - int64_t(start);  // <= 0: an empty sub-item
      const float r = work_item<Op, kMap, U>(p.x + off, kMap ? p.y + off : nullptr,
                                             valid < (int64_t(1) << sl) ? valid : (int64_t(1) << sl),
                                             int64_t(1) << sl, p.a, p.b, lane);
      if (lane == 0) p.fin.sub[u] = r;
      unit = p.dynamic ? nwarps + __shfl_sync(kFull, claim, 0) : unit + nwarps;
      continue;
    }
#pragma unroll 1
    for (uint64_t item = unit * kPer; item < umin((unit + 1) * kPer, p.nitems); ++item) {
      const uint32_t s = p.item_seg[item];
      const uint64_t blk = item - p.first_item[s];
      const uint64_t off = p.begin[s] + (blk << p.item_log2);
      const int64_t item_floats = int64_t(1) << p.item_log2;
      const int64_t valid = int64_t(umin(uint64_t(item_floats), p.len[s] - (blk << p.item_log2)));
      const float r =
          work_item<Op, kMap, U>(p.x + off, kMap ? p.y + off : nullptr, valid, item_floats, p.a, p.b, lane);
      if (lane == 0) p.partial[item] = r;
    }
    unit = p.dynamic ? nwarps + __shfl_sync(kFull, claim, 0) : unit + nwarps;
  }
  if (!p.finish) return;
  __shared__ TreeSmem sm;
  __shared__ uint32_t ticket;
  const uint32_t G = gridDim.x;
  const uint32_t F = p.fin.finishers ? p.fin.finishers : uint32_t(umin(G, p.fin.nseg ? p.fin.nseg : 1));
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    ticket = atomicAdd(p.fin.done, 1u);
  }
  __syncthreads();
  if (ticket + F < G) return;
  if (p.early) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (!p.early_top) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    // every CTA is resident (cooperative launch), so the others finish their
    // stream; a wait of kPeerWaitNs cannot happen — trap rather than reduce
    // item roots that are not all written
    const uint64_t t0 = global_ns();
    uint32_t spins = 0;
    while (ld_acquire_gpu(p.fin.done) < G) {
      __nanosleep(32);
      if ((++spins & 1023) == 0 && global_ns() - t0 > kPeerWaitNs) __trap();
    }
  }
  __syncthreads();
  segment_values<Op>(p.fin, ticket + F - G, F, sm);
  stage2<Op>(p.fin, F, sm);
}

// Stand-alone finish (tables with no work items, or UCG_SEPARATE_FINISH=1):
// one CTA per segment, then stage 2 by the last CTA.
template <class Op>
__global__ void __launch_bounds__(kTreeThreads) k_segment_finish(const __grid_constant__ FinishArgs p) {
  __shared__ TreeSmem sm;
  const uint32_t F = gridDim.x;
  if (blockIdx.x < p.nseg) segment_values<Op>(p, blockIdx.x, F, sm);
  stage2<Op>(p, F, sm);
}

// reduce_cl stage 2 alone over partition values already in `out` (one CTA):
// with an exchange context, the sharded NVLink exchange + the tree over all
// ranks' values (the e2e path, whose partials come from per-chunk launches).
template <class Op>
__global__ void __launch_bounds__(kTreeThreads) k_stage2_only(const __grid_constant__ FinishArgs p) {
  __shared__ TreeSmem sm;
  stage2<Op>(p, 1, sm);
}

template <class Op>
__global__ void __launch_bounds__(kTreeThreads) k_tree(const float* __restrict__ x, uint64_t n, float* __restrict__ out) {
  __shared__ TreeSmem sm;
  const float r = n ? cta_tree<Op>(x, n, sm) : Op::empty();
  if (threadIdx.x == 0) out[0] = r;
}

// ---- elementwise ---------------------------------------------------------------

__global__ void __launch_bounds__(256) k_affine(const float4* __restrict__ x, float4* __restrict__ y, uint64_t n4,
                                                float a, float b) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  // 4-way unrolled grid-stride loop: 4 independent 128-bit loads in flight
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 v0 = ld_stream(x + i), v1 = ld_stream(x + i + stride), v2 = ld_stream(x + i + 2 * stride),
           v3 = ld_stream(x + i + 3 * stride);
#define UCG_AFF(v) v.x = affine(v.x, a, b); v.y = affine(v.y, a, b); v.z = affine(v.z, a, b); v.w = affine(v.w, a, b);
    UCG_AFF(v0) UCG_AFF(v1) UCG_AFF(v2) UCG_AFF(v3)
    st_stream(y + i, v0);
    st_stream(y + i + stride, v1);
    st_stream(y + i + 2 * stride, v2);
    st_stream(y + i + 3 * stride, v3);
  }
  for (; i < n4; i += stride) {
    float4 v = ld_stream(x + i);
    UCG_AFF(v)
#undef UCG_AFF
    st_stream(y + i, v);
  }
}

// Map-only stream with claimed work items: a warp claims 16 KB items (4
// chunks of 1024 floats, 8 LDG.128 per lane per chunk) from a counter, the
// next chunk's loads in flight while the current one is mapped and stored;
// the next claim is issued when an item starts and consumed when it ends.
// Same access pattern as the fused reduction kernel (which reaches ~1.04 of
// the copy peak this way), without the tree.
constexpr int kAffItemChunks = 4;
__global__ void __launch_bounds__(kWarps * 32, 2) k_affine_items(const float* __restrict__ x, float* __restrict__ y,
                                                                  uint64_t nitems, float a, float b,
                                                                  unsigned long long* __restrict__ ctr) {
  constexpr int U = 8, kChunk = 128 * U;
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = uint64_t(gridDim.x) * kWarps;
  uint64_t item = uint64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  while (item < nitems) {
    unsigned long long claim = 0;
    if (lane == 0) claim = atomicAdd(ctr, 1ull);
    const float* xs = x + item * (kAffItemChunks * kChunk);
    float* ys = y + item * (kAffItemChunks * kChunk);
    float4 cur[U], nxt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = ld_stream(reinterpret_cast<const float4*>(xs + 128 * u + 4 * lane));
#pragma unroll
    for (int c = 0; c < kAffItemChunks; ++c) {
      if (c + 1 < kAffItemChunks) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          nxt[u] = ld_stream(reinterpret_cast<const float4*>(xs + (c + 1) * kChunk + 128 * u + 4 * lane));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float4 v = cur[u];
        v.x = affine(v.x, a, b);
        v.y = affine(v.y, a, b);
        v.z = affine(v.z, a, b);
        v.w = affine(v.w, a, b);
        st_stream(reinterpret_cast<float4*>(ys + c * kChunk + 128 * u + 4 * lane), v);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = nxt[u];
    }
    item = nwarps + __shfl_sync(kFull, claim, 0);
  }
}

__global__ void k_affine_tail(const float* __restrict__ x, float* __restrict__ y, uint64_t from, uint64_t n,
                              float a, float b) {
  const uint64_t i = from + threadIdx.x;
  if (i < n) y[i] = affine(x[i], a, b);
}

template <class Op>
__global__ void __launch_bounds__(256) k_elementwise2(const float* __restrict__ a, const float* __restrict__ b,
                                                      float* __restrict__ c, uint64_t n) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    c[i] = Op::apply(a[i], b[i]);
}
__global__ void __launch_bounds__(256) k_add_i64(const int64_t* __restrict__ a, const int64_t* __restrict__ b,
                                                 int64_t* __restrict__ c, uint64_t n) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    c[i] = int64_t(uint64_t(a[i]) + uint64_t(b[i]));
}

// ---- reduce_cl over vector elements (stage 1 fold + stage 2 tree, per lane) ----

struct I64Add {
  static __device__ __forceinline__ int64_t apply(int64_t a, int64_t b) { return int64_t(uint64_t(a) + uint64_t(b)); }
};
struct F32SumE {
  static __device__ __forceinline__ float apply(float a, float b) { return __fadd_rn(a, b); }
};
struct F32MaxE {
  static __device__ __forceinline__ float apply(float a, float b) { return (a < b) ? b : a; }
};

// reduce_cl over vector elements, in two launches:
//  stage 1 (engine.hpp:144-170): every non-empty partition's elements folded
//    left to right, all partitions and lanes in parallel —
//    short vectors (len < 32): one WARP per (partition, lane): the lanes load
//      32 consecutive elements' values (the next 32 in flight) and lane 0's
//      fold consumes them in order through shuffles, so a chain of 2^18
//      one-float elements runs at shuffle + add latency, not load latency;
//    long vectors: one thread per (partition, lane) with loads 8 ahead;
//  stage 2 (engine.hpp:172-190): one thread per lane, the pairing tree over
//    the partition partials in partition order (binary-counter stack of
//    aligned subtrees, folded right to left).
constexpr int kStage2Depth = 64;  // binary-counter stack: one slot per bit of the partition count

template <class T, class Op>
__global__ void __launch_bounds__(256) k_fold_warp(const T* const* __restrict__ elems,
                                                   const uint64_t* __restrict__ part_first, uint64_t nonempty,
                                                   uint64_t len, T* __restrict__ partials) {
  const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nonempty * len) return;
  const uint64_t k = w / len, j = w % len;
  const uint64_t e0 = part_first[k], e1 = part_first[k + 1];
  T acc = elems[e0][j];
  uint64_t base = e0 + 1;
  T v = base + lane < e1 ? elems[base + lane][j] : T{};
  while (base < e1) {
    const uint64_t nb = base + 32;
    const T nv = nb + lane < e1 ? elems[nb + lane][j] : T{};  // next batch in flight
    const int cnt = int(umin(32, e1 - base));
    for (int i = 0; i < cnt; ++i) acc = Op::apply(acc, __shfl_sync(0xffffffffu, v, i));
    v = nv;
    base = nb;
  }
  if (lane == 0) partials[k * len + j] = acc;
}

template <class T, class Op>
__global__ void __launch_bounds__(128) k_fold_thread(const T* const* __restrict__ elems,
                                                     const uint64_t* __restrict__ part_first, uint64_t nonempty,
                                                     uint64_t len, T* __restrict__ partials) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nonempty * len) return;
  const uint64_t k = t / len, j = t % len;
  const uint64_t e0 = part_first[k], e1 = part_first[k + 1];
  T acc = elems[e0][j];
  uint64_t e = e0 + 1;
  for (; e + 8 <= e1; e += 8) {
    T v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = elems[e + i][j];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc = Op::apply(acc, v[i]);
  }
  for (; e < e1; ++e) acc = Op::apply(acc, elems[e][j]);
  partials[k * len + j] = acc;
}

template <class T, class Op>
__global__ void __launch_bounds__(128) k_stage2(const T* __restrict__ partials, uint64_t nonempty, uint64_t len,
                                                T* __restrict__ out) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= len) return;
  T stk[kStage2Depth];  // slot l holds an aligned subtree of 2^l partials (no partition limit)
  for (uint64_t k = 0; k < nonempty; ++k) {
    T acc = partials[k * len + j];
    int lvl = 0;
#pragma unroll 1
    while ((k >> lvl) & 1) {
      acc = Op::apply(stk[lvl], acc);
      ++lvl;
    }
    stk[lvl] = acc;
  }
  bool have = false;
  T acc{};
#pragma unroll 1
  for (int lvl = 0; lvl < kStage2Depth; ++lvl) {
    if ((nonempty >> lvl) & 1) {
      acc = have ? Op::apply(stk[lvl], acc) : stk[lvl];
      have = true;
    }
  }
  out[j] = acc;
}

// Pass-1 variants (chunk width U, CTAs per SM). The default was chosen by a
// sweep on B200 (tools/microbench.py); UCG_PASS1_VARIANT overrides it for
// tuning runs.
struct Pass1Variant {
  int u, minb;
};
constexpr Pass1Variant kPass1Variants[] = {{8, 2}, {4, 3}, {4, 4}, {2, 8}, {2, 6}, {8, 3}};
constexpr int kPass1Default = 0;

inline int pass1_variant() {
  static int v = [] {
    const char* e = getenv("UCG_PASS1_VARIANT");
    int k = e ? atoi(e) : kPass1Default;
    return (k < 0 || k >= int(sizeof(kPass1Variants) / sizeof(kPass1Variants[0]))) ? kPass1Default : k;
  }();
  return v;
}

template <class Op, bool kMap, int U, int MINB>
cudaError_t launch_pass1(const Pass1Args& args, const ucg_segtab* t, cudaStream_t st) {
  const uint64_t want = (t->nitems + kWarps - 1) / kWarps;
  const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(sm_count()) * MINB)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kWarps * 32);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  // co-residency is needed only when several finisher CTAs wait for the
  // whole grid; a single finisher is the last CTA out and never waits, so
  // that launch instead overlaps its ramp with the previous step's tail
  // (programmatic dependent launch; C1: the whole step is ~6 us)
  static const bool no_pdl = getenv("UCG_NO_PDL") != nullptr;
  // UCG_PDL_MULTI=1 (A/B): the multi-finisher launch too is a PDL launch
  // instead of a cooperative one. Its grid never exceeds the co-resident
  // capacity (2 CTAs x 148 SMs at the occupancy the cooperative launch
  // validates), and the next step's CTAs park in griddepcontrol.wait only in
  // slots this grid has left, so every CTA of this grid is already resident.
  static const bool pdl_multi = getenv("UCG_PDL_MULTI") != nullptr;
  // An early-mode launch is a PDL launch (its CTAs become resident as the
  // previous step's CTAs leave; its finishers wait only for CTAs of its own
  // grid, which all get slots once the previous finishers exit).
  if (args.finish && args.fin.finishers != 1 && !args.early && !(pdl_multi && !no_pdl)) {
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.numAttrs = 1;
  } else if (!no_pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, k_segment_pass1<Op, kMap, U, MINB>, args);
}

template <class Op, bool kMap>
cudaError_t dispatch_pass1(const Pass1Args& args, const ucg_segtab* t, cudaStream_t st) {
  switch (pass1_variant()) {
    case 1: return launch_pass1<Op, kMap, 4, 3>(args, t, st);
    case 2: return launch_pass1<Op, kMap, 4, 4>(args, t, st);
    case 3: return launch_pass1<Op, kMap, 2, 8>(args, t, st);
    case 4: return launch_pass1<Op, kMap, 2, 6>(args, t, st);
    case 5: return launch_pass1<Op, kMap, 8, 3>(args, t, st);
    default: return launch_pass1<Op, kMap, 8, 2>(args, t, st);
  }
}

// Items are claimed dynamically by default (UCG_DYNAMIC_ITEMS=0: grid-stride).
// Measured on B200 (tools/scaling_probe.py, ncu dram__throughput): 2^30 fp32
// fused map+psum 1.266 ms / 82.4% of DRAM peak claimed vs 1.380 ms / 75.6%
// grid-stride — warps stay on one compact, advancing address window instead
// of drifting apart, and the last items balance across SMs.
inline bool dynamic_items() {
  static const bool v = [] {
    const char* e = getenv("UCG_DYNAMIC_ITEMS");
    return !e || atoi(e) != 0;
  }();
  return v;
}

inline bool separate_finish() {
  static const bool v = [] {
    const char* e = getenv("UCG_SEPARATE_FINISH");
    return e && atoi(e) != 0;
  }();
  return v;
}

// Early mode is safe when the kernel just before this one in the stream is
// the same fused step (same table, buffers, map and op): then the only early
// overlap is that step's partition trees, and this step's stream touches
// nothing they read. Any other pass-1 launch on the stream breaks the chain;
// other kernels and copies never trigger their dependents early, so a
// programmatic launch after them starts only when they have completed.
// UCG_NO_EARLY (A/B): never.
inline bool repeat_of_last_pass1(cudaStream_t st, const ucg_segtab* t, const float* x, const float* y, float a,
                                 float b, const float* out, const float* result, const ucg_xchg* xg, int op) {
  struct Key {
    const void* t;
    const void *x, *y, *out, *result, *xg;
    float a, b;
    int op;
    bool operator==(const Key& o) const {
      return t == o.t && x == o.x && y == o.y && out == o.out && result == o.result && xg == o.xg &&
             std::memcmp(&a, &o.a, 4) == 0 && std::memcmp(&b, &o.b, 4) == 0 && op == o.op;
    }
  };
  static const bool off = getenv("UCG_NO_EARLY") != nullptr || getenv("UCG_NO_PDL") != nullptr;
  static std::mutex mu;
  static std::unordered_map<cudaStream_t, Key> last;
  const Key k{t, x, y, out, result, xg, a, b, op};
  std::lock_guard<std::mutex> lock(mu);
  auto it = last.find(st);
  const bool same = it != last.end() && it->second == k;
  last[st] = k;
  return same && !off;
}

// Pass 1 with the partition trees and reduce_cl stage 2 folded into its tail
// (one launch per step); a table without work items launches the stand-alone
// finish kernel instead.
template <class Op>
int segment_reduce(const float* x, float* y, const ucg_segtab* t, float a, float b, float* scratch, float* out,
                   float* result, ucg_xchg* xg, cudaStream_t st) {
  int dev = -1;
  UCG_CUDA(cudaGetDevice(&dev));
  if (dev != t->device) {
    return fail(UCG_ERR_ARG, "segment table was created on device " + std::to_string(t->device) +
                                 ", current device is " + std::to_string(dev));
  }
  // launch parity: alternate launches use alternate counter sets and scratch
  // halves, so a step may stream while the previous one finishes
  const uint64_t par = t->launches++ & 1;
  scratch += par * scratch_half(t);
  uint32_t* done = t->d_done + 4 * par;
  FinishArgs f{scratch, t->d_first_item, t->nseg, out, done, t->d_gen + 2 * par, result, 1, 0, 0, t->nseg, nullptr, 0, nullptr, nullptr, 0, 0, 0, 0};
  if (xg) {
    f.world = xg->world;
    f.rank = xg->rank;
    f.part_offset = xg->part_offset;
    f.p_total = xg->p_total;
    f.peers = xg->d_peers;
    f.flags_offset = xg->flags_offset;
    f.epoch = xg->d_epoch;
    static const bool flags_xchg = getenv("UCG_XCHG_FLAGS") != nullptr;  // A/B: the fenced flag protocol
    static const bool late_send = getenv("UCG_XCHG_LATE_SEND") != nullptr;  // A/B: stage 2 sends everything
    f.flag_exchange = flags_xchg ? 1 : 0;
    f.early_send = (flags_xchg || late_send) ? 0 : 1;
    f.err = xg->d_err;
  }
  if (y && t->ntaper) {  // tapered tail of the map stream (scratch: item roots, then the sub-roots)
    f.sub = scratch + ((t->nitems + 4) & ~uint64_t(3));  // 16-byte aligned
    f.taper_first = t->nitems - t->ntaper;
    f.ntaper = t->ntaper;
  }
  const bool fused_finish = t->nitems && !separate_finish();
  if (!fused_finish) f.gen = nullptr;  // only fused launches take parity tickets and release
  // many partitions of few items: a warp per partition tree (the fused tail
  // has only min(G, P) finisher CTAs; G = 2 CTAs per SM)
  f.warp_mode = fused_finish && t->nseg > uint64_t(sm_count()) * 4 &&
                t->max_items_per_seg <= (uint64_t(256) << kWarpTreeDepth);
  // small tables (C1: 4 partitions of 2^8 items): the last CTA to leave the
  // stream runs every partition tree (one warp each) and stage 2 itself, when
  // that is at most two rounds of one 256-value block per warp — no finisher
  // phase, no second wait. Saves ~2 us of a ~10 us step.
  if (fused_finish && !getenv("UCG_MULTI_FINISHER")) {
    const uint64_t rounds = (t->nseg + kWarps - 1) / kWarps, blocks = (t->max_items_per_seg + 255) / 256;
    if (rounds * blocks <= 2) {
      f.warp_mode = 1;
      f.finishers = 1;
    }
  }
  if (t->nitems) {
    Pass1Args args{x, y, t->d_begin, t->d_len, t->d_first_item, t->d_item_seg, t->nitems, t->item_log2,
                   a, b, scratch, fused_finish ? 1 : 0, dynamic_items() ? 1 : 0, 0, 0, f};
    // every pass-1 launch updates the tracker (a different launch in between
    // breaks the chain); only a fused one may run early
    const bool repeat = repeat_of_last_pass1(st, t, x, y, a, b, out, result, xg, Op::kId);
    args.early = fused_finish && repeat ? 1 : 0;
    // the next step is triggered at the top (default; C1 4.93 -> 4.38 us,
    // 8-GPU shard 163.7 -> 160.4 us, same box); UCG_EARLY_LATE_TRIGGER=1
    // (A/B): only after this step's stream and the previous step's completion
    static const bool early_top = getenv("UCG_EARLY_LATE_TRIGGER") == nullptr;
    args.early_top = args.early && early_top ? 1 : 0;
    const cudaError_t e = y ? dispatch_pass1<Op, true>(args, t, st) : dispatch_pass1<Op, false>(args, t, st);
    UCG_CUDA(e);
    UCG_LAUNCHED();
  }
  if (!fused_finish && (t->nseg || result)) {
    k_segment_finish<Op><<<unsigned(std::max<uint64_t>(1, t->nseg)), kTreeThreads, 0, st>>>(f);
    UCG_LAUNCHED();
  }
  return UCG_OK;
}

template <class T, class Op>
int reduce_cl(const T* const* elem_ptrs, uint64_t count, uint64_t len, const uint64_t* part_counts,
              uint64_t nparts, T* out, cudaStream_t st) {
  uint64_t total = 0;
  std::vector<uint64_t> first(1, 0);
  for (uint64_t p = 0; p < nparts; ++p) {
    total += part_counts[p];
    if (part_counts[p]) first.push_back(total);
  }
  if (total != count) return fail(UCG_ERR_ARG, "part_counts do not sum to count");
  if (count == 0) return fail(UCG_ERR_EMPTY, "reduce_cl needs at least one element");
  const uint64_t nonempty = first.size() - 1;
  if (len == 0) return UCG_OK;
  uint64_t* d_first = nullptr;
  T* d_part = nullptr;
  UCG_CUDA(cudaMallocAsync(&d_first, first.size() * 8, st));
  UCG_CUDA(cudaMallocAsync(&d_part, nonempty * len * sizeof(T), st));
  // (the pageable-source copy is staged before cudaMemcpyAsync returns)
  UCG_CUDA(cudaMemcpyAsync(d_first, first.data(), first.size() * 8, cudaMemcpyHostToDevice, st));
  const uint64_t chains = nonempty * len;
  if (len < 32) {
    const unsigned grid = unsigned((chains * 32 + 255) / 256);
    k_fold_warp<T, Op><<<grid, 256, 0, st>>>(elem_ptrs, d_first, nonempty, len, d_part);
  } else {
    const unsigned grid = unsigned((chains + 127) / 128);
    k_fold_thread<T, Op><<<grid, 128, 0, st>>>(elem_ptrs, d_first, nonempty, len, d_part);
  }
  UCG_LAUNCHED();
  k_stage2<T, Op><<<unsigned((len + 127) / 128), 128, 0, st>>>(d_part, nonempty, len, out);
  UCG_LAUNCHED();
  UCG_CUDA(cudaFreeAsync(d_first, st));
  UCG_CUDA(cudaFreeAsync(d_part, st));
  return UCG_OK;
}

}  // namespace
}  // namespace ucg

using namespace ucg;

extern "C" {

int ucg_map_affine_f32(const float* x, float* y, uint64_t n, float a, float b, void* stream) {
  if (int rc = check_device()) return rc;
  if (!n) return UCG_OK;
  if (!x || !y) return fail(UCG_ERR_ARG, "x/y is null");
  if (!aligned16(x) || !aligned16(y)) return fail(UCG_ERR_ARG, "x/y must be 16-byte aligned");
  cudaStream_t st = as_stream(stream);
  constexpr uint64_t kItem = kAffItemChunks * 1024;  // floats per claimed item
  const uint64_t nitems = n / kItem;
  uint64_t done = 0;
  if (nitems >= uint64_t(sm_count()) * 16) {  // large maps: claimed 16 KB items
    unsigned long long* ctr = claim_counter();
    if (!ctr) return fail(UCG_ERR_CUDA, "map: counter allocation failed");
    UCG_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
    const unsigned grid = unsigned(std::min<uint64_t>((nitems + kWarps - 1) / kWarps, uint64_t(sm_count()) * 2));
    k_affine_items<<<grid, kWarps * 32, 0, st>>>(x, y, nitems, a, b, ctr);
    UCG_LAUNCHED();
    done = nitems * kItem;
    x += done;
    y += done;
    n -= done;
  }
  const uint64_t n4 = n / 4;
  if (n4) {
    const uint64_t want = (n4 + 255) / 256;
    const unsigned grid = unsigned(std::min<uint64_t>(want, uint64_t(sm_count()) * 8));
    k_affine<<<grid, 256, 0, st>>>(reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), n4, a, b);
    UCG_LAUNCHED();
  }
  if (n % 4) {
    k_affine_tail<<<1, 32, 0, st>>>(x, y, n4 * 4, n, a, b);
    UCG_LAUNCHED();
  }
  return UCG_OK;
}

int ucg_elementwise2_f32(const float* a, const float* b, float* c, uint64_t n, int op, void* stream) {
  if (int rc = check_device()) return rc;
  if (!n) return UCG_OK;
  if (!a || !b || !c) return fail(UCG_ERR_ARG, "null argument");
  const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(sm_count()) * 8));
  if (op == UCG_OP_SUM) k_elementwise2<OpSum><<<grid, 256, 0, as_stream(stream)>>>(a, b, c, n);
  else if (op == UCG_OP_MAX) k_elementwise2<OpMax><<<grid, 256, 0, as_stream(stream)>>>(a, b, c, n);
  else return fail(UCG_ERR_ARG, "unknown op");
  UCG_LAUNCHED();
  return UCG_OK;
}

int ucg_elementwise2_i64(const int64_t* a, const int64_t* b, int64_t* c, uint64_t n, void* stream) {
  if (int rc = check_device()) return rc;
  if (!n) return UCG_OK;
  if (!a || !b || !c) return fail(UCG_ERR_ARG, "null argument");
  const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(sm_count()) * 8));
  k_add_i64<<<grid, 256, 0, as_stream(stream)>>>(a, b, c, n);
  UCG_LAUNCHED();
  return UCG_OK;
}

int ucg_segment_reduce_f32(const float* x, const ucg_segtab* t, int op, float* scratch, float* out,
                           void* stream) {
  if (int rc = check_device()) return rc;
  if (!t) return fail(UCG_ERR_ARG, "segment table is null");
  if (t->nseg && (!out || (t->nitems && (!x || !scratch)))) return fail(UCG_ERR_ARG, "null argument");
  if (t->nitems && !aligned16(x)) return fail(UCG_ERR_ARG, "x must be 16-byte aligned");
  if (op == UCG_OP_SUM)
    return segment_reduce<OpSum>(x, nullptr, t, 0.f, 0.f, scratch, out, nullptr, nullptr, as_stream(stream));
  if (op == UCG_OP_MAX)
    return segment_reduce<OpMax>(x, nullptr, t, 0.f, 0.f, scratch, out, nullptr, nullptr, as_stream(stream));
  return fail(UCG_ERR_ARG, "unknown op");
}

int ucg_map_affine_segment_reduce_f32(const float* x, float* y, const ucg_segtab* t, float a, float b, int op,
                                      float* scratch, float* out, void* stream) {
  if (int rc = check_device()) return rc;
  if (!t) return fail(UCG_ERR_ARG, "segment table is null");
  if (t->nseg && (!out || (t->nitems && (!x || !y || !scratch)))) return fail(UCG_ERR_ARG, "null argument");
  if (t->nitems && (!aligned16(x) || !aligned16(y))) return fail(UCG_ERR_ARG, "x/y must be 16-byte aligned");
  if (op == UCG_OP_SUM) return segment_reduce<OpSum>(x, y, t, a, b, scratch, out, nullptr, nullptr, as_stream(stream));
  if (op == UCG_OP_MAX) return segment_reduce<OpMax>(x, y, t, a, b, scratch, out, nullptr, nullptr, as_stream(stream));
  return fail(UCG_ERR_ARG, "unknown op");
}

int ucg_segment_reduce_cl_f32(const float* x, float* y, const ucg_segtab* t, float a, float b, int op,
                              float* scratch, float* partials, ucg_xchg* xchg, float* result, void* stream) {
  if (int rc = check_device()) return rc;
  if (!t || !result) return fail(UCG_ERR_ARG, "segment table / result is null");
  if (t->nseg && (!partials || (t->nitems && (!x || !scratch)))) return fail(UCG_ERR_ARG, "null argument");
  if (t->nitems && (!aligned16(x) || (y && !aligned16(y)))) return fail(UCG_ERR_ARG, "x/y must be 16-byte aligned");
  if (xchg && (!xchg->opened || xchg->nloc != t->nseg)) return fail(UCG_ERR_ARG, "exchange not opened for this shard");
  if (xchg) {
    if (int rc = xchg_guard(xchg)) return rc;
  }
  if (op == UCG_OP_SUM) return segment_reduce<OpSum>(x, y, t, a, b, scratch, partials, result, xchg, as_stream(stream));
  if (op == UCG_OP_MAX) return segment_reduce<OpMax>(x, y, t, a, b, scratch, partials, result, xchg, as_stream(stream));
  return fail(UCG_ERR_ARG, "unknown op");
}

int ucg_reduce_cl_xchg_f32(float* partials, uint64_t nloc, int op, ucg_xchg* xchg, float* result, void* stream) {
  if (int rc = check_device()) return rc;
  if (!xchg || !result || (nloc && !partials)) return fail(UCG_ERR_ARG, "null argument");
  if (!xchg->opened || xchg->nloc != nloc) return fail(UCG_ERR_ARG, "exchange not opened for this shard");
  if (int rc = xchg_guard(xchg)) return rc;
  int dev = -1;
  UCG_CUDA(cudaGetDevice(&dev));
  if (dev != xchg->device) return fail(UCG_ERR_ARG, "exchange context belongs to another device");
  // one CTA: the stage-2 tail with F = 1 (no ticket); done counters unused
  static unsigned int* scratch_done[64] = {};
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!scratch_done[dev]) UCG_CUDA(cudaMalloc(&scratch_done[dev], 3 * sizeof(unsigned int)));
  }
  FinishArgs f{nullptr, nullptr, nloc, partials, scratch_done[dev], nullptr, result, xchg->world, xchg->rank,
               xchg->part_offset, xchg->p_total, xchg->d_peers, xchg->flags_offset, xchg->d_epoch, xchg->d_err, 0, 1,
               getenv("UCG_XCHG_FLAGS") ? 1 : 0, 0};
  cudaStream_t st = as_stream(stream);
  if (op == UCG_OP_SUM) k_stage2_only<OpSum><<<1, kTreeThreads, 0, st>>>(f);
  else if (op == UCG_OP_MAX) k_stage2_only<OpMax><<<1, kTreeThreads, 0, st>>>(f);
  else return fail(UCG_ERR_ARG, "unknown op");
  UCG_LAUNCHED();
  return UCG_OK;
}

int ucg_tree_reduce_f32(const float* x, uint64_t n, int op, float* out, void* stream) {
  if (int rc = check_device()) return rc;
  if (!out || (n && !x)) return fail(UCG_ERR_ARG, "null argument");
  if (op == UCG_OP_SUM) k_tree<OpSum><<<1, kTreeThreads, 0, as_stream(stream)>>>(x, n, out);
  else if (op == UCG_OP_MAX) k_tree<OpMax><<<1, kTreeThreads, 0, as_stream(stream)>>>(x, n, out);
  else return fail(UCG_ERR_ARG, "unknown op");
  UCG_LAUNCHED();
  return UCG_OK;
}

int ucg_reduce_cl_f32(const float* const* elem_ptrs, uint64_t count, uint64_t len, const uint64_t* part_counts,
                      uint64_t nparts, int op, float* out, void* stream) {
  if (int rc = check_device()) return rc;
  if ((count && !elem_ptrs) || (nparts && !part_counts) || (len && !out)) return fail(UCG_ERR_ARG, "null argument");
  if (op == UCG_OP_SUM)
    return reduce_cl<float, F32SumE>(elem_ptrs, count, len, part_counts, nparts, out, as_stream(stream));
  if (op == UCG_OP_MAX)
    return reduce_cl<float, F32MaxE>(elem_ptrs, count, len, part_counts, nparts, out, as_stream(stream));
  return fail(UCG_ERR_ARG, "unknown op");
}

int ucg_reduce_cl_i64(const int64_t* const* elem_ptrs, uint64_t count, uint64_t len, const uint64_t* part_counts,
                      uint64_t nparts, int64_t* out, void* stream) {
  if (int rc = check_device()) return rc;
  if ((count && !elem_ptrs) || (nparts && !part_counts) || (len && !out)) return fail(UCG_ERR_ARG, "null argument");
  return reduce_cl<int64_t, I64Add>(elem_ptrs, count, len, part_counts, nparts, out, as_stream(stream));
}

}  // extern "C"
