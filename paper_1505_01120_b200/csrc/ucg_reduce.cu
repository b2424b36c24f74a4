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
// Data movement: one warp owns a work item of 2^14 floats of one segment and
// streams it in 1024-float chunks (8 coalesced LDG.128 per lane, 16 KB per
// chunk per warp in flight). A chunk is reduced with a value-halving
// butterfly: 12 shuffles per 1024 floats instead of 40.
#include <cuda_runtime.h>

#include <algorithm>
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

// Reduce one 1024-float chunk at `x` (16B aligned). Lane l holds floats
// [128u + 4l, 128u + 4l + 4) of sub-block u (u = 0..7). kGuard: only the
// first `valid` floats exist (the rest are the identity). kMap: the chunk is
// first mapped through y = fl(fl(a*x)+b) and the mapped values are stored to
// y before being reduced. Returns the chunk's tree value in every lane.
template <class Op, bool kMap, bool kGuard>
__device__ __forceinline__ float chunk1024(const float* __restrict__ x, float* __restrict__ y,
                                           int64_t valid, float a, float b, int lane) {
  float s[8];
  float4 v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
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
#pragma unroll
  for (int u = 0; u < 8; ++u) {
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
  // value-halving butterfly over lane bits 0,1,2 (8-, 16-, 32-float nodes)
  const bool b0 = lane & 1, b1 = lane & 2, b2 = lane & 4;
  float t[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float keep = b0 ? s[j + 4] : s[j];
    const float send = b0 ? s[j] : s[j + 4];
    t[j] = lr<Op>(keep, __shfl_xor_sync(kFull, send, 1), !b0);
  }
  float q[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const float keep = b1 ? t[j + 2] : t[j];
    const float send = b1 ? t[j] : t[j + 2];
    q[j] = lr<Op>(keep, __shfl_xor_sync(kFull, send, 2), !b1);
  }
  float r;
  {
    const float keep = b2 ? q[1] : q[0];
    const float send = b2 ? q[0] : q[1];
    r = lr<Op>(keep, __shfl_xor_sync(kFull, send, 4), !b2);
  }
  // lane now holds sub-block (4*b0 + 2*b1 + b2) over its 8-lane group; finish
  // the 64- and 128-float nodes across lane bits 3, 4.
  r = lr<Op>(r, __shfl_xor_sync(kFull, r, 8), !(lane & 8));
  r = lr<Op>(r, __shfl_xor_sync(kFull, r, 16), !(lane & 16));
  // tree over the 8 sub-blocks: (u, u^1) differ in lane bit 2, then bit 1, then bit 0
  r = lr<Op>(r, __shfl_xor_sync(kFull, r, 4), !b2);
  r = lr<Op>(r, __shfl_xor_sync(kFull, r, 2), !b1);
  r = lr<Op>(r, __shfl_xor_sync(kFull, r, 1), !b0);
  return r;
}

// Reduce one work item: `valid` floats at x (<= kItemFloats), as 16 chunks
// combined by a binary-counter stack (aligned power-of-two subtrees).
template <class Op, bool kMap>
__device__ __forceinline__ float work_item(const float* __restrict__ x, float* __restrict__ y,
                                           int64_t valid, float a, float b, int lane) {
  constexpr int kChunks = int(kItemFloats / 1024);
  constexpr int kDepth = kItemLog2 - 10;
  float stk[kDepth];
#pragma unroll
  for (int j = 0; j < kDepth; ++j) stk[j] = Op::identity();
  float v = Op::identity();
  const bool full = valid >= int64_t(kItemFloats);
#pragma unroll 1
  for (int c = 0; c < kChunks; ++c) {
    const int64_t rem = valid - int64_t(c) * 1024;
    if (full || rem >= 1024) {
      v = chunk1024<Op, kMap, false>(x + c * 1024, y + c * 1024, 1024, a, b, lane);
    } else if (rem > 0) {
      v = chunk1024<Op, kMap, true>(x + c * 1024, y + c * 1024, rem, a, b, lane);
    } else {
      v = Op::identity();
    }
#pragma unroll
    for (int j = 0; j < kDepth; ++j) {
      if (c & (1 << j)) {
        v = Op::apply(stk[j], v);
      } else {
        stk[j] = v;
        break;
      }
    }
  }
  return v;  // c = kChunks-1 has all bits set: v is the root
}

// Pass 1: one warp per work item (grid-stride over items).
template <class Op, bool kMap>
__global__ void __launch_bounds__(kWarps * 32)
    k_segment_pass1(const float* __restrict__ x, float* __restrict__ y, const uint64_t* __restrict__ begin,
                    const uint64_t* __restrict__ len, const uint64_t* __restrict__ first_item,
                    const uint32_t* __restrict__ item_seg, uint64_t nitems, float a, float b,
                    float* __restrict__ partial) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = uint64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = uint64_t(gridDim.x) * kWarps;
  for (uint64_t item = warp; item < nitems; item += nwarps) {
    const uint32_t s = item_seg[item];
    const uint64_t blk = item - first_item[s];
    const uint64_t off = begin[s] + (blk << kItemLog2);
    const int64_t valid = int64_t(umin(kItemFloats, len[s] - (blk << kItemLog2)));
    const float r = work_item<Op, kMap>(x + off, kMap ? y + off : nullptr, valid, a, b, lane);
    if (lane == 0) partial[item] = r;
  }
}

// Tree over n values in global memory by ONE CTA (blockDim 256), padded to a
// power of two with the identity. Values are consumed in aligned blocks of
// 2048 whose roots are merged with a binary-counter stack.
constexpr int kTreeThreads = 256;
constexpr int kTreeBlock = 2048;

template <class Op>
__device__ float cta_tree(const float* __restrict__ vals, uint64_t n, float* sm /*kTreeBlock*/,
                          float* stk /*64*/) {
  const int tid = threadIdx.x;
  const uint64_t nblocks = (n + kTreeBlock - 1) / kTreeBlock;
  // one block of 2048 is the whole tree when n <= 2048 (padded size = pow2 >= n)
  float root = Op::identity();
  for (uint64_t bi = 0; bi < nblocks; ++bi) {
    const uint64_t base = bi * kTreeBlock;
    const uint64_t cnt = umin(kTreeBlock, n - base);
    // a partial block padded to any power of two >= cnt has the same root
    int size = 1;
    while (uint64_t(size) < cnt) size <<= 1;
    for (int i = tid; i < size; i += kTreeThreads)
      sm[i] = uint64_t(i) < cnt ? vals[base + i] : Op::identity();
    __syncthreads();
    for (int w = size / 2; w >= 1; w >>= 1) {
      for (int i = tid; i < w; i += kTreeThreads) sm[i] = Op::apply(sm[2 * i], sm[2 * i + 1]);
      __syncthreads();
    }
    if (tid == 0) {
      float v = sm[0];
      int j = 0;
      // binary-counter merge of this block (index bi) into the stack
      while ((bi >> j) & 1) {
        v = Op::apply(stk[j], v);
        ++j;
      }
      stk[j] = v;
    }
    __syncthreads();
  }
  if (tid == 0 && nblocks) {
    // fold the remaining stack right to left: smaller (right) subtrees first
    bool have = false;
    float acc = Op::identity();
    for (int j = 0; j < 64; ++j) {
      if ((nblocks >> j) & 1) {
        acc = have ? Op::apply(stk[j], acc) : stk[j];
        have = true;
      }
    }
    root = acc;
  }
  return root;  // valid in thread 0
}

// Pass 2: one CTA per segment; tree over the segment's work-item values.
template <class Op>
__global__ void __launch_bounds__(kTreeThreads)
    k_segment_pass2(const float* __restrict__ partial, const uint64_t* __restrict__ first_item,
                    float* __restrict__ out) {
  __shared__ float sm[kTreeBlock];
  __shared__ float stk[64];
  const uint64_t s = blockIdx.x;
  const uint64_t f = first_item[s], n = first_item[s + 1] - f;
  if (n == 0) {
    if (threadIdx.x == 0) out[s] = Op::empty();
    return;
  }
  const float r = cta_tree<Op>(partial + f, n, sm, stk);
  if (threadIdx.x == 0) out[s] = r;
}

template <class Op>
__global__ void __launch_bounds__(kTreeThreads) k_tree(const float* __restrict__ x, uint64_t n, float* __restrict__ out) {
  __shared__ float sm[kTreeBlock];
  __shared__ float stk[64];
  if (n == 0) {
    if (threadIdx.x == 0) out[0] = Op::empty();
    return;
  }
  const float r = cta_tree<Op>(x, n, sm, stk);
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

constexpr int kMaxParts = 4096;  // per launch (host splits larger trees)

// One thread per lane j. part_first[p]..part_first[p+1]: element range of the
// p-th NON-EMPTY partition (nonempty entries). Stage 1 folds left to right,
// stage 2 merges partials with a binary-counter stack (aligned subtrees),
// then folds the stack right to left — the pairing tree with promotion.
template <class T, class Op>
__global__ void __launch_bounds__(128) k_reduce_cl(const T* const* __restrict__ elems, const uint64_t* __restrict__ part_first,
                                                   uint64_t nonempty, uint64_t len, T* __restrict__ out) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= len) return;
  T stk[13];  // nonempty <= 4096 -> depth <= 12
  uint64_t k = 0;
  for (; k < nonempty; ++k) {
    uint64_t e = part_first[k];
    T acc = elems[e][j];
    for (++e; e < part_first[k + 1]; ++e) acc = Op::apply(acc, elems[e][j]);
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
  for (int lvl = 0; lvl < 13; ++lvl) {
    if ((nonempty >> lvl) & 1) {
      acc = have ? Op::apply(stk[lvl], acc) : stk[lvl];
      have = true;
    }
  }
  out[j] = acc;
}

template <class Op>
int segment_reduce(const float* x, float* y, const ucg_segtab* t, float a, float b, float* scratch, float* out,
                   cudaStream_t st) {
  if (t->nitems) {
    const uint64_t want = (t->nitems + kWarps - 1) / kWarps;
    const unsigned grid = unsigned(std::min<uint64_t>(want, uint64_t(sm_count()) * 4));
    if (y)
      k_segment_pass1<Op, true><<<grid, kWarps * 32, 0, st>>>(x, y, t->d_begin, t->d_len, t->d_first_item,
                                                             t->d_item_seg, t->nitems, a, b, scratch);
    else
      k_segment_pass1<Op, false><<<grid, kWarps * 32, 0, st>>>(x, y, t->d_begin, t->d_len, t->d_first_item,
                                                              t->d_item_seg, t->nitems, a, b, scratch);
    UCG_LAUNCHED();
  }
  if (t->nseg) {
    k_segment_pass2<Op><<<unsigned(t->nseg), kTreeThreads, 0, st>>>(scratch, t->d_first_item, out);
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
  if (nonempty > kMaxParts) return fail(UCG_ERR_ARG, "more than 4096 non-empty partitions");
  if (len == 0) return UCG_OK;
  uint64_t* d_first = nullptr;
  UCG_CUDA(cudaMallocAsync(&d_first, first.size() * 8, st));
  UCG_CUDA(cudaMemcpyAsync(d_first, first.data(), first.size() * 8, cudaMemcpyHostToDevice, st));
  const unsigned grid = unsigned((len + 127) / 128);
  k_reduce_cl<T, Op><<<grid, 128, 0, st>>>(elem_ptrs, d_first, nonempty, len, out);
  UCG_LAUNCHED();
  // (the pageable-source copy above is staged before cudaMemcpyAsync returns)
  UCG_CUDA(cudaFreeAsync(d_first, st));
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
  if (op == UCG_OP_SUM) return segment_reduce<OpSum>(x, nullptr, t, 0.f, 0.f, scratch, out, as_stream(stream));
  if (op == UCG_OP_MAX) return segment_reduce<OpMax>(x, nullptr, t, 0.f, 0.f, scratch, out, as_stream(stream));
  return fail(UCG_ERR_ARG, "unknown op");
}

int ucg_map_affine_segment_reduce_f32(const float* x, float* y, const ucg_segtab* t, float a, float b, int op,
                                      float* scratch, float* out, void* stream) {
  if (int rc = check_device()) return rc;
  if (!t) return fail(UCG_ERR_ARG, "segment table is null");
  if (t->nseg && (!out || (t->nitems && (!x || !y || !scratch)))) return fail(UCG_ERR_ARG, "null argument");
  if (t->nitems && (!aligned16(x) || !aligned16(y))) return fail(UCG_ERR_ARG, "x/y must be 16-byte aligned");
  if (op == UCG_OP_SUM) return segment_reduce<OpSum>(x, y, t, a, b, scratch, out, as_stream(stream));
  if (op == UCG_OP_MAX) return segment_reduce<OpMax>(x, y, t, a, b, scratch, out, as_stream(stream));
  return fail(UCG_ERR_ARG, "unknown op");
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
