// ucg_text.cu — WordCount word-start flags.
//
// flags[gid] = 1 iff byte[gid] is a word character and (gid == 0 or
// byte[gid-1] is a delimiter); delimiters are ASCII space, tab, LF, CR
// (ucores/dataset.hpp:87-89). Lanes own 16-byte words (128-bit loads and
// stores, 4 in flight per lane); the byte before a word comes from the
// neighbouring lane by shuffle. 2 B/byte of HBM traffic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "ucg_common.cuh"

namespace ucg {
namespace {

// 1 in each byte lane that is a delimiter, 0 otherwise. Exact SWAR zero-byte
// test per delimiter c (no carries cross bytes: (x & 0x7f) + 0x7f <= 0xfe):
// byte b == c  iff  the high bit of ~(((b ^ c) & 0x7f) + 0x7f | (b ^ c)) is
// set. ~4 integer ops per delimiter instead of an emulated __vcmpeq4.
template <uint32_t C>
__device__ __forceinline__ uint32_t eq_byte_hi(uint32_t w, uint32_t wl) {
  const uint32_t t = (wl ^ (C & 0x7f7f7f7fu)) + 0x7f7f7f7fu;
  return ~(t | (w ^ C)) & 0x80808080u;
}
__device__ __forceinline__ uint32_t delim_mask(uint32_t w) {
  const uint32_t wl = w & 0x7f7f7f7fu;
  const uint32_t hi = eq_byte_hi<0x20202020u>(w, wl) | eq_byte_hi<0x09090909u>(w, wl) |
                      eq_byte_hi<0x0a0a0a0au>(w, wl) | eq_byte_hi<0x0d0d0d0du>(w, wl);
  return hi >> 7;
}

// flags of one 16-byte word given its delimiter masks and the delimiter flag
// (0/1) of the byte before it
__device__ __forceinline__ uint4 word_flags16(const uint4& w, uint32_t prev_delim) {
  const uint32_t d[4] = {delim_mask(w.x), delim_mask(w.y), delim_mask(w.z), delim_mask(w.w)};
  uint32_t f[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    // delimiter flags of the byte before each byte of word k
    const uint32_t before = (d[k] << 8) | (k ? d[k - 1] >> 24 : prev_delim);
    f[k] = (d[k] ^ 0x01010101u) & before;  // word char preceded by a delimiter
  }
  return make_uint4(f[0], f[1], f[2], f[3]);
}

// A warp walks blocks of kWU x 512 contiguous bytes (grid-stride) and loads
// the next block while it finishes the current one: lane l holds the 16-byte
// words (u*32 + l), u < kWU. The byte before lane
// l's word is the last byte of lane l-1's word (shuffle); lane 0 takes it
// from lane 31 of the previous row, and a block's first byte looks back with
// one scalar load.
template <int kWU>
__global__ void __launch_bounds__(256) k_word_flags(const uint8_t* __restrict__ in, uint8_t* __restrict__ flags,
                                                    uint64_t n16) {
  const int lane = threadIdx.x & 31;
  const uint64_t nblk = n16 / (32 * kWU);
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint4* src = reinterpret_cast<const uint4*>(in);
  uint4* dst = reinterpret_cast<uint4*>(flags);
  uint64_t b = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  uint4 w[kWU];
  if (b < nblk) {
#pragma unroll
    for (int u = 0; u < kWU; ++u) w[u] = __ldcs(src + b * 32 * kWU + u * 32 + lane);
  }
  while (b < nblk) {
    const uint64_t nb = b + nwarps;
    uint4 nx[kWU];
    if (nb < nblk) {
#pragma unroll
      for (int u = 0; u < kWU; ++u) nx[u] = __ldcs(src + nb * 32 * kWU + u * 32 + lane);
    }
    const uint64_t w0 = b * 32 * kWU;
    // previous byte's delimiter flag; "before the text" counts as a delimiter
    uint32_t carry = 1;
    if (lane == 0 && w0 > 0) carry = delim_mask(in[16 * w0 - 1]) & 1u;
#pragma unroll
    for (int u = 0; u < kWU; ++u) {
      const uint32_t last = delim_mask(w[u].w) >> 24;  // this lane's last byte
      const uint32_t up = __shfl_up_sync(0xffffffffu, last, 1);
      const uint32_t prev = lane ? up : carry;
      carry = __shfl_sync(0xffffffffu, last, 31);     // for lane 0 of the next row
      __stcs(dst + w0 + u * 32 + lane, word_flags16(w[u], prev));
    }
#pragma unroll
    for (int u = 0; u < kWU; ++u) w[u] = nx[u];
    b = nb;
  }
  // words past the last full block: one per thread
  const uint64_t tail0 = nblk * 32 * kWU;
  for (uint64_t i = tail0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 v = __ldcs(src + i);
    const uint32_t prev = i > 0 ? (delim_mask(in[16 * i - 1]) & 1u) : 1u;
    __stcs(dst + i, word_flags16(v, prev));
  }
}

// Claimed variant: a warp claims units of kClaim consecutive blocks (16 KB)
// from a per-launch counter and walks them with the same prefetch.
template <int kWU, int kClaim>
__global__ void __launch_bounds__(256) k_word_flags_claim(const uint8_t* __restrict__ in, uint8_t* __restrict__ flags,
                                                          uint64_t n16, unsigned long long* __restrict__ ctr) {
  const int lane = threadIdx.x & 31;
  const uint64_t nblk = n16 / (32 * kWU);
  const uint64_t nunits = (nblk + kClaim - 1) / kClaim;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint4* src = reinterpret_cast<const uint4*>(in);
  uint4* dst = reinterpret_cast<uint4*>(flags);
  uint64_t unit = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  while (unit < nunits) {
    unsigned long long claim = 0;
    if (lane == 0) claim = atomicAdd(ctr, 1ull);
    const uint64_t b0 = unit * kClaim, b1 = b0 + kClaim < nblk ? b0 + kClaim : nblk;
    uint4 w[kWU];
#pragma unroll
    for (int u = 0; u < kWU; ++u) w[u] = __ldcs(src + b0 * 32 * kWU + u * 32 + lane);
    for (uint64_t b = b0; b < b1; ++b) {
      uint4 nx[kWU];
      if (b + 1 < b1) {
#pragma unroll
        for (int u = 0; u < kWU; ++u) nx[u] = __ldcs(src + (b + 1) * 32 * kWU + u * 32 + lane);
      }
      const uint64_t w0 = b * 32 * kWU;
      uint32_t carry = 1;
      if (lane == 0 && w0 > 0) carry = delim_mask(in[16 * w0 - 1]) & 1u;
#pragma unroll
      for (int u = 0; u < kWU; ++u) {
        const uint32_t last = delim_mask(w[u].w) >> 24;
        const uint32_t up = __shfl_up_sync(0xffffffffu, last, 1);
        const uint32_t prev = lane ? up : carry;
        carry = __shfl_sync(0xffffffffu, last, 31);
        __stcs(dst + w0 + u * 32 + lane, word_flags16(w[u], prev));
      }
#pragma unroll
      for (int u = 0; u < kWU; ++u) w[u] = nx[u];
    }
    unit = nwarps + __shfl_sync(0xffffffffu, claim, 0);
  }
  const uint64_t tail0 = nblk * 32 * kWU;
  for (uint64_t i = tail0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 v = __ldcs(src + i);
    const uint32_t prev = i > 0 ? (delim_mask(in[16 * i - 1]) & 1u) : 1u;
    __stcs(dst + i, word_flags16(v, prev));
  }
  // ctr[1] counts CTAs out: the last one returns the claim pair to zero for
  // its next user (claim_pair_selfreset: no memset launch per call)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1ull) == gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
}

__global__ void __launch_bounds__(256) k_word_flags_bytes(const uint8_t* __restrict__ in, uint8_t* __restrict__ flags,
                                                          uint64_t from, uint64_t n) {
  auto is_delim = [](uint8_t b) { return b == ' ' || b == '\t' || b == '\n' || b == '\r'; };
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = from + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    flags[i] = uint8_t(!is_delim(in[i]) && (i == 0 || is_delim(in[i - 1])));
}

}  // namespace
}  // namespace ucg

using namespace ucg;

extern "C" int ucg_word_start_flags(const uint8_t* bytes, uint64_t n, uint8_t* flags, void* stream) {
  if (int rc = check_device()) return rc;
  if (!n) return UCG_OK;
  if (!bytes || !flags) return fail(UCG_ERR_ARG, "null argument");
  cudaStream_t st = as_stream(stream);
  uint64_t done = 0;
  if (aligned16(bytes) && aligned16(flags) && n >= 16) {
    const uint64_t n16 = n / 16;
    // default: claimed 16 KB units (round 1: 1 GiB in 0.394 ms, 0.85 of
    // HBM); UCG_WC_VARIANT=1: grid-stride blocks (0.406 ms)
    static const int variant = [] {
      const char* e = getenv("UCG_WC_VARIANT");
      return e ? atoi(e) : 0;
    }();
    const uint64_t warps = std::max<uint64_t>(1, n16 / (32 * 4));
    if (variant == 1) {
      const unsigned grid = unsigned(std::min<uint64_t>((warps + 7) / 8, uint64_t(sm_count()) * 8));
      k_word_flags<4><<<grid, 256, 0, st>>>(bytes, flags, n16);
    } else {
      unsigned long long* ctr = claim_pair_selfreset();  // zero at launch, re-zeroed by the last CTA
      if (!ctr) return fail(UCG_ERR_CUDA, "word flags: counter allocation failed");
      // 16-byte words per lane per block: 8 (default; 4 KB blocks, 4 per
      // claim: twice the bytes in flight of 4 — 1 GiB in 333.5 vs 346.9 us,
      // 0.985 vs 0.946 of the copy peak, same box) or 4 (UCG_WC_WU=4, A/B)
      static const int wu = [] {
        const char* e = getenv("UCG_WC_WU");
        return e && atoi(e) == 4 ? 4 : 8;
      }();
      const unsigned grid = unsigned(std::min<uint64_t>((warps / 8 + 7) / 8 + 1, uint64_t(sm_count()) * 8));
      if (wu == 8) k_word_flags_claim<8, 4><<<grid, 256, 0, st>>>(bytes, flags, n16, ctr);
      else k_word_flags_claim<4, 8><<<grid, 256, 0, st>>>(bytes, flags, n16, ctr);
    }
    UCG_LAUNCHED();
    done = n16 * 16;
  }
  if (done < n) {
    const unsigned grid = unsigned(std::min<uint64_t>((n - done + 255) / 256, uint64_t(sm_count()) * 8));
    k_word_flags_bytes<<<grid, 256, 0, st>>>(bytes, flags, done, n);
    UCG_LAUNCHED();
  }
  return UCG_OK;
}
