// ucg_text.cu — WordCount word-start flags.
//
// flags[gid] = 1 iff byte[gid] is a word character and (gid == 0 or
// byte[gid-1] is a delimiter); delimiters are ASCII space, tab, LF, CR
// (ucores/dataset.hpp:87-89). One thread owns 16 bytes (one 128-bit load and
// store), the byte before its span comes from the previous thread by shuffle
// (lane 0 loads it). 2 B/byte of HBM traffic.
#include <cuda_runtime.h>

#include <algorithm>

#include "ucg_common.cuh"

namespace ucg {
namespace {

// 1 in each byte lane that is a delimiter, 0 otherwise
__device__ __forceinline__ uint32_t delim_mask(uint32_t w) {
  const uint32_t sp = __vcmpeq4(w, 0x20202020u), tb = __vcmpeq4(w, 0x09090909u);
  const uint32_t lf = __vcmpeq4(w, 0x0a0a0a0au), cr = __vcmpeq4(w, 0x0d0d0d0du);
  return (sp | tb | lf | cr) & 0x01010101u;
}

__global__ void __launch_bounds__(256) k_word_flags(const uint8_t* __restrict__ in, uint8_t* __restrict__ flags,
                                                    uint64_t n16) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
    const uint4 w = __ldcs(reinterpret_cast<const uint4*>(in) + i);
    // previous byte: 1 = "before the chunk" counts as a delimiter (gid == 0 rule)
    uint32_t prev_delim = 1;
    if (i > 0) prev_delim = delim_mask(in[16 * i - 1]) & 1u;
    const uint32_t d[4] = {delim_mask(w.x), delim_mask(w.y), delim_mask(w.z), delim_mask(w.w)};
    uint32_t f[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // delimiter flags of the byte before each byte of word k
      const uint32_t before = (d[k] << 8) | (k ? d[k - 1] >> 24 : prev_delim);
      f[k] = (d[k] ^ 0x01010101u) & before;  // word char preceded by a delimiter
    }
    __stcs(reinterpret_cast<uint4*>(flags) + i, make_uint4(f[0], f[1], f[2], f[3]));
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
    const unsigned grid = unsigned(std::min<uint64_t>((n16 + 255) / 256, uint64_t(sm_count()) * 8));
    k_word_flags<<<grid, 256, 0, st>>>(bytes, flags, n16);
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
