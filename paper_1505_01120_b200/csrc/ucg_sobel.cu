// ucg_sobel.cu — 3x3 Sobel over row bands (workload C4), u8 -> u8.
//
// out(r,c) = min(255, |Gx|+|Gy|) over the band's halo'd input, zero outside
// the image columns (oracle/ucores_oracle.c orc_sobel_band_u8). Separable
// form: with dh(c) = p(c+1)-p(c-1) and sh(c) = p(c-1)+2p(c)+p(c+1) per row,
// Gx = dh(r0)+2dh(r1)+dh(r2) and Gy = sh(r2)-sh(r0).
//
// Data movement: one thread owns 16 consecutive columns (one 128-bit load
// per input row) and walks down a strip of kStrip output rows keeping the
// 3-row window in registers, so each input row is read from HBM once (plus
// 2 halo rows per strip); the left/right neighbour bytes come from the
// adjacent lanes by shuffle. One 128-bit store per output row.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "ucg_common.cuh"

namespace ucg {
namespace {

constexpr int kSobelThreads = 128;
constexpr int kStrip = 32;   // output rows per thread
constexpr int kMaxBands = 512;

struct SobelBands {
  uint64_t in_off[kMaxBands];
  uint64_t out_off[kMaxBands];
  uint64_t rows[kMaxBands];
  uint64_t first_strip[kMaxBands + 1];
  uint32_t nbands;
};

struct RowTerms {
  int dh[16];
  int sh[16];
};

// Load one input row segment (16 px at column c0) and build its dh/sh terms.
__device__ __forceinline__ void load_row(const uint8_t* __restrict__ row, uint64_t width, uint64_t c0, int lane,
                                         bool active, RowTerms& t) {
  uint4 w = make_uint4(0, 0, 0, 0);
  if (active) w = *reinterpret_cast<const uint4*>(row + c0);
  // neighbour bytes: byte 15 of lane-1, byte 0 of lane+1 (edge lanes read directly)
  uint32_t left = __shfl_up_sync(0xffffffffu, w.w, 1) >> 24;
  uint32_t right = __shfl_down_sync(0xffffffffu, w.x, 1) & 0xffu;
  if (lane == 0) left = (active && c0 > 0) ? row[c0 - 1] : 0u;
  if (lane == 31 || !active) right = (active && c0 + 16 < width) ? row[c0 + 16] : 0u;
  // a lane past the row end contributes zeros; the lane before it must see 0 too
  int p[18];
  p[0] = int(left);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 16; ++i) p[i + 1] = int((ws[i >> 2] >> (8 * (i & 3))) & 0xffu);
  p[17] = int(right);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    t.dh[i] = p[i + 2] - p[i];
    t.sh[i] = p[i] + 2 * p[i + 1] + p[i + 2];
  }
}

__global__ void __launch_bounds__(kSobelThreads)
    k_sobel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, const __grid_constant__ SobelBands bands,
            uint64_t width, uint64_t nstrips) {
  const int lane = threadIdx.x & 31;
  const uint64_t lanes_per_row = (width + 15) / 16;
  const uint64_t warps_per_row = (lanes_per_row + 31) / 32;
  const uint64_t nwarps = uint64_t(gridDim.x) * (kSobelThreads / 32);
  const uint64_t total = nstrips * warps_per_row;
  for (uint64_t wi = uint64_t(blockIdx.x) * (kSobelThreads / 32) + (threadIdx.x >> 5); wi < total; wi += nwarps) {
    const uint64_t strip = wi / warps_per_row;
    const uint64_t wcol = wi % warps_per_row;
    uint32_t lo = 0, hi = bands.nbands;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (bands.first_strip[mid] <= strip) lo = mid;
      else hi = mid;
    }
    const uint64_t r0 = (strip - bands.first_strip[lo]) * kStrip;
    const uint64_t nrows = umin(kStrip, bands.rows[lo] - r0);
    const uint8_t* src = in + bands.in_off[lo] + r0 * width;  // input row r0 = halo row above output r0
    uint8_t* dst = out + bands.out_off[lo] + r0 * width;
    const uint64_t c0 = (wcol * 32 + lane) * 16;
    const bool active = c0 < width;
    RowTerms a, b, c;
    load_row(src, width, c0, lane, active, a);
    load_row(src + width, width, c0, lane, active, b);
    for (uint64_t r = 0; r < nrows; ++r) {
      load_row(src + (r + 2) * width, width, c0, lane, active, c);
      uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int gx = a.dh[i] + 2 * b.dh[i] + c.dh[i];
        const int gy = c.sh[i] - a.sh[i];
        const int m = min(255, abs(gx) + abs(gy));
        o[i >> 2] |= uint32_t(m) << (8 * (i & 3));
      }
      if (active) st_stream(reinterpret_cast<float4*>(dst + r * width + c0),
                            make_float4(__uint_as_float(o[0]), __uint_as_float(o[1]), __uint_as_float(o[2]),
                                        __uint_as_float(o[3])));
      a = b;
      b = c;
    }
  }
}

// Generic path for widths that are not a multiple of 16 (rows not 16-byte
// aligned): one thread per output pixel, nine byte loads.
__global__ void __launch_bounds__(256)
    k_sobel_generic(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, const __grid_constant__ SobelBands bands,
                    uint64_t width, uint64_t npix) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < npix; i += stride) {
    // first_strip holds cumulative pixel counts in this mode
    uint32_t lo = 0, hi = bands.nbands;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (bands.first_strip[mid] <= i) lo = mid;
      else hi = mid;
    }
    const uint64_t k = i - bands.first_strip[lo];
    const uint64_t r = k / width;
    const int64_t c = int64_t(k % width);
    const uint8_t* src = in + bands.in_off[lo];
    auto px = [&](uint64_t rr, int64_t cc) -> int {
      return (cc < 0 || uint64_t(cc) >= width) ? 0 : int(src[rr * width + uint64_t(cc)]);
    };
    const int gx = (px(r, c + 1) - px(r, c - 1)) + 2 * (px(r + 1, c + 1) - px(r + 1, c - 1)) +
                   (px(r + 2, c + 1) - px(r + 2, c - 1));
    const int gy = (px(r + 2, c - 1) + 2 * px(r + 2, c) + px(r + 2, c + 1)) -
                   (px(r, c - 1) + 2 * px(r, c) + px(r, c + 1));
    out[bands.out_off[lo] + k] = uint8_t(min(255, abs(gx) + abs(gy)));
  }
}

}  // namespace
}  // namespace ucg

using namespace ucg;

extern "C" {

int ucg_sobel_bands_u8(const uint8_t* in, const uint64_t* in_off, uint8_t* out, const uint64_t* out_off,
                       const uint64_t* rows, uint64_t nbands, uint64_t width, void* stream) {
  if (int rc = check_device()) return rc;
  if (!nbands || !width) return UCG_OK;
  if (!in || !out || !in_off || !out_off || !rows) return fail(UCG_ERR_ARG, "null argument");
  cudaStream_t st = as_stream(stream);
  bool vec = width % 16 == 0 && aligned16(in) && aligned16(out);
  for (uint64_t i = 0; i < nbands && vec; ++i) vec = in_off[i] % 16 == 0 && out_off[i] % 16 == 0;
  for (uint64_t b0 = 0; b0 < nbands; b0 += kMaxBands) {
    const uint32_t nb = uint32_t(std::min<uint64_t>(kMaxBands, nbands - b0));
    SobelBands p;
    p.nbands = nb;
    p.first_strip[0] = 0;
    if (!vec) {
      for (uint32_t i = 0; i < nb; ++i) {
        p.in_off[i] = in_off[b0 + i];
        p.out_off[i] = out_off[b0 + i];
        p.rows[i] = rows[b0 + i];
        p.first_strip[i + 1] = p.first_strip[i] + rows[b0 + i] * width;
      }
      const uint64_t npix = p.first_strip[nb];
      if (!npix) continue;
      const unsigned grid = unsigned(std::min<uint64_t>((npix + 255) / 256, uint64_t(sm_count()) * 8));
      k_sobel_generic<<<grid, 256, 0, st>>>(in, out, p, width, npix);
      UCG_LAUNCHED();
      continue;
    }
    for (uint32_t i = 0; i < nb; ++i) {
      p.in_off[i] = in_off[b0 + i];
      p.out_off[i] = out_off[b0 + i];
      p.rows[i] = rows[b0 + i];
      p.first_strip[i + 1] = p.first_strip[i] + (rows[b0 + i] + kStrip - 1) / kStrip;
    }
    const uint64_t nstrips = p.first_strip[nb];
    if (!nstrips) continue;
    const uint64_t warps_per_row = ((width + 15) / 16 + 31) / 32;
    const uint64_t warps = nstrips * warps_per_row;
    const unsigned grid =
        unsigned(std::min<uint64_t>((warps + kSobelThreads / 32 - 1) / (kSobelThreads / 32), uint64_t(sm_count()) * 16));
    k_sobel<<<grid, kSobelThreads, 0, st>>>(in, out, p, width, nstrips);
    UCG_LAUNCHED();
  }
  return UCG_OK;
}

int ucg_sobel_band_u8(const uint8_t* in, uint8_t* out, uint64_t rows_out, uint64_t width, void* stream) {
  const uint64_t zero = 0;
  return ucg_sobel_bands_u8(in, &zero, out, &zero, &rows_out, 1, width, stream);
}

}  // extern "C"
