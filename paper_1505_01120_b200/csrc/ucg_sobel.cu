// ucg_sobel.cu — 3x3 Sobel over row bands (workload C4), u8 -> u8.
//
// out(r,c) = min(255, |Gx|+|Gy|) over the band's halo'd input, zero outside
// the image columns (oracle/ucores_oracle.c orc_sobel_band_u8). Separable
// form: with dh(c) = p(c+1)-p(c-1) and sh(c) = p(c-1)+2p(c)+p(c+1) per row,
// Gx = dh(r0)+2dh(r1)+dh(r2) and Gy = sh(r2)-sh(r0). Arithmetic is packed two
// pixels per 32-bit register (biased 16-bit halves, byte permutes to build
// the neighbour vectors, sm_100 packed 16x2 min/max), ~7 integer ops/pixel.
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

// Row terms for 16 pixels as 8 packed pairs (pixel 2i in the low 16 bits,
// pixel 2i+1 in the high 16 bits), biased so no half ever borrows:
//   dh = p(c+1) - p(c-1) + 256   in [1, 511]
//   sh = p(c-1) + 2p(c) + p(c+1) in [0, 1020]
struct RowTerms {
  uint32_t dh[8];
  uint32_t sh[8];
};

// A fetched input row segment: the thread's 16 bytes plus, for the warp's
// edge lanes, the neighbour byte outside the warp's 512-byte span.
struct RawRow {
  uint4 w;
  uint32_t edge;
};

__device__ __forceinline__ RawRow fetch_row(const uint8_t* __restrict__ row, uint64_t width, uint64_t c0, int lane,
                                            bool active, bool exists) {
  RawRow q{make_uint4(0, 0, 0, 0), 0u};
  if (exists && active) q.w = __ldcs(reinterpret_cast<const uint4*>(row + c0));
  if (exists && active) {
    if (lane == 0 && c0 > 0) q.edge = row[c0 - 1];
    if (lane == 31 && c0 + 16 < width) q.edge = row[c0 + 16];
  }
  return q;
}

// Build the row terms from a fetched row (neighbour bytes by shuffle).
__device__ __forceinline__ void make_terms(const RawRow& q, int lane, RowTerms& t) {
  uint32_t left = __shfl_up_sync(0xffffffffu, q.w.w, 1) >> 24;
  uint32_t right = __shfl_down_sync(0xffffffffu, q.w.x, 1) & 0xffu;
  // a lane past the row end holds zeros, which is the out-of-image value
  if (lane == 0) left = q.edge;
  if (lane == 31) right = q.edge;
  const uint32_t ws[6] = {left << 24, q.w.x, q.w.y, q.w.z, q.w.w, right};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t cur = ws[k + 1];
    const uint32_t sl = __byte_perm(ws[k], cur, 0x6543);      // p(4k-1) .. p(4k+2)
    const uint32_t sr = __byte_perm(cur, ws[k + 2], 0x4321);  // p(4k+1) .. p(4k+4)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t sel = h ? 0x4342u : 0x4140u;  // bytes (2h, 2h+1) -> 16-bit halves
      const uint32_t E = __byte_perm(cur, 0, sel);
      const uint32_t L = __byte_perm(sl, 0, sel);
      const uint32_t R = __byte_perm(sr, 0, sel);
      t.dh[2 * k + h] = R - L + 0x01000100u;
      t.sh[2 * k + h] = L + R + (E << 1);
    }
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
    // output row r from input rows (top, mid, bottom) = (r, r+1, r+2)
    auto emit = [&](uint64_t r, const RowTerms& a, const RowTerms& b, const RowTerms& c) {
      uint32_t o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        // per half: gx' = Gx + 1024, gy' = Gy + 1024, both in [4, 2044]
        const uint32_t gx = a.dh[i] + c.dh[i] + (b.dh[i] << 1);
        const uint32_t gy = c.sh[i] - a.sh[i] + 0x04000400u;
        // |G| + 1024 = max(g', 2048 - g') per half
        const uint32_t ax = __vmaxu2(gx, 0x08000800u - gx);
        const uint32_t ay = __vmaxu2(gy, 0x08000800u - gy);
        // min(|Gx|+|Gy|, 255) + 2048 per half; its low byte is the output pixel
        o[i] = __vminu2(__vadd2(ax, ay), 0x08FF08FFu);
      }
      if (active) {
        const uint32_t q0 = __byte_perm(o[0], o[1], 0x6420), q1 = __byte_perm(o[2], o[3], 0x6420);
        const uint32_t q2 = __byte_perm(o[4], o[5], 0x6420), q3 = __byte_perm(o[6], o[7], 0x6420);
        st_stream(reinterpret_cast<float4*>(dst + r * width + c0),
                  make_float4(__uint_as_float(q0), __uint_as_float(q1), __uint_as_float(q2), __uint_as_float(q3)));
      }
    };
    // 3-row register window rotated by unrolling (no copies); the raw loads of
    // the next 3 input rows are issued before the current 3 are computed, so
    // every warp keeps 3 x 512 B of loads in flight.
    const uint64_t last_in = nrows + 1;  // input rows 0..nrows+1 exist for this strip
    auto fetch = [&](uint64_t i) { return fetch_row(src + i * width, width, c0, lane, active, i <= last_in); };
    RowTerms t0, t1, t2;
    make_terms(fetch(0), lane, t0);
    make_terms(fetch(1), lane, t1);
    RawRow p0 = fetch(2), p1 = fetch(3), p2 = fetch(4);
    uint64_t r = 0;
    for (; r + 3 <= nrows; r += 3) {
      const RawRow n0 = fetch(r + 5), n1 = fetch(r + 6), n2 = fetch(r + 7);
      make_terms(p0, lane, t2);
      emit(r, t0, t1, t2);
      make_terms(p1, lane, t0);
      emit(r + 1, t1, t2, t0);
      make_terms(p2, lane, t1);
      emit(r + 2, t2, t0, t1);
      p0 = n0;
      p1 = n1;
      p2 = n2;
    }
    if (r < nrows) {
      make_terms(p0, lane, t2);
      emit(r, t0, t1, t2);
      if (r + 1 < nrows) {
        make_terms(p1, lane, t0);
        emit(r + 1, t1, t2, t0);
      }
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
