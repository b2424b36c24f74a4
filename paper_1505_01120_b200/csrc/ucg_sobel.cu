// ucg_sobel.cu — 3x3 Sobel over row bands (workload C4), u8 -> u8.
//
// out(r,c) = min(255, |Gx|+|Gy|) over the band's halo'd input, zero outside
// the image columns (oracle/ucores_oracle.c orc_sobel_band_u8). Separable
// form: with dh(c) = p(c+1)-p(c-1) and sh(c) = p(c-1)+2p(c)+p(c+1) per row,
// Gx = dh(r0)+2dh(r1)+dh(r2) and Gy = sh(r2)-sh(r0). Arithmetic is packed two
// pixels per 32-bit register (16-bit halves, byte permutes build the
// neighbour vectors); by default the halves are read as fp16 subnormals and
// added exactly with HADD2/HFMA2 (see word_terms / out_pair below).
//
// Three kernels: the default TMA-tiled persistent kernel (k_sobel_tma, tiles
// claimed from a self-resetting counter pair), a row-streaming TMA kernel
// (k_sobel_rows, A/B) and a register-streaming kernel without TMA (k_sobel,
// below: one thread owns 16 consecutive columns and walks down a strip of
// kStrip output rows, the neighbour bytes by shuffle; A/B).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
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

// ---- TMA-tiled path -----------------------------------------------------------
// A CTA tile is 256 output columns x 64 output rows of one band. TMA copies the
// 66 x 256 input rows plus 16-byte side boxes at x-16 and x+256 into shared
// memory; side boxes that fall outside the image are zero-filled by the TMA
// unit, which is exactly the zero-outside-columns rule. Persistent CTAs double
// buffer: the next tile is requested as soon as a buffer is free. Each
// of the 128 threads owns 16 columns x 8 output rows (10 input rows, 3-row
// window in registers), reads its bytes with LDS.128 and the neighbour bytes
// from the side columns, and stores 16 output bytes per row.
constexpr int kTW = 256, kTH = 64, kTIn = kTH + 2;
constexpr uint32_t kCenterBytes = kTW * kTIn;          // 16896
constexpr uint32_t kSideBytes = 16 * kTIn;             // 1056
constexpr uint32_t kSideStride = 1152;                 // side boxes at 128-byte aligned offsets
constexpr uint32_t kBufBytes = 19200;                  // center + 2 sides, 128-aligned
constexpr int kTmaThreads = 128;

struct SobelTiles {
  uint32_t in_row0[kMaxBands];      // first input row of band b in the 2-D view
  uint64_t out_off[kMaxBands];
  uint32_t rows[kMaxBands];
  uint32_t first_tile[kMaxBands + 1];
  uint32_t nbands;
  uint32_t col_tiles;
  uint32_t mul[3];  // {1, 2, 0xFFFFFFFF} (see k_sobel_tma)
};

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
// d = a*b + c on the FMA pipe (IMAD), leaving the ALU pipe to PRMT / VIMNMX
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// ---- the per-pixel arithmetic, two forms ----------------------------------------
// Both work on even/odd planes of packed 16-bit halves (E = pixels 4k, 4k+2;
// O = 4k+1, 4k+3; Le / Ro = the left neighbours of the even pixels and the
// right neighbours of the odd ones).
//
// fp16 forms (kArith 1-3; 2 is the default): each 16-bit half holding a
// byte p is read as the fp16 SUBNORMAL p * 2^-24, and more generally any
// integer v in [0, 2048) stored in a half IS the fp16 value v * 2^-24. Every
// intermediate (dh, sh, Gx, Gy, |Gx|+|Gy|) is an integer multiple of 2^-24 of
// magnitude <= 2040, so HADD2/HFMA2 are exact; |.| is a free operand
// modifier of HADD2, the clamp is one HMNMX2, and min(|Gx|+|Gy|, 255) * 2^-24
// has the output byte as its low byte. The non-negative sh terms can equally
// be added as plain u16x2 integers on the ALU pipe (forms 2 and 3), which
// balances the ALU and fp16 pipes — both half rate.
// Integer form (kArith 0, round 1): biased u16x2 lanes, IMAD on the FMA pipe
// and VIMNMX/IADD3 on the ALU pipe; slowest at the power cap (IMAD as an
// adder costs more power than HADD2, so the clocks drop further).
__device__ __forceinline__ __half2 h2_of(uint32_t u) {
  __half2 h;
  memcpy(&h, &u, 4);
  return h;
}
__device__ __forceinline__ uint32_t u_of(__half2 h) {
  uint32_t u;
  memcpy(&u, &h, 4);
  return u;
}

// row terms of one 4-pixel word: dh = R - L, sh = L + 2C + R for the even and
// the odd plane (integer form: unbiased, exact mod 2^32 on the packed word)
template <int kArith>
__device__ __forceinline__ void word_terms(uint32_t E, uint32_t O, uint32_t Le, uint32_t Ro, uint32_t one,
                                           uint32_t two, uint32_t m1, uint32_t& dhe, uint32_t& dho, uint32_t& she,
                                           uint32_t& sho) {
  if constexpr (kArith != 0) {
    const __half2 e = h2_of(E), o = h2_of(O), l = h2_of(Le), r = h2_of(Ro), k2 = __float2half2_rn(2.f);
    dhe = u_of(__hsub2(o, l));
    dho = u_of(__hsub2(r, e));
    // sh is non-negative and < 2048: its integer bits ARE the fp16 value
    // sh * 2^-24, so arithmetic forms 2 / 3 add it on the ALU pipe instead
    // (plain u16x2 adds, no carries) to balance the two half-rate pipes
    if constexpr (kArith >= 2) she = Le + O + E + E;
    else she = u_of(__hfma2(e, k2, __hadd2(l, o)));
    if constexpr (kArith == 3) sho = E + Ro + O + O;
    else sho = u_of(__hfma2(o, k2, __hadd2(e, r)));
  } else {
    dhe = mad_u32(Le, m1, O);
    dho = mad_u32(E, m1, Ro);
    she = mad_u32(E, two, mad_u32(Le, one, O));
    sho = mad_u32(O, two, mad_u32(E, one, Ro));
  }
}

// one packed output pair from input rows (a, b, c) = (r, r+1, r+2); the
// output bytes are the low bytes of the two halves
template <int kArith>
__device__ __forceinline__ uint32_t out_pair(uint32_t adh, uint32_t bdh, uint32_t cdh, uint32_t ash, uint32_t csh,
                                             uint32_t two, uint32_t m1) {
  if constexpr (kArith != 0) {
    const __half2 gx = __hfma2(h2_of(bdh), __float2half2_rn(2.f), __hadd2(h2_of(adh), h2_of(cdh)));
    const __half2 gy = __hsub2(h2_of(csh), h2_of(ash));
    return u_of(__hmin2(__hadd2(__habs2(gx), __habs2(gy)), h2_of(0x00FF00FFu)));
  } else {
    // per half: gx' = Gx + 1024, gy' = Gy + 1024, both in [4, 2044]
    const uint32_t gx = mad_u32(bdh, two, adh + cdh + 0x04000400u);
    const uint32_t gy = csh - ash + 0x04000400u;
    // |G| + 1024 = max(g', 2048 - g') per half
    const uint32_t ax = __vmaxu2(gx, mad_u32(gx, m1, 0x08000800u));
    const uint32_t ay = __vmaxu2(gy, mad_u32(gy, m1, 0x08000800u));
    return __vminu2(__vadd2(ax, ay), 0x08FF08FFu);  // min(|Gx|+|Gy|, 255) + 2048
  }
}

__device__ __forceinline__ void tile_of(const SobelTiles& p, uint32_t t, uint32_t& b, uint32_t& rb, uint32_t& cb) {
  uint32_t lo = 0, hi = p.nbands;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p.first_tile[mid] <= t) lo = mid;
    else hi = mid;
  }
  b = lo;
  const uint32_t k = t - p.first_tile[lo];
  rb = k / p.col_tiles;
  cb = k % p.col_tiles;
}

struct SobelMaps {
  CUtensorMap center;  // box {256 B, 66 rows}
  CUtensorMap side;    // box {16 B, 66 rows}
};

// Where a buffer's tile lies: written by the issuing thread before the TMA
// and published to the CTA by the buffer's mbarrier phase (the arrive has
// release semantics), so only that thread runs the band search.
struct TileInfo {
  uint32_t b, rb, cb, valid;
};

__device__ __forceinline__ void issue_tile(const SobelMaps* maps, const SobelTiles& p, uint32_t t, uint8_t* buf,
                                           uint64_t* bar, TileInfo* info) {
  if (t >= p.first_tile[p.nbands]) {
    // no tile left: complete the buffer's phase with a plain arrive, so the
    // consumers wake up, see valid == 0 and leave
    *info = TileInfo{0, 0, 0, 0};
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(bar)) : "memory");
    return;
  }
  uint32_t b, rb, cb;
  tile_of(p, t, b, rb, cb);
  *info = TileInfo{b, rb, cb, 1};
  const int x = int(cb) * kTW, y = int(p.in_row0[b] + rb * kTH);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)),
               "r"(kCenterBytes + 2 * kSideBytes) : "memory");
  const int xs[3] = {x, x - 16, x + kTW};
  const uint32_t dst[3] = {sa(buf), sa(buf + kCenterBytes), sa(buf + kCenterBytes + kSideStride)};
#pragma unroll
  for (int k = 0; k < 3; ++k)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst[k]), "l"(k ? &maps->side : &maps->center), "r"(xs[k]), "r"(y), "r"(sa(bar))
        : "memory");
}

template <int kArith>
__global__ void __launch_bounds__(kTmaThreads)
    k_sobel_tma(const __grid_constant__ SobelMaps maps, uint8_t* __restrict__ out, const __grid_constant__ SobelTiles p,
                uint64_t width, unsigned long long* __restrict__ ctr) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) uint64_t full[2];
  __shared__ TileInfo info[2];
  const int tid = threadIdx.x, cg = tid & 15, rg = tid >> 4;
  const SobelMaps* map = &maps;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[1])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t it = 0;
  if (tid == 0) {
    issue_tile(map, p, blockIdx.x, smem, &full[0], &info[0]);
    issue_tile(map, p, blockIdx.x + gridDim.x, smem + kBufBytes, &full[1], &info[1]);
  }
  // Tiles after the first two per CTA: claimed from a counter (ctr[0]) when a
  // buffer frees up, so SMs that run ahead take more tiles and the grid ends
  // together; ctr == null: the static round-robin t += gridDim.x. Claims only
  // grow, so the first empty buffer ends the CTA with no copy in flight.
  uint32_t t = blockIdx.x;
  for (;; ++it) {
    const uint32_t bi = it & 1;
    uint8_t* buf = smem + bi * kBufBytes;
    asm volatile("{\n .reg .pred q;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W;\n}\n" ::"r"(
                     sa(&full[bi])), "r"((it >> 1) & 1)
                 : "memory");
    if (!info[bi].valid) {
      // the last CTA out returns the claim pair to zero for its next user
      if (ctr && tid == 0) {
        __threadfence();
        if (atomicAdd(ctr + 1, 1ull) == gridDim.x - 1) {
          ctr[0] = 0;
          ctr[1] = 0;
        }
      }
      break;
    }
    const uint32_t b = info[bi].b, rb = info[bi].rb, cb = info[bi].cb;
    const uint32_t valid_rows = min(uint32_t(kTH), p.rows[b] - rb * kTH);
    const uint64_t col = uint64_t(cb) * kTW + cg * 16;
    const uint8_t* center = buf;
    const uint8_t* left = buf + kCenterBytes;
    const uint8_t* right = left + kSideStride;
    // smem reads through explicit shared-window addresses (LDS, not generic LD)
    const uint32_t c_s = sa(center), l_s = sa(left), r_s = sa(right);
    // multipliers opaque to the compiler (kernel parameters): x*k+y stays an
    // IMAD on the FMA pipe instead of becoming an IADD3/LEA on the ALU pipe
    const uint32_t one = p.mul[0], two = p.mul[1], m1 = p.mul[2];
    // Row terms in even/odd planes: for word k (pixels 4k..4k+3) the even
    // plane holds pixels (4k, 4k+2) and the odd plane (4k+1, 4k+3) as 16-bit
    // halves, so the right neighbours of even pixels ARE the odd plane and
    // the left neighbours of odd pixels ARE the even plane; only the other
    // two neighbour vectors need one byte permute each (4 PRMT per 4 pixels
    // instead of 8). Terms are left unbiased: every linear step is exact
    // mod 2^32 on the packed word (a negative low half borrows from the high
    // half consistently), and emit adds the bias that makes both halves
    // non-negative before the per-half min/max.
    auto terms = [&](int i, RowTerms& tr) {
      const uint32_t row = c_s + uint32_t(i * kTW + cg * 16);
      uint4 w;
      uint32_t pw, nw;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "r"(row));
      // the 4-byte words holding pixel -1 (byte 3) and pixel 16 (byte 0)
      const uint32_t pa = cg ? row - 4 : l_s + uint32_t(i * 16 + 12);
      const uint32_t na = cg < 15 ? row + 16 : r_s + uint32_t(i * 16);
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pw) : "r"(pa));
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(nw) : "r"(na));
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      uint32_t E[4], O[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        E[k] = __byte_perm(ws[k], 0, 0x4240);  // (p[4k], p[4k+2])
        O[k] = __byte_perm(ws[k], 0, 0x4341);  // (p[4k+1], p[4k+3])
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // left of the even pixels (p[4k-1], p[4k+1]); right of the odd ones (p[4k+2], p[4k+4])
        const uint32_t Le = k ? __byte_perm(O[k - 1], O[k], 0x5432) : __byte_perm(pw, O[0], 0x5453);
        const uint32_t Ro = k < 3 ? __byte_perm(E[k], E[k + 1], 0x5432) : __byte_perm(E[3], nw, 0x1432);
        word_terms<kArith>(E[k], O[k], Le, Ro, one, two, m1, tr.dh[2 * k], tr.dh[2 * k + 1], tr.sh[2 * k],
                          tr.sh[2 * k + 1]);
      }
    };
    uint8_t* dst = out + p.out_off[b] + (uint64_t(rb) * kTH + rg * 8) * width + col;
    auto emit = [&](int r, const RowTerms& a, const RowTerms& bb, const RowTerms& c) {
      if (uint32_t(rg * 8 + r) >= valid_rows || col >= width) return;
      uint32_t o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = out_pair<kArith>(a.dh[i], bb.dh[i], c.dh[i], a.sh[i], c.sh[i], two, m1);
      // interleave the planes back: bytes (even lo, odd lo, even hi, odd hi)
      const uint32_t q0 = __byte_perm(o[0], o[1], 0x6240), q1 = __byte_perm(o[2], o[3], 0x6240);
      const uint32_t q2 = __byte_perm(o[4], o[5], 0x6240), q3 = __byte_perm(o[6], o[7], 0x6240);
      st_stream(reinterpret_cast<float4*>(dst + uint64_t(r) * width),
                make_float4(__uint_as_float(q0), __uint_as_float(q1), __uint_as_float(q2), __uint_as_float(q3)));
    };
    const int i0 = rg * 8;
    RowTerms t0, t1, t2;
    terms(i0, t0);
    terms(i0 + 1, t1);
    terms(i0 + 2, t2);
    emit(0, t0, t1, t2);
    terms(i0 + 3, t0);
    emit(1, t1, t2, t0);
    terms(i0 + 4, t1);
    emit(2, t2, t0, t1);
    terms(i0 + 5, t2);
    emit(3, t0, t1, t2);
    terms(i0 + 6, t0);
    emit(4, t1, t2, t0);
    terms(i0 + 7, t1);
    emit(5, t2, t0, t1);
    terms(i0 + 8, t2);
    emit(6, t0, t1, t2);
    terms(i0 + 9, t0);
    emit(7, t1, t2, t0);
    __syncthreads();  // buffer bi fully read
    if (tid == 0) {
      t = ctr ? 2 * gridDim.x + uint32_t(atomicAdd(ctr, 1ull)) : t + gridDim.x;
      issue_tile(map, p, ctr ? t : t + gridDim.x, buf, &full[bi], &info[bi]);
    }
  }
}

// ---- row-streaming path (default for widths that are multiples of 16) -----------
// Each warp owns a 512-column segment (16 columns per lane) and walks DOWN a
// balanced range of output rows, so every input row's terms are computed
// once (the tiled kernel above computes 10 input rows' terms per 8 output
// rows) and the 3-row window lives in registers. Input rows stream in through
// a per-warp ring of kSlots smem slots of 3 rows each, filled by 1-D bulk
// copies (cp.async.bulk, one per row: the segment plus 16 bytes either side,
// the out-of-image side left zero) completing on the slot's mbarrier; lane 0
// refills a slot as soon as the warp has read it. One wait and one refill per
// 3 rows, and the 3-row groups line up with the register window's rotation,
// so the loop body is straight-line code. No CTA-wide barrier anywhere. The
// work split is static: the output rows of all bands, concatenated, divided
// evenly among the warps of one column segment.
constexpr int kRowThreads = 128;

// Geometry of a lane owning kCols columns (16 or 8): a warp segment is
// 32 * kCols columns, a ring row holds it plus 16 bytes either side, a TMA
// box is 3 such rows, a slot is the box rounded up to 128 bytes.
template <int kCols>
struct RowGeom {
  static constexpr uint32_t seg = 32 * kCols;
  static constexpr uint32_t row_bytes = seg + 32;
  static constexpr uint32_t box_bytes = 3 * row_bytes;
  static constexpr uint32_t slot_bytes = (box_bytes + 127) / 128 * 128;
};

template <int kW>  // kW 4-byte words = 4 kW pixels per lane
struct RowTermsW {
  uint32_t dh[2 * kW];
  uint32_t sh[2 * kW];
};

struct SobelRows {
  uint32_t in_row0[kMaxBands];        // first input row of band b in the 2-D view of the input
  uint64_t out_off[kMaxBands];
  uint32_t first_row[kMaxBands + 1];  // output rows before band b (prefix sums)
  uint32_t nbands;
  uint32_t segs;                      // column segments per row
  uint32_t mul[3];                    // {1, 2, 0xFFFFFFFF}, opaque to the compiler
};

template <int kMinBlocks, int kSlots, int kCols, int kArith>
__global__ void __launch_bounds__(kRowThreads, kMinBlocks)
    k_sobel_rows(const __grid_constant__ CUtensorMap rows3, uint8_t* __restrict__ out,
                 const __grid_constant__ SobelRows p, uint64_t width) {
  using G = RowGeom<kCols>;
  constexpr int kW = kCols / 4;
  extern __shared__ __align__(128) uint8_t dyn[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t one = p.mul[0], two = p.mul[1], m1 = p.mul[2];
  uint8_t* ring = dyn + wib * (kSlots * G::slot_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(dyn + (kRowThreads / 32) * kSlots * G::slot_bytes) + wib * kSlots;
  if (lane == 0) {
    for (int k = 0; k < kSlots; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  const uint32_t gw = blockIdx.x * (kRowThreads / 32) + wib, nw = gridDim.x * (kRowThreads / 32);
  const uint32_t seg = gw % p.segs, slot_w = gw / p.segs, nslot = nw / p.segs;
  if (slot_w >= nslot) return;  // the leftover warps of an uneven split
  const uint32_t total = p.first_row[p.nbands];
  const uint32_t g0 = uint32_t(uint64_t(total) * slot_w / nslot), g1 = uint32_t(uint64_t(total) * (slot_w + 1) / nslot);
  const int64_t c0 = int64_t(seg) * G::seg;
  const uint64_t col = uint64_t(c0) + lane * kCols;
  const bool active = col < width;
  // this warp's window in every row: image columns [c0 - 16, c0 + seg + 16)
  // as 8-byte elements; the parts outside the image are zero-filled by the TMA
  const int x8 = int(c0 / 8) - 2;
  uint32_t q = 0;  // row groups consumed by this warp: group q uses slot q % kSlots, phase (q / kSlots) & 1

  uint32_t b = 0;
  {
    uint32_t l = 0, h = p.nbands;  // band holding output row g0
    while (h - l > 1) {
      const uint32_t m = (l + h) >> 1;
      if (p.first_row[m] <= g0) l = m;
      else h = m;
    }
    b = l;
  }
  for (uint32_t g = g0; g < g1; ++b) {
    const uint32_t r0 = g - p.first_row[b];  // first local output row of this piece
    const uint32_t r1 = min(g1, p.first_row[b + 1]) - p.first_row[b];
    g += r1 - r0;
    if (r1 <= r0) continue;
    const int y0 = int(p.in_row0[b] + r0);  // input row r0 of the band (the halo above output row r0)
    uint8_t* dst = out + p.out_off[b] + uint64_t(r0) * width + col;
    const uint32_t nin = r1 - r0 + 2, ngroups = (nin + 2) / 3;
    // lane 0: input rows 3j..3j+2 of this piece into slot (q + j) % kSlots —
    // one 2-D TMA box (a last partial group reads rows past the piece: in the
    // 2-D view those are the next band's rows or zero fill, never used)
    auto fill = [&](uint32_t j) {
      const uint32_t k = (q + j) % kSlots;
      const uint32_t bar = sa(&full[k]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(G::box_bytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              sa(ring + k * G::slot_bytes)),
          "l"(&rows3), "r"(x8), "r"(y0 + int(3 * j)), "r"(bar)
          : "memory");
    };
    if (lane == 0)
      for (uint32_t j = 0; j < min(uint32_t(kSlots), ngroups); ++j) fill(j);
    auto terms = [&](uint32_t row_s, RowTermsW<kW>& tr) {
      uint32_t ws[kW];
      uint32_t pw, nw2;
      if constexpr (kW == 4) {
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(ws[0]), "=r"(ws[1]), "=r"(ws[2]), "=r"(ws[3]) : "r"(row_s));
      } else {
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(ws[0]), "=r"(ws[1]) : "r"(row_s));
      }
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pw) : "r"(row_s - 4));
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(nw2) : "r"(row_s + 4 * kW));
      uint32_t E[kW], O[kW];
#pragma unroll
      for (int kk = 0; kk < kW; ++kk) {
        E[kk] = __byte_perm(ws[kk], 0, 0x4240);
        O[kk] = __byte_perm(ws[kk], 0, 0x4341);
      }
#pragma unroll
      for (int kk = 0; kk < kW; ++kk) {
        const uint32_t Le = kk ? __byte_perm(O[kk - 1], O[kk], 0x5432) : __byte_perm(pw, O[0], 0x5453);
        const uint32_t Ro = kk < kW - 1 ? __byte_perm(E[kk], E[kk + 1], 0x5432) : __byte_perm(E[kW - 1], nw2, 0x1432);
        word_terms<kArith>(E[kk], O[kk], Le, Ro, one, two, m1, tr.dh[2 * kk], tr.dh[2 * kk + 1], tr.sh[2 * kk],
                          tr.sh[2 * kk + 1]);
      }
    };
    auto emit = [&](uint32_t r, const RowTermsW<kW>& a, const RowTermsW<kW>& bb, const RowTermsW<kW>& c) {
      uint32_t o[2 * kW];
#pragma unroll
      for (int i = 0; i < 2 * kW; ++i) o[i] = out_pair<kArith>(a.dh[i], bb.dh[i], c.dh[i], a.sh[i], c.sh[i], two, m1);
      if (active) {
        uint32_t x[kW];
#pragma unroll
        for (int kk = 0; kk < kW; ++kk) x[kk] = __byte_perm(o[2 * kk], o[2 * kk + 1], 0x6240);
        if constexpr (kW == 4) {
          st_stream(reinterpret_cast<float4*>(dst + uint64_t(r) * width),
                    make_float4(__uint_as_float(x[0]), __uint_as_float(x[1]), __uint_as_float(x[2]), __uint_as_float(x[3])));
        } else {
          __stcs(reinterpret_cast<uint2*>(dst + uint64_t(r) * width), make_uint2(x[0], x[1]));
        }
      }
    };
    // group j = input rows 3j, 3j+1, 3j+2 -> window slots t0, t1, t2 (output
    // row i-2 needs input rows i-2, i-1, i)
    RowTermsW<kW> t0, t1, t2;
    for (uint32_t j = 0; j < ngroups; ++j) {
      const uint32_t k = (q + j) % kSlots;
      asm volatile("{\n .reg .pred w;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 w, [%0], %1;\n @!w bra W;\n}\n" ::"r"(
                       sa(&full[k])), "r"(((q + j) / kSlots) & 1)
                   : "memory");
      const uint32_t base = sa(ring + k * G::slot_bytes + 16 + lane * kCols);
      const uint32_t i0 = 3 * j;
      terms(base, t0);
      if (i0 >= 2) emit(i0 - 2, t1, t2, t0);
      if (i0 + 1 < nin) {
        terms(base + G::row_bytes, t1);
        if (i0 + 1 >= 2) emit(i0 - 1, t2, t0, t1);
        if (i0 + 2 < nin) {
          terms(base + 2 * G::row_bytes, t2);
          emit(i0, t0, t1, t2);
        }
      }
      __syncwarp();  // every lane has read slot k
      if (lane == 0 && j + kSlots < ngroups) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        fill(j + kSlots);
      }
    }
    q += ngroups;
  }
}

template <int kSlots, int kCols>
constexpr uint32_t sobel_rows_smem() {
  return (kRowThreads / 32) * kSlots * (RowGeom<kCols>::slot_bytes + 8) + 128;
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
  // UCG_SOBEL_VARIANT (A/B runs): 1 = TMA tiles (default), 0 = row streaming
  // (measured equal: 100.8 vs 99.9 us at 16384^2 — both ALU-pipe bound, see
  // DESIGN.md §5), 2 = register streaming without TMA
  static const int variant = [] {
    const char* e = getenv("UCG_SOBEL_VARIANT");
    return e ? atoi(e) : (getenv("UCG_SOBEL_NO_TMA") ? 2 : 1);
  }();
  // Arithmetic form (UCG_SOBEL_ARITH for A/B runs): mix (default) = fp16-
  // subnormal with the even plane's sh terms added on the ALU pipe; half =
  // all fp16; mix2 = both planes' sh on the ALU pipe; int = the round-1
  // biased-integer form. Same box, claimed tiles (profiles/r02/sobel_claim/):
  // bench line (1 s soak, power-capped ~1.7 GHz) mix 95.5-96.8 us, half
  // 99.2, mix2 97.6, int 107.9; 2000 back-to-back launches mix 90.2-91.1,
  // half 91.9-92.7, int 102.1; alone under ncu mix 86.7, half 89.2. The fp16
  // adds cost less power than IMAD-as-adder (clocks stay higher at the cap)
  // and balance the FMA and ALU pipes, which both run at half rate.
  static const int arith = [] {
    const char* e = getenv("UCG_SOBEL_ARITH");
    if (!e) return 2;
    if (strcmp(e, "int") == 0) return 0;
    if (strcmp(e, "half") == 0) return 1;
    if (strcmp(e, "mix2") == 0) return 3;
    return 2;
  }();
  bool rows_ok = vec && variant == 0 && width < (1ull << 31);
  for (uint64_t i = 0; i < nbands && rows_ok; ++i) rows_ok = in_off[i] % width == 0;
  if (rows_ok) {
    // A/B knobs: UCG_SOBEL_COLS (columns per lane, 16 or 8), UCG_SOBEL_SLOTS
    // (3-row slots per warp, 4 or 6)
    static const int cols = [] {
      const char* e = getenv("UCG_SOBEL_COLS");
      return e && atoi(e) == 8 ? 8 : 16;
    }();
    static const int slots = [] {
      const char* e = getenv("UCG_SOBEL_SLOTS");
      return e && atoi(e) == 6 ? 6 : 4;
    }();
    // row streaming (A/B only): 16 or 8 columns per lane (4 row slots), or
    // 16 columns with 6 slots; integer, fp16 or mixed form
    auto kern = cols == 8 ? (arith == 0 ? k_sobel_rows<8, 4, 8, 0> : k_sobel_rows<8, 4, 8, 2>)
                : slots == 6 ? (arith == 0 ? k_sobel_rows<5, 6, 16, 0> : k_sobel_rows<5, 6, 16, 2>)
                : arith == 0 ? k_sobel_rows<5, 4, 16, 0>
                : arith == 1 ? k_sobel_rows<5, 4, 16, 1>
                : arith == 3 ? k_sobel_rows<5, 4, 16, 3>
                             : k_sobel_rows<5, 4, 16, 2>;
    const uint32_t smem = cols == 16 ? (slots == 6 ? sobel_rows_smem<6, 16>() : sobel_rows_smem<4, 16>())
                                     : (slots == 6 ? sobel_rows_smem<6, 8>() : sobel_rows_smem<4, 8>());
    const uint32_t seg_cols = 32u * uint32_t(cols);
    static std::atomic<uint64_t> occ_seen{0};
    static int per_sm = 1;
    if (first_on_device(occ_seen)) {
      UCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      UCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowThreads, smem));
    }
    for (uint64_t b0 = 0; b0 < nbands; b0 += kMaxBands) {
      const uint32_t nb = uint32_t(std::min<uint64_t>(kMaxBands, nbands - b0));
      SobelRows p;
      p.nbands = nb;
      p.segs = uint32_t((width + seg_cols - 1) / seg_cols);
      uint64_t in_rows = 0;
      for (uint32_t i = 0; i < nb; ++i) {
        if (in_off[b0 + i] % width) return fail(UCG_ERR_ARG, "sobel: bands must start on a row boundary");
        p.in_row0[i] = uint32_t(in_off[b0 + i] / width);
        in_rows = std::max<uint64_t>(in_rows, in_off[b0 + i] / width + rows[b0 + i] + 2);
      }
      if (in_rows >= (1ull << 31)) return fail(UCG_ERR_ARG, "sobel: input too tall for a tensor map");
      CUtensorMap rows3;
      {
        auto enc = tmap_encode_fn();
        if (!enc) return fail(UCG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        cuuint64_t dims[2] = {width / 8, in_rows};
        cuuint64_t strides[1] = {width};
        cuuint32_t box[2] = {(seg_cols + 32) / 8, 3}, estr[2] = {1, 1};
        if (enc(&rows3, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint8_t*>(in), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
          return fail(UCG_ERR_CUDA, "sobel rows tensor map encode failed");
      }
      p.mul[0] = 1;
      p.mul[1] = 2;
      p.mul[2] = 0xFFFFFFFFu;
      p.first_row[0] = 0;
      uint64_t tot = 0;
      for (uint32_t i = 0; i < nb; ++i) {
        p.out_off[i] = out_off[b0 + i];
        tot += rows[b0 + i];
        if (tot >= (1ull << 32)) return fail(UCG_ERR_ARG, "sobel: more than 2^32 output rows in one launch");
        p.first_row[i + 1] = uint32_t(tot);
      }
      if (!tot) continue;
      // every resident warp streams; a column segment's warps split its rows
      // evenly, at least 8 rows each so a band's halo overhead stays small
      const uint64_t warps_fill = uint64_t(sm_count()) * std::max(1, per_sm) * (kRowThreads / 32);
      const uint64_t per_seg = std::max<uint64_t>(1, std::min<uint64_t>(warps_fill / p.segs, (tot + 7) / 8));
      const uint64_t warps = per_seg * p.segs;
      const unsigned grid = unsigned((warps + kRowThreads / 32 - 1) / (kRowThreads / 32));
      kern<<<grid, kRowThreads, smem, st>>>(rows3, out, p, width);
      UCG_LAUNCHED();
    }
    return UCG_OK;
  }
  bool tma = vec && width >= 16 && width < (1ull << 31) && variant == 1;
  uint64_t total_rows = 0;
  for (uint64_t i = 0; i < nbands && tma; ++i) {
    tma = in_off[i] % width == 0 && rows[i] < (1u << 30);
    total_rows = std::max<uint64_t>(total_rows, in_off[i] / width + rows[i] + 2);
  }
  if (tma && total_rows < (1ull << 31)) {
    auto enc = tmap_encode_fn();
    if (!enc) return fail(UCG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    SobelMaps maps;
    cuuint64_t dims[2] = {width, total_rows};
    cuuint64_t strides[1] = {width};
    cuuint32_t estr[2] = {1, 1};
    cuuint32_t boxc[2] = {uint32_t(kTW), uint32_t(kTIn)}, boxs[2] = {16u, uint32_t(kTIn)};
    CUresult r1 = enc(&maps.center, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(in), dims, strides, boxc,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc(&maps.side, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(in), dims, strides, boxs,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) return fail(UCG_ERR_CUDA, "sobel tensor map encode failed");
    auto tkern = arith == 0 ? k_sobel_tma<0> : arith == 2 ? k_sobel_tma<2> : arith == 3 ? k_sobel_tma<3> : k_sobel_tma<1>;
    static std::atomic<uint64_t> attr{0};
    if (first_on_device(attr))
      UCG_CUDA(cudaFuncSetAttribute(tkern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(2 * kBufBytes + 128)));
    const uint32_t col_tiles = uint32_t((width + kTW - 1) / kTW);
    for (uint64_t b0 = 0; b0 < nbands; b0 += kMaxBands) {
      const uint32_t nb = uint32_t(std::min<uint64_t>(kMaxBands, nbands - b0));
      SobelTiles p;
      p.nbands = nb;
      p.col_tiles = col_tiles;
      p.mul[0] = 1;
      p.mul[1] = 2;
      p.mul[2] = 0xFFFFFFFFu;
      p.first_tile[0] = 0;
      for (uint32_t i = 0; i < nb; ++i) {
        p.in_row0[i] = uint32_t(in_off[b0 + i] / width);
        p.out_off[i] = out_off[b0 + i];
        p.rows[i] = uint32_t(rows[b0 + i]);
        p.first_tile[i + 1] = p.first_tile[i] + uint32_t((rows[b0 + i] + kTH - 1) / kTH) * col_tiles;
      }
      const uint32_t ntiles = p.first_tile[nb];
      if (!ntiles) continue;
      const unsigned grid = unsigned(std::min<uint64_t>(ntiles, uint64_t(sm_count()) * 5));
      // UCG_SOBEL_STATIC (A/B runs): round-robin tiles instead of claimed ones
      static const bool static_tiles = getenv("UCG_SOBEL_STATIC") != nullptr;
      unsigned long long* ctr = nullptr;
      if (!static_tiles) {
        ctr = claim_pair_selfreset();  // zero at launch; the kernel's last CTA re-zeroes it
        if (!ctr) return fail(UCG_ERR_CUDA, "sobel: claim counter unavailable");
      }
      tkern<<<grid, kTmaThreads, 2 * kBufBytes + 128, st>>>(maps, out, p, width, ctr);
      UCG_LAUNCHED();
    }
    return UCG_OK;
  }
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
