/*
 * ucores_oracle.c — TEST INFRASTRUCTURE ONLY (see ucores_oracle.h).
 *
 * CPU restatement of the reference semantics for the mapCL / mapCLPartition /
 * reduceCL hot path. Compiled with -ffp-contract=off so every float
 * expression rounds exactly as written.
 */
#include "ucores_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9E3779B97F4A7C15ull

/* SplitMix64 finaliser, constants per SPEC.md:465. */
uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t orc_stream_u64(uint64_t seed, uint64_t i) { return orc_mix64(seed + (i + 1) * GAMMA); }

void orc_fill_uniform_f32(uint64_t seed, uint64_t first, uint64_t n, float* out) {
  for (uint64_t i = 0; i < n; ++i) {
    out[i] = (float)(orc_stream_u64(seed, first + i) >> 40) * (1.0f / 16777216.0f);
  }
}

uint64_t orc_fnv64(const void* data, uint64_t n) {
  const unsigned char* b = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* element k holds values (k*len + i) mod 1000. */
void orc_fill_vectoradd(uint64_t k, uint64_t len, float* out) {
  for (uint64_t i = 0; i < len; ++i) out[i] = (float)((k * len + i) % 1000u);
}

/* ucores/dataset.hpp:64-82 create_dataset: base = n/P, the first n%P
 * partitions take one extra element (ceiling-first, contiguous, in order). */
int orc_partition_sizes(uint64_t n, uint64_t P, uint64_t* sizes) {
  if (P < 1) return -1; /* InvalidPartitionCount (dataset.hpp:65-68) */
  const uint64_t base = n / P, extra = n % P;
  for (uint64_t p = 0; p < P; ++p) sizes[p] = base + (p < extra ? 1 : 0);
  return 0;
}

/* axpb run() body: y[gid] = a*x[gid] + b, evaluated as two IEEE roundings. */
void orc_map_affine_f32(const float* x, uint64_t n, float a, float b, float* y) {
  for (uint64_t i = 0; i < n; ++i) {
    const float t = a * x[i];
    y[i] = t + b;
  }
}

static inline float combine_f32(float a, float b, int op) {
  if (op == ORC_OP_MAX) return (a < b) ? b : a; /* std::max(a,b) */
  return a + b;
}

/* ucores/engine.hpp:172-190, stage 2: while more than one value remains,
 * pair (0,1),(2,3),... in the current order; a trailing unpaired value is
 * promoted unchanged to the end of the next round. Restated literally, level
 * by level, on a scratch copy. */
float orc_tree_reduce_f32(const float* x, uint64_t n, int op) {
  if (n == 0) return op == ORC_OP_MAX ? -INFINITY : 0.0f;
  float* cur = (float*)malloc(n * sizeof(float));
  memcpy(cur, x, n * sizeof(float));
  uint64_t m = n;
  while (m > 1) {
    uint64_t k = 0;
    for (uint64_t i = 0; i + 1 < m; i += 2) cur[k++] = combine_f32(cur[i], cur[i + 1], op);
    if (m % 2 == 1) cur[k++] = cur[m - 1];
    m = k;
  }
  const float r = cur[0];
  free(cur);
  return r;
}

int64_t orc_tree_reduce_i64(const int64_t* x, uint64_t n) {
  if (n == 0) return 0;
  int64_t* cur = (int64_t*)malloc(n * sizeof(int64_t));
  memcpy(cur, x, n * sizeof(int64_t));
  uint64_t m = n;
  while (m > 1) {
    uint64_t k = 0;
    for (uint64_t i = 0; i + 1 < m; i += 2)
      cur[k++] = (int64_t)((uint64_t)cur[i] + (uint64_t)cur[i + 1]);
    if (m % 2 == 1) cur[k++] = cur[m - 1];
    m = k;
  }
  const int64_t r = cur[0];
  free(cur);
  return r;
}

/* ucores/engine.hpp:121-192 reduce_cl with an elementwise binary kernel
 * (the Fig-3 vectoradd body c[gid] = a[gid] (op) b[gid], kernel.hpp:208-215):
 *   stage 1 (:144-170): acc = e0; acc = k(acc, e_i) left to right per
 *   non-empty partition; stage 2 (:172-190): the pairing tree over partials.
 * The tree is applied lane by lane, which is exactly what pairing whole
 * vectors elementwise does. */
int orc_reduce_cl_f32(const float* elems, uint64_t len, const uint64_t* part_counts,
                      uint64_t P, int op, float* out) {
  uint64_t count = 0, nonempty = 0;
  for (uint64_t p = 0; p < P; ++p) {
    count += part_counts[p];
    nonempty += part_counts[p] ? 1 : 0;
  }
  if (count == 0) return -1; /* EmptyDataset (engine.hpp:124) */
  float* partial = (float*)malloc((nonempty ? nonempty : 1) * len * sizeof(float));
  uint64_t e = 0, q = 0;
  for (uint64_t p = 0; p < P; ++p) {
    if (!part_counts[p]) continue;
    float* acc = partial + q * len;
    memcpy(acc, elems + e * len, len * sizeof(float));
    for (uint64_t j = 1; j < part_counts[p]; ++j) {
      const float* r = elems + (e + j) * len;
      for (uint64_t i = 0; i < len; ++i) acc[i] = combine_f32(acc[i], r[i], op);
    }
    e += part_counts[p];
    ++q;
  }
  float* lane = (float*)malloc((nonempty ? nonempty : 1) * sizeof(float));
  for (uint64_t i = 0; i < len; ++i) {
    for (uint64_t k = 0; k < nonempty; ++k) lane[k] = partial[k * len + i];
    out[i] = orc_tree_reduce_f32(lane, nonempty, op);
  }
  free(lane);
  free(partial);
  return 0;
}

int orc_reduce_cl_i64(const int64_t* elems, uint64_t len, const uint64_t* part_counts,
                      uint64_t P, int64_t* out) {
  uint64_t count = 0, nonempty = 0;
  for (uint64_t p = 0; p < P; ++p) {
    count += part_counts[p];
    nonempty += part_counts[p] ? 1 : 0;
  }
  if (count == 0) return -1;
  int64_t* partial = (int64_t*)malloc((nonempty ? nonempty : 1) * len * sizeof(int64_t));
  uint64_t e = 0, q = 0;
  for (uint64_t p = 0; p < P; ++p) {
    if (!part_counts[p]) continue;
    int64_t* acc = partial + q * len;
    memcpy(acc, elems + e * len, len * sizeof(int64_t));
    for (uint64_t j = 1; j < part_counts[p]; ++j) {
      const int64_t* r = elems + (e + j) * len;
      for (uint64_t i = 0; i < len; ++i) acc[i] = (int64_t)((uint64_t)acc[i] + (uint64_t)r[i]);
    }
    e += part_counts[p];
    ++q;
  }
  int64_t* lane = (int64_t*)malloc((nonempty ? nonempty : 1) * sizeof(int64_t));
  for (uint64_t i = 0; i < len; ++i) {
    for (uint64_t k = 0; k < nonempty; ++k) lane[k] = partial[k * len + i];
    out[i] = orc_tree_reduce_i64(lane, nonempty);
  }
  free(lane);
  free(partial);
  return 0;
}

/* state s0 = task_seed XOR (gid*gamma); z1 = mix(s0+gamma),
 * z2 = mix(s0+2*gamma); x = (z1>>32)/2^32, y = (z2>>32)/2^32 as doubles;
 * hit iff x*x + y*y <= 1 in IEEE double (no contraction). */
int orc_pi_hit(uint64_t task_seed, uint64_t gid) {
  const uint64_t s0 = task_seed ^ (gid * GAMMA);
  const uint64_t z1 = orc_mix64(s0 + GAMMA);
  const uint64_t z2 = orc_mix64(s0 + 2 * GAMMA);
  const double x = (double)(z1 >> 32) / 4294967296.0;
  const double y = (double)(z2 >> 32) / 4294967296.0;
  const double xx = x * x;
  const double yy = y * y;
  const double s = xx + yy;
  return s <= 1.0;
}

uint64_t orc_pi_hits(uint64_t task_seed, uint64_t samples) {
  uint64_t h = 0;
  for (uint64_t g = 0; g < samples; ++g) h += (uint64_t)orc_pi_hit(task_seed, g);
  return h;
}

static inline int px(const uint8_t* in, uint64_t width, uint64_t r, int64_t c) {
  if (c < 0 || (uint64_t)c >= width) return 0;
  return in[r * width + (uint64_t)c];
}

/* Sobel band kernel (workload C4; not in the reference — definition frozen
 * here and in DESIGN.md): Gx = [-1 0 1; -2 0 2; -1 0 1],
 * Gy = [-1 -2 -1; 0 0 0; 1 2 1], zero outside the image columns, halo rows
 * supplied by the band element. */
void orc_sobel_band_u8(const uint8_t* in, uint64_t rows_out, uint64_t width, uint8_t* out) {
  for (uint64_t r = 0; r < rows_out; ++r) {
    for (uint64_t c = 0; c < width; ++c) {
      const int64_t cc = (int64_t)c;
      const int gx = -px(in, width, r, cc - 1) + px(in, width, r, cc + 1) -
                     2 * px(in, width, r + 1, cc - 1) + 2 * px(in, width, r + 1, cc + 1) -
                     px(in, width, r + 2, cc - 1) + px(in, width, r + 2, cc + 1);
      const int gy = -px(in, width, r, cc - 1) - 2 * px(in, width, r, cc) -
                     px(in, width, r, cc + 1) + px(in, width, r + 2, cc - 1) +
                     2 * px(in, width, r + 2, cc) + px(in, width, r + 2, cc + 1);
      int m = abs(gx) + abs(gy);
      out[r * width + c] = (uint8_t)(m > 255 ? 255 : m);
    }
  }
}

static inline int is_delim(uint8_t b) { return b == ' ' || b == '\t' || b == '\n' || b == '\r'; }

/* WordCount run() body with the dataset.hpp:87-89 delimiters. */
void orc_word_start_flags(const uint8_t* b, uint64_t n, uint8_t* flags) {
  for (uint64_t i = 0; i < n; ++i) flags[i] = (uint8_t)(!is_delim(b[i]) && (i == 0 || is_delim(b[i - 1])));
}

/* ucores/dataset.hpp:94-112 chunk_offsets: a tentative cut at start+target is
 * advanced past the next delimiter so no word spans two chunks. */
uint64_t orc_chunk_offsets(const uint8_t* data, uint64_t n, uint64_t target, uint64_t* pairs, uint64_t max_chunks) {
  uint64_t start = 0, k = 0;
  while (start < n) {
    const uint64_t tentative = start + target;
    uint64_t cut;
    if (tentative >= n) {
      cut = n;
    } else {
      uint64_t d = tentative;
      while (d < n && !is_delim(data[d])) ++d;
      cut = d < n ? d + 1 : n;
    }
    if (k < max_chunks) {
      pairs[2 * k] = start;
      pairs[2 * k + 1] = cut;
    }
    ++k;
    start = cut;
  }
  return k;
}

/* Matmul class-D body: C[gid] with gid = i*n + j, fp32 accumulate over k in
 * ascending order (workload C5; not in the reference). */
void orc_matmul_f32(const float* A, const float* B, uint64_t n, float* C) {
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < n; ++j) {
      float acc = 0.0f;
      for (uint64_t k = 0; k < n; ++k) {
        const float t = A[i * n + k] * B[k * n + j];
        acc = acc + t;
      }
      C[i * n + j] = acc;
    }
}

double orc_matmul_entry_f64(const float* A, const float* B, uint64_t n, uint64_t i, uint64_t j) {
  double acc = 0.0;
  for (uint64_t k = 0; k < n; ++k) acc += (double)A[i * n + k] * (double)B[k * n + j];
  return acc;
}
