/*
 * ucores_oracle.h — CPU restatement of the reference's mapCL / mapCLPartition /
 * reduceCL semantics and of the workload kernels.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it. The product path (paper_1505_01120_b200/) never links or calls it.
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to the reference root (proj/include/ucores/X.hpp written ucores/X.hpp).
 * Parity is pinned against oracle/_ref (the reference headers compiled here,
 * see oracle/Makefile) through tests/golden/ref_golden.json.
 */
#ifndef UCORES_ORACLE_H
#define UCORES_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- deterministic input generation (shared definition with the CUDA fill) */
uint64_t orc_mix64(uint64_t z);
/* i-th output of the SplitMix64 stream whose state starts at `seed`. */
uint64_t orc_stream_u64(uint64_t seed, uint64_t i);
/* out[i] = uniform [0,1) float from orc_stream_u64(seed, first + i) >> 40. */
void orc_fill_uniform_f32(uint64_t seed, uint64_t first, uint64_t n, float* out);
/* SPEC.md:474 vectoradd fill: element k, value i = (k*len + i) mod 1000. */
void orc_fill_vectoradd(uint64_t k, uint64_t len, float* out);

/* FNV-1a 64 over bytes (the digest the golden vectors record). */
uint64_t orc_fnv64(const void* data, uint64_t n);

/* ---- data model */
/* create_dataset ceiling-first sizes (ucores/dataset.hpp:64-82). 0 ok, -1 if P<1. */
int orc_partition_sizes(uint64_t n, uint64_t num_partitions, uint64_t* sizes_out);

/* ---- map kernels */
/* axpb map body: y = fl(fl(a*x) + b) — two roundings, no contraction. */
void orc_map_affine_f32(const float* x, uint64_t n, float a, float b, float* y);

/* ---- the reduce tree (ucores/engine.hpp:172-190 pairing rule) */
enum { ORC_OP_SUM = 0, ORC_OP_MAX = 1 };
/* Pairwise tree over x[0..n): each round pairs (0,1),(2,3),...; an unpaired
 * trailing value is promoted unchanged. op SUM: a+b; op MAX: (a<b)?b:a
 * (std::max). Empty input: 0.0f (SUM) / -INF (MAX). */
float orc_tree_reduce_f32(const float* x, uint64_t n, int op);
int64_t orc_tree_reduce_i64(const int64_t* x, uint64_t n);

/* reduce_cl over vector elements (ucores/engine.hpp:121-192): stage 1 left
 * fold inside each partition, stage 2 pairing tree over partials. Elements
 * are `count` vectors of `len` floats laid out back to back in `elems`;
 * part_counts[p] = number of elements in partition p. Elementwise op.
 * Returns 0, -1 on empty dataset (EmptyDataset). */
int orc_reduce_cl_f32(const float* elems, uint64_t len, const uint64_t* part_counts,
                      uint64_t num_partitions, int op, float* out);
int orc_reduce_cl_i64(const int64_t* elems, uint64_t len, const uint64_t* part_counts,
                      uint64_t num_partitions, int64_t* out);

/* ---- Monte-Carlo pi */
int orc_pi_hit(uint64_t task_seed, uint64_t gid);
uint64_t orc_pi_hits(uint64_t task_seed, uint64_t samples);

/* ---- 3x3 Sobel on a row band with one halo row above and below. in has
 * rows_in = rows_out + 2 rows of `width` bytes; columns outside the image are
 * zero. out(r,c) = min(255, |Gx|+|Gy|). */
void orc_sobel_band_u8(const uint8_t* in, uint64_t rows_out, uint64_t width, uint8_t* out);

/* ---- WordCount: flags[i] = byte i is a word character and
 * (i == 0 or byte i-1 is a delimiter); delimiters: space, tab, LF, CR
 * (ucores/dataset.hpp:87-89). */
void orc_word_start_flags(const uint8_t* bytes, uint64_t n, uint8_t* flags);
/* create_from_text chunk boundaries (ucores/dataset.hpp:94-112): writes up to
 * max_chunks [begin,end) pairs, returns the number of chunks. */
uint64_t orc_chunk_offsets(const uint8_t* data, uint64_t n, uint64_t target, uint64_t* pairs, uint64_t max_chunks);

/* ---- dense matmul: C = A·B (n×n row-major). fp32 sequential-k accumulate
 * (the class-D run() body) and an fp64 entry for tolerance checks. */
void orc_matmul_f32(const float* A, const float* B, uint64_t n, float* C);
double orc_matmul_entry_f64(const float* A, const float* B, uint64_t n, uint64_t i, uint64_t j);

#ifdef __cplusplus
}
#endif
#endif
