/*
 * ucores_cuda.h — C-ABI of libucores_cuda.so, the B200 (sm_100a) engine for
 * the reference's mapCL / mapCLPartition / reduceCL hot path.
 *
 * Reference = the header-only C++20 `ucores` library (proj/include/ucores/,
 * abbreviated ucores/X.hpp). The reference has no FFI; these entry points are
 * what its two seams bind:
 *   seam B  KernelExecutor::execute          ucores/kernel.hpp:219-234
 *   seam A  ClusterDriver::run_wave          ucores/engine.hpp:34-39
 * The C++ drop-in adapters that call them live in
 * paper_1505_01120_b200/host/ucores_b200/ (see INTEGRATION.md).
 *
 * Conventions
 *  - Every function returns int: 0 (UCG_OK) or a negative UCG_ERR_* code;
 *    ucg_last_error() returns the thread-local message of the last failure.
 *    The C++ adapter rethrows these as ucores::KernelPanic("run", msg), the
 *    reference's error for a failing run phase (device.hpp:360,400,430).
 *  - Device work runs on the CURRENT CUDA device (ucg_set_device) and is
 *    enqueued on `stream` (a cudaStream_t passed as void*, NULL = legacy
 *    default stream). Calls are asynchronous unless stated otherwise.
 *  - Device pointers are caller-owned (ucg_malloc or any CUDA allocation);
 *    float arrays must be 16-byte aligned. Host pointers are caller-owned.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry returns UCG_ERR_NODEV.
 */
#ifndef UCORES_CUDA_H
#define UCORES_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UCG_ABI_VERSION 1

enum {
  UCG_OK = 0,
  UCG_ERR_CUDA = -1,     /* CUDA runtime / launch error (message has cudaGetErrorString) */
  UCG_ERR_ARG = -2,      /* invalid argument (null, misaligned, bad size) */
  UCG_ERR_NODEV = -3,    /* no CUDA device, or not compute capability 10.x */
  UCG_ERR_LENGTH = -4,   /* element lengths differ (reference LengthMismatch, errors.hpp:112) */
  UCG_ERR_EMPTY = -5,    /* reduce over zero elements (reference EmptyDataset, errors.hpp:80) */
  UCG_ERR_NCCL = -6,     /* collective failure */
  UCG_ERR_PEER = -7      /* a sharded exchange timed out in an earlier launch: a peer never
                            published (that launch wrote NaN / -1 and kept its epoch); every
                            call on the exchange fails until ucg_xchg_reset */
};

/* reduce operators: the combine of the binary kernels sum2 / max2 / isum2 */
enum { UCG_OP_SUM = 0, UCG_OP_MAX = 1 };

/* ------------------------------------------------------------------------ */
/* runtime                                                                   */
/* ------------------------------------------------------------------------ */

const char* ucg_last_error(void);
int ucg_abi_version(void);

/* Replaces the inventory enumeration of GPU devices
 * (ucores/device.hpp:212-242 default_inventory / enumerate_platforms). */
int ucg_device_count(int* n_out);

typedef struct ucg_device_info {
  char name[128];
  int ordinal;
  int cc_major, cc_minor;
  int sm_count;
  uint64_t hbm_bytes;
  uint64_t l2_bytes;
} ucg_device_info;
int ucg_device_info_get(int ordinal, ucg_device_info* out);
int ucg_set_device(int ordinal);
/** The calling thread's current device (cudaGetDevice). */
int ucg_get_device(int* ordinal_out);

/* Device / pinned-host memory and copies (the partition upload path; replaces
 * the host copies at ucores/kernel.hpp:103-112 bind and :137-147 take). */
int ucg_malloc(void** dptr, uint64_t bytes);
int ucg_free(void* dptr);
int ucg_host_alloc(void** hptr, uint64_t bytes); /* page-locked */
int ucg_host_free(void* hptr);
int ucg_host_register(void* hptr, uint64_t bytes);
int ucg_host_unregister(void* hptr);
int ucg_memcpy_h2d(void* dst, const void* src, uint64_t bytes, void* stream);
int ucg_memcpy_d2h(void* dst, const void* src, uint64_t bytes, void* stream);
int ucg_memcpy_d2d(void* dst, const void* src, uint64_t bytes, void* stream);
/* Strided copy (cudaMemcpy2DAsync, direction inferred from the pointers, so
 * host, device and peer-device addresses all work): `rows` rows of
 * `width_bytes`, source / destination rows `spitch` / `dpitch` bytes apart. */
int ucg_memcpy2d(void* dst, uint64_t dpitch, const void* src, uint64_t spitch, uint64_t width_bytes,
                 uint64_t rows, void* stream);
int ucg_memset(void* dst, int value, uint64_t bytes, void* stream);
int ucg_stream_create(void** stream_out);
int ucg_stream_destroy(void* stream);
int ucg_stream_synchronize(void* stream);
int ucg_event_create(void** ev_out);
int ucg_event_destroy(void* ev);
int ucg_event_record(void* ev, void* stream);
int ucg_event_synchronize(void* ev);
int ucg_stream_wait_event(void* stream, void* ev);
int ucg_event_elapsed_ms(void* ev_start, void* ev_end, float* ms_out); /* synchronizes on ev_end */
int ucg_device_synchronize(void);

/* Number of kernel launches this library issued on this process (all
 * devices). Used by bench.py for gpu_launches. */
uint64_t ucg_launch_count(void);

/* ------------------------------------------------------------------------ */
/* synthetic inputs (bench / tests; not on the hot path)                      */
/* ------------------------------------------------------------------------ */

/* out[i] = float(mix64(seed + (first+i+1)*GAMMA) >> 40) * 2^-24  in [0,1) */
int ucg_fill_uniform_f32(float* out, uint64_t n, uint64_t seed, uint64_t first, void* stream);
/* out[i] = byte(mix64(seed + (first+i+1)*GAMMA) >> 56) */
int ucg_fill_bytes_u8(uint8_t* out, uint64_t n, uint64_t seed, uint64_t first, void* stream);

/* ------------------------------------------------------------------------ */
/* segment tables: the device mirror of a Dataset's partitions                */
/* ------------------------------------------------------------------------ */

/* A segment = one partition's concatenated payload (ucores/engine.hpp:102,
 * Element::concat element.hpp:132-174) stored contiguously in a device buffer
 * at float offset begin[s] (multiple of 4) with len[s] floats. The table is
 * uploaded once (synchronously) on the current device and reused by every
 * launch over that layout on that device; it also carries the launches'
 * work-item counters (two sets, used by alternate launches), so it serves
 * one stream at a time: launches on it are stream-ordered, and a repeated
 * step may overlap only the step before it (see ucg_segtab_scratch_floats). */
typedef struct ucg_segtab ucg_segtab;
int ucg_segtab_create(const uint64_t* begin, const uint64_t* len, uint64_t nseg, ucg_segtab** out);
int ucg_segtab_destroy(ucg_segtab* t);
/* scratch floats the segment reductions need for a table: two halves of
 * work-item partials, used by alternate launches on the table, so a repeated
 * step (same table, buffers, map and op as the kernel before it in the
 * stream) streams while the previous step's partition trees finish. The
 * scratch must stay the same buffer across such repeated steps. */
int ucg_segtab_scratch_floats(const ucg_segtab* t, uint64_t* n_out);

/* ------------------------------------------------------------------------ */
/* hot path: map kernels (mapCL, ucores/engine.hpp:54-85)                     */
/* ------------------------------------------------------------------------ */

/* axpb run() body over n floats: y[i] = fl(fl(a*x[i]) + b) (no FMA
 * contraction, bit-identical to the host executor). x, y 16-byte aligned;
 * y may equal x. Large maps hand out 16 KB work items from a per-launch
 * counter (a memset node precedes the kernel). */
int ucg_map_affine_f32(const float* x, float* y, uint64_t n, float a, float b, void* stream);

/* Fig-3 vectoradd body: c = a (op) b. */
int ucg_elementwise2_f32(const float* a, const float* b, float* c, uint64_t n, int op, void* stream);
int ucg_elementwise2_i64(const int64_t* a, const int64_t* b, int64_t* c, uint64_t n, void* stream);

/* ------------------------------------------------------------------------ */
/* hot path: partition reductions (mapCLPartition psum/pmax,                  */
/* ucores/engine.hpp:89-114) and the reduceCL tree (engine.hpp:121-192)       */
/* ------------------------------------------------------------------------ */

/* out[s] = pairing-tree reduction (engine.hpp:172-190 rule applied to the
 * elements of segment s; op SUM: a+b, MAX: std::max) of segment s of x.
 * Empty segment: +0.0f (SUM) / -inf (MAX). scratch: ucg_segtab_scratch_floats
 * floats of device memory. Bit-identical to the host psum/pmax kernels.
 * One launch (work items claimed from the table's counter, trees in the
 * kernel's tail). */
int ucg_segment_reduce_f32(const float* x, const ucg_segtab* t, int op, float* scratch,
                           float* out, void* stream);

/* Fused mapCL(axpb) -> mapCLPartition(psum|pmax): y = fl(fl(a*x)+b) is
 * written for every element of every segment AND out[s] is the tree
 * reduction of y over segment s, in one pass over HBM (8 B/elem instead of
 * 12). Results are bit-identical to the unfused pair. */
int ucg_map_affine_segment_reduce_f32(const float* x, float* y, const ucg_segtab* t, float a,
                                      float b, int op, float* scratch, float* out, void* stream);

/* Peer-exchange context for a reduce_cl over a collection sharded across
 * GPUs, one process per GPU (replaces the ReducePair waves of stage 2 that
 * combine partials living on different workers, engine.hpp:172-190). Each
 * rank owns nloc consecutive partitions starting at part_offset of p_total.
 * Setup: create -> export the IPC handle (ucg_xchg_handle_bytes bytes) ->
 * exchange handles out of band (e.g. torch.distributed all_gather) -> open
 * with all ranks' handles in rank order. */
typedef struct ucg_xchg ucg_xchg;
int ucg_xchg_create(int world, int rank, uint64_t nloc, uint64_t part_offset, uint64_t p_total, ucg_xchg** out);
uint64_t ucg_xchg_handle_bytes(void);
int ucg_xchg_export(const ucg_xchg* x, void* handle_out);
int ucg_xchg_open(ucg_xchg* x, const void* all_handles);
int ucg_xchg_error(const ucg_xchg* x, int* err_out); /* 1 if a peer never arrived (synchronous) */
/* The same error word read without synchronizing (it is host-mapped: the
 * value of every launch that has completed so far). */
int ucg_xchg_poll(const ucg_xchg* x, int* err_out);
/* Recovery after UCG_ERR_PEER, called by EVERY rank between two barriers,
 * with no exchange launch in flight: clears the error word, the epoch and
 * this rank's region (its slots and flags). */
int ucg_xchg_reset(ucg_xchg* x);
int ucg_xchg_destroy(ucg_xchg* x);

/* mapCLPartition(psum|pmax) + reduceCL stage 2 in ONE launch: the kernel
 * streams the segments' work items (fused with the axpb map when y != NULL:
 * y is written), then — in its tail, under a cooperative launch — reduces
 * each segment to `partials` and runs the pairing tree over all partitions
 * into `result` (device, one float). With xchg != NULL the last CTA first
 * stores this rank's partials into every peer's buffer over NVLink and waits
 * for all ranks' epoch flags, so every rank obtains the same,
 * reference-ordered result with no separate collective launch. The table
 * holds the launch's counters: a segment table / exchange must not be used
 * by two launches concurrently (the calls on one stream serialise). */
int ucg_segment_reduce_cl_f32(const float* x, float* y, const ucg_segtab* t, float a, float b, int op,
                              float* scratch, float* partials, ucg_xchg* xchg, float* result, void* stream);

/* reduce_cl stage 2 alone, sharded: this rank's nloc partition values
 * (device, already computed — e.g. by per-chunk launches overlapping an
 * upload) go through the same NVLink exchange as ucg_segment_reduce_cl_f32's
 * tail, and *result (device) is the reference pairing tree over all ranks'
 * values in partition order. One single-CTA launch, no collective call. */
int ucg_reduce_cl_xchg_f32(float* partials, uint64_t nloc, int op, ucg_xchg* xchg, float* result, void* stream);

/* Sharded map_cl(pi) + reduce_cl(isum2) (C3 over GPUs, one process per
 * GPU): ucg_pi_hits_total over this rank's tasks, and the last CTA of the
 * launch exchanges the rank totals over NVLink (8-byte P2P stores into every
 * peer's region + epoch flags, as ucg_segment_reduce_cl_f32) so *total_out
 * ends as the sum over ALL ranks — no collective call. xchg: created with
 * nloc = 2, part_offset = 2*rank, p_total = 2*world, opened. A rank with no
 * tasks still joins the exchange. */
int ucg_pi_hits_total_xchg(const uint64_t* seeds, const uint64_t* samples, uint64_t ntasks, int64_t* hits_out,
                           int64_t* total_out, ucg_xchg* xchg, void* stream);

/* reduceCL stage 2 over n one-float partials in partition order: the pairing
 * tree with odd promotion (engine.hpp:172-190). out: one float (device). */
int ucg_tree_reduce_f32(const float* x, uint64_t n, int op, float* out, void* stream);

/* Full reduceCL over vector elements with an elementwise binary kernel
 * (sum2 / max2 / vectoradd / isum2): stage 1 left fold inside each partition
 * (engine.hpp:144-170), stage 2 pairing tree over partition partials
 * (engine.hpp:172-190), lane by lane. elem_ptrs: device array of `count`
 * device pointers to elements of `len` values each, in collect() order;
 * part_counts: HOST array of per-partition element counts (nparts entries).
 * Returns UCG_ERR_EMPTY when count == 0. */
int ucg_reduce_cl_f32(const float* const* elem_ptrs, uint64_t count, uint64_t len,
                      const uint64_t* part_counts, uint64_t nparts, int op, float* out,
                      void* stream);
int ucg_reduce_cl_i64(const int64_t* const* elem_ptrs, uint64_t count, uint64_t len,
                      const uint64_t* part_counts, uint64_t nparts, int64_t* out, void* stream);

/* ------------------------------------------------------------------------ */
/* Monte-Carlo pi: one task per element {seed, samples}     */
/* ------------------------------------------------------------------------ */

/* hits_out[t] (device int64) = number of gids in [0, samples[t]) whose
 * SplitMix64 point (seed[t] ^ gid*GAMMA) lies in the unit quarter circle,
 * bit-identical to the IEEE-double host test. seeds / samples: HOST arrays. */
int ucg_pi_hits(const uint64_t* seeds, const uint64_t* samples, uint64_t ntasks, int64_t* hits_out,
                void* stream);
/* Same launch, plus the reduce_cl(isum2) of the task results into *total_out
 * (device int64, overwritten): the sum over all tasks' hits (integer, so any
 * tree order gives the same value — engine.hpp:121-192). total_out may be
 * NULL. */
int ucg_pi_hits_total(const uint64_t* seeds, const uint64_t* samples, uint64_t ntasks, int64_t* hits_out,
                      int64_t* total_out, void* stream);
/* Class-D form for the seam-B executor: flags[gid] = hit(seed, gid) (device u8). */
int ucg_pi_flags(uint64_t seed, uint64_t samples, uint8_t* flags, void* stream);

/* ------------------------------------------------------------------------ */
/* 3x3 Sobel on row bands (workload C4)                                       */
/* ------------------------------------------------------------------------ */

/* in: (rows_out+2) x width bytes (one halo row above and below), out:
 * rows_out x width bytes. out = min(255, |Gx|+|Gy|), zero outside columns. */
int ucg_sobel_band_u8(const uint8_t* in, uint8_t* out, uint64_t rows_out, uint64_t width,
                      void* stream);
/* nbands bands in one launch; band b input at in + in_off[b], output at
 * out + out_off[b], rows[b] output rows; offsets/rows are HOST arrays. */
int ucg_sobel_bands_u8(const uint8_t* in, const uint64_t* in_off, uint8_t* out,
                       const uint64_t* out_off, const uint64_t* rows, uint64_t nbands,
                       uint64_t width, void* stream);

/* ------------------------------------------------------------------------ */
/* WordCount word-start flags                */
/* ------------------------------------------------------------------------ */

/* The wordcount kernel's run() over one chunk: flags[gid] = 1 iff bytes[gid]
 * is a word character and (gid == 0 or bytes[gid-1] is a delimiter: space,
 * tab, LF, CR — ucores/dataset.hpp:87-89), else 0. Device u8 arrays.
 * create_from_text chunks end on a delimiter, so one call over consecutive
 * chunks equals the per-chunk calls. */
int ucg_word_start_flags(const uint8_t* bytes, uint64_t n, uint8_t* flags, void* stream);

/* ------------------------------------------------------------------------ */
/* dense matmul (workload C5): tcgen05 tensor cores                           */
/* ------------------------------------------------------------------------ */

/* C = A * B, n x n row-major fp32 in, fp32 out, TF32 tensor-core math with
 * fp32 accumulation in TMEM. n must be a multiple of 128. */
int ucg_gemm_tf32(const float* A, const float* B, float* C, uint64_t n, void* stream);

/* Same product, fp32-faithful ("3xTF32"): A and B are split into TF32
 * hi + lo halves (hi = round-to-nearest TF32, lo = x - hi, exact) and the
 * tensor cores accumulate Ahi*Bhi + Ahi*Blo + Alo*Bhi in fp32 (TMEM) — the
 * k range is cut into chunks of 256, each accumulated from zero in TMEM and
 * added to C with an fp32 round-to-nearest add (the tensor core's own fp32
 * accumulation truncates). Error: rms 2.7e-6 of rms(C) at any n (cuBLAS
 * SGEMM: 0.3-1.6e-6; TF32: 7e-4), at ~a third of the TF32 rate. Finite data
 * only: an inf operand turns into nan (inf * the zero lo half of an exact
 * partner). Workspace 4 n^2 floats from the stream-ordered pool. */
int ucg_gemm_f32(const float* A, const float* B, float* C, uint64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* UCORES_CUDA_H */
