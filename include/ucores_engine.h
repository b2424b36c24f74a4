/*
 * ucores_engine.h — C-ABI of libucores_engine.so: the C++ drop-in
 * (GpuClusterDriver / CudaExecutor under the unmodified reference
 * ucores::Engine) exposed to FFI callers such as Python's ctypes (bench.py
 * uses it to time the end-to-end path through the reference API).
 *
 * Status convention as ucores_cuda.h: 0 ok, <0 error, message in
 * ucd_last_error(). Reference exceptions map to codes:
 *   UCD_ERR_JOB_FAILED  ucores::JobFailed     (errors.hpp:84-87)
 *   UCD_ERR_EMPTY       ucores::EmptyDataset  (errors.hpp:80-83)
 *   UCD_ERR_ARITY       ucores::ArityMismatch (errors.hpp:45-48)
 *   UCD_ERR_UNKNOWN     ucores::UnknownKernel (errors.hpp:41-44)
 *   UCD_ERR_OTHER       any other ucores::Error / std::exception
 */
#ifndef UCORES_ENGINE_H
#define UCORES_ENGINE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  UCD_OK = 0,
  UCD_ERR_JOB_FAILED = -10,
  UCD_ERR_EMPTY = -11,
  UCD_ERR_ARITY = -12,
  UCD_ERR_UNKNOWN = -13,
  UCD_ERR_OTHER = -14
};

/* BATCHED: Engine + GpuClusterDriver (seam A, one launch per kernel per GPU
 * per wave); PER_TASK: Engine + GpuWorkerRuntime/CudaExecutor (seam B);
 * DEVICE: DeviceEngine (device_dataset.hpp) — the dataset is
 * uploaded once and the chain stays in HBM. */
enum { UCD_MODE_BATCHED = 0, UCD_MODE_PER_TASK = 1, UCD_MODE_DEVICE = 2 };

const char* ucd_last_error(void);

/* The C2 pipeline through ucores::Engine (engine.hpp:54-192) with the GPU
 * drivers: x holds `nparts` partitions back to back (part_lens[p] floats
 * each, one F32Array element per partition);
 *   y = map_cl(x, "axpb"(a,b)); ps = map_cl_partition(y, "psum"|"pmax");
 *   r = reduce_cl(ps, "sum2"|"max2")
 * y_out (nullable, sum(part_lens) floats) receives the collected y,
 * partials_out (nullable, nparts) the psum/pmax dataset, result_out the
 * reduced value. seconds_out: wall time from the built host Dataset to the
 * result Element (the reference arm times its Engine the same way). gpus <= 0:
 * every visible GPU. */
int ucd_pipeline_f32(const float* x, const uint64_t* part_lens, uint64_t nparts, float a, float b, int op,
                     int gpus, int mode, float* y_out, float* partials_out, float* result_out,
                     double* seconds_out);

/* ucd_pipeline_f32 (BATCHED mode) with a time breakdown, for profiling the
 * drop-in: out8 = {map_cl seconds, of which inside the driver's run_wave,
 * map_cl_partition seconds, of which run_wave, reduce_cl seconds, of which
 * run_wave, the whole chain, the result's fp32 bit pattern}. Time outside
 * run_wave is the reference Engine's own work (task input copies,
 * Element::concat, result assembly). */
int ucd_pipeline_breakdown_f32(const float* x, const uint64_t* part_lens, uint64_t nparts, float a, float b, int op,
                               int gpus, double* out8);

/* The C1 literal form: n one-float elements x[i] in nparts
 * partitions (create_dataset, ceiling-first), then the same chain as
 * ucd_pipeline_f32. map_cl is one task per element in the reference; the GPU
 * paths batch the wave (BATCHED) or keep the dataset in HBM (DEVICE).
 * seconds_out: wall time from the host array to the result (Dataset
 * construction included). */
int ucd_literal_f32(const float* x, uint64_t n, uint64_t nparts, float a, float b, int op, int gpus, int mode,
                    float* result_out, double* seconds_out);

/* Monte-Carlo pi through Engine::map_cl(d, "pi") over `tasks` elements
 * {seed + t, samples split ceiling-first}: hits_out receives the total. */
int ucd_pi(uint64_t samples, uint64_t tasks, uint64_t seed, int gpus, int64_t* hits_out, double* seconds_out);

#ifdef __cplusplus
}
#endif
#endif /* UCORES_ENGINE_H */
