// ucg_common.cuh — shared internals of libucores_cuda.so (sm_100a only).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>

#include "ucores_cuda.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libucores_cuda targets sm_100a only"
#endif

struct ucg_xchg;

namespace ucg {

// ---- error state ------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
int check_device();  // UCG_OK when the current device is compute capability 10.x
int xchg_guard(const ::ucg_xchg* x);  // UCG_ERR_PEER once a peer wait has timed out
int sm_count();      // SMs of the current device (cached per device)
extern std::atomic<uint64_t> g_launches;

// An 8-byte claim counter on the current device for one launch of a kernel
// that hands out work items dynamically (the next slot of a per-device ring;
// the caller zeroes it on its stream before the launch). Null if the ring
// cannot be allocated.
unsigned long long* claim_counter();

// A {claims, exit tickets} pair of 8-byte counters for a kernel that resets
// them itself (the last CTA to exit zeroes both), from a ring zeroed once at
// allocation: no memset launch before each use. Null if the ring cannot be
// allocated.
unsigned long long* claim_pair_selfreset();

// True the first time it is called on the current device for this flag word.
// Kernel attributes (cudaFuncSetAttribute) are per device: a process driving
// several GPUs (the seam-A driver) must set them on each one.
inline bool first_on_device(std::atomic<uint64_t>& seen) {
  int d = 0;
  cudaGetDevice(&d);
  const uint64_t bit = 1ull << (d & 63);
  return !(seen.fetch_or(bit) & bit);
}

#define UCG_CUDA(call)                                  \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return ::ucg::cuda_fail(_e, #call); \
  } while (0)

// after a <<<>>> launch
#define UCG_LAUNCHED()                                          \
  do {                                                          \
    ::ucg::g_launches.fetch_add(1, std::memory_order_relaxed);  \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::ucg::cuda_fail(_e, "kernel launch"); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- device helpers -----------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t umin(uint64_t a, uint64_t b) { return a < b ? a : b; }
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// The two reduce combines. SUM: IEEE a+b (identity -0.0f, exact for every
// operand); MAX: std::max(a,b) == (a<b)?b:a (identity -inf as right operand).
struct OpSum {
  static constexpr int kId = 0;
  static __device__ __forceinline__ float apply(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float identity() { return -0.0f; }
  static __device__ __forceinline__ float empty() { return 0.0f; }
};
struct OpMax {
  static constexpr int kId = 1;
  static __device__ __forceinline__ float apply(float a, float b) { return (a < b) ? b : a; }
  static __device__ __forceinline__ float identity() { return __int_as_float(0xff800000); }
  static __device__ __forceinline__ float empty() { return __int_as_float(0xff800000); }
};

// streaming 128-bit global accesses (data is touched exactly once)
// Peer waits give up (and raise the exchange's error flag) after this long:
// generous, so a rank that is late to its first step (lazy module loading,
// graph capture, host-side set-up) is waited for, while a dead peer still
// surfaces as an error instead of a hang.
constexpr uint64_t kPeerWaitNs = 30ull * 1000 * 1000 * 1000;
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }

}  // namespace ucg

// segment table (opaque to C callers)
struct ucg_segtab {
  int device;
  uint64_t nseg;
  uint64_t nitems;         // work items over all segments
  uint64_t* d_begin;       // [nseg]
  uint64_t* d_len;         // [nseg]
  uint64_t* d_first_item;  // [nseg+1]
  uint32_t* d_item_seg;    // [nitems]
  uint64_t max_items_per_seg;
  int item_log2;           // work-item size (floats) = 2^item_log2, chosen per table
  uint32_t* d_done;        // [2][4] pass-1 exit / finisher / item counters per launch parity
                           // (zero between launches of that parity)
  uint64_t ntaper;         // trailing items the fused map streams as 4 sub-items each (0: none)
  unsigned long long* d_gen;  // [2][2] per parity: start tickets, completed fused grids (never reset)
  mutable uint64_t launches = 0;  // pass-1 launches so far: parity selects the counter and scratch half
};

// Peer-exchange context of a sharded reduce_cl (one process per GPU).
struct ucg_xchg {
  int device;
  int world, rank;
  uint64_t nloc, part_offset, p_total;
  uint64_t region_bytes, flags_offset;
  uint8_t* region;          // this rank's IPC-exported buffer: [2 x p_total floats | flags[world]]
                            // (value buffer by epoch parity: a rank one step ahead never
                            // overwrites values a peer may still be reading)
  uint64_t* d_peers;        // [world] device addresses of every rank's region (mapped)
  uint8_t** peer_ptrs;      // host copy (opened IPC handles, own region at [rank])
  uint32_t* h_err;          // error word in mapped pinned host memory: kernels store 1 on a
  uint32_t* d_err;          // peer timeout (d_err = its device alias); entry points read h_err
                            // without a sync and refuse to launch while it is set
  uint32_t* d_epoch;        // exchanges completed by this rank (advanced on the device, so
                            // sharded steps can be replayed from CUDA graphs)
  bool opened;
};

namespace ucg {
// Floats of scratch one pass-1 launch uses (item roots, then the tapered
// tail's sub-roots), rounded to 16 bytes; the caller's scratch holds two such
// halves, used by alternate launches so a step's stream can overlap the
// previous step's partition trees (ucg_reduce.cu segment_reduce).
inline uint64_t scratch_half(const ucg_segtab* t) {
  const uint64_t n = t->ntaper ? ((t->nitems + 4) & ~uint64_t(3)) + 4 * t->ntaper : t->nitems + 1;
  return (n + 3) & ~uint64_t(3);
}
// Work item = one aligned block of 2^item_log2 floats of one segment (the
// last item of a segment may be partial). The size is picked per segment
// table in [2^11, 2^14] so the last wave of warps is nearly full.
constexpr int kMinItemLog2 = 10;  // one 1024-float chunk
constexpr int kMaxItemLog2 = 14;
}  // namespace ucg
