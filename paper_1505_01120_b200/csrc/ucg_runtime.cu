// ucg_runtime.cu — device runtime of libucores_cuda.so: error state, device
// enumeration (the GPU half of ucores/device.hpp:212-242), memory, streams,
// events, synthetic-input fills and segment tables.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include <algorithm>

#include "ucg_common.cuh"

namespace ucg {

static thread_local std::string t_last_error;
std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { t_last_error = msg; }

int fail(int code, const std::string& msg) {
  t_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  t_last_error = std::string(what) + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e);
  return e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? UCG_ERR_NODEV : UCG_ERR_CUDA;
}

namespace {
struct DevCache {
  int sms = 0;
  int major = 0;
};
std::mutex g_dev_mu;
DevCache g_dev[64];

const DevCache* dev_cache(int* dev_out) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  *dev_out = dev;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (g_dev[dev].sms == 0) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return nullptr;
    g_dev[dev].sms = p.multiProcessorCount;
    g_dev[dev].major = p.major;
    // stream-ordered workspaces (reduce_cl partials, the 3xTF32 split) stay
    // mapped in the device's default pool between calls instead of being
    // unmapped at every synchronize (a 1 GB re-map costs milliseconds)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
  return &g_dev[dev];
}
}  // namespace

// Entry-point guard of every launch on an exchange (reads the host-mapped
// error word: no device sync).
int xchg_guard(const ucg_xchg* x) {
  if (*reinterpret_cast<volatile uint32_t*>(x->h_err))
    return fail(UCG_ERR_PEER, "peer exchange timed out in an earlier launch (ucg_xchg_reset on every rank to recover)");
  return UCG_OK;
}

int check_device() {
  int dev = -1;
  const DevCache* c = dev_cache(&dev);
  if (!c) {
    cudaGetLastError();
    return fail(UCG_ERR_NODEV, "no usable CUDA device (libucores_cuda has no CPU fallback)");
  }
  if (c->major != 10) {
    return fail(UCG_ERR_NODEV, "device " + std::to_string(dev) +
                                   " is not compute capability 10.x (built for sm_100a only)");
  }
  return UCG_OK;
}

unsigned long long* claim_counter() {
  // a ring of 2^16 counters per device (512 KB): each launch takes the next
  // slot, so concurrent launches (any streams) use distinct counters unless
  // 65536 launches are in flight at once
  constexpr uint64_t kSlots = 1u << 16;
  static std::mutex mu;
  static unsigned long long* ring[64] = {};
  static uint64_t next[64] = {};
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!ring[d]) {
    if (cudaMalloc(&ring[d], kSlots * sizeof(unsigned long long)) != cudaSuccess) {
      ring[d] = nullptr;
      return nullptr;
    }
  }
  return ring[d] + (next[d]++ % kSlots);
}

unsigned long long* claim_pair_selfreset() {
  // every user of this ring leaves its pair at zero when its launch ends, so
  // a slot handed out again (after 2^15 later launches) is clean
  constexpr uint64_t kPairs = 1u << 15;
  static std::mutex mu;
  static unsigned long long* ring[64] = {};
  static uint64_t next[64] = {};
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!ring[d]) {
    unsigned long long* r = nullptr;
    if (cudaMalloc(&r, kPairs * 2 * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    if (cudaMemset(r, 0, kPairs * 2 * sizeof(unsigned long long)) != cudaSuccess) {
      cudaFree(r);
      return nullptr;
    }
    ring[d] = r;
  }
  return ring[d] + 2 * (next[d]++ % kPairs);
}

int sm_count() {
  int dev = -1;
  const DevCache* c = dev_cache(&dev);
  return c ? c->sms : 148;
}

// ---- fills -------------------------------------------------------------------
__global__ void k_fill_uniform(float* __restrict__ out, uint64_t n, uint64_t seed, uint64_t first) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    out[i] = float(mix64(seed + (first + i + 1) * kGamma) >> 40) * (1.0f / 16777216.0f);
  }
}
__global__ void k_fill_bytes(uint8_t* __restrict__ out, uint64_t n, uint64_t seed, uint64_t first) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    out[i] = uint8_t(mix64(seed + (first + i + 1) * kGamma) >> 56);
  }
}

// ---- segment table -------------------------------------------------------------
}  // namespace ucg

using namespace ucg;

extern "C" {

const char* ucg_last_error(void) { return t_last_error.c_str(); }
int ucg_abi_version(void) { return UCG_ABI_VERSION; }

int ucg_device_count(int* n_out) {
  if (!n_out) return fail(UCG_ERR_ARG, "n_out is null");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *n_out = 0;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return UCG_OK;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *n_out = n;
  return UCG_OK;
}

int ucg_device_info_get(int ordinal, ucg_device_info* out) {
  if (!out) return fail(UCG_ERR_ARG, "out is null");
  cudaDeviceProp p;
  UCG_CUDA(cudaGetDeviceProperties(&p, ordinal));
  std::memset(out, 0, sizeof *out);
  std::strncpy(out->name, p.name, sizeof out->name - 1);
  out->ordinal = ordinal;
  out->cc_major = p.major;
  out->cc_minor = p.minor;
  out->sm_count = p.multiProcessorCount;
  out->hbm_bytes = p.totalGlobalMem;
  out->l2_bytes = p.l2CacheSize;
  return UCG_OK;
}

int ucg_set_device(int ordinal) {
  UCG_CUDA(cudaSetDevice(ordinal));
  return UCG_OK;
}
int ucg_get_device(int* ordinal_out) {
  if (!ordinal_out) return fail(UCG_ERR_ARG, "ordinal_out is null");
  UCG_CUDA(cudaGetDevice(ordinal_out));
  return UCG_OK;
}

int ucg_malloc(void** dptr, uint64_t bytes) {
  if (!dptr) return fail(UCG_ERR_ARG, "dptr is null");
  *dptr = nullptr;
  if (bytes == 0) return UCG_OK;
  UCG_CUDA(cudaMalloc(dptr, bytes));
  return UCG_OK;
}
int ucg_free(void* dptr) {
  if (dptr) UCG_CUDA(cudaFree(dptr));
  return UCG_OK;
}
int ucg_host_alloc(void** hptr, uint64_t bytes) {
  if (!hptr) return fail(UCG_ERR_ARG, "hptr is null");
  *hptr = nullptr;
  if (bytes == 0) return UCG_OK;
  UCG_CUDA(cudaHostAlloc(hptr, bytes, cudaHostAllocPortable));
  return UCG_OK;
}
int ucg_host_free(void* hptr) {
  if (hptr) UCG_CUDA(cudaFreeHost(hptr));
  return UCG_OK;
}
int ucg_host_register(void* hptr, uint64_t bytes) {
  if (!hptr || !bytes) return UCG_OK;
  UCG_CUDA(cudaHostRegister(hptr, bytes, cudaHostRegisterPortable));
  return UCG_OK;
}
int ucg_host_unregister(void* hptr) {
  if (hptr) UCG_CUDA(cudaHostUnregister(hptr));
  return UCG_OK;
}
int ucg_memcpy_h2d(void* dst, const void* src, uint64_t bytes, void* stream) {
  if (!bytes) return UCG_OK;
  UCG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream)));
  return UCG_OK;
}
int ucg_memcpy_d2h(void* dst, const void* src, uint64_t bytes, void* stream) {
  if (!bytes) return UCG_OK;
  UCG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
  return UCG_OK;
}
int ucg_memcpy_d2d(void* dst, const void* src, uint64_t bytes, void* stream) {
  if (!bytes) return UCG_OK;
  UCG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, as_stream(stream)));
  return UCG_OK;
}
int ucg_memcpy2d(void* dst, uint64_t dpitch, const void* src, uint64_t spitch, uint64_t width_bytes,
                 uint64_t rows, void* stream) {
  if (!width_bytes || !rows) return UCG_OK;
  if (!dst || !src) return fail(UCG_ERR_ARG, "null pointer");
  UCG_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width_bytes, rows, cudaMemcpyDefault, as_stream(stream)));
  return UCG_OK;
}
int ucg_memset(void* dst, int value, uint64_t bytes, void* stream) {
  if (!bytes) return UCG_OK;
  UCG_CUDA(cudaMemsetAsync(dst, value, bytes, as_stream(stream)));
  return UCG_OK;
}
int ucg_stream_create(void** s) {
  if (!s) return fail(UCG_ERR_ARG, "stream_out is null");
  cudaStream_t st;
  UCG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  *s = st;
  return UCG_OK;
}
int ucg_stream_destroy(void* s) {
  if (s) UCG_CUDA(cudaStreamDestroy(as_stream(s)));
  return UCG_OK;
}
int ucg_stream_synchronize(void* s) {
  UCG_CUDA(cudaStreamSynchronize(as_stream(s)));
  return UCG_OK;
}
int ucg_event_create(void** ev) {
  if (!ev) return fail(UCG_ERR_ARG, "ev_out is null");
  cudaEvent_t e;
  UCG_CUDA(cudaEventCreate(&e));
  *ev = e;
  return UCG_OK;
}
int ucg_event_destroy(void* ev) {
  if (ev) UCG_CUDA(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(ev)));
  return UCG_OK;
}
int ucg_event_record(void* ev, void* stream) {
  UCG_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev), as_stream(stream)));
  return UCG_OK;
}
int ucg_event_synchronize(void* ev) {
  UCG_CUDA(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(ev)));
  return UCG_OK;
}
int ucg_stream_wait_event(void* stream, void* ev) {
  UCG_CUDA(cudaStreamWaitEvent(as_stream(stream), reinterpret_cast<cudaEvent_t>(ev), 0));
  return UCG_OK;
}
int ucg_event_elapsed_ms(void* a, void* b, float* ms) {
  if (!ms) return fail(UCG_ERR_ARG, "ms_out is null");
  UCG_CUDA(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(b)));
  UCG_CUDA(cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(a), reinterpret_cast<cudaEvent_t>(b)));
  return UCG_OK;
}
int ucg_device_synchronize(void) {
  UCG_CUDA(cudaDeviceSynchronize());
  return UCG_OK;
}
uint64_t ucg_launch_count(void) { return g_launches.load(); }

int ucg_fill_uniform_f32(float* out, uint64_t n, uint64_t seed, uint64_t first, void* stream) {
  if (int rc = check_device()) return rc;
  if (!n) return UCG_OK;
  if (!out) return fail(UCG_ERR_ARG, "out is null");
  const unsigned grid = unsigned(sm_count()) * 8;
  k_fill_uniform<<<grid, 256, 0, as_stream(stream)>>>(out, n, seed, first);
  UCG_LAUNCHED();
  return UCG_OK;
}
int ucg_fill_bytes_u8(uint8_t* out, uint64_t n, uint64_t seed, uint64_t first, void* stream) {
  if (int rc = check_device()) return rc;
  if (!n) return UCG_OK;
  if (!out) return fail(UCG_ERR_ARG, "out is null");
  const unsigned grid = unsigned(sm_count()) * 8;
  k_fill_bytes<<<grid, 256, 0, as_stream(stream)>>>(out, n, seed, first);
  UCG_LAUNCHED();
  return UCG_OK;
}

int ucg_segtab_create(const uint64_t* begin, const uint64_t* len, uint64_t nseg, ucg_segtab** out) {
  if (!out) return fail(UCG_ERR_ARG, "out is null");
  *out = nullptr;
  if (int rc = check_device()) return rc;
  if (nseg && (!begin || !len)) return fail(UCG_ERR_ARG, "begin/len is null");
  if (nseg >= (1ull << 32)) return fail(UCG_ERR_ARG, "too many segments");
  // work-item size: 2^12 floats (16 KB; items are claimed dynamically, so no
  // wave quantisation to fit), halved while that leaves fewer items than
  // resident warps. Sweeps (tools/scaling_probe.py, tools/kernel_times.py,
  // 2^27..2^30 floats): the fused map+reduce is best at 2^12 (smaller last
  // items at 8-GPU shard sizes); the read-only reduce claims two items per
  // atomic, since one claim per 2^12 items saturates the counter.
  int item_log2 = 12;
  while (item_log2 > kMinItemLog2) {
    uint64_t items = 0;
    for (uint64_t s = 0; s < nseg; ++s) items += (len[s] + (1ull << item_log2) - 1) >> item_log2;
    if (items >= uint64_t(sm_count()) * 16) break;
    --item_log2;
  }
  if (const char* e = getenv("UCG_ITEM_LOG2")) {  // tuning override (tools/)
    const int L = atoi(e);
    if (L >= kMinItemLog2 && L <= kMaxItemLog2) item_log2 = L;
  }
  std::vector<uint64_t> first(nseg + 1, 0);
  uint64_t maxi = 0;
  for (uint64_t s = 0; s < nseg; ++s) {
    if (begin[s] % 4) return fail(UCG_ERR_ARG, "segment " + std::to_string(s) + " begin is not 16-byte aligned");
    const uint64_t items = (len[s] + (1ull << item_log2) - 1) >> item_log2;
    first[s + 1] = first[s] + items;
    if (items > maxi) maxi = items;
  }
  const uint64_t nitems = first[nseg];
  std::vector<uint32_t> item_seg(nitems);
  for (uint64_t s = 0; s < nseg; ++s)
    for (uint64_t i = first[s]; i < first[s + 1]; ++i) item_seg[i] = uint32_t(s);
  auto* t = new ucg_segtab{};
  cudaGetDevice(&t->device);
  t->nseg = nseg;
  t->nitems = nitems;
  t->max_items_per_seg = maxi;
  t->item_log2 = item_log2;
  // tapered tail (A/B knob, off by default): UCG_TAPER=k streams the last k
  // items of the fused map as 4 aligned sub-items each and the finishers
  // recombine the sub-roots into the item roots (same association, results
  // bit-identical). Measured slower at every k (8-GPU shard: 168.4 us per
  // step off, 168.6 / 169.4 / 170.1 us at k = 148 / 592 / 1184): one-chunk
  // sub-items have no next chunk in flight, and the tail is not item-bound.
  {
    static const char* e = getenv("UCG_TAPER");
    const uint64_t want = e ? uint64_t(atoll(e)) : 0;
    t->ntaper = item_log2 >= 12 ? std::min<uint64_t>(nitems / 4, want) : 0;
  }
  auto cleanup = [&](cudaError_t e, const char* what) {
    cudaFree(t->d_begin);
    cudaFree(t->d_len);
    cudaFree(t->d_first_item);
    cudaFree(t->d_item_seg);
    cudaFree(t->d_done);
    cudaFree(t->d_gen);
    delete t;
    return cuda_fail(e, what);
  };
  cudaError_t e;
  if ((e = cudaMalloc(&t->d_begin, (nseg + 1) * 8)) != cudaSuccess) return cleanup(e, "cudaMalloc");
  if ((e = cudaMalloc(&t->d_len, (nseg + 1) * 8)) != cudaSuccess) return cleanup(e, "cudaMalloc");
  if ((e = cudaMalloc(&t->d_first_item, (nseg + 1) * 8)) != cudaSuccess) return cleanup(e, "cudaMalloc");
  if ((e = cudaMalloc(&t->d_item_seg, (nitems + 1) * 4)) != cudaSuccess) return cleanup(e, "cudaMalloc");
  if ((e = cudaMalloc(&t->d_done, 32)) != cudaSuccess) return cleanup(e, "cudaMalloc");
  if ((e = cudaMemset(t->d_done, 0, 32)) != cudaSuccess) return cleanup(e, "cudaMemset");
  if ((e = cudaMalloc(&t->d_gen, 32)) != cudaSuccess) return cleanup(e, "cudaMalloc");
  if ((e = cudaMemset(t->d_gen, 0, 32)) != cudaSuccess) return cleanup(e, "cudaMemset");
  if (nseg) {
    if ((e = cudaMemcpy(t->d_begin, begin, nseg * 8, cudaMemcpyHostToDevice)) != cudaSuccess) return cleanup(e, "cudaMemcpy");
    if ((e = cudaMemcpy(t->d_len, len, nseg * 8, cudaMemcpyHostToDevice)) != cudaSuccess) return cleanup(e, "cudaMemcpy");
  }
  if ((e = cudaMemcpy(t->d_first_item, first.data(), (nseg + 1) * 8, cudaMemcpyHostToDevice)) != cudaSuccess) return cleanup(e, "cudaMemcpy");
  if (nitems && (e = cudaMemcpy(t->d_item_seg, item_seg.data(), nitems * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
    return cleanup(e, "cudaMemcpy");
  *out = t;
  return UCG_OK;
}

int ucg_segtab_destroy(ucg_segtab* t) {
  if (!t) return UCG_OK;
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != t->device) cudaSetDevice(t->device);  // free on the table's own device
  cudaFree(t->d_begin);
  cudaFree(t->d_len);
  cudaFree(t->d_first_item);
  cudaFree(t->d_item_seg);
  cudaFree(t->d_done);
  cudaFree(t->d_gen);
  if (cur >= 0 && cur != t->device) cudaSetDevice(cur);
  delete t;
  return UCG_OK;
}

// ---- peer exchange (sharded reduce_cl over NVLink) ------------------------------

int ucg_xchg_create(int world, int rank, uint64_t nloc, uint64_t part_offset, uint64_t p_total, ucg_xchg** out) {
  if (!out) return fail(UCG_ERR_ARG, "out is null");
  *out = nullptr;
  if (int rc = check_device()) return rc;
  if (world < 1 || world > 64 || rank < 0 || rank >= world || part_offset + nloc > p_total)
    return fail(UCG_ERR_ARG, "bad exchange geometry");
  auto* x = new ucg_xchg{};
  cudaGetDevice(&x->device);
  x->world = world;
  x->rank = rank;
  x->nloc = nloc;
  x->part_offset = part_offset;
  x->p_total = p_total;
  // [2 parity buffers of p_total 64-bit {epoch, value} slots | p_total gathered
  //  floats | pad | flags[world]] (the flag protocol uses the first 2*p_total*4 B)
  x->flags_offset = (20 * p_total + 255) / 256 * 256;
  x->region_bytes = x->flags_offset + 256;
  x->peer_ptrs = new uint8_t*[world]();
  cudaError_t e;
  if ((e = cudaMalloc(&x->region, x->region_bytes)) != cudaSuccess || (e = cudaMemset(x->region, 0, x->region_bytes)) != cudaSuccess ||
      (e = cudaMalloc(&x->d_peers, world * 8)) != cudaSuccess || (e = cudaMalloc(&x->d_epoch, 4)) != cudaSuccess ||
      (e = cudaMemset(x->d_epoch, 0, 4)) != cudaSuccess ||
      (e = cudaHostAlloc(&x->h_err, 4, cudaHostAllocMapped)) != cudaSuccess ||
      (e = cudaHostGetDevicePointer(&x->d_err, x->h_err, 0)) != cudaSuccess) {
    cudaFree(x->region);
    cudaFree(x->d_peers);
    cudaFree(x->d_epoch);
    if (x->h_err) cudaFreeHost(x->h_err);
    delete[] x->peer_ptrs;
    delete x;
    return cuda_fail(e, "ucg_xchg_create");
  }
  *x->h_err = 0;
  *out = x;
  return UCG_OK;
}

uint64_t ucg_xchg_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int ucg_xchg_export(const ucg_xchg* x, void* handle_out) {
  if (!x || !handle_out) return fail(UCG_ERR_ARG, "null argument");
  cudaIpcMemHandle_t h;
  UCG_CUDA(cudaIpcGetMemHandle(&h, x->region));
  std::memcpy(handle_out, &h, sizeof h);
  return UCG_OK;
}

int ucg_xchg_open(ucg_xchg* x, const void* all_handles) {
  if (!x || !all_handles) return fail(UCG_ERR_ARG, "null argument");
  if (x->opened) return UCG_OK;
  const auto* hs = static_cast<const cudaIpcMemHandle_t*>(all_handles);
  std::vector<uint64_t> addrs(x->world);
  for (int r = 0; r < x->world; ++r) {
    if (r == x->rank) {
      x->peer_ptrs[r] = x->region;
    } else {
      void* p = nullptr;
      UCG_CUDA(cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess));
      x->peer_ptrs[r] = static_cast<uint8_t*>(p);
    }
    addrs[r] = reinterpret_cast<uint64_t>(x->peer_ptrs[r]);
  }
  UCG_CUDA(cudaMemcpy(x->d_peers, addrs.data(), x->world * 8, cudaMemcpyHostToDevice));
  x->opened = true;
  return UCG_OK;
}

int ucg_xchg_error(const ucg_xchg* x, int* err_out) {
  if (!x || !err_out) return fail(UCG_ERR_ARG, "null argument");
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != x->device) UCG_CUDA(cudaSetDevice(x->device));
  const cudaError_t e = cudaDeviceSynchronize();
  if (cur >= 0 && cur != x->device) cudaSetDevice(cur);
  UCG_CUDA(e);
  *err_out = int(*reinterpret_cast<volatile uint32_t*>(x->h_err));
  return UCG_OK;
}

int ucg_xchg_poll(const ucg_xchg* x, int* err_out) {
  if (!x || !err_out) return fail(UCG_ERR_ARG, "null argument");
  *err_out = int(*reinterpret_cast<volatile uint32_t*>(x->h_err));
  return UCG_OK;
}

int ucg_xchg_reset(ucg_xchg* x) {
  if (!x) return fail(UCG_ERR_ARG, "null argument");
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != x->device) UCG_CUDA(cudaSetDevice(x->device));
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemset(x->region, 0, x->region_bytes);
  if (e == cudaSuccess) e = cudaMemset(x->d_epoch, 0, 4);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (cur >= 0 && cur != x->device) cudaSetDevice(cur);
  UCG_CUDA(e);
  *reinterpret_cast<volatile uint32_t*>(x->h_err) = 0;
  return UCG_OK;
}

int ucg_xchg_destroy(ucg_xchg* x) {
  if (!x) return UCG_OK;
  for (int r = 0; r < x->world; ++r)
    if (x->peer_ptrs[r] && r != x->rank) cudaIpcCloseMemHandle(x->peer_ptrs[r]);
  cudaFree(x->region);
  cudaFree(x->d_peers);
  cudaFree(x->d_epoch);
  cudaFreeHost(x->h_err);
  delete[] x->peer_ptrs;
  delete x;
  return UCG_OK;
}

int ucg_segtab_scratch_floats(const ucg_segtab* t, uint64_t* n_out) {
  if (!t || !n_out) return fail(UCG_ERR_ARG, "null argument");
  *n_out = 2 * ucg::scratch_half(t);  // one half per launch parity (consecutive steps overlap)
  return UCG_OK;
}

}  // extern "C"
