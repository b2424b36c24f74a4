// device_dataset.hpp — SURVEY §8(f)1: a device-resident Dataset and an engine
// whose map_cl / map_cl_partition / reduce_cl keep every payload in HBM
// between calls. upload() and collect() are the only host<->device payload
// transfers; a chain map_cl -> map_cl_partition -> reduce_cl moves one result
// element back to the host.
//
// Semantics are those of ucores::Engine (engine.hpp:54-192) with the workload
// kernels of kernels.hpp, and results are bit-identical to it (matmul: TF32
// tolerance):
//   * map_cl: one output element per input element, structure preserved;
//   * map_cl_partition: the partition's elements concatenated (element.hpp:
//     132-174), one output element per partition; an empty partition
//     concatenates to an empty ByteArray and fails the job, as in the
//     reference;
//   * reduce_cl: stage-1 left fold per partition, stage-2 pairing tree over
//     the partials in partition order, EmptyDataset on zero elements and the
//     element itself for one (engine.hpp:121-192).
// Task failures surface as ucores::JobFailed with the reference message shape
// (scheduler.hpp:290-302); kernels without a device body as UnknownKernel.
//
// Layout: partition p lives on GPU p*G/P (contiguous blocks, as
// GpuClusterDriver); a GPU's partitions share one allocation, each starting
// at an aligned offset with its elements stored back to back, so a
// partition's bytes ARE its concatenation. One host thread drives all GPUs
// through their streams; every call returns with its results complete.
#pragma once

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <list>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "ucores/dataset.hpp"
#include "ucores_b200/trace.hpp"
#include "ucores/element.hpp"
#include "ucores/errors.hpp"
#include "ucores_b200/device_ops.hpp"
#include "ucores_b200/gpu_context.hpp"

namespace ucores_b200 {

inline std::size_t entry_bytes(ucores::ElementKind k) {
  switch (k) {
    case ucores::ElementKind::F32Array: return 4;
    case ucores::ElementKind::F64Array: return 8;
    case ucores::ElementKind::I32Array: return 4;
    case ucores::ElementKind::I64Array: return 8;
    case ucores::ElementKind::ByteArray: return 1;
    default: throw ucores::ElementKindError("key count tables stay on the host (no device layout)");
  }
}

/// Per-engine cache of device blocks: an engine op allocates its outputs and
/// temporaries from here and released blocks are reused by size instead of
/// going back through cudaMalloc / cudaFree (which synchronises the device).
class DevicePool {
 public:
  DevicePool() = default;
  DevicePool(const DevicePool&) = delete;
  DevicePool& operator=(const DevicePool&) = delete;
  ~DevicePool() {
    for (const Block& b : free_) release(b);
  }
  void* get(int ordinal, std::uint64_t& bytes) {
    bytes = round(bytes);
    {
      std::lock_guard<std::mutex> lock(mu_);
      auto best = free_.end();
      for (auto it = free_.begin(); it != free_.end(); ++it)
        if (it->ordinal == ordinal && it->bytes >= bytes && it->bytes <= 2 * bytes &&
            (best == free_.end() || it->bytes < best->bytes))
          best = it;
      if (best != free_.end()) {
        void* p = best->ptr;
        bytes = best->bytes;
        free_.erase(best);
        return p;
      }
    }
    DeviceGuard guard;
    check(ucg_set_device(ordinal));
    void* p = nullptr;
    if (ucg_malloc(&p, bytes) != UCG_OK) {  // out of memory: drop the cache of this GPU, retry once
      trim(ordinal);
      check(ucg_malloc(&p, bytes));
    }
    return p;
  }
  void put(int ordinal, void* p, std::uint64_t bytes) {
    std::lock_guard<std::mutex> lock(mu_);
    free_.push_back({ordinal, p, bytes});
  }
  void trim(int ordinal) {
    std::vector<Block> drop;
    {
      std::lock_guard<std::mutex> lock(mu_);
      for (auto it = free_.begin(); it != free_.end();) {
        if (it->ordinal == ordinal) {
          drop.push_back(*it);
          it = free_.erase(it);
        } else {
          ++it;
        }
      }
    }
    for (const Block& b : drop) release(b);
  }

 private:
  struct Block {
    int ordinal;
    void* ptr;
    std::uint64_t bytes;
  };
  static std::uint64_t round(std::uint64_t b) {
    const std::uint64_t g = b >= (1u << 21) ? (1u << 21) : 256;  // 2 MiB granules for large blocks
    return std::max<std::uint64_t>(256, (b + g - 1) / g * g);
  }
  static void release(const Block& b) {
    DeviceGuard guard;
    ucg_set_device(b.ordinal);
    ucg_free(b.ptr);
  }
  std::mutex mu_;
  std::vector<Block> free_;
};

/// A device block on one GPU ordinal, returned to its pool on destruction.
class GpuAlloc {
 public:
  GpuAlloc(std::shared_ptr<DevicePool> pool, int ordinal, std::uint64_t bytes)
      : pool_(std::move(pool)), ordinal_(ordinal), bytes_(bytes) {
    ptr_ = pool_->get(ordinal_, bytes_);
  }
  GpuAlloc(const GpuAlloc&) = delete;
  GpuAlloc& operator=(const GpuAlloc&) = delete;
  ~GpuAlloc() {
    if (ptr_) pool_->put(ordinal_, ptr_, bytes_);
  }
  std::uint8_t* at(std::uint64_t off) const { return static_cast<std::uint8_t*>(ptr_) + off; }

 private:
  std::shared_ptr<DevicePool> pool_;
  int ordinal_;
  std::uint64_t bytes_;
  void* ptr_ = nullptr;
};

/// One partition of a DeviceDataset: all elements of one kind, back to back.
struct DevicePartition {
  std::size_t gpu = 0;                               // engine GPU index
  ucores::ElementKind kind = ucores::ElementKind::ByteArray;
  std::uint64_t offset = 0;                          // byte offset in that GPU's allocation
  std::vector<std::uint64_t> sizes;                  // entries per element
  std::uint64_t entries() const { return std::accumulate(sizes.begin(), sizes.end(), std::uint64_t(0)); }
  std::uint64_t bytes() const { return entries() * entry_bytes(kind); }
};

/// A partitioned collection resident in HBM (the device twin of
/// ucores::Dataset, dataset.hpp:17-59). Immutable; cheap to copy (shares
/// its allocations).
class DeviceDataset {
 public:
  std::size_t partition_count() const { return parts_.size(); }
  std::size_t count() const {
    std::size_t n = 0;
    for (const DevicePartition& p : parts_) n += p.sizes.size();
    return n;
  }
  const std::vector<DevicePartition>& partitions() const { return parts_; }
  /// Device address of partition p's first entry.
  std::uint8_t* data(std::size_t p) const { return bufs_.at(parts_.at(p).gpu)->at(parts_[p].offset); }

 private:
  friend class DeviceEngine;
  std::vector<DevicePartition> parts_;
  std::vector<std::shared_ptr<GpuAlloc>> bufs_;  // one per engine GPU (may be null)
};

class DeviceEngine {
 public:
  explicit DeviceEngine(WorkloadParams params = {}, int max_gpus = -1) : params_(params) {
    for (auto& g : open_gpus(max_gpus)) gpus_.push_back(std::move(g));
    // bring-up: each GPU's transfer pipeline (pinned slot rings, copy
    // streams) and the host copy threads exist before the first upload, as a
    // worker's resources exist before its first task
    for (auto& g : gpus_) g->attached<HostPipe>();
    work_pool();
  }
  std::size_t gpu_count() const { return gpus_.size(); }
  /// Kernel parameters for later calls (axpb's a, b; sobel width; matmul n).
  void set_params(const WorkloadParams& p) { params_ = p; }

  /// Host Dataset -> HBM. Each partition must hold one element kind (a
  /// partition's bytes are its concatenation); tables stay on the host.
  DeviceDataset upload(const ucores::Dataset& d) {
    TraceRange trace("ucores.upload");
    std::vector<DevicePartition> parts(d.partition_count());
    for (std::size_t p = 0; p < parts.size(); ++p) {
      const auto& els = d.partitions()[p].elements;
      parts[p].gpu = gpu_of(p, parts.size());
      parts[p].kind = els.empty() ? ucores::ElementKind::ByteArray : els.front().kind();
      for (const ucores::Element& e : els) {
        if (e.kind() != parts[p].kind) {
          throw ucores::MixedElementVariants("device partitions hold one element kind (partition " +
                                             std::to_string(p) + ")");
        }
        entry_bytes(e.kind());
        parts[p].sizes.push_back(e.size());
      }
    }
    DeviceDataset out = allocate(std::move(parts));
    // every GPU's partitions through its pipe, the GPUs concurrently (one
    // host thread each): a partition's elements land back to back, so its
    // bytes are its concatenation; small elements share a pinned slot
    run_per_gpu([&](std::size_t g) {
      HostPipe& pipe = gpus_[g]->attached<HostPipe>();
      for (std::size_t p = 0; p < out.parts_.size(); ++p) {
        if (out.parts_[p].gpu != g) continue;
        std::vector<std::span<const std::uint8_t>> pieces;
        std::vector<std::uint64_t> off;
        std::uint64_t at = 0;
        for (const ucores::Element& e : d.partitions()[p].elements) {
          pieces.emplace_back(static_cast<const std::uint8_t*>(host_bytes(e)), e.byte_size());
          off.push_back(at);
          at += e.byte_size();
        }
        pipe.upload_pieces(out.data(p), pieces, off);
      }
      // the GPU's stream waits for the last DMA by event: the first operator
      // is enqueued while the tail of the upload is still in flight (the
      // host payloads are already in pinned slots, so the caller may drop
      // the host Dataset as soon as upload() returns)
      pipe.compute_after_upload();
    });
    return out;
  }

  /// Ingestion without host Elements: the device twin of
  /// ucores::create_dataset (dataset.hpp:64-82) over caller-owned host
  /// arrays — element i is `elements[i]` (kind `kind`, bytes), distributed
  /// over `num_partitions` contiguous partitions ceiling-first, and copied
  /// straight from the caller's memory through each GPU's transfer
  /// pipeline. Errors as create_dataset: InvalidPartitionCount for 0
  /// partitions. The caller's arrays may be reused once this returns.
  DeviceDataset create_dataset(const std::vector<std::span<const std::uint8_t>>& elements, ucores::ElementKind kind,
                               std::size_t num_partitions) {
    TraceRange trace("ucores.create_dataset");
    if (num_partitions < 1)
      throw ucores::InvalidPartitionCount("num_partitions must be >= 1, got " + std::to_string(num_partitions));
    const std::size_t eb = entry_bytes(kind), n = elements.size();
    const std::size_t base = n / num_partitions, extra = n % num_partitions;
    std::vector<DevicePartition> parts(num_partitions);
    std::vector<std::size_t> first(num_partitions + 1, 0);
    for (std::size_t p = 0; p < num_partitions; ++p) {
      const std::size_t take = base + (p < extra ? 1 : 0);
      first[p + 1] = first[p] + take;
      parts[p].gpu = gpu_of(p, num_partitions);
      parts[p].kind = take ? kind : ucores::ElementKind::ByteArray;  // an empty partition concatenates to bytes
      for (std::size_t i = first[p]; i < first[p + 1]; ++i) {
        if (elements[i].size() % eb)
          throw ucores::ElementKindError("element " + std::to_string(i) + " is not a whole number of entries");
        parts[p].sizes.push_back(elements[i].size() / eb);
      }
    }
    DeviceDataset out = allocate(std::move(parts));
    run_per_gpu([&](std::size_t g) {
      HostPipe& pipe = gpus_[g]->attached<HostPipe>();
      for (std::size_t p = 0; p < num_partitions; ++p) {
        if (out.parts_[p].gpu != g) continue;
        std::vector<std::span<const std::uint8_t>> pieces(elements.begin() + first[p], elements.begin() + first[p + 1]);
        std::vector<std::uint64_t> off;
        std::uint64_t at = 0;
        for (const auto& e : pieces) {
          off.push_back(at);
          at += e.size();
        }
        pipe.upload_pieces(out.data(p), pieces, off);
      }
      pipe.compute_after_upload();
    });
    return out;
  }

  /// HBM -> host Dataset (the lazy collect of SURVEY §8(f)1).
  ucores::Dataset collect(const DeviceDataset& d) {
    TraceRange trace("ucores.collect");
    std::vector<ucores::Partition> parts(d.partition_count());
    std::vector<std::vector<std::uint8_t>> staging(d.partition_count());
    for (std::size_t p = 0; p < parts.size(); ++p) {
      const DevicePartition& dp = d.parts_[p];
      staging[p].resize(dp.bytes());
      Gpu& g = *gpus_[dp.gpu];
      DeviceGuard guard;
      g.bind();
      check(ucg_memcpy_d2h(staging[p].data(), d.data(p), staging[p].size(), g.stream()));
    }
    sync_all();
    for (std::size_t p = 0; p < parts.size(); ++p) {
      const DevicePartition& dp = d.parts_[p];
      const std::uint8_t* src = staging[p].data();
      for (std::uint64_t n : dp.sizes) {
        parts[p].elements.push_back(make_element(dp.kind, src, n));
        src += n * entry_bytes(dp.kind);
      }
    }
    return ucores::Dataset(std::move(parts));
  }

  /// Engine::map_cl (engine.hpp:54-85): axpb, psum, pmax, pi, sobel, matmul.
  DeviceDataset map_cl(const DeviceDataset& d, const std::string& kernel) {
    TraceRange trace("ucores.map_cl:" + kernel);
    return unary(d, kernel, false);
  }

  /// Engine::map_cl_partition (engine.hpp:89-114) over the concatenated
  /// partitions: axpb, psum, pmax, sobel (pi / matmul fail as in the
  /// reference unless a partition holds exactly one element).
  DeviceDataset map_cl_partition(const DeviceDataset& d, const std::string& kernel) {
    TraceRange trace("ucores.map_cl_partition:" + kernel);
    for (std::size_t p = 0; p < d.parts_.size(); ++p) {
      if (d.parts_[p].sizes.empty()) {
        fail(p, "map_parameters: element kind mismatch, have bytes (empty partition concatenates to an empty "
                "ByteArray, element.hpp:133)");
      }
    }
    return unary(d, kernel, true);
  }

  /// Engine::reduce_cl (engine.hpp:121-192): sum2, max2, vectoradd, isum2.
  ucores::Element reduce_cl(const DeviceDataset& d, const std::string& kernel) {
    TraceRange trace("ucores.reduce_cl:" + kernel);
    const bool i64 = kernel == "isum2";
    if (!i64 && kernel != "sum2" && kernel != "max2" && kernel != "vectoradd") {
      throw ucores::UnknownKernel("no device reduce_cl body for kernel '" + kernel + "'");
    }
    const std::size_t count = d.count();
    if (count == 0) throw ucores::EmptyDataset("reduce_cl needs at least one element");
    if (count == 1) {
      for (std::size_t p = 0; p < d.parts_.size(); ++p) {
        if (!d.parts_[p].sizes.empty()) return collect_one(d, p);
      }
    }
    const auto want = i64 ? ucores::ElementKind::I64Array : ucores::ElementKind::F32Array;
    std::uint64_t len = 0;
    bool have_len = false;
    for (std::size_t p = 0; p < d.parts_.size(); ++p) {
      const DevicePartition& dp = d.parts_[p];
      if (dp.sizes.empty()) continue;
      if (dp.kind != want) fail(p, std::string("map_parameters: element kind mismatch, have ") + ucores::to_string(dp.kind));
      for (std::uint64_t n : dp.sizes) {
        if (!have_len) len = n, have_len = true;
        if (n != len) fail(p, "map_parameters: vector lengths differ");
      }
    }
    const int op = kernel == "max2" ? UCG_OP_MAX : UCG_OP_SUM;
    const std::uint64_t eb = entry_bytes(want);
    // stage 1 on each partition's GPU: the left fold of its elements
    std::vector<std::size_t> nonempty;
    for (std::size_t p = 0; p < d.parts_.size(); ++p)
      if (!d.parts_[p].sizes.empty()) nonempty.push_back(p);
    const std::uint64_t row = std::max<std::uint64_t>(eb * len, 1);
    const std::uint64_t stride = (row + 255) / 256 * 256;
    std::vector<std::shared_ptr<GpuAlloc>> partials(gpus_.size()), ptrs(gpus_.size());
    std::vector<std::vector<std::uint64_t>> host_ptrs(gpus_.size());
    std::vector<std::vector<std::size_t>> on_gpu(gpus_.size());
    for (std::size_t k = 0; k < nonempty.size(); ++k) on_gpu[d.parts_[nonempty[k]].gpu].push_back(k);
    for (std::size_t g = 0; g < gpus_.size(); ++g) {
      if (on_gpu[g].empty()) continue;
      DeviceGuard guard;
      gpus_[g]->bind();
      partials[g] = std::make_shared<GpuAlloc>(pool_, gpus_[g]->ordinal(), stride * on_gpu[g].size());
      for (std::size_t k : on_gpu[g]) {
        const DevicePartition& dp = d.parts_[nonempty[k]];
        for (std::size_t e = 0; e < dp.sizes.size(); ++e)
          host_ptrs[g].push_back(reinterpret_cast<std::uint64_t>(d.data(nonempty[k]) + e * eb * len));
      }
      ptrs[g] = std::make_shared<GpuAlloc>(pool_, gpus_[g]->ordinal(), host_ptrs[g].size() * 8);
      check(ucg_memcpy_h2d(ptrs[g]->at(0), host_ptrs[g].data(), host_ptrs[g].size() * 8, gpus_[g]->stream()));
      std::uint64_t first = 0;
      for (std::size_t j = 0; j < on_gpu[g].size(); ++j) {
        const DevicePartition& dp = d.parts_[nonempty[on_gpu[g][j]]];
        const std::uint64_t c = dp.sizes.size();
        reduce_vectors(i64, reinterpret_cast<const void* const*>(ptrs[g]->at(first * 8)), c, len, &c, 1, op,
                       partials[g]->at(j * stride), gpus_[g]->stream());
        first += c;
      }
    }
    // stage 2 on GPU 0: the partials gathered in partition order, then the tree
    Gpu& g0 = *gpus_[0];
    DeviceGuard guard;
    g0.bind();
    std::vector<std::uint64_t> slot(nonempty.size());
    for (std::size_t g = 0; g < gpus_.size(); ++g)
      for (std::size_t j = 0; j < on_gpu[g].size(); ++j) slot[on_gpu[g][j]] = j;
    sync_all();
    GpuAlloc gathered(pool_, g0.ordinal(), stride * nonempty.size()), gptrs(pool_, g0.ordinal(), nonempty.size() * 8),
        out(pool_, g0.ordinal(), row);
    std::vector<std::uint64_t> gp(nonempty.size());
    for (std::size_t k = 0; k < nonempty.size(); ++k) {
      const std::size_t g = d.parts_[nonempty[k]].gpu;
      check(ucg_memcpy2d(gathered.at(k * stride), stride, partials[g]->at(slot[k] * stride), stride, row, 1,
                         g0.stream()));
      gp[k] = reinterpret_cast<std::uint64_t>(gathered.at(k * stride));
    }
    check(ucg_memcpy_h2d(gptrs.at(0), gp.data(), gp.size() * 8, g0.stream()));
    std::vector<std::uint64_t> ones(nonempty.size(), 1);
    reduce_vectors(i64, reinterpret_cast<const void* const*>(gptrs.at(0)), nonempty.size(), len, ones.data(),
                   ones.size(), op, out.at(0), g0.stream());
    std::vector<std::uint8_t> host(eb * len);
    check(ucg_memcpy_d2h(host.data(), out.at(0), host.size(), g0.stream()));
    g0.sync();
    return make_element(want, host.data(), len);
  }

 private:
  // -- layout -------------------------------------------------------------------
  std::size_t gpu_of(std::size_t p, std::size_t P) const { return P ? p * gpus_.size() / P : 0; }

  std::uint64_t align_for(ucores::ElementKind k) const {
    // byte bands start on a row boundary so the Sobel kernel takes its TMA path
    const std::uint64_t w = params_.sobel_width;
    if (k == ucores::ElementKind::ByteArray && w && w % 256 == 0 && w <= (1u << 20)) return w;
    return 256;
  }

  DeviceDataset allocate(std::vector<DevicePartition> parts) {
    DeviceDataset out;
    std::vector<std::uint64_t> used(gpus_.size(), 0);
    for (DevicePartition& p : parts) {
      const std::uint64_t a = align_for(p.kind);
      p.offset = (used[p.gpu] + a - 1) / a * a;
      used[p.gpu] = p.offset + p.bytes();
    }
    out.bufs_.resize(gpus_.size());
    for (std::size_t g = 0; g < gpus_.size(); ++g) {
      bool any = false;
      for (const DevicePartition& p : parts) any |= p.gpu == g;
      if (any) out.bufs_[g] = std::make_shared<GpuAlloc>(pool_, gpus_[g]->ordinal(), (used[g] + 255) / 256 * 256);
    }
    out.parts_ = std::move(parts);
    return out;
  }

  std::uint64_t used_bytes(const DeviceDataset& d, std::size_t g) const {
    std::uint64_t u = 0;
    for (const DevicePartition& p : d.parts_)
      if (p.gpu == g) u = std::max(u, p.offset + p.bytes());
    return u;
  }

  // -- map_cl / map_cl_partition --------------------------------------------------
  // A unit is one element (map_cl) or one whole partition (map_cl_partition).
  struct Unit {
    std::size_t part;
    std::uint64_t in_off, entries;  // byte offset in the GPU allocation, entries
  };

  std::vector<Unit> units_of(const DeviceDataset& d, std::size_t g, bool per_partition) const {
    std::vector<Unit> u;
    for (std::size_t p = 0; p < d.parts_.size(); ++p) {
      const DevicePartition& dp = d.parts_[p];
      if (dp.gpu != g) continue;
      if (per_partition) {
        u.push_back({p, dp.offset, dp.entries()});
        continue;
      }
      std::uint64_t off = dp.offset;
      for (std::uint64_t n : dp.sizes) {
        u.push_back({p, off, n});
        off += n * entry_bytes(dp.kind);
      }
    }
    return u;
  }

  DeviceDataset unary(const DeviceDataset& d, const std::string& kernel, bool per_partition) {
    using K = ucores::ElementKind;
    K in_kind, out_kind;
    std::function<std::uint64_t(std::uint64_t)> out_size;
    const std::uint64_t w = params_.sobel_width, mn = params_.matmul_n;
    if (kernel == "axpb") {
      in_kind = out_kind = K::F32Array;
      out_size = [](std::uint64_t n) { return n; };
    } else if (kernel == "psum" || kernel == "pmax") {
      in_kind = out_kind = K::F32Array;
      out_size = [](std::uint64_t) { return std::uint64_t(1); };
    } else if (kernel == "sobel") {
      in_kind = out_kind = K::ByteArray;
      out_size = [w](std::uint64_t n) { return n - 2 * w; };
    } else if (kernel == "pi") {
      in_kind = out_kind = K::I64Array;
      out_size = [](std::uint64_t) { return std::uint64_t(2); };
    } else if (kernel == "matmul") {
      in_kind = out_kind = K::F32Array;
      out_size = [mn](std::uint64_t) { return mn * mn; };
    } else {
      throw ucores::UnknownKernel("no device body for kernel '" + kernel + "' in DeviceEngine");
    }
    // map_parameters checks (kernels.hpp), per unit
    for (std::size_t g = 0; g < gpus_.size(); ++g) {
      for (const Unit& u : units_of(d, g, per_partition)) {
        const DevicePartition& dp = d.parts_[u.part];
        if (dp.kind != in_kind)
          fail(u.part, std::string("map_parameters: element kind mismatch, have ") + ucores::to_string(dp.kind));
        if (kernel == "sobel" && (w == 0 || u.entries % w != 0 || u.entries / w < 2))
          fail(u.part, "map_parameters: band is not (rows+2) x width");
        if (kernel == "pi" && u.entries != 2) fail(u.part, "map_parameters: pi element must be {task_seed, samples}");
        if (kernel == "matmul" && (u.entries != 2 * mn * mn || mn % 256 != 0))
          fail(u.part, "map_parameters: matmul element must hold A||B (n a multiple of 256)");
      }
    }
    // output structure
    std::vector<DevicePartition> parts(d.parts_.size());
    for (std::size_t p = 0; p < parts.size(); ++p) {
      const DevicePartition& dp = d.parts_[p];
      parts[p].gpu = dp.gpu;
      parts[p].kind = out_kind;
      if (per_partition) {
        parts[p].sizes.push_back(out_size(dp.entries()));
      } else {
        for (std::uint64_t n : dp.sizes) parts[p].sizes.push_back(out_size(n));
      }
    }
    DeviceDataset out = allocate(std::move(parts));
    // temporaries live until every GPU's stream is drained (sync_all below),
    // so the GPUs run concurrently and no block returns to the pool early
    std::vector<std::shared_ptr<GpuAlloc>> keep;
    for (std::size_t g = 0; g < gpus_.size(); ++g) {
      const std::vector<Unit> units = units_of(d, g, per_partition);
      if (units.empty()) continue;
      Gpu& gpu = *gpus_[g];
      DeviceGuard guard;
      gpu.bind();
      void* st = gpu.stream();
      const std::vector<Unit> ounits = units_of(out, g, per_partition);
      std::uint8_t* ib = d.bufs_[g]->at(0);
      std::uint8_t* ob = out.bufs_[g]->at(0);
      if (kernel == "axpb") {
        // same byte layout in and out: one launch over the GPU's whole span
        check(ucg_map_affine_f32(reinterpret_cast<const float*>(ib), reinterpret_cast<float*>(ob),
                                 used_bytes(d, g) / 4, params_.a, params_.b, st));
      } else if (kernel == "psum" || kernel == "pmax") {
        std::vector<std::uint64_t> begin, len;
        for (const Unit& u : units) begin.push_back(u.in_off / 4), len.push_back(u.entries);
        std::vector<std::size_t> realign;  // units whose floats are not 16-byte aligned
        for (std::size_t i = 0; i < units.size(); ++i)
          if (begin[i] % 4) realign.push_back(i);
        std::shared_ptr<GpuAlloc> tmp;  // kept alive through `keep`
        const float* base = reinterpret_cast<const float*>(ib);
        if (!realign.empty()) {  // map_cl over packed elements: copy them to aligned segments first
          std::uint64_t total = 0;
          for (std::size_t i = 0; i < units.size(); ++i) total += (len[i] + 63) / 64 * 64;
          tmp = std::make_shared<GpuAlloc>(pool_, gpu.ordinal(), total * 4);
          std::uint64_t at = 0;
          for (std::size_t i = 0; i < units.size(); ++i) {
            check(ucg_memcpy_d2d(tmp->at(at * 4), ib + units[i].in_off, len[i] * 4, st));
            begin[i] = at;
            at += (len[i] + 63) / 64 * 64;
          }
          base = reinterpret_cast<const float*>(tmp->at(0));
          keep.push_back(tmp);
        }
        ucg_segtab* tab = segtab(g, begin, len);
        std::uint64_t nscratch = 0;
        check(ucg_segtab_scratch_floats(tab, &nscratch));
        auto scratch = std::make_shared<GpuAlloc>(pool_, gpu.ordinal(), nscratch * 4);
        auto vals = std::make_shared<GpuAlloc>(pool_, gpu.ordinal(), units.size() * 4);
        keep.push_back(scratch);
        keep.push_back(vals);
        check(ucg_segment_reduce_f32(base, tab, kernel == "pmax" ? UCG_OP_MAX : UCG_OP_SUM,
                                     reinterpret_cast<float*>(scratch->at(0)), reinterpret_cast<float*>(vals->at(0)),
                                     st));
        // the values of one partition's units are contiguous on both sides:
        // one copy per partition, not one per unit
        for (std::size_t i = 0; i < units.size();) {
          std::size_t j = i + 1;
          while (j < units.size() && units[j].part == units[i].part) ++j;
          check(ucg_memcpy_d2d(ob + ounits[i].in_off, vals->at(i * 4), (j - i) * 4, st));
          i = j;
        }
      } else if (kernel == "sobel") {
        std::vector<std::uint64_t> in_off, out_off, rows;
        for (std::size_t i = 0; i < units.size(); ++i) {
          in_off.push_back(units[i].in_off);
          out_off.push_back(ounits[i].in_off);
          rows.push_back(units[i].entries / w - 2);
        }
        check(ucg_sobel_bands_u8(ib, in_off.data(), ob, out_off.data(), rows.data(), rows.size(), w, st));
      } else if (kernel == "pi") {
        // {seed, samples} of one partition's units are contiguous: one copy each
        std::vector<std::int64_t> params(units.size() * 2);
        for (std::size_t i = 0; i < units.size();) {
          std::size_t j = i + 1;
          while (j < units.size() && units[j].part == units[i].part) ++j;
          check(ucg_memcpy_d2h(&params[2 * i], ib + units[i].in_off, (j - i) * 16, st));
          i = j;
        }
        check(ucg_stream_synchronize(st));
        std::vector<std::uint64_t> seeds(units.size()), samples(units.size());
        for (std::size_t i = 0; i < units.size(); ++i) {
          seeds[i] = static_cast<std::uint64_t>(params[2 * i]);
          samples[i] = static_cast<std::uint64_t>(params[2 * i + 1]);
        }
        auto hits = std::make_shared<GpuAlloc>(pool_, gpu.ordinal(), units.size() * 8);
        keep.push_back(hits);
        check(ucg_pi_hits(seeds.data(), samples.data(), units.size(), reinterpret_cast<std::int64_t*>(hits->at(0)),
                          st));
        // outputs {hits, samples}: the hits come back once, the pairs go up
        // once per partition
        std::vector<std::int64_t> h(units.size()), pairs(2 * units.size());
        check(ucg_memcpy_d2h(h.data(), hits->at(0), h.size() * 8, st));
        check(ucg_stream_synchronize(st));
        for (std::size_t i = 0; i < units.size(); ++i) {
          pairs[2 * i] = h[i];
          pairs[2 * i + 1] = static_cast<std::int64_t>(samples[i]);
        }
        for (std::size_t i = 0; i < units.size();) {
          std::size_t j = i + 1;
          while (j < units.size() && units[j].part == units[i].part) ++j;
          // pageable source: staged before the call returns
          check(ucg_memcpy_h2d(ob + ounits[i].in_off, &pairs[2 * i], (j - i) * 16, st));
          i = j;
        }
        check(ucg_stream_synchronize(st));
      } else {  // matmul
        for (std::size_t i = 0; i < units.size(); ++i) {
          const float* a = reinterpret_cast<const float*>(ib + units[i].in_off);
          check((params_.matmul_fp32 ? ucg_gemm_f32 : ucg_gemm_tf32)(
              a, a + mn * mn, reinterpret_cast<float*>(ob + ounits[i].in_off), mn, st));
        }
      }
    }
    sync_all();
    return out;
  }

  // -- host threads ------------------------------------------------------------------
  // fn(g) for every GPU, each on its own host thread (GPU 0 on the caller's)
  void run_per_gpu(const std::function<void(std::size_t)>& fn) {
    std::vector<std::thread> t;
    std::vector<std::exception_ptr> err(gpus_.size());
    auto one = [&](std::size_t g) {
      try {
        DeviceGuard guard;
        gpus_[g]->bind();
        fn(g);
      } catch (...) {
        err[g] = std::current_exception();
      }
    };
    for (std::size_t g = 1; g < gpus_.size(); ++g) t.emplace_back(one, g);
    one(0);
    for (auto& x : t) x.join();
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
  }

  // -- helpers ----------------------------------------------------------------------
  static void reduce_vectors(bool i64, const void* const* ptrs, std::uint64_t count, std::uint64_t len,
                             const std::uint64_t* part_counts, std::uint64_t nparts, int op, void* out, void* st) {
    if (i64) {
      check(ucg_reduce_cl_i64(reinterpret_cast<const std::int64_t* const*>(ptrs), count, len, part_counts, nparts,
                              static_cast<std::int64_t*>(out), st));
    } else {
      check(ucg_reduce_cl_f32(reinterpret_cast<const float* const*>(ptrs), count, len, part_counts, nparts, op,
                              static_cast<float*>(out), st));
    }
  }

  [[noreturn]] void fail(std::size_t partition, const std::string& why) const {
    // the reference's failed-task message shape (scheduler.hpp:290-302); the
    // device path does not retry a deterministic kernel-contract failure
    throw ucores::JobFailed("task for partition " + std::to_string(partition) + " failed after 1 attempts (" + why +
                            ")");
  }

  static const void* host_bytes(const ucores::Element& e) {
    switch (e.kind()) {
      case ucores::ElementKind::F32Array: return e.as_f32().data();
      case ucores::ElementKind::F64Array: return e.as_f64().data();
      case ucores::ElementKind::I32Array: return e.as_i32().data();
      case ucores::ElementKind::I64Array: return e.as_i64().data();
      default: return e.as_bytes().data();
    }
  }

  static ucores::Element make_element(ucores::ElementKind k, const std::uint8_t* src, std::uint64_t n) {
    auto vec = [&](auto tag) {
      using T = decltype(tag);
      std::vector<T> v(n);
      if (n) std::memcpy(v.data(), src, n * sizeof(T));
      return v;
    };
    switch (k) {
      case ucores::ElementKind::F32Array: return ucores::Element::f32(vec(float{}));
      case ucores::ElementKind::F64Array: return ucores::Element::f64(vec(double{}));
      case ucores::ElementKind::I32Array: return ucores::Element::i32(vec(std::int32_t{}));
      case ucores::ElementKind::I64Array: return ucores::Element::i64(vec(std::int64_t{}));
      default: return ucores::Element::bytes(vec(std::uint8_t{}));
    }
  }

  ucores::Element collect_one(const DeviceDataset& d, std::size_t p) {
    const DevicePartition& dp = d.parts_[p];
    std::vector<std::uint8_t> host(dp.bytes());
    Gpu& g = *gpus_[dp.gpu];
    DeviceGuard guard;
    g.bind();
    check(ucg_memcpy_d2h(host.data(), d.data(p), host.size(), g.stream()));
    g.sync();
    return make_element(dp.kind, host.data(), dp.sizes.front());
  }

  /// Segment tables by layout (uploading one costs a cudaMalloc): a chain
  /// over the same dataset shape reuses them. Ops run one at a time per
  /// engine and finish before returning, so a table is never in flight twice.
  ucg_segtab* segtab(std::size_t g, const std::vector<std::uint64_t>& begin, const std::vector<std::uint64_t>& len) {
    // keyed by (GPU, FNV-1a of the layout); the layout itself confirms a hit.
    // At most kMaxTabs live tables, least recently used evicted first.
    std::uint64_t h = 0xcbf29ce484222325ull ^ g;
    for (const auto* v : {&begin, &len})
      for (std::uint64_t x : *v) h = (h ^ x) * 0x100000001b3ull;
    for (auto it = tabs_.begin(); it != tabs_.end(); ++it) {
      if (it->gpu == g && it->hash == h && it->begin == begin && it->len == len) {
        tabs_.splice(tabs_.begin(), tabs_, it);  // most recent first
        return tabs_.front().tab.get();
      }
    }
    ucg_segtab* tab = nullptr;
    check(ucg_segtab_create(begin.data(), len.data(), begin.size(), &tab));
    if (tabs_.size() >= kMaxTabs) tabs_.pop_back();
    tabs_.push_front(Tab{g, h, begin, len, std::unique_ptr<ucg_segtab, TabFree>(tab)});
    return tab;
  }
  struct TabFree {
    void operator()(ucg_segtab* t) const { ucg_segtab_destroy(t); }
  };
  struct Tab {
    std::size_t gpu;
    std::uint64_t hash;
    std::vector<std::uint64_t> begin, len;
    std::unique_ptr<ucg_segtab, TabFree> tab;
  };
  static constexpr std::size_t kMaxTabs = 16;

  void sync_all() {
    for (auto& g : gpus_) {
      DeviceGuard guard;
      g->bind();
      g->sync();
    }
  }

  WorkloadParams params_;
  std::vector<std::shared_ptr<Gpu>> gpus_;
  std::shared_ptr<DevicePool> pool_ = std::make_shared<DevicePool>();
  std::list<Tab> tabs_;
};

}  // namespace ucores_b200
