// cuda_executor.hpp — seam B: a KernelExecutor (ucores/kernel.hpp:219-234)
// that runs the run() phase on a B200, and GpuWorkerRuntime, the reference
// WorkerRuntime::execute semantics (ucores/worker.hpp:40-72) bound to it.
//
// The reference executor only sees the KernelContext and a run_item closure
// over the host run(); the device body is found by kernel name (DeviceOp
// registry). The name travels through a thread-local set by the worker for
// the duration of one task — the one-line hook a maintainer adds to
// WorkerRuntime::execute.
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <string_view>
#include <utility>

#include "ucores/device.hpp"
#include "ucores/kernel.hpp"
#include "ucores/task.hpp"
#include "ucores/wire.hpp"
#include "ucores/worker.hpp"
#include "ucores_b200/device_ops.hpp"
#include "ucores_b200/gpu_context.hpp"
#include "ucores_b200/trace.hpp"

namespace ucores_b200 {

namespace detail {
inline std::string& current_kernel_slot() {
  thread_local std::string name;
  return name;
}
}  // namespace detail

/// RAII: the kernel name the CudaExecutor resolves on this thread.
class KernelScope {
 public:
  explicit KernelScope(std::string name) : prev_(std::exchange(detail::current_kernel_slot(), std::move(name))) {}
  ~KernelScope() { detail::current_kernel_slot() = std::move(prev_); }
  KernelScope(const KernelScope&) = delete;
  KernelScope& operator=(const KernelScope&) = delete;

 private:
  std::string prev_;
};

inline const std::string& current_kernel() { return detail::current_kernel_slot(); }

/// run() phase on one GPU. Metrics follow note_launch (kernel.hpp:227-233);
/// failures surface as KernelPanic("run", ...) like the host executors
/// (device.hpp:360,400,430). No host fallback.
class CudaExecutor : public ucores::KernelExecutor {
 public:
  CudaExecutor(std::shared_ptr<Gpu> gpu, const DeviceOpRegistry& ops) : gpu_(std::move(gpu)), ops_(&ops) {}

  std::string_view kind() const override { return "cuda-sm100a"; }

  void execute(ucores::KernelContext& ctx, const std::function<void(std::size_t)>&) override {
    note_launch(ctx);
    const std::string& name = current_kernel();
    const DeviceOp* op = ops_->find(name);
    if (!op || !op->run_phase) {
      throw ucores::KernelPanic("run", "no device body for kernel '" + name + "' (the GPU path has no CPU fallback)");
    }
    if (ctx.range().global_size == 0) return;
    TraceRange trace("ucores.run " + name);
    std::lock_guard<std::mutex> lock(gpu_->mutex());
    DeviceGuard guard;
    gpu_->bind();
    op->run_phase(*gpu_, ctx);
  }

  Gpu& gpu() { return *gpu_; }

 private:
  std::shared_ptr<Gpu> gpu_;
  const DeviceOpRegistry* ops_;
};

/// The device descriptor a B200 presents in the reference inventory
/// (device.hpp:53-65): type GPU, 148-SM width.
inline ucores::DeviceDescriptor b200_descriptor(int ordinal) {
  ucores::DeviceDescriptor d;
  d.device_id = "cuda:" + std::to_string(ordinal);
  d.device_type = ucores::ExecutionMode::GPU;
  ucg_device_info info{};
  d.parallel_width = ucg_device_info_get(ordinal, &info) == UCG_OK ? static_cast<std::uint32_t>(info.sm_count) : 148;
  d.cost = ucores::default_accelerator_cost();
  return d;
}

/// The GPU platform of the inventory (device.hpp:212-242 default_inventory
/// lists only the host): one STD platform, arch = device name, one GPU
/// device per visible B200.
inline ucores::PlatformDescriptor gpu_platform() {
  ucores::PlatformDescriptor p;
  p.impl_kind = ucores::ImplKind::STD;
  ucg_device_info info{};
  p.arch = gpu_count() > 0 && ucg_device_info_get(0, &info) == UCG_OK ? std::string(info.name) : "NVIDIA";
  for (int i = 0; i < gpu_count(); ++i) p.devices.push_back(b200_descriptor(i));
  return p;
}

/// Process-wide Gpu for a descriptor "cuda:N" (what make_executor needs when
/// patched, INTEGRATION.md seam B).
inline std::shared_ptr<Gpu> gpu_for(const ucores::DeviceDescriptor& d) {
  static std::mutex mu;
  static std::map<int, std::shared_ptr<Gpu>> gpus;
  int ordinal = 0;
  if (d.device_id.rfind("cuda:", 0) == 0) ordinal = std::stoi(d.device_id.substr(5));
  std::lock_guard<std::mutex> lock(mu);
  auto& g = gpus[ordinal];
  if (!g) g = std::make_shared<Gpu>(ordinal);
  return g;
}

/// Process-wide registry holding the device bodies of the workload kernels.
inline const DeviceOpRegistry& default_device_ops() {
  static const DeviceOpRegistry ops = [] {
    ucores::KernelRegistry unused;
    DeviceOpRegistry r;
    register_workload(unused, r);
    return r;
  }();
  return ops;
}

/// WorkerRuntime (worker.hpp:18-82) with the run phase on a B200: provision
/// through the per-worker ProgramCache, fresh kernel instance per task, the
/// strict three-phase lifecycle, "host-fallback" when the kernel declines
/// device execution, and failures returned as TaskErrorMsg{phase}. Never throws.
class GpuWorkerRuntime {
 public:
  GpuWorkerRuntime(std::string worker_id, const ucores::KernelRegistry& registry, const DeviceOpRegistry& ops,
                   std::shared_ptr<Gpu> gpu)
      : worker_id_(std::move(worker_id)),
        registry_(&registry),
        device_(b200_descriptor(gpu->ordinal())),
        executor_(std::move(gpu), ops) {}

  const std::string& worker_id() const { return worker_id_; }
  const ucores::DeviceDescriptor& device() const { return device_; }
  const ucores::ProgramCache& cache() const { return cache_; }

  ucores::Message execute(const ucores::Task& task) {
    try {
      ucores::provision_program(cache_, *registry_, device_, task.kernel_name,
                                ucores::Provisioning::BuildFromSource);
      KernelScope scope(task.kernel_name);
      ucores::TaskResult result;
      result.job_id = task.job_id;
      result.task_id = task.task_id;
      result.worker_id = worker_id_;
      if (task.kind == ucores::TaskKind::ReducePair) {
        if (task.inputs.size() != 2) throw ucores::Error("REDUCE_PAIR task must carry 2 inputs");
        auto kernel = registry_->instantiate_binary(task.kernel_name);
        result.output = ucores::execute_kernel_lifecycle(*kernel, task.inputs[0], task.inputs[1], executor_,
                                                         &result.metrics);
      } else {
        if (task.inputs.size() != 1) throw ucores::Error("task must carry 1 input");
        auto kernel = registry_->instantiate_unary(task.kernel_name);
        result.output = ucores::execute_kernel_lifecycle(*kernel, task.inputs[0], executor_, &result.metrics);
      }
      if (result.metrics.executor_kind.empty()) result.metrics.executor_kind = "host-fallback";
      return ucores::TaskResultMsg{std::move(result)};
    } catch (const ucores::KernelPanic& e) {
      return ucores::TaskErrorMsg{task.job_id, task.task_id, e.phase(), e.what()};
    } catch (const std::exception& e) {
      return ucores::TaskErrorMsg{task.job_id, task.task_id, "dispatch", e.what()};
    }
  }

 private:
  std::string worker_id_;
  const ucores::KernelRegistry* registry_;
  ucores::DeviceDescriptor device_;
  CudaExecutor executor_;
  ucores::ProgramCache cache_;
};

}  // namespace ucores_b200
