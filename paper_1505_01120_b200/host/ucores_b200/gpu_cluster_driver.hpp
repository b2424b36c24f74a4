// gpu_cluster_driver.hpp — seam A: a ClusterDriver (ucores/engine.hpp:34-39)
// that executes every wave the unmodified reference Engine plans on the
// B200s of one box.
//
// Partition -> device scheduling (replaces Scheduler::take_assignments,
// scheduler.hpp:94-117): the tasks of one kernel in a wave are split into
// contiguous blocks, task i of T on GPU floor(i*G/T) (partition p of a
// map_cl_partition wave lands on GPU floor(p*G/P)), and each
// GPU runs its block as ONE batched device launch (DeviceOp::run_tasks) on
// its own host thread. Wave contract kept from DriverCore
// (scheduler.hpp:229-302): results sorted by task_id, the wave is a barrier,
// a failing task is retried up to max_retries times (here on the next GPU)
// and then the job fails with JobFailed naming task, job and attempts.
// Mode::PerTask instead runs every task through GpuWorkerRuntime (the host
// lifecycle with the run phase on the GPU, seam B).
#pragma once

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <memory>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "ucores/engine.hpp"
#include "ucores/errors.hpp"
#include "ucores/task.hpp"
#include "ucores/wire.hpp"
#include "ucores_b200/cuda_executor.hpp"
#include "ucores_b200/device_ops.hpp"
#include "ucores_b200/gpu_context.hpp"
#include "ucores_b200/trace.hpp"

namespace ucores_b200 {

class GpuClusterDriver : public ucores::ClusterDriver {
 public:
  enum class Mode { Batched, PerTask };

  struct Options {
    int max_gpus = -1;  // -1: every visible GPU
    Mode mode = Mode::Batched;
  };

  GpuClusterDriver(const ucores::KernelRegistry& registry, const DeviceOpRegistry& ops)
      : GpuClusterDriver(registry, ops, Options{}) {}

  GpuClusterDriver(const ucores::KernelRegistry& registry, const DeviceOpRegistry& ops, Options opt)
      : registry_(&registry), ops_(&ops), opt_(opt) {
    for (auto& g : open_gpus(opt.max_gpus)) gpus_.push_back(std::shared_ptr<Gpu>(std::move(g)));
    for (auto& g : gpus_) {
      worker_ids_.push_back("gpu" + std::to_string(g->ordinal()));
      workers_.push_back(std::make_unique<GpuWorkerRuntime>(worker_ids_.back(), registry, ops, g));
    }
    // bring-up, as a worker's resources exist before its first task: each
    // GPU's transfer pipeline (pinned slot rings, copy streams) and the host
    // copy threads
    if (opt.mode == Mode::Batched) {
      for (auto& g : gpus_) g->attached<HostPipe>();
      work_pool();
    }
  }

  std::uint64_t new_job_id() override { return ++job_id_; }

  std::vector<ucores::TaskResult> run_wave(std::vector<ucores::Task> tasks, int max_retries) override {
    if (tasks.empty()) return {};
    TraceRange trace("ucores.run_wave");
    // results are filled in place (a wave of the C1 literal form is 2^20
    // tasks: no per-task optional / failure slots)
    Wave w;
    w.out.resize(tasks.size());
    if (opt_.mode == Mode::PerTask) {
      run_per_task(tasks, max_retries, w);
    } else {
      // group by kernel name, keeping task order inside each group
      std::map<std::string, std::vector<std::size_t>> groups;
      for (std::size_t i = 0; i < tasks.size(); ++i) groups[tasks[i].kernel_name].push_back(i);
      for (auto& [name, idx] : groups) run_group(tasks, name, idx, max_retries, w);
    }
    // results sorted by task_id (scheduler.hpp:274-287); a wave the Engine
    // planned in task order already is (sorting 2^20 results costs ~0.1 s)
    auto by_id = [](const ucores::TaskResult& a, const ucores::TaskResult& b) { return a.task_id < b.task_id; };
    if (!std::is_sorted(w.out.begin(), w.out.end(), by_id)) std::sort(w.out.begin(), w.out.end(), by_id);
    waves_ += 1;
    tasks_ += tasks.size();
    return std::move(w.out);
  }

  // -- observability (mirrors LocalClusterDriver's hooks) ---------------------
  std::size_t gpu_count() const { return gpus_.size(); }
  std::uint64_t waves_run() const { return waves_; }
  std::uint64_t tasks_run() const { return tasks_; }
  std::uint64_t retries() const { return retries_; }
  const std::vector<std::uint64_t>& tasks_per_gpu() const { return per_gpu_; }
  Gpu& gpu(std::size_t i) { return *gpus_.at(i); }

 private:
  struct Failure {
    std::string phase, detail;
  };
  // One wave's results (in task order) and its failed tasks (sparse;
  // guarded, batches of different GPUs report concurrently).
  struct Wave {
    std::vector<ucores::TaskResult> out;
    std::map<std::size_t, Failure> failed;
    std::mutex mu;
    void fail(std::size_t i, Failure f) {
      std::lock_guard<std::mutex> lk(mu);
      failed[i] = std::move(f);
    }
  };

  // Run tasks idx[lo,hi) of one kernel on GPU g as one batch. On failure the
  // batch is re-run task by task so only the failing tasks are retried.
  void run_batch(const std::vector<ucores::Task>& tasks, const DeviceOp& op, const std::vector<std::size_t>& idx,
                 std::size_t lo, std::size_t hi, std::size_t g, Wave& w) {
    if (lo >= hi) return;
    TraceRange trace("ucores.batch " + tasks[idx[lo]].kernel_name + " gpu" + std::to_string(g));
    std::vector<const ucores::Task*> batch;
    batch.reserve(hi - lo);
    for (std::size_t k = lo; k < hi; ++k) batch.push_back(&tasks[idx[k]]);
    Gpu& gpu = *gpus_[g];
    auto attempt = [&](std::span<const ucores::Task* const> b) {
      std::lock_guard<std::mutex> lock(gpu.mutex());
      DeviceGuard guard;
      gpu.bind();
      return op.run_tasks(gpu, b);
    };
    try {
      std::vector<ucores::Element> outs = attempt(batch);
      for (std::size_t k = 0; k < batch.size(); ++k) fill_result(w.out[idx[lo + k]], *batch[k], std::move(outs[k]), g);
    } catch (const std::exception&) {
      for (std::size_t k = 0; k < batch.size(); ++k) {
        try {
          std::vector<ucores::Element> one = attempt(std::span<const ucores::Task* const>(&batch[k], 1));
          fill_result(w.out[idx[lo + k]], *batch[k], std::move(one.at(0)), g);
        } catch (const TaskFailure& f) {
          w.fail(idx[lo + k], Failure{f.phase(), f.what()});
        } catch (const ucores::KernelPanic& e) {
          w.fail(idx[lo + k], Failure{e.phase(), e.what()});
        } catch (const std::exception& e) {
          w.fail(idx[lo + k], Failure{"run", e.what()});
        }
      }
    }
    per_gpu_[g] += hi - lo;
  }

  void run_group(const std::vector<ucores::Task>& tasks, const std::string& name, const std::vector<std::size_t>& idx,
                 int max_retries, Wave& w) {
    per_gpu_.resize(gpus_.size(), 0);
    const DeviceOp* op = ops_->find(name);
    if (!op || !op->run_tasks) {
      for (std::size_t i : idx) w.fail(i, Failure{"run", "no device body for kernel '" + name + "' (no CPU fallback)"});
    } else {
      const std::size_t T = idx.size(), G = std::min(gpus_.size(), T);
      std::vector<std::thread> threads;
      std::vector<std::exception_ptr> errs(G);
      for (std::size_t g = 1; g < G; ++g) {
        threads.emplace_back([&, g] {
          try {
            run_batch(tasks, *op, idx, g * T / G, (g + 1) * T / G, g, w);
          } catch (...) {
            errs[g] = std::current_exception();
          }
        });
      }
      run_batch(tasks, *op, idx, 0, T / G, 0, w);
      for (auto& t : threads) t.join();
      for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    }
    // retries: attempt 1..max_retries on the next GPU (scheduler.hpp:290-302)
    std::map<std::size_t, Failure> failed;
    failed.swap(w.failed);
    for (auto& [i, first] : failed) {
      std::optional<Failure> last = first;
      for (int a = 1; a <= max_retries && last; ++a) {
        ++retries_;
        const std::size_t g = (i + a) % gpus_.size();
        last.reset();
        if (op && op->run_tasks) {
          std::vector<std::size_t> one{i};
          run_batch(tasks, *op, one, 0, 1, g, w);
          if (auto it = w.failed.find(i); it != w.failed.end()) {
            last = it->second;
            w.failed.erase(it);
          }
        } else {
          last = first;
        }
      }
      if (last) {
        throw ucores::JobFailed("task " + std::to_string(tasks[i].task_id) + " of job " +
                                std::to_string(tasks[i].job_id) + " failed after " + std::to_string(max_retries + 1) +
                                " attempts (phase " + last->phase + ": " + last->detail + ")");
      }
    }
  }

  void run_per_task(const std::vector<ucores::Task>& tasks, int max_retries, Wave& w) {
    per_gpu_.resize(gpus_.size(), 0);
    const std::size_t T = tasks.size(), G = std::min(gpus_.size(), T);
    std::vector<std::optional<std::string>> failure(T);
    auto work = [&](std::size_t g) {
      for (std::size_t i = g * T / G; i < (g + 1) * T / G; ++i) {
        for (int a = 0;; ++a) {
          const std::size_t gg = (g + a) % gpus_.size();
          ucores::Message m = workers_[gg]->execute(tasks[i]);
          if (auto* r = std::get_if<ucores::TaskResultMsg>(&m)) {
            w.out[i] = std::move(r->result);
            break;
          }
          const auto& e = std::get<ucores::TaskErrorMsg>(m);
          if (a >= max_retries) {
            failure[i] = "task " + std::to_string(tasks[i].task_id) + " of job " + std::to_string(tasks[i].job_id) +
                         " failed after " + std::to_string(a + 1) + " attempts (phase " + e.phase + ": " + e.detail + ")";
            break;
          }
        }
        per_gpu_[g] += 1;
      }
    };
    std::vector<std::thread> threads;
    for (std::size_t g = 1; g < G; ++g) threads.emplace_back(work, g);
    work(0);
    for (auto& t : threads) t.join();
    for (auto& f : failure)
      if (f) throw ucores::JobFailed(*f);
  }

  void fill_result(ucores::TaskResult& r, const ucores::Task& t, ucores::Element out, std::size_t g) const {
    r.job_id = t.job_id;
    r.task_id = t.task_id;
    r.worker_id = worker_ids_[g];
    std::uint64_t in_bytes = 0, items = 0;
    for (const auto& e : t.inputs) {
      in_bytes += e.byte_size();
      items = std::max<std::uint64_t>(items, e.size());
    }
    r.metrics.items = items;
    r.metrics.bytes_moved = in_bytes + out.byte_size();
    r.metrics.executor_kind = "cuda-sm100a";
    r.metrics.device_invocations = 1;
    r.output = std::move(out);
  }

  const ucores::KernelRegistry* registry_;
  const DeviceOpRegistry* ops_;
  Options opt_;
  std::vector<std::shared_ptr<Gpu>> gpus_;
  std::vector<std::unique_ptr<GpuWorkerRuntime>> workers_;
  std::vector<std::string> worker_ids_;
  std::atomic<std::uint64_t> job_id_{0};
  std::uint64_t waves_ = 0, tasks_ = 0, retries_ = 0;
  std::vector<std::uint64_t> per_gpu_;
};

}  // namespace ucores_b200
