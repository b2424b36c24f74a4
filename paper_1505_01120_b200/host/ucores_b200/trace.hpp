// trace.hpp — NVTX ranges around the host-side stages of the path (SURVEY §5
// tracing): the driver's waves and per-GPU batches (seam A), the executor's
// run phase (seam B), DeviceEngine's operators and transfers. They show up in
// nsys timelines and filter ncu captures (`ncu --nvtx --nvtx-include
// "ucores.map_cl_partition:psum/"`; names avoid '/', ncu's nesting
// separator). nvtx3 is header-only and binds a tool lazily: with no
// tool attached a range is one predicted branch.
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <string>

namespace ucores_b200 {

class TraceRange {
 public:
  explicit TraceRange(const char* name) { nvtxRangePushA(name); }
  explicit TraceRange(const std::string& name) { nvtxRangePushA(name.c_str()); }
  ~TraceRange() { nvtxRangePop(); }
  TraceRange(const TraceRange&) = delete;
  TraceRange& operator=(const TraceRange&) = delete;
};

}  // namespace ucores_b200
