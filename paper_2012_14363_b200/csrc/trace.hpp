// trace.hpp -- NVTX ranges around the C-ABI entry points (nsys / ncu
// --nvtx show engine calls by name). nvtx3 is header-only and resolves its
// tool library lazily: with no profiler attached a range costs a branch.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace spb {
struct TraceRange {
  explicit TraceRange(const char *name) { nvtxRangePushA(name); }
  ~TraceRange() { nvtxRangePop(); }
  TraceRange(const TraceRange &) = delete;
  TraceRange &operator=(const TraceRange &) = delete;
};
} // namespace spb

#define SPB_TRACE_CAT2(a, b) a##b
#define SPB_TRACE_CAT(a, b) SPB_TRACE_CAT2(a, b)
#define SPB_TRACE(name) ::spb::TraceRange SPB_TRACE_CAT(spb_trace_, __LINE__)(name)
