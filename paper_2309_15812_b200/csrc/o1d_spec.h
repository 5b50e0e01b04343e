// o1d_spec.h — runtime-specialised (JIT) kernels: one case per distinct tap
// table, with the taps compiled in as constants so the register-blocked tap
// loops get static register indexing.
#pragma once
#include <string>

#include "o1d_internal.h"

namespace o1d {
// buffers of one launch; which are used depends on the pass:
//   0 forward: x, w -> y      1 backward_input: dy, w -> dx      2 backward_weight: x, dy -> dW (ws)
//   3 fused backward: x, dy, w -> dx, dW (ws)
struct RunArgs {
    const void *x = nullptr, *dy = nullptr;
    const float *w = nullptr;
    void *y = nullptr, *dx = nullptr;
    float *dW = nullptr, *ws = nullptr;
};
o1d_status spec_create(o1d_plan *pl);  // may leave pl->spec == nullptr (generic only)
// generated CUDA source of one pass (host only; diagnostics)
o1d_status spec_source(const o1d_plan *pl, int pass, std::string *out);
void spec_destroy(o1d_plan *pl);
bool spec_has(const o1d_plan *pl, int pass);
bool spec_step_fused(const o1d_plan *pl);  // o1d_step runs forward + the fused backward
int spec_launches(const o1d_plan *pl, int pass);
size_t spec_workspace_bytes(const o1d_plan *pl);
// diagnostics: copy (and reset) the O1D_TRACE event buffer; returns bytes copied (0: tracing off)
size_t spec_trace(const o1d_plan *pl, void *host, size_t bytes);
// n0/nlen: batch window (planes n in [n0, n0 + nlen), nlen = 0: all); finalize: passes 2/3 also
// launch the dW finalize (set false for all but the last window, see spec_finalize); nowait: the
// inputs do not come from the preceding kernel on the stream (o1d_step)
o1d_status spec_run(const o1d_plan *pl, int pass, const RunArgs &a, void *stream, int n0 = 0, int nlen = 0,
                    bool finalize = true, bool nowait = false);
bool spec_window_ok(const o1d_plan *pl);
o1d_status spec_finalize(const o1d_plan *pl, int pass, float *dW, const float *ws, void *stream);
}  // namespace o1d
