// o1d_spec.h — runtime-specialised (JIT) kernels: one case per distinct tap
// table, with the taps compiled in as constants so the register-blocked tap
// loops get static register indexing.
#pragma once
#include <string>

#include "o1d_internal.h"

namespace o1d {
o1d_status spec_create(o1d_plan *pl);  // may leave pl->spec == nullptr (generic only)
// generated CUDA source of one pass (host only; diagnostics)
o1d_status spec_source(const o1d_plan *pl, int pass, std::string *out);
void spec_destroy(o1d_plan *pl);
bool spec_has(const o1d_plan *pl, int pass);
int spec_launches(const o1d_plan *pl, int pass);
size_t spec_workspace_bytes(const o1d_plan *pl);
// diagnostics: copy (and reset) the O1D_TRACE event buffer; returns bytes copied (0: tracing off)
size_t spec_trace(const o1d_plan *pl, void *host, size_t bytes);
// pass 0: a=x, w, b=y; pass 1: a=dy, w, b=dx; pass 2: a=x, b=dy, dW, ws
// n0/nlen: batch window (planes n in [n0, n0 + nlen), nlen = 0: all); finalize: pass 2 also
// launches the dW finalize (set false for all but the last window, see spec_finalize)
o1d_status spec_run(const o1d_plan *pl, int pass, const void *a, const float *w, const void *b, float *dW,
                    float *ws, void *stream, int n0 = 0, int nlen = 0, bool finalize = true, bool nowait = false);
bool spec_window_ok(const o1d_plan *pl);
o1d_status spec_finalize(const o1d_plan *pl, float *dW, const float *ws, void *stream);
}  // namespace o1d
