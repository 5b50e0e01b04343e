// o1d_spec.cpp — placeholder until the specialised kernels land: every plan
// uses the generic kernels.
#include "o1d_spec.h"

namespace o1d {
o1d_status spec_create(o1d_plan *pl) { pl->spec = nullptr; return O1D_OK; }
void spec_destroy(o1d_plan *) {}
bool spec_has(const o1d_plan *, int) { return false; }
int spec_launches(const o1d_plan *, int) { return 0; }
size_t spec_workspace_bytes(const o1d_plan *) { return 0; }
o1d_status spec_run(const o1d_plan *, int, const void *, const float *, const void *, float *, float *, void *) {
    return fail(O1D_UNSUPPORTED, "no specialised kernels");
}
}  // namespace o1d
