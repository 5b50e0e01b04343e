// o1d_internal.h — plan structure and helpers shared by the host code and the
// CUDA launchers of liboriented1d (never exposed through the C ABI).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/oriented1d.h"

namespace o1d {

// Thread-local error message behind o1d_last_error().
void set_error(const std::string &msg);
o1d_status fail(o1d_status st, const std::string &msg);

// Tap rule of P:1263-1264 with reading R3 (floor of the exact real value).
void make_taps_one(int K, int pad, double theta_deg, int16_t *oh, int16_t *ow);

// Geometry of one "stencil launch": an output plane of Ho x Wo computed from an
// input plane of Hi x Wi with stride `str` and per-channel taps (dh, dw):
//   out[p][q] = sum_k in[str*p + dh_k][str*q + dw_k] * wt[k]   (zero outside)
// forward: in = x, out = y, taps (oh, ow).  backward_input (str == 1): in = dy,
// out = dx, taps (-oh, -ow): dx[h][w] = sum_k dy[h-oh_k][w-ow_k] w_k.
struct Stencil {
    int Hi, Wi, Ho, Wo, str, K;
    int minDH, maxDH, minDW, maxDW;  // over all channels
    const int16_t *d_dh, *d_dw;      // device [C][K]
};

// Specialised (JIT) kernel handle, one per distinct tap table and pass.
struct JitKernel;

struct SpecSet;  // JIT-specialised kernels for one plan (o1d_jit.cpp)

}  // namespace o1d

struct o1d_plan {
    o1d_desc d;
    int P, Q, pad;
    int device;
    std::vector<double> angles;
    std::vector<int16_t> oh, ow;      // host [C][K]
    int minOH, maxOH, minOW, maxOW;   // over all channels
    int n_distinct;                   // distinct tap tables
    std::vector<int32_t> table_of;    // channel -> distinct table index
    // device copies, one allocation
    void *d_block = nullptr;
    int16_t *d_oh = nullptr, *d_ow = nullptr, *d_noh = nullptr, *d_now = nullptr;
    o1d::Stencil fwd, bwd_in;
    // generic backward_weight band height (output rows per CTA) and band count
    int bw_band = 0, bw_bands = 0;
    int fwd_band = 0, bi_band = 0;
    size_t ws_bytes = 0;
    o1d::SpecSet *spec = nullptr;     // null => generic kernels only
    void *aux_stream = nullptr;       // o1d_step_host's second stream (cudaStream_t)
    void *aux_ev[2] = {nullptr, nullptr};
    void *aux_stream2 = nullptr;      // o1d_step_host's third stream (device -> host copies, pipelined path)
    static constexpr int kChunkEv = 3 * 16;
    void *chunk_ev[kChunkEv] = {};    // per batch chunk: inputs on device x / dy, outputs ready
    std::string describe;
};

namespace o1d {
// launchers (o1d_kernels.cu); return O1D_OK or O1D_CUDA_ERROR (message set)
o1d_status generic_stencil(const o1d_plan *pl, const Stencil &st, int band, const void *in, const float *w,
                           void *out, void *stream);
o1d_status generic_bwd_input_strided(const o1d_plan *pl, const void *dy, const float *w, void *dx, void *stream);
o1d_status generic_bwd_weight(const o1d_plan *pl, const void *x, const void *dy, float *dW, float *ws,
                              void *stream);
int generic_band_rows(const o1d_plan *pl, const Stencil &st, int extra_rows_per_out);
size_t dtype_size(int dt);
// GPC id per %smid (probe with thread-block clusters; cached); false if unavailable
bool gpc_map(int device, std::vector<int> *gpc_of_smid);
}  // namespace o1d
