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
void make_taps_one(int K, double pad, double theta_deg, int16_t *oh, int16_t *ow);

// Geometry of one "stencil launch": an output plane of Ho x Wo computed from an
// input plane of Hi x Wi with stride `str` and per-channel WEIGHTED taps: KE
// entries e per channel, each an offset (dh, dw), a source tap index k and a
// coefficient (rotation / shear: KE = K, k = e, coef = 1; bilinear: up to four
// neighbours per tap with the interpolation weights, reading R14):
//   out[p][q] = sum_e in[str*p + dh_e][str*q + dw_e] * coef_e * wt[k_e]   (zero outside)
// forward: in = x, out = y, taps (dh, dw).  backward_input (str == 1): in = dy,
// out = dx, negated taps: dx[h][w] = sum_e dy[h-dh_e][w-dw_e] coef_e w_{k_e}.
struct Stencil {
    int Hi, Wi, Ho, Wo, str, KE;
    int minDH, maxDH, minDW, maxDW;  // over all channels
    const int16_t *d_dh, *d_dw;      // device [C][KE]
    // input rows the taps can reach are every rstep-th row of a tile (str > 1 and every dh congruent
    // mod str, e.g. the stem's horizontal stride-2 layer): the others are never staged
    int rstep = 1;
};

struct SpecSet;  // JIT-specialised kernels for one plan (o1d_spec.cpp)

}  // namespace o1d

struct o1d_plan {
    o1d_desc d;
    int P, Q;
    double pad;
    int device;
    int disc;                         // O1D_TAPS_ROTATION / _SHEAR / _BILINEAR
    std::vector<double> angles;
    std::vector<int16_t> oh, ow;      // host [C][K]: the floor taps (bilinear: the base corner)
    // expanded weighted taps, host [C][KE] (see o1d::Stencil)
    int KE = 0;
    std::vector<int16_t> eoh, eow, ek;
    std::vector<float> ecoef;
    int minOH, maxOH, minOW, maxOW;   // over all channels, expanded taps
    int n_distinct;                   // distinct (expanded) tap tables
    std::vector<int32_t> table_of;    // channel -> distinct table index
    // device copies, one allocation: eoh, eow, -eoh, -eow, ek (int16 [C][KE]) then coef (f32 [C][KE])
    void *d_block = nullptr;
    int16_t *d_oh = nullptr, *d_ow = nullptr, *d_noh = nullptr, *d_now = nullptr, *d_ek = nullptr;
    float *d_coef = nullptr;
    o1d::Stencil fwd, bwd_in;
    // generic backward_weight band height (output rows per CTA) and band count
    int bw_band = 0, bw_bands = 0;
    int fwd_band = 0, bi_band = 0;
    size_t ws_bytes = 0;
    o1d::SpecSet *spec = nullptr;     // null => generic kernels only
    double plan_ms = 0.0;             // host time of o1d_plan_create (incl. JIT or cache hit)
    bool jit_cache_hit = false;
    int e2e_chunks = 8;               // o1d_step_host batch chunks (O1D_E2E_CHUNKS at plan creation)
    void *aux_stream = nullptr;       // o1d_step_host's second stream (cudaStream_t)
    void *aux_ev[2] = {nullptr, nullptr};
    void *aux_stream2 = nullptr;      // o1d_step_host's third stream (device -> host copies, pipelined path)
    static constexpr int kChunkEv = 3 * 16;
    void *chunk_ev[kChunkEv] = {};    // per batch chunk: inputs on device x / dy, outputs ready
    std::string describe;
};

namespace o1d {
// launchers (o1d_generic.cu); return O1D_OK or O1D_CUDA_ERROR (message set)
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
