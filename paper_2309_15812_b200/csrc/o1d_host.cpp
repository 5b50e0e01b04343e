// o1d_host.cpp — host side of liboriented1d: the C ABI entry points, tap
// generation (P:1263-1264 with reading R3), plan creation and validation.
#include <cuda_runtime.h>
#include <quadmath.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "o1d_internal.h"
#include "o1d_spec.h"

namespace o1d {

static thread_local std::string g_err;

static int env_int_host(const char *n, int dflt) {
    const char *v = getenv(n);
    return (v && *v) ? atoi(v) : dflt;
}

void set_error(const std::string &msg) { g_err = msg; }
o1d_status fail(o1d_status st, const std::string &msg) {
    g_err = msg;
    return st;
}

// Tap rule of P:1263-1264 evaluated as the floor of the EXACT real value
// (reading R3).  The angle is a binary double, i.e. a rational number of
// degrees t, so by Niven's theorem sin(t) is rational only at t = 0, 30, 90,
// 150, 180, 210, 270, 330 (mod 360) and cos(t) only at t = 0, 60, 90, 120, 180,
// 240, 270, 300; there the product m*sin / m*cos is evaluated exactly.  Any other
// product is irrational, never an integer: f64 gives its floor unless it lies
// within 1e-9 of an integer, in which case it is re-evaluated in binary128
// (__float128, 113-bit significand), exact unless the angle lies within ~1e-28
// degrees of one of the Niven angles above.
static bool niven_sin(double t, double *v) {  // t in [0, 360)
    static const double a[8] = {0, 30, 90, 150, 180, 210, 270, 330};
    static const double s[8] = {0, 0.5, 1, 0.5, 0, -0.5, -1, -0.5};
    for (int i = 0; i < 8; ++i)
        if (t == a[i]) { *v = s[i]; return true; }
    return false;
}
static bool niven_cos(double t, double *v) {
    static const double a[8] = {0, 60, 90, 120, 180, 240, 270, 300};
    static const double c[8] = {1, 0.5, 0, -0.5, -1, -0.5, 0, 0.5};
    for (int i = 0; i < 8; ++i)
        if (t == a[i]) { *v = c[i]; return true; }
    return false;
}

// floor(m * f(t)) for f = sin (is_sin) or cos, t in degrees reduced to [0, 360)
static int floor_trig_times(int m, double t, bool is_sin) {
    if (m == 0) return 0;
    double r;
    if (is_sin ? niven_sin(t, &r) : niven_cos(t, &r)) return (int)std::floor((double)m * r);  // exact: r in {0,+-1/2,+-1}
    const double rad = t * (M_PI / 180.0);
    const double v = (double)m * (is_sin ? std::sin(rad) : std::cos(rad));
    const double n = std::nearbyint(v);
    if (std::fabs(v - n) >= 1e-9) return (int)std::floor(v);
    const __float128 radq = (__float128)t * (acosq((__float128)-1) / 180);
    const __float128 vq = (__float128)m * (is_sin ? sinq(radq) : cosq(radq));
    return (int)floorq(vq);
}


// Shear form (reading R13): offset = m (-sin t, cos t) / max(|sin t|, |cos t|).
// The grid coordinate is exact (+-m); the other one is floor(-+m tan t) / floor(+-m cot t).
// tan t of a rational angle is rational only at t = 0, 45, 135 (mod 180) (Niven): exact
// there; elsewhere irrational, floored from f64 unless within 1e-9 of an integer, then in
// binary128.
static int floor_m_tan(int m, double t, bool cot) {  // floor(m * tan(t)) or floor(m * cot(t)), t in [0, 360)
    if (m == 0) return 0;
    const double u = std::fmod(t, 180.0);
    if (!cot && (u == 0.0)) return 0;
    if (!cot && (u == 45.0)) return m;
    if (!cot && (u == 135.0)) return -m;
    if (cot && u == 90.0) return 0;
    if (cot && u == 45.0) return m;
    if (cot && u == 135.0) return -m;
    const double rad = t * (M_PI / 180.0);
    const double v = (double)m * (cot ? std::cos(rad) / std::sin(rad) : std::tan(rad));
    const double n = std::nearbyint(v);
    if (std::fabs(v - n) >= 1e-9) return (int)std::floor(v);
    const __float128 radq = (__float128)t * (acosq((__float128)-1) / 180);
    const __float128 vq = (__float128)m * (cot ? cosq(radq) / sinq(radq) : tanq(radq));
    return (int)floorq(vq);
}

void make_taps_one_shear(int K, int pad, double theta_deg, int16_t *oh, int16_t *ow) {
    double t = std::fmod(theta_deg, 360.0);  // exact
    if (t < 0) t += 360.0;
    if (t >= 360.0) t -= 360.0;
    const double u = std::fmod(t, 180.0);
    const bool cols = u <= 45.0 || u >= 135.0;  // |cos t| >= |sin t|
    const int sgn_cos = (t < 90.0 || t > 270.0) ? 1 : ((t > 90.0 && t < 270.0) ? -1 : 0);
    const int sgn_sin = (t > 0.0 && t < 180.0) ? 1 : (t > 180.0 ? -1 : 0);
    for (int k = 0; k < K; ++k) {
        const int m = k - pad;
        if (cols) {  // delta_w = m sgn(cos t), delta_h = -m tan(t) sgn(cos t)
            ow[k] = (int16_t)(m * sgn_cos);
            oh[k] = (int16_t)floor_m_tan(-m * sgn_cos, t, false);
        } else {     // delta_h = -m sgn(sin t), delta_w = m cot(t) sgn(sin t)
            oh[k] = (int16_t)(-m * sgn_sin);
            ow[k] = (int16_t)floor_m_tan(m * sgn_sin, t, true);
        }
    }
}

void make_taps_one(int K, int pad, double theta_deg, int16_t *oh, int16_t *ow) {
    double t = std::fmod(theta_deg, 360.0);  // exact
    if (t < 0) t += 360.0;
    if (t >= 360.0) t -= 360.0;
    for (int k = 0; k < K; ++k) {
        const int m = k - pad;
        oh[k] = (int16_t)floor_trig_times(-m, t, true);   // floor(-(k-pad) sin t)
        ow[k] = (int16_t)floor_trig_times(m, t, false);   // floor( (k-pad) cos t)
    }
}

}  // namespace o1d

using namespace o1d;

extern "C" {

const char *o1d_last_error(void) { return g_err.c_str(); }
const char *o1d_version(void) { return "liboriented1d 0.1 (sm_100a)"; }

o1d_status o1d_make_taps(int32_t K, int32_t pad, int32_t C, const double *angles_deg, int16_t *oh, int16_t *ow) {
    if (!angles_deg || !oh || !ow) return fail(O1D_INVALID_ARG, "o1d_make_taps: NULL pointer");
    if (K < 1) return fail(O1D_INVALID_CONFIG, "o1d_make_taps: K < 1");
    if (C < 1) return fail(O1D_INVALID_SHAPE, "o1d_make_taps: C < 1");
    if (pad < 0) pad = K / 2;
    if (pad >= K) return fail(O1D_INVALID_CONFIG, "o1d_make_taps: pad >= K");
    for (int c = 0; c < C; ++c) {
        if (!std::isfinite(angles_deg[c])) return fail(O1D_INVALID_ARG, "o1d_make_taps: non-finite angle");
        make_taps_one(K, pad, angles_deg[c], oh + (size_t)c * K, ow + (size_t)c * K);
    }
    return O1D_OK;
}

o1d_status o1d_make_taps_ex(int32_t K, int32_t pad, int32_t C, const double *angles_deg, int32_t mode, int16_t *oh,
                            int16_t *ow) {
    if (mode == O1D_TAPS_ROTATION) return o1d_make_taps(K, pad, C, angles_deg, oh, ow);
    if (mode != O1D_TAPS_SHEAR) return fail(O1D_INVALID_ARG, "o1d_make_taps_ex: mode must be O1D_TAPS_ROTATION or O1D_TAPS_SHEAR");
    if (!angles_deg || !oh || !ow) return fail(O1D_INVALID_ARG, "o1d_make_taps_ex: NULL pointer");
    if (K < 1) return fail(O1D_INVALID_CONFIG, "o1d_make_taps_ex: K < 1");
    if (C < 1) return fail(O1D_INVALID_SHAPE, "o1d_make_taps_ex: C < 1");
    if (pad < 0) pad = K / 2;
    if (pad >= K) return fail(O1D_INVALID_CONFIG, "o1d_make_taps_ex: pad >= K");
    for (int c = 0; c < C; ++c) {
        if (!std::isfinite(angles_deg[c])) return fail(O1D_INVALID_ARG, "o1d_make_taps_ex: non-finite angle");
        make_taps_one_shear(K, pad, angles_deg[c], oh + (size_t)c * K, ow + (size_t)c * K);
    }
    return O1D_OK;
}

o1d_status o1d_direction_angles(int32_t D, int32_t C, int32_t assign, double shift_deg, double *out) {
    if (!out) return fail(O1D_INVALID_ARG, "o1d_direction_angles: NULL out");
    if (C < 1) return fail(O1D_INVALID_SHAPE, "o1d_direction_angles: C < 1");
    if (D < 1 || (C % D != 0 && D != C)) return fail(O1D_INVALID_CONFIG, "o1d_direction_angles: D must divide C (or D == C)");
    if (assign != O1D_ASSIGN_CONTIGUOUS && assign != O1D_ASSIGN_CYCLED)
        return fail(O1D_INVALID_ARG, "o1d_direction_angles: bad assign");
    for (int c = 0; c < C; ++c) {
        const long g = assign == O1D_ASSIGN_CONTIGUOUS ? ((long)c * D) / C : c % D;
        // i*180/D is exact in f64 whenever D's odd part divides 180*i exactly or is a power of 2 times it
        double a = (180.0 * (double)g) / (double)D;
        if (shift_deg != 0.0) {
            a = std::fmod(a + shift_deg, 180.0);
            if (a < 0) a += 180.0;
        }
        out[c] = a;
    }
    return O1D_OK;
}

static o1d_status validate_desc(const o1d_desc *d) {
    if (!d) return fail(O1D_INVALID_ARG, "NULL descriptor");
    if (d->N < 1 || d->C < 1 || d->H < 1 || d->W < 1) return fail(O1D_INVALID_SHAPE, "N, C, H, W must be >= 1");
    if (d->K < 1) return fail(O1D_INVALID_CONFIG, "K must be >= 1");
    if (d->stride < 1) return fail(O1D_INVALID_CONFIG, "stride must be >= 1");
    if (d->pad >= d->K) return fail(O1D_INVALID_CONFIG, "pad must be < K");
    if (d->pad < -1) return fail(O1D_INVALID_CONFIG, "pad must be >= 0 (or -1 for floor(K/2))");
    if (d->dtype != O1D_F32 && d->dtype != O1D_BF16 && d->dtype != O1D_F16)
        return fail(O1D_UNSUPPORTED, "dtype must be O1D_F32, O1D_BF16 or O1D_F16");
    if (d->layout != O1D_NCHW) return fail(O1D_UNSUPPORTED, "only the NCHW-contiguous layout is implemented");
    if ((long)d->N * d->C * d->H * d->W > (1L << 40)) return fail(O1D_UNSUPPORTED, "tensor too large");
    if (d->K > 1023) return fail(O1D_UNSUPPORTED, "K > 1023");
    if (d->flags & ~(O1D_FLAG_FORCE_GENERIC | O1D_FLAG_NO_TMA | O1D_FLAG_SHEAR))
        return fail(O1D_INVALID_ARG, "unknown bits in o1d_desc.flags");
    return O1D_OK;
}

// Host-only part of plan creation: taps, distinct tables, halo extents.
static o1d_status plan_host_init(const o1d_desc *d, const double *angles_deg, o1d_plan *pl) {
    if (o1d_status st = validate_desc(d)) return st;
    if (!angles_deg) return fail(O1D_INVALID_ARG, "o1d_plan_create: NULL angles");
    pl->d = *d;
    pl->pad = d->pad < 0 ? d->K / 2 : d->pad;
    pl->d.pad = pl->pad;
    pl->P = (d->H - 1) / d->stride + 1;
    pl->Q = (d->W - 1) / d->stride + 1;
    const int C = d->C, K = d->K;
    pl->angles.assign(angles_deg, angles_deg + C);
    pl->oh.resize((size_t)C * K);
    pl->ow.resize((size_t)C * K);
    if (o1d_status st = o1d_make_taps_ex(K, pl->pad, C, angles_deg, (d->flags & O1D_FLAG_SHEAR) ? O1D_TAPS_SHEAR : O1D_TAPS_ROTATION,
                                         pl->oh.data(), pl->ow.data()))
        return st;
    std::map<std::vector<int16_t>, int> ids;
    pl->table_of.resize(C);
    pl->minOH = pl->minOW = 1 << 20;
    pl->maxOH = pl->maxOW = -(1 << 20);
    for (int c = 0; c < C; ++c) {
        std::vector<int16_t> key(2 * K);
        for (int k = 0; k < K; ++k) {
            key[2 * k] = pl->oh[c * K + k];
            key[2 * k + 1] = pl->ow[c * K + k];
            pl->minOH = std::min<int>(pl->minOH, pl->oh[c * K + k]);
            pl->maxOH = std::max<int>(pl->maxOH, pl->oh[c * K + k]);
            pl->minOW = std::min<int>(pl->minOW, pl->ow[c * K + k]);
            pl->maxOW = std::max<int>(pl->maxOW, pl->ow[c * K + k]);
        }
        auto it = ids.find(key);
        if (it == ids.end()) it = ids.emplace(key, (int)ids.size()).first;
        pl->table_of[c] = it->second;
    }
    pl->n_distinct = (int)ids.size();
    return O1D_OK;
}

size_t o1d_debug_trace(const o1d_plan *pl, void *host, size_t bytes) {
    if (!pl || !host) return 0;
    return spec_trace(pl, host, bytes);
}

o1d_status o1d_spec_source(const o1d_desc *d, const double *angles_deg, int32_t pass, char *buf, size_t *len) {
    if (!len) return fail(O1D_INVALID_ARG, "o1d_spec_source: NULL len");
    o1d_plan pl;
    if (o1d_status st = plan_host_init(d, angles_deg, &pl)) return st;
    std::string src;
    if (o1d_status st = spec_source(&pl, pass, &src)) return st;
    if (buf && *len > src.size()) memcpy(buf, src.c_str(), src.size() + 1);
    *len = src.size() + 1;
    return O1D_OK;
}

o1d_status o1d_plan_create(const o1d_desc *d, const double *angles_deg, o1d_plan **out) {
    if (!out) return fail(O1D_INVALID_ARG, "o1d_plan_create: NULL out");
    *out = nullptr;
    if (o1d_status st = validate_desc(d)) return st;
    o1d_plan *pl = new (std::nothrow) o1d_plan();
    if (!pl) return fail(O1D_INVALID_ARG, "out of host memory");
    if (o1d_status st = plan_host_init(d, angles_deg, pl)) {
        delete pl;
        return st;
    }
    const int C = d->C, K = d->K;
    // device tables: oh, ow, -oh, -ow
    if (cudaGetDevice(&pl->device) != cudaSuccess) {
        delete pl;
        return fail(O1D_CUDA_ERROR, std::string("cudaGetDevice: ") + cudaGetErrorString(cudaGetLastError()));
    }
    const size_t tb = sizeof(int16_t) * (size_t)C * K;
    std::vector<int16_t> host(4 * (size_t)C * K);
    for (size_t i = 0; i < (size_t)C * K; ++i) {
        host[i] = pl->oh[i];
        host[(size_t)C * K + i] = pl->ow[i];
        host[2 * (size_t)C * K + i] = (int16_t)-pl->oh[i];
        host[3 * (size_t)C * K + i] = (int16_t)-pl->ow[i];
    }
    if (cudaMalloc(&pl->d_block, 4 * tb) != cudaSuccess ||
        cudaMemcpy(pl->d_block, host.data(), 4 * tb, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaError_t e = cudaGetLastError();
        if (pl->d_block) cudaFree(pl->d_block);
        delete pl;
        return fail(O1D_CUDA_ERROR, std::string("plan tables: ") + cudaGetErrorString(e));
    }
    int16_t *base = static_cast<int16_t *>(pl->d_block);
    pl->d_oh = base;
    pl->d_ow = base + (size_t)C * K;
    pl->d_noh = base + 2 * (size_t)C * K;
    pl->d_now = base + 3 * (size_t)C * K;
    // stencil geometry of the forward and (stride 1) backward_input passes
    pl->fwd = Stencil{d->H, d->W, pl->P, pl->Q, d->stride, K, pl->minOH, pl->maxOH, pl->minOW, pl->maxOW,
                      pl->d_oh, pl->d_ow};
    pl->bwd_in = Stencil{pl->P, pl->Q, d->H, d->W, 1, K, -pl->maxOH, -pl->minOH, -pl->maxOW, -pl->minOW,
                         pl->d_noh, pl->d_now};
    pl->fwd_band = generic_band_rows(pl, pl->fwd, 0);
    pl->bi_band = d->stride == 1 ? generic_band_rows(pl, pl->bwd_in, 0) : 1;
    pl->bw_band = generic_band_rows(pl, pl->fwd, 1);
    if (pl->fwd_band == 0 || pl->bi_band == 0 || pl->bw_band == 0) {
        o1d_plan_destroy(pl);
        return fail(O1D_UNSUPPORTED, "image row (plus halo) does not fit in shared memory");
    }
    pl->bw_bands = (pl->P + pl->bw_band - 1) / pl->bw_band;
    {
        cudaStream_t s2 = nullptr;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&e0, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) != cudaSuccess) {
            o1d_plan_destroy(pl);
            return fail(O1D_CUDA_ERROR, "stream/event creation failed");
        }
        pl->aux_stream = s2;
        pl->aux_ev[0] = e0;
        pl->aux_ev[1] = e1;
        cudaStream_t s3 = nullptr;
        bool ok = cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking) == cudaSuccess;
        pl->aux_stream2 = s3;
        for (int i = 0; ok && i < o1d_plan::kChunkEv; ++i) {
            cudaEvent_t e = nullptr;
            ok = cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
            pl->chunk_ev[i] = e;
        }
        if (!ok) {
            o1d_plan_destroy(pl);
            return fail(O1D_CUDA_ERROR, "stream/event creation failed");
        }
    }
    pl->ws_bytes = sizeof(float) * (size_t)d->N * C * pl->bw_bands * K;
    char buf[256];
    snprintf(buf, sizeof buf, "generic(fwd band %d, bwd_in band %d, bwd_w band %d), %d distinct tap tables",
             pl->fwd_band, pl->bi_band, pl->bw_band, pl->n_distinct);
    pl->describe = buf;
    if (!(d->flags & O1D_FLAG_FORCE_GENERIC)) {
        o1d_status st = spec_create(pl);
        if (st != O1D_OK) {
            o1d_plan_destroy(pl);
            return st;
        }
    }
    *out = pl;
    return O1D_OK;
}

void o1d_plan_destroy(o1d_plan *pl) {
    if (!pl) return;
    spec_destroy(pl);
    if (pl->aux_stream) cudaStreamDestroy(static_cast<cudaStream_t>(pl->aux_stream));
    if (pl->aux_stream2) cudaStreamDestroy(static_cast<cudaStream_t>(pl->aux_stream2));
    for (void *e : pl->chunk_ev)
        if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
    for (void *e : pl->aux_ev)
        if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
    if (pl->d_block) cudaFree(pl->d_block);
    delete pl;
}

o1d_status o1d_plan_out_shape(const o1d_plan *pl, int32_t *P, int32_t *Q) {
    if (!pl || !P || !Q) return fail(O1D_INVALID_ARG, "o1d_plan_out_shape: NULL pointer");
    *P = pl->P;
    *Q = pl->Q;
    return O1D_OK;
}

o1d_status o1d_plan_get_taps(const o1d_plan *pl, int16_t *oh, int16_t *ow) {
    if (!pl || !oh || !ow) return fail(O1D_INVALID_ARG, "o1d_plan_get_taps: NULL pointer");
    std::memcpy(oh, pl->oh.data(), pl->oh.size() * sizeof(int16_t));
    std::memcpy(ow, pl->ow.data(), pl->ow.size() * sizeof(int16_t));
    return O1D_OK;
}

const char *o1d_plan_describe(const o1d_plan *pl) { return pl ? pl->describe.c_str() : ""; }

size_t o1d_workspace_bytes(const o1d_plan *pl) {
    if (!pl) return 0;
    return std::max(pl->ws_bytes, spec_workspace_bytes(pl));
}

static o1d_status check_ptr(const void *p, const char *name) {
    if (!p) return fail(O1D_INVALID_ARG, std::string(name) + " is NULL");
    if (reinterpret_cast<uintptr_t>(p) & 15) return fail(O1D_MISALIGNED, std::string(name) + " is not 16-byte aligned");
    return O1D_OK;
}

static o1d_status check_device(const o1d_plan *pl) {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(O1D_CUDA_ERROR, "cudaGetDevice failed");
    if (dev != pl->device) return fail(O1D_INVALID_ARG, "current device differs from the plan's device");
    return O1D_OK;
}

o1d_status o1d_forward(const o1d_plan *pl, const void *x, const float *w, void *y, void *stream) {
    if (!pl) return fail(O1D_INVALID_ARG, "NULL plan");
    if (o1d_status st = check_ptr(x, "x")) return st;
    if (o1d_status st = check_ptr(w, "w")) return st;
    if (o1d_status st = check_ptr(y, "y")) return st;
    if (o1d_status st = check_device(pl)) return st;
    if (pl->spec && spec_has(pl, 0)) return spec_run(pl, 0, x, w, y, nullptr, nullptr, stream);
    return generic_stencil(pl, pl->fwd, pl->fwd_band, x, w, y, stream);
}

o1d_status o1d_backward_input(const o1d_plan *pl, const void *dy, const float *w, void *dx, void *stream) {
    if (!pl) return fail(O1D_INVALID_ARG, "NULL plan");
    if (o1d_status st = check_ptr(dy, "dy")) return st;
    if (o1d_status st = check_ptr(w, "w")) return st;
    if (o1d_status st = check_ptr(dx, "dx")) return st;
    if (o1d_status st = check_device(pl)) return st;
    if (pl->spec && spec_has(pl, 1)) return spec_run(pl, 1, dy, w, dx, nullptr, nullptr, stream);
    if (pl->d.stride == 1) return generic_stencil(pl, pl->bwd_in, pl->bi_band, dy, w, dx, stream);
    return generic_bwd_input_strided(pl, dy, w, dx, stream);
}

o1d_status o1d_backward_weight(const o1d_plan *pl, const void *x, const void *dy, float *dW, void *ws,
                               size_t ws_bytes, void *stream) {
    if (!pl) return fail(O1D_INVALID_ARG, "NULL plan");
    if (o1d_status st = check_ptr(x, "x")) return st;
    if (o1d_status st = check_ptr(dy, "dy")) return st;
    if (o1d_status st = check_ptr(dW, "dW")) return st;
    if (o1d_status st = check_ptr(ws, "ws")) return st;
    if (ws_bytes < o1d_workspace_bytes(pl))
        return fail(O1D_WORKSPACE_TOO_SMALL, "ws_bytes < o1d_workspace_bytes(plan)");
    if (o1d_status st = check_device(pl)) return st;
    if (pl->spec && spec_has(pl, 2)) return spec_run(pl, 2, x, nullptr, dy, dW, static_cast<float *>(ws), stream);
    return generic_bwd_weight(pl, x, dy, dW, static_cast<float *>(ws), stream);
}

o1d_status o1d_step(const o1d_plan *pl, const void *x, const float *w, const void *dy, void *y, void *dx, float *dW,
                    void *ws, size_t ws_bytes, void *stream) {
    if (!pl) return fail(O1D_INVALID_ARG, "NULL plan");
    for (const void *q : {x, (const void *)w, dy, (const void *)y, (const void *)dx, (const void *)dW, (const void *)ws})
        if (o1d_status st = check_ptr(q, "o1d_step buffer")) return st;
    if (ws_bytes < o1d_workspace_bytes(pl)) return fail(O1D_WORKSPACE_TOO_SMALL, "ws_bytes < o1d_workspace_bytes(plan)");
    if (o1d_status st = check_device(pl)) return st;
    if (!(pl->spec && spec_has(pl, 0) && spec_has(pl, 1) && spec_has(pl, 2))) {
        if (o1d_status st = o1d_forward(pl, x, w, y, stream)) return st;
        if (o1d_status st = o1d_backward_input(pl, dy, w, dx, stream)) return st;
        return o1d_backward_weight(pl, x, dy, dW, ws, ws_bytes, stream);
    }
    // The three passes of a step read only the step's inputs (x, w, dy) and write disjoint
    // outputs, so backward_input and backward_weight need not wait for the preceding pass:
    // they start on the SMs the preceding pass frees (its tail) instead of after it.  The
    // forward still waits for whatever preceded the step on the stream.
    if (o1d_status st = spec_run(pl, 0, x, w, y, nullptr, nullptr, stream)) return st;
    if (o1d_status st = spec_run(pl, 1, dy, w, dx, nullptr, nullptr, stream, 0, 0, true, true)) return st;
    return spec_run(pl, 2, x, nullptr, dy, dW, static_cast<float *>(ws), stream, 0, 0, true, true);
}

int32_t o1d_launches_per_call(const o1d_plan *pl, int32_t pass) {
    if (!pl) return 0;
    if (pl->spec && spec_has(pl, pass)) return spec_launches(pl, pass);
    return pass == 2 ? 2 : 1;
}

static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

size_t o1d_step_host_workspace_bytes(const o1d_plan *pl) {
    if (!pl) return 0;
    const size_t es = dtype_size(pl->d.dtype);
    const size_t nx = (size_t)pl->d.N * pl->d.C * pl->d.H * pl->d.W * es;
    const size_t ny = (size_t)pl->d.N * pl->d.C * pl->P * pl->Q * es;
    const size_t nw = sizeof(float) * (size_t)pl->d.C * pl->d.K;
    return 2 * align256(nx) + 2 * align256(ny) + 2 * align256(nw) + align256(o1d_workspace_bytes(pl));
}

o1d_status o1d_step_host(const o1d_plan *pl, const void *x_h, const float *w_h, const void *dy_h, void *y_h,
                         void *dx_h, float *dW_h, void *dev_ws, size_t dev_ws_bytes, void *stream) {
    if (!pl || !x_h || !w_h || !dy_h || !y_h || !dx_h || !dW_h) return fail(O1D_INVALID_ARG, "o1d_step_host: NULL pointer");
    if (o1d_status st = check_ptr(dev_ws, "dev_ws")) return st;
    if (dev_ws_bytes < o1d_step_host_workspace_bytes(pl))
        return fail(O1D_WORKSPACE_TOO_SMALL, "dev_ws_bytes < o1d_step_host_workspace_bytes(plan)");
    if (o1d_status st = check_device(pl)) return st;
    const size_t es = dtype_size(pl->d.dtype);
    const size_t nx = (size_t)pl->d.N * pl->d.C * pl->d.H * pl->d.W * es;
    const size_t ny = (size_t)pl->d.N * pl->d.C * pl->P * pl->Q * es;
    const size_t nw = sizeof(float) * (size_t)pl->d.C * pl->d.K;
    char *b = static_cast<char *>(dev_ws);
    void *x = b; b += align256(nx);
    void *dx = b; b += align256(nx);
    void *y = b; b += align256(ny);
    void *dy = b; b += align256(ny);
    float *w = reinterpret_cast<float *>(b); b += align256(nw);
    float *dW = reinterpret_cast<float *>(b); b += align256(nw);
    void *ws = b;
    const int nch = pl->spec && spec_window_ok(pl) && pl->d.N >= 2 && env_int_host("O1D_E2E_CHUNKS", 8) > 1
                        ? std::min(std::min(pl->d.N, env_int_host("O1D_E2E_CHUNKS", 8)), 16)
                        : 0;
    if (nch > 1) {
        // Pipelined over batch chunks (the kernels take a batch window, so no sub-plans and the
        // dW partials land in the full workspace: dW is bitwise that of the unchunked step):
        //   s2 (H2D): w, then per chunk x_i -> ev x_i, dy_i -> ev dy_i
        //   s  (compute): per chunk: wait x_i: forward_i; wait dy_i: backward_input_i,
        //                 backward_weight_i (no finalize) -> ev out_i; then the finalize, D2H dW
        //   s3 (D2H): per chunk: wait out_i: y_i, dx_i
        // so the two PCIe directions stream concurrently and the kernels fill the gaps.
        cudaStream_t s = static_cast<cudaStream_t>(stream), s2 = static_cast<cudaStream_t>(pl->aux_stream),
                     s3 = static_cast<cudaStream_t>(pl->aux_stream2);
        cudaEvent_t e0 = static_cast<cudaEvent_t>(pl->aux_ev[0]), e1 = static_cast<cudaEvent_t>(pl->aux_ev[1]);
        auto cu = [](cudaError_t e, const char *what) -> o1d_status {
            if (e != cudaSuccess) return fail(O1D_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
            return O1D_OK;
        };
        auto ev = [&](int kind, int i) { return static_cast<cudaEvent_t>(pl->chunk_ev[kind * 16 + i]); };
        const size_t px = (size_t)pl->d.C * pl->d.H * pl->d.W * es, py = (size_t)pl->d.C * pl->P * pl->Q * es;
        if (o1d_status st = cu(cudaEventRecord(e0, s), "event")) return st;  // after prior work on s
        if (o1d_status st = cu(cudaStreamWaitEvent(s2, e0, 0), "wait")) return st;
        if (o1d_status st = cu(cudaStreamWaitEvent(s3, e0, 0), "wait")) return st;
        if (o1d_status st = cu(cudaMemcpyAsync(w, w_h, nw, cudaMemcpyHostToDevice, s2), "H2D w")) return st;
        int n0s[16], nls[16];
        for (int i = 0, n0 = 0; i < nch; ++i) {
            const int nl = pl->d.N / nch + (i < pl->d.N % nch ? 1 : 0);
            n0s[i] = n0, nls[i] = nl, n0 += nl;
        }
        for (int i = 0; i < nch; ++i) {
            const size_t ox = (size_t)n0s[i] * px, oy = (size_t)n0s[i] * py;
            if (o1d_status st = cu(cudaMemcpyAsync(static_cast<char *>(x) + ox, static_cast<const char *>(x_h) + ox,
                                                   (size_t)nls[i] * px, cudaMemcpyHostToDevice, s2), "H2D x"))
                return st;
            if (o1d_status st = cu(cudaEventRecord(ev(0, i), s2), "event")) return st;
            if (o1d_status st = cu(cudaMemcpyAsync(static_cast<char *>(dy) + oy, static_cast<const char *>(dy_h) + oy,
                                                   (size_t)nls[i] * py, cudaMemcpyHostToDevice, s2), "H2D dy"))
                return st;
            if (o1d_status st = cu(cudaEventRecord(ev(1, i), s2), "event")) return st;
        }
        for (int i = 0; i < nch; ++i) {
            if (o1d_status st = cu(cudaStreamWaitEvent(s, ev(0, i), 0), "wait")) return st;
            if (o1d_status st = spec_run(pl, 0, x, w, y, nullptr, nullptr, s, n0s[i], nls[i], true)) return st;
            if (o1d_status st = cu(cudaStreamWaitEvent(s, ev(1, i), 0), "wait")) return st;
            if (o1d_status st = spec_run(pl, 1, dy, w, dx, nullptr, nullptr, s, n0s[i], nls[i], true)) return st;
            if (o1d_status st = spec_run(pl, 2, x, nullptr, dy, dW, static_cast<float *>(ws), s, n0s[i], nls[i], false))
                return st;
            if (o1d_status st = cu(cudaEventRecord(ev(2, i), s), "event")) return st;
            const size_t ox = (size_t)n0s[i] * px, oy = (size_t)n0s[i] * py;
            if (o1d_status st = cu(cudaStreamWaitEvent(s3, ev(2, i), 0), "wait")) return st;
            if (o1d_status st = cu(cudaMemcpyAsync(static_cast<char *>(y_h) + oy, static_cast<char *>(y) + oy,
                                                   (size_t)nls[i] * py, cudaMemcpyDeviceToHost, s3), "D2H y"))
                return st;
            if (o1d_status st = cu(cudaMemcpyAsync(static_cast<char *>(dx_h) + ox, static_cast<char *>(dx) + ox,
                                                   (size_t)nls[i] * px, cudaMemcpyDeviceToHost, s3), "D2H dx"))
                return st;
        }
        if (o1d_status st = spec_finalize(pl, dW, static_cast<float *>(ws), s)) return st;
        if (o1d_status st = cu(cudaMemcpyAsync(dW_h, dW, nw, cudaMemcpyDeviceToHost, s), "D2H dW")) return st;
        if (o1d_status st = cu(cudaEventRecord(e1, s3), "event")) return st;
        if (o1d_status st = cu(cudaStreamWaitEvent(s, e1, 0), "wait")) return st;
        return cu(cudaStreamSynchronize(s), "o1d_step_host");
    }
    // Two streams so the PCIe directions overlap with each other and with the
    // kernels:  s  : H2D w, x  -> forward        -> D2H y
    //           s2 : H2D dy    -> backward_input -> D2H dx -> (x ready) backward_weight -> D2H dW
    cudaStream_t s = static_cast<cudaStream_t>(stream), s2 = static_cast<cudaStream_t>(pl->aux_stream);
    cudaEvent_t e_in = static_cast<cudaEvent_t>(pl->aux_ev[0]), e_out = static_cast<cudaEvent_t>(pl->aux_ev[1]);
    auto cu = [](cudaError_t e, const char *what) -> o1d_status {
        if (e != cudaSuccess) return fail(O1D_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
        return O1D_OK;
    };
    if (o1d_status st = cu(cudaEventRecord(e_out, s), "event")) return st;  // s2 starts after prior work on s
    if (o1d_status st = cu(cudaStreamWaitEvent(s2, e_out, 0), "wait")) return st;
    if (o1d_status st = cu(cudaMemcpyAsync(w, w_h, nw, cudaMemcpyHostToDevice, s), "H2D w")) return st;
    if (o1d_status st = cu(cudaMemcpyAsync(x, x_h, nx, cudaMemcpyHostToDevice, s), "H2D x")) return st;
    if (o1d_status st = cu(cudaEventRecord(e_in, s), "event")) return st;
    if (o1d_status st = cu(cudaMemcpyAsync(dy, dy_h, ny, cudaMemcpyHostToDevice, s2), "H2D dy")) return st;
    if (o1d_status st = o1d_forward(pl, x, w, y, stream)) return st;
    if (o1d_status st = cu(cudaMemcpyAsync(y_h, y, ny, cudaMemcpyDeviceToHost, s), "D2H y")) return st;
    if (o1d_status st = cu(cudaStreamWaitEvent(s2, e_in, 0), "wait")) return st;  // w and x are on the device
    if (o1d_status st = o1d_backward_input(pl, dy, w, dx, s2)) return st;
    if (o1d_status st = cu(cudaMemcpyAsync(dx_h, dx, nx, cudaMemcpyDeviceToHost, s2), "D2H dx")) return st;
    if (o1d_status st = o1d_backward_weight(pl, x, dy, dW, ws, o1d_workspace_bytes(pl), s2)) return st;
    if (o1d_status st = cu(cudaMemcpyAsync(dW_h, dW, nw, cudaMemcpyDeviceToHost, s2), "D2H dW")) return st;
    if (o1d_status st = cu(cudaEventRecord(e_out, s2), "event")) return st;
    if (o1d_status st = cu(cudaStreamWaitEvent(s, e_out, 0), "wait")) return st;
    return cu(cudaStreamSynchronize(s), "o1d_step_host");
}

}  // extern "C"
