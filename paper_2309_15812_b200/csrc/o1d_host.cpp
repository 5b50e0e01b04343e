// o1d_host.cpp — host side of liboriented1d: the C ABI entry points, tap
// generation (P:1263-1264 with reading R3), plan creation and validation.
#include <cuda_runtime.h>
#include <quadmath.h>

#include <algorithm>
#include <chrono>
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

// floor(m * f(t)) for f = sin (is_sin) or cos, t in degrees reduced to [0, 360); m = k - pad
// is a binary double (an integer for the default pad): m * r is exact for r in {0, +-1/2, +-1}
static int floor_trig_times(double m, double t, bool is_sin) {
    if (m == 0) return 0;
    double r;
    if (is_sin ? niven_sin(t, &r) : niven_cos(t, &r)) return (int)std::floor(m * r);  // exact: r in {0,+-1/2,+-1}
    const double rad = t * (M_PI / 180.0);
    const double v = m * (is_sin ? std::sin(rad) : std::cos(rad));
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

void make_taps_one_shear(int K, int pad, double theta_deg, int16_t *oh, int16_t *ow) {  // integer pad (R13)
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

static double reduce360(double theta_deg) {
    double t = std::fmod(theta_deg, 360.0);  // exact
    if (t < 0) t += 360.0;
    if (t >= 360.0) t -= 360.0;
    return t;
}

void make_taps_one(int K, double pad, double theta_deg, int16_t *oh, int16_t *ow) {
    const double t = reduce360(theta_deg);
    for (int k = 0; k < K; ++k) {
        const double m = (double)k - pad;
        oh[k] = (int16_t)floor_trig_times(-m, t, true);   // floor(-(k-pad) sin t)
        ow[k] = (int16_t)floor_trig_times(m, t, false);   // floor( (k-pad) cos t)
    }
}

// Bilinear discretisation (reading R14): the real offset (u, v) = (-(k-pad) sin t,
// (k-pad) cos t); base corner = the exact floors (make_taps_one), fractional parts in [0, 1]:
// exact at the Niven angles (m * r with r in {0, +-1/2, +-1}), else f64 trig minus the exact
// floor, clamped (an f64 value within rounding of an integer gives a ~0 or ~1 fraction:
// the interpolation is continuous there).
static double frac_of(double m, double t, bool is_sin, int fl) {
    if (m == 0) return 0.0;
    double r;
    if (is_sin ? niven_sin(t, &r) : niven_cos(t, &r)) return m * r - (double)fl;  // exact
    const double rad = t * (M_PI / 180.0);
    const double v = m * (is_sin ? std::sin(rad) : std::cos(rad));
    return std::min(1.0, std::max(0.0, v - (double)fl));
}

void make_bilinear_one(int K, double pad, double theta_deg, int16_t *h0, int16_t *w0, double *fa, double *fb) {
    const double t = reduce360(theta_deg);
    make_taps_one(K, pad, theta_deg, h0, w0);
    for (int k = 0; k < K; ++k) {
        const double m = (double)k - pad;
        fa[k] = frac_of(-m, t, true, h0[k]);
        fb[k] = frac_of(m, t, false, w0[k]);
    }
}

}  // namespace o1d

using namespace o1d;

extern "C" {

const char *o1d_last_error(void) { return g_err.c_str(); }
const char *o1d_version(void) { return "liboriented1d 0.1 (sm_100a)"; }

static o1d_status check_taps_args(const char *fn, int32_t K, double *pad, int32_t C, const void *a, const void *b,
                                  const void *c) {
    if (!a || !b || !c) return fail(O1D_INVALID_ARG, std::string(fn) + ": NULL pointer");
    if (K < 1) return fail(O1D_INVALID_CONFIG, std::string(fn) + ": K < 1");
    if (C < 1) return fail(O1D_INVALID_SHAPE, std::string(fn) + ": C < 1");
    if (!std::isfinite(*pad)) return fail(O1D_INVALID_ARG, std::string(fn) + ": non-finite pad");
    if (*pad < 0) *pad = (double)(K / 2);
    if (*pad > 4096.0) return fail(O1D_INVALID_CONFIG, std::string(fn) + ": |pad| > 4096");
    return O1D_OK;
}

o1d_status o1d_make_taps(int32_t K, double pad, int32_t C, const double *angles_deg, int16_t *oh, int16_t *ow) {
    if (o1d_status st = check_taps_args("o1d_make_taps", K, &pad, C, angles_deg, oh, ow)) return st;
    for (int c = 0; c < C; ++c) {
        if (!std::isfinite(angles_deg[c])) return fail(O1D_INVALID_ARG, "o1d_make_taps: non-finite angle");
        make_taps_one(K, pad, angles_deg[c], oh + (size_t)c * K, ow + (size_t)c * K);
    }
    return O1D_OK;
}

o1d_status o1d_make_taps_ex(int32_t K, double pad, int32_t C, const double *angles_deg, int32_t mode, int16_t *oh,
                            int16_t *ow) {
    if (mode == O1D_TAPS_ROTATION || mode == O1D_TAPS_BILINEAR) return o1d_make_taps(K, pad, C, angles_deg, oh, ow);
    if (mode != O1D_TAPS_SHEAR)
        return fail(O1D_INVALID_ARG, "o1d_make_taps_ex: mode must be O1D_TAPS_ROTATION, _SHEAR or _BILINEAR");
    if (o1d_status st = check_taps_args("o1d_make_taps_ex", K, &pad, C, angles_deg, oh, ow)) return st;
    if (pad != std::floor(pad)) return fail(O1D_UNSUPPORTED, "o1d_make_taps_ex: the shear form takes an integer pad");
    for (int c = 0; c < C; ++c) {
        if (!std::isfinite(angles_deg[c])) return fail(O1D_INVALID_ARG, "o1d_make_taps_ex: non-finite angle");
        make_taps_one_shear(K, (int)pad, angles_deg[c], oh + (size_t)c * K, ow + (size_t)c * K);
    }
    return O1D_OK;
}

o1d_status o1d_make_bilinear(int32_t K, double pad, int32_t C, const double *angles_deg, int16_t *h0, int16_t *w0,
                             double *fa, double *fb) {
    if (o1d_status st = check_taps_args("o1d_make_bilinear", K, &pad, C, angles_deg, h0, w0)) return st;
    if (!fa || !fb) return fail(O1D_INVALID_ARG, "o1d_make_bilinear: NULL pointer");
    for (int c = 0; c < C; ++c) {
        if (!std::isfinite(angles_deg[c])) return fail(O1D_INVALID_ARG, "o1d_make_bilinear: non-finite angle");
        const size_t o = (size_t)c * K;
        make_bilinear_one(K, pad, angles_deg[c], h0 + o, w0 + o, fa + o, fb + o);
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
    if (!std::isfinite(d->pad)) return fail(O1D_INVALID_ARG, "pad must be finite");
    if (d->pad > d->K - 1) return fail(O1D_INVALID_CONFIG, "pad must be <= K - 1 (or negative for floor(K/2))");
    if (d->dtype != O1D_F32 && d->dtype != O1D_BF16 && d->dtype != O1D_F16)
        return fail(O1D_UNSUPPORTED, "dtype must be O1D_F32, O1D_BF16 or O1D_F16");
    if (d->layout != O1D_NCHW) return fail(O1D_UNSUPPORTED, "only the NCHW-contiguous layout is implemented");
    if ((long)d->N * d->C * d->H * d->W > (1L << 40)) return fail(O1D_UNSUPPORTED, "tensor too large");
    if (d->K > 1023) return fail(O1D_UNSUPPORTED, "K > 1023");
    if (d->flags & ~(O1D_FLAG_FORCE_GENERIC | O1D_FLAG_NO_TMA | O1D_FLAG_SHEAR | O1D_FLAG_BILINEAR))
        return fail(O1D_INVALID_ARG, "unknown bits in o1d_desc.flags");
    if ((d->flags & O1D_FLAG_SHEAR) && (d->flags & O1D_FLAG_BILINEAR))
        return fail(O1D_INVALID_CONFIG, "O1D_FLAG_SHEAR and O1D_FLAG_BILINEAR are exclusive");
    if ((d->flags & O1D_FLAG_SHEAR) && d->pad >= 0 && d->pad != std::floor(d->pad))
        return fail(O1D_UNSUPPORTED, "the shear form takes an integer pad");
    return O1D_OK;
}

// Host-only part of plan creation: taps, expanded weighted taps, distinct tables, halo extents.
static o1d_status plan_host_init(const o1d_desc *d, const double *angles_deg, o1d_plan *pl) {
    if (o1d_status st = validate_desc(d)) return st;
    if (!angles_deg) return fail(O1D_INVALID_ARG, "o1d_plan_create: NULL angles");
    pl->d = *d;
    pl->pad = d->pad < 0 ? (double)(d->K / 2) : d->pad;
    pl->d.pad = pl->pad;
    pl->P = (d->H - 1) / d->stride + 1;
    pl->Q = (d->W - 1) / d->stride + 1;
    pl->disc = (d->flags & O1D_FLAG_SHEAR) ? O1D_TAPS_SHEAR : (d->flags & O1D_FLAG_BILINEAR) ? O1D_TAPS_BILINEAR
                                                                                             : O1D_TAPS_ROTATION;
    const int C = d->C, K = d->K;
    pl->angles.assign(angles_deg, angles_deg + C);
    pl->oh.resize((size_t)C * K);
    pl->ow.resize((size_t)C * K);
    std::vector<double> fa, fb;
    if (pl->disc == O1D_TAPS_BILINEAR) {
        fa.resize((size_t)C * K);
        fb.resize((size_t)C * K);
        if (o1d_status st = o1d_make_bilinear(K, pl->pad, C, angles_deg, pl->oh.data(), pl->ow.data(), fa.data(), fb.data()))
            return st;
    } else if (o1d_status st = o1d_make_taps_ex(K, pl->pad, C, angles_deg, pl->disc, pl->oh.data(), pl->ow.data())) {
        return st;
    }
    // expanded weighted taps: one entry per tap (rotation / shear) or one per bilinear
    // neighbour with a non-zero weight, padded to the widest channel with
    // zero-weight entries at offset (0, 0)
    struct E { int16_t dh, dw, k; float coef; };
    std::vector<std::vector<E>> ex(C);
    for (int c = 0; c < C; ++c)
        for (int k = 0; k < K; ++k) {
            const size_t i = (size_t)c * K + k;
            if (pl->disc != O1D_TAPS_BILINEAR) {
                ex[c].push_back({pl->oh[i], pl->ow[i], (int16_t)k, 1.0f});
                continue;
            }
            const double a = fa[i], b = fb[i];
            const double wq[4] = {(1 - a) * (1 - b), (1 - a) * b, a * (1 - b), a * b};
            for (int q = 0; q < 4; ++q)
                if (wq[q] != 0.0)
                    ex[c].push_back({(int16_t)(pl->oh[i] + (q >> 1)), (int16_t)(pl->ow[i] + (q & 1)), (int16_t)k, (float)wq[q]});
        }
    int KE = 1;
    for (auto &v : ex) KE = std::max(KE, (int)v.size());
    pl->KE = KE;
    pl->eoh.assign((size_t)C * KE, 0);
    pl->eow.assign((size_t)C * KE, 0);
    pl->ek.assign((size_t)C * KE, 0);
    pl->ecoef.assign((size_t)C * KE, 0.0f);
    std::map<std::vector<int32_t>, int> ids;
    pl->table_of.resize(C);
    pl->minOH = pl->minOW = 1 << 20;
    pl->maxOH = pl->maxOW = -(1 << 20);
    for (int c = 0; c < C; ++c) {
        std::vector<int32_t> key;
        for (size_t e = 0; e < ex[c].size(); ++e) {
            const E &t = ex[c][e];
            const size_t i = (size_t)c * KE + e;
            pl->eoh[i] = t.dh, pl->eow[i] = t.dw, pl->ek[i] = t.k, pl->ecoef[i] = t.coef;
            int32_t cb;
            std::memcpy(&cb, &t.coef, 4);
            key.insert(key.end(), {t.dh, t.dw, t.k, cb});
        }
        for (int e = 0; e < KE; ++e) {
            const size_t i = (size_t)c * KE + e;
            pl->minOH = std::min<int>(pl->minOH, pl->eoh[i]);
            pl->maxOH = std::max<int>(pl->maxOH, pl->eoh[i]);
            pl->minOW = std::min<int>(pl->minOW, pl->eow[i]);
            pl->maxOW = std::max<int>(pl->maxOW, pl->eow[i]);
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
    const auto t_start = std::chrono::steady_clock::now();
    if (!out) return fail(O1D_INVALID_ARG, "o1d_plan_create: NULL out");
    *out = nullptr;
    if (o1d_status st = validate_desc(d)) return st;
    o1d_plan *pl = new (std::nothrow) o1d_plan();
    if (!pl) return fail(O1D_INVALID_ARG, "out of host memory");
    if (o1d_status st = plan_host_init(d, angles_deg, pl)) {
        delete pl;
        return st;
    }
    const int C = d->C, KE = pl->KE;
    // device tables: eoh, eow, -eoh, -eow, ek (int16 [C][KE]), coef (f32 [C][KE])
    if (cudaGetDevice(&pl->device) != cudaSuccess) {
        delete pl;
        return fail(O1D_CUDA_ERROR, std::string("cudaGetDevice: ") + cudaGetErrorString(cudaGetLastError()));
    }
    const size_t n = (size_t)C * KE;
    const size_t tb = (sizeof(int16_t) * 5 * n + 15) & ~(size_t)15;
    std::vector<unsigned char> host(tb + sizeof(float) * n, 0);
    int16_t *h16 = reinterpret_cast<int16_t *>(host.data());
    for (size_t i = 0; i < n; ++i) {
        h16[i] = pl->eoh[i];
        h16[n + i] = pl->eow[i];
        h16[2 * n + i] = (int16_t)-pl->eoh[i];
        h16[3 * n + i] = (int16_t)-pl->eow[i];
        h16[4 * n + i] = pl->ek[i];
    }
    std::memcpy(host.data() + tb, pl->ecoef.data(), sizeof(float) * n);
    if (cudaMalloc(&pl->d_block, host.size()) != cudaSuccess ||
        cudaMemcpy(pl->d_block, host.data(), host.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaError_t e = cudaGetLastError();
        if (pl->d_block) cudaFree(pl->d_block);
        delete pl;
        return fail(O1D_CUDA_ERROR, std::string("plan tables: ") + cudaGetErrorString(e));
    }
    int16_t *base = static_cast<int16_t *>(pl->d_block);
    pl->d_oh = base;
    pl->d_ow = base + n;
    pl->d_noh = base + 2 * n;
    pl->d_now = base + 3 * n;
    pl->d_ek = base + 4 * n;
    pl->d_coef = reinterpret_cast<float *>(static_cast<unsigned char *>(pl->d_block) + tb);
    // stencil geometry of the forward and (stride 1) backward_input passes
    pl->fwd = Stencil{d->H, d->W, pl->P, pl->Q, d->stride, KE, pl->minOH, pl->maxOH, pl->minOW, pl->maxOW,
                      pl->d_oh, pl->d_ow};
    pl->bwd_in = Stencil{pl->P, pl->Q, d->H, d->W, 1, KE, -pl->maxOH, -pl->minOH, -pl->maxOW, -pl->minOW,
                         pl->d_noh, pl->d_now};
    if (d->stride > 1) {  // only rows str*p + dh are read: skip the others when every dh agrees mod str
        bool cong = true;
        for (size_t e = 0; e < pl->eoh.size() && cong; ++e) cong = ((pl->eoh[e] - pl->minOH) % d->stride) == 0;
        if (cong) pl->fwd.rstep = d->stride;
    }
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
    pl->ws_bytes = sizeof(float) * (size_t)d->N * C * pl->bw_bands * KE;
    pl->e2e_chunks = env_int_host("O1D_E2E_CHUNKS", 8);
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
    pl->plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    *out = pl;
    return O1D_OK;
}

o1d_status o1d_plan_stats(const o1d_plan *pl, double *create_ms, int32_t *jit_cache_hit) {
    if (!pl || !create_ms || !jit_cache_hit) return fail(O1D_INVALID_ARG, "o1d_plan_stats: NULL pointer");
    *create_ms = pl->plan_ms;
    *jit_cache_hit = pl->spec ? (pl->jit_cache_hit ? 1 : 0) : -1;
    return O1D_OK;
}

void o1d_plan_destroy(o1d_plan *pl) {
    if (!pl) return;
    // launches may still reference the plan's tables, counters and modules: finish them on
    // the plan's device first (and restore the caller's device)
    int prev = -1;
    const bool have_prev = cudaGetDevice(&prev) == cudaSuccess;
    if (cudaSetDevice(pl->device) == cudaSuccess) cudaDeviceSynchronize();
    cudaGetLastError();
    spec_destroy(pl);
    if (pl->aux_stream) cudaStreamDestroy(static_cast<cudaStream_t>(pl->aux_stream));
    if (pl->aux_stream2) cudaStreamDestroy(static_cast<cudaStream_t>(pl->aux_stream2));
    for (void *e : pl->chunk_ev)
        if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
    for (void *e : pl->aux_ev)
        if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
    if (pl->d_block) cudaFree(pl->d_block);
    if (have_prev) cudaSetDevice(prev);
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
    if (spec_has(pl, 0)) {
        RunArgs a;
        a.x = x, a.w = w, a.y = y;
        return spec_run(pl, 0, a, stream);
    }
    return generic_stencil(pl, pl->fwd, pl->fwd_band, x, w, y, stream);
}

o1d_status o1d_backward_input(const o1d_plan *pl, const void *dy, const float *w, void *dx, void *stream) {
    if (!pl) return fail(O1D_INVALID_ARG, "NULL plan");
    if (o1d_status st = check_ptr(dy, "dy")) return st;
    if (o1d_status st = check_ptr(w, "w")) return st;
    if (o1d_status st = check_ptr(dx, "dx")) return st;
    if (o1d_status st = check_device(pl)) return st;
    if (spec_has(pl, 1)) {
        RunArgs a;
        a.dy = dy, a.w = w, a.dx = dx;
        return spec_run(pl, 1, a, stream);
    }
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
    if (spec_has(pl, 2)) {
        RunArgs a;
        a.x = x, a.dy = dy, a.dW = dW, a.ws = static_cast<float *>(ws);
        return spec_run(pl, 2, a, stream);
    }
    return generic_bwd_weight(pl, x, dy, dW, static_cast<float *>(ws), stream);
}

o1d_status o1d_backward(const o1d_plan *pl, const void *x, const void *dy, const float *w, void *dx, float *dW,
                        void *ws, size_t ws_bytes, void *stream) {
    if (!pl) return fail(O1D_INVALID_ARG, "NULL plan");
    for (const void *q : {x, dy, (const void *)w, (const void *)dx, (const void *)dW, (const void *)ws})
        if (o1d_status st = check_ptr(q, "o1d_backward buffer")) return st;
    if (ws_bytes < o1d_workspace_bytes(pl)) return fail(O1D_WORKSPACE_TOO_SMALL, "ws_bytes < o1d_workspace_bytes(plan)");
    if (o1d_status st = check_device(pl)) return st;
    if (spec_has(pl, 3)) {
        RunArgs a;
        a.x = x, a.dy = dy, a.w = w, a.dx = dx, a.dW = dW, a.ws = static_cast<float *>(ws);
        return spec_run(pl, 3, a, stream);
    }
    if (o1d_status st = o1d_backward_input(pl, dy, w, dx, stream)) return st;
    return o1d_backward_weight(pl, x, dy, dW, ws, ws_bytes, stream);
}

o1d_status o1d_step(const o1d_plan *pl, const void *x, const float *w, const void *dy, void *y, void *dx, float *dW,
                    void *ws, size_t ws_bytes, void *stream) {
    if (!pl) return fail(O1D_INVALID_ARG, "NULL plan");
    for (const void *q : {x, (const void *)w, dy, (const void *)y, (const void *)dx, (const void *)dW, (const void *)ws})
        if (o1d_status st = check_ptr(q, "o1d_step buffer")) return st;
    if (ws_bytes < o1d_workspace_bytes(pl)) return fail(O1D_WORKSPACE_TOO_SMALL, "ws_bytes < o1d_workspace_bytes(plan)");
    if (o1d_status st = check_device(pl)) return st;
    if (!(spec_has(pl, 0) && spec_has(pl, 1) && spec_has(pl, 2))) {
        if (o1d_status st = o1d_forward(pl, x, w, y, stream)) return st;
        return o1d_backward(pl, x, dy, w, dx, dW, ws, ws_bytes, stream);
    }
    // The passes of a step read only the step's inputs (x, w, dy) and write disjoint outputs,
    // so the backward pass(es) need not wait for the preceding pass: they start on the SMs
    // the preceding pass frees (its tail) instead of after it.  The forward still waits for
    // whatever preceded the step on the stream.
    RunArgs a;
    a.x = x, a.w = w, a.y = y, a.dy = dy, a.dx = dx, a.dW = dW, a.ws = static_cast<float *>(ws);
    if (o1d_status st = spec_run(pl, 0, a, stream)) return st;
    if (spec_step_fused(pl)) return spec_run(pl, 3, a, stream, 0, 0, true, true);
    if (o1d_status st = spec_run(pl, 1, a, stream, 0, 0, true, true)) return st;
    return spec_run(pl, 2, a, stream, 0, 0, true, true);
}

int32_t o1d_launches_per_call(const o1d_plan *pl, int32_t pass) {
    if (!pl || pass < 0 || pass > 3) return 0;
    if (spec_has(pl, pass)) return spec_launches(pl, pass);
    if (pass == 3) return o1d_launches_per_call(pl, 1) + o1d_launches_per_call(pl, 2);
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
    const int nch = spec_window_ok(pl) && pl->d.N >= 2 && pl->e2e_chunks > 1
                        ? std::min(std::min(pl->d.N, pl->e2e_chunks), 16)
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
        RunArgs ra;
        ra.x = x, ra.w = w, ra.y = y, ra.dy = dy, ra.dx = dx, ra.dW = dW, ra.ws = static_cast<float *>(ws);
        const bool fused = spec_step_fused(pl);
        for (int i = 0; i < nch; ++i) {
            if (o1d_status st = cu(cudaStreamWaitEvent(s, ev(0, i), 0), "wait")) return st;
            if (o1d_status st = spec_run(pl, 0, ra, s, n0s[i], nls[i], true)) return st;
            if (o1d_status st = cu(cudaStreamWaitEvent(s, ev(1, i), 0), "wait")) return st;
            if (fused) {
                if (o1d_status st = spec_run(pl, 3, ra, s, n0s[i], nls[i], false)) return st;
            } else {
                if (o1d_status st = spec_run(pl, 1, ra, s, n0s[i], nls[i], true)) return st;
                if (o1d_status st = spec_run(pl, 2, ra, s, n0s[i], nls[i], false)) return st;
            }
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
        if (o1d_status st = spec_finalize(pl, fused ? 3 : 2, dW, static_cast<float *>(ws), s)) return st;
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
    if (o1d_status st = o1d_backward(pl, x, dy, w, dx, dW, ws, o1d_workspace_bytes(pl), s2)) return st;
    if (o1d_status st = cu(cudaMemcpyAsync(dx_h, dx, nx, cudaMemcpyDeviceToHost, s2), "D2H dx")) return st;
    if (o1d_status st = cu(cudaMemcpyAsync(dW_h, dW, nw, cudaMemcpyDeviceToHost, s2), "D2H dW")) return st;
    if (o1d_status st = cu(cudaEventRecord(e_out, s2), "event")) return st;
    if (o1d_status st = cu(cudaStreamWaitEvent(s, e_out, 0), "wait")) return st;
    return cu(cudaStreamSynchronize(s), "o1d_step_host");
}

}  // extern "C"
