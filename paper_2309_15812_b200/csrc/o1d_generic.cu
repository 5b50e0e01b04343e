// o1d_generic.cu — runtime-tap ("generic") kernels of liboriented1d.
//
// These kernels take the tap table at run time, so they serve every plan
// (arbitrary per-channel angles, any K, any stride, every discretisation: the
// plan's expanded weighted taps (dh, dw, k, coef) -- one per tap for the
// rotation / shear forms, up to four per tap for bilinear interpolation).  They stage the input band
// plus the angle-dependent halo in shared memory once (zero-filled outside the
// image: reading R1), so every tap read is a shared-memory read — the paper's
// "load the whole input in shared GPU memory ... cut the image into bands"
// — but they get no register reuse across taps.  The JIT-specialised
// kernels (o1d_spec_*.cuh) are the fast path; these are the fallback.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <functional>
#include <string>

#include "o1d_internal.h"

namespace o1d {
namespace {

template <typename T> __device__ __forceinline__ float ld_act(const T *p);
template <> __device__ __forceinline__ float ld_act<float>(const float *p) { return *p; }
template <> __device__ __forceinline__ float ld_act<__nv_bfloat16>(const __nv_bfloat16 *p) {
    return __bfloat162float(*p);
}
template <> __device__ __forceinline__ float ld_act<__half>(const __half *p) { return __half2float(*p); }

template <typename T> __device__ __forceinline__ T to_act(float v);
template <> __device__ __forceinline__ float to_act<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 to_act<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ __half to_act<__half>(float v) { return __float2half_rn(v); }

constexpr int kThreads = 256;
constexpr int kSmemBudget = 96 * 1024;
// preferred shared memory per CTA when choosing a band height: small enough for several CTAs per
// SM, so the staging loads of one CTA overlap the compute of the others (O1D_GENERIC_KB)
size_t pref_budget() {
    static const size_t kb = [] {
        const char *v = getenv("O1D_GENERIC_KB");
        const int k = (v && *v) ? atoi(v) : 48;
        return (size_t)std::max(4, std::min(96, k)) * 1024;
    }();
    return kb;
}
int pick_band(int rows, const std::function<size_t(int)> &smem_for) {
    int band = rows;
    while (band > 1 && smem_for(band) > pref_budget()) band = (band + 1) / 2;
    if (smem_for(band) <= pref_budget()) return band;
    band = rows;
    while (band > 1 && smem_for(band) > (size_t)kSmemBudget) band = (band + 1) / 2;
    return smem_for(band) <= (size_t)kSmemBudget ? band : 0;
}

// tile[r][j] = plane[h0 + r][v0 + j] as fp32 (zero outside the Hi x Wi image, reading R1), r < rows,
// j < cols; only rows r that are multiples of rstep (the rows the taps read, Stencil::rstep).  Image
// rows whose byte length is a multiple of 16 are read in 16-byte vectors (the activations may be
// 2-byte bf16/fp16: one vector load instead of eight scalar ones).
template <typename T>
__device__ __forceinline__ void stage_tile(float *tile, int pitch, const T *plane, int Hi, int Wi, int h0, int rows,
                                           int v0, int cols, int rstep = 1) {
    const int tid = threadIdx.x, nt = blockDim.x;
    constexpr int V = 16 / sizeof(T);
    const bool vec = ((Wi * (int)sizeof(T)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(plane) & 15) == 0);
    const int nr = (rows + rstep - 1) / rstep;  // staged rows: r = k * rstep, k < nr
    if (!vec) {
        for (int i = tid; i < nr * cols; i += nt) {
            const int k = i / cols, j = i - k * cols, r = k * rstep;
            const int h = h0 + r, v = v0 + j;
            tile[r * pitch + j] = (h >= 0 && h < Hi && v >= 0 && v < Wi) ? ld_act<T>(plane + (size_t)h * Wi + v) : 0.f;
        }
        return;
    }
    const int ja = max(0, -v0), jb = min(cols, Wi - v0);  // in-image columns, tile coordinates
    if (ja >= jb) {
        for (int i = tid; i < nr * cols; i += nt) tile[(i / cols) * rstep * pitch + i % cols] = 0.f;
        return;
    }
    // staged rows inside the image: k in [ka, kb)  (h0 + k * rstep in [0, Hi))
    const int ka = min(nr, (max(0, -h0) + rstep - 1) / rstep);
    const int kb = max(ka, min(nr, (Hi - h0 + rstep - 1) / rstep));
    {  // zero halo (no loads): whole rows outside the image, the side columns of the others
        const int side = ja + (cols - jb);
        for (int i = tid; i < (kb - ka) * side; i += nt) {
            const int k = ka + i / side, m = i % side;
            tile[k * rstep * pitch + (m < ja ? m : jb + (m - ja))] = 0.f;
        }
        const int nout = ka + (nr - kb);  // staged rows outside the image: [0, ka) and [kb, nr)
        for (int i = tid; i < nout * cols; i += nt) {
            const int o = i / cols, k = o < ka ? o : kb + (o - ka);
            tile[k * rstep * pitch + (i - o * cols)] = 0.f;
        }
    }
    const int ma = (v0 + ja) / V, mb = (v0 + jb + V - 1) / V;  // 16-byte chunks covering the columns
    const int nm = mb - ma, total = (kb - ka) * nm;
    constexpr int U = 4;  // four independent 16-byte loads in flight per thread
    for (int i0 = tid; i0 < total; i0 += U * nt) {
        uint4 u[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int i = i0 + q * nt;
            if (i < total) {
                const int rr = i / nm, m = ma + (i - rr * nm);
                u[q] = __ldg(reinterpret_cast<const uint4 *>(plane + (size_t)(h0 + (ka + rr) * rstep) * Wi) + m);
            }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int i = i0 + q * nt;
            if (i >= total) break;
            const int rr = i / nm, m = ma + (i - rr * nm), r = (ka + rr) * rstep;
            const T *e = reinterpret_cast<const T *>(&u[q]);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const int j = m * V + k - v0;
                if (j >= ja && j < jb) tile[r * pitch + j] = ld_act<T>(e + k);
            }
        }
    }
}

struct StencilArgs {
    const void *in;
    const float *w;
    void *out;
    const int16_t *dh, *dw, *ek;
    const float *coef;
    int C, Hi, Wi, Ho, Wo, str, K, KE;
    int minDH, maxDH, minDW;
    int band, bands;
    int tileRows, tileCols, pitch;
    int rstep;  // Stencil::rstep
};

// out[p][q] = sum_e in[str*p + dh_e][str*q + dw_e] * coef_e * w_{k_e}, one CTA per (plane, band of output rows)
// KC > 0: at most KC expanded taps, their offsets and weights held in registers (short kernels
// such as the stem's K=5); KC = 0: any count, read from shared memory per tap
template <typename T, int KC>
__global__ void __launch_bounds__(kThreads) stencil_generic_kernel(StencilArgs a) {
    extern __shared__ float sm[];
    const int tid = threadIdx.x;
    const int plane = blockIdx.x / a.bands;
    const int bnd = blockIdx.x - plane * a.bands;
    const int c = plane % a.C;
    const int p0 = bnd * a.band;
    const int nrows = min(a.band, a.Ho - p0);
    float *tile = sm;
    int *toff = reinterpret_cast<int *>(tile + a.tileRows * a.pitch + 8 * a.str + a.pitch);
    float *wk = reinterpret_cast<float *>(toff + a.KE);
    for (int e = tid; e < a.KE; e += blockDim.x) {
        const int i = c * a.KE + e;
        toff[e] = (a.dh[i] - a.minDH) * a.pitch + (a.dw[i] - a.minDW);
        wk[e] = a.coef[i] * a.w[c * a.K + a.ek[i]];
    }
    const T *in = static_cast<const T *>(a.in) + (size_t)plane * a.Hi * a.Wi;
    const int h0 = a.str * p0 + a.minDH;
    const int rows = a.str * (nrows - 1) + 1 + (a.maxDH - a.minDH);
    stage_tile<T>(tile, a.pitch, in, a.Hi, a.Wi, h0, rows, a.minDW, a.tileCols, a.rstep);
    __syncthreads();
    T *out = static_cast<T *>(a.out) + (size_t)plane * a.Ho * a.Wo;
    // a warp computes 32 consecutive outputs of a row, 4 times 32 apart (q = qc + 32 j): the lanes read
    // consecutive shared-memory words (the round-2 map of 4 consecutive outputs per thread put lanes 4
    // words apart: 4-way bank conflicts, x str for strided planes -- ncu: 74% of the shared-memory
    // wavefronts were conflicts at the stem's 112^2 layer)
    // J outputs per lane (J = 1..4, as many 32-wide columns as the row needs), chunks of 32 J outputs
    const int J = min(4, (a.Wo + 31) >> 5), cw = 32 * J, nch = (a.Wo + cw - 1) / cw;
    int roff[KC > 0 ? KC : 1];
    float rw[KC > 0 ? KC : 1];
    if constexpr (KC > 0) {
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            roff[k] = k < a.KE ? toff[k] : 0;
            rw[k] = k < a.KE ? wk[k] : 0.f;
        }
    }
    if (a.Wo <= 32) {
        // narrow rows (J = 1 would feed one FMA per tap-offset / weight read): 4 consecutive outputs per
        // thread as in round 2 (bank conflicts, but the tap reads are amortised: 28^2 K=31 270 vs 354 us)
        const int qg = (a.Wo + 3) >> 2;
        for (int g = tid; g < nrows * qg; g += blockDim.x) {
            const int pr = g / qg, q0 = (g - pr * qg) * 4;
            const float *base = tile + pr * a.str * a.pitch + q0 * a.str;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            if constexpr (KC > 0) {
#pragma unroll
                for (int k = 0; k < KC; ++k) {
                    if (k >= a.KE) break;
                    const float *s = base + roff[k];
                    const float wv = rw[k];
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[j] = fmaf(s[j * a.str], wv, acc[j]);
                }
            } else {
                for (int k = 0; k < a.KE; ++k) {
                    const float *s = base + toff[k];
                    const float wv = wk[k];
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[j] = fmaf(s[j * a.str], wv, acc[j]);
                }
            }
            T *orow = out + (size_t)(p0 + pr) * a.Wo + q0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (q0 + j < a.Wo) orow[j] = to_act<T>(acc[j]);
        }
        return;
    }
    for (int g = tid; g < nrows * nch * 32; g += blockDim.x) {  // blockDim.x is a multiple of 32
        const int t = g >> 5, pr = nch == 1 ? t : t / nch, qc = (t - pr * nch) * cw + (g & 31);
        const float *row = tile + pr * a.str * a.pitch;
        // outputs past the row (last chunk) read in-row columns and are not stored
        const int lim = min(a.Wo - 1, qc - (g & 31) + cw - 1);  // this chunk's last in-row output
        const float *b0 = row + min(qc, lim) * a.str, *b1 = row + min(qc + 32, lim) * a.str;
        const float *b2 = row + min(qc + 64, lim) * a.str, *b3 = row + min(qc + 96, lim) * a.str;
        float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
        if constexpr (KC > 0) {
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                if (k >= a.KE) break;  // (no padding taps: 0 * inf would leak a non-finite input)
                const int o = roff[k];
                const float wv = rw[k];
                acc0 = fmaf(b0[o], wv, acc0);
                if (J > 1) acc1 = fmaf(b1[o], wv, acc1);
                if (J > 2) acc2 = fmaf(b2[o], wv, acc2);
                if (J > 3) acc3 = fmaf(b3[o], wv, acc3);
            }
        } else {
            for (int k = 0; k < a.KE; ++k) {
                const int o = toff[k];
                const float wv = wk[k];
                acc0 = fmaf(b0[o], wv, acc0);
                if (J > 1) acc1 = fmaf(b1[o], wv, acc1);
                if (J > 2) acc2 = fmaf(b2[o], wv, acc2);
                if (J > 3) acc3 = fmaf(b3[o], wv, acc3);
            }
        }
        T *orow = out + (size_t)(p0 + pr) * a.Wo;
        if (qc <= lim) orow[qc] = to_act<T>(acc0);
        if (J > 1 && qc + 32 <= lim) orow[qc + 32] = to_act<T>(acc1);
        if (J > 2 && qc + 64 <= lim) orow[qc + 64] = to_act<T>(acc2);
        if (J > 3 && qc + 96 <= lim) orow[qc + 96] = to_act<T>(acc3);
    }
}

// dx[h][w] = sum_e [str | h-oh_e, str | w-ow_e, in range] dy[(h-oh_e)/str][(w-ow_e)/str] * coef_e * w_{k_e}
template <typename T>
__global__ void __launch_bounds__(kThreads) bwd_input_strided_kernel(const T *dy, const float *w, T *dx,
                                                                     const int16_t *oh, const int16_t *ow,
                                                                     const int16_t *ek, const float *coef,
                                                                     int C, int H, int W, int P, int Q, int K,
                                                                     int KE, int str, long total) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int v = (int)(i % W);
    const int h = (int)((i / W) % H);
    const long plane = i / ((long)W * H);
    const int c = (int)(plane % C);
    const T *g = dy + plane * P * Q;
    float acc = 0.f;
    for (int e = 0; e < KE; ++e) {
        const int i = c * KE + e;
        const int a = h - oh[i], b = v - ow[i];
        if (a < 0 || b < 0 || a % str || b % str) continue;
        const int p = a / str, q = b / str;
        if (p >= P || q >= Q) continue;
        acc = fmaf(ld_act<T>(g + p * Q + q), coef[i] * w[c * K + ek[i]], acc);
    }
    dx[i] = to_act<T>(acc);
}

// Strided backward_input, tiled: one CTA per (plane, band of dx rows); the dy rows and columns the
// band can reach are staged in shared memory (zero outside), then every thread produces 4
// consecutive dx outputs of a row: dx[h][w] = sum_e dy[(h-oh_e)/s][(w-ow_e)/s] c_e w_{k_e} over the
// taps with s | h-oh_e and s | w-ow_e (the divisibility test of a row is shared by the 4 outputs).
struct BwdInArgs {
    const void *dy;
    const float *w;
    void *dx;
    const int16_t *oh, *ow, *ek;
    const float *coef;
    int C, H, W, P, Q, str, K, KE;
    int minOH, maxOH, minOW, maxOW;
    int band, bands;
    int tileRows, tileCols, pitch;  // dy tile
};

// SC: the stride as a compile-time constant (2: the Depthwise 1D Stem) or 0 (run time)
template <typename T, int SC>
__global__ void __launch_bounds__(kThreads) bwd_input_strided_tiled_kernel(BwdInArgs a) {
    extern __shared__ float sm[];
    const int tid = threadIdx.x;
    const int plane = blockIdx.x / a.bands;
    const int bnd = blockIdx.x - plane * a.bands;
    const int c = plane % a.C;
    const int hb = bnd * a.band, nrows = min(a.band, a.H - hb);
    const int s = SC ? SC : a.str;
    // dy rows a with hb - maxOH <= s*a <= hb + nrows - 1 - minOH: a0 = ceil((hb - maxOH) / s)
    const int an = hb - a.maxOH;
    const int a0 = an >= 0 ? (an + s - 1) / s : -((-an) / s);
    const int bn = -a.maxOW;
    const int b0 = bn >= 0 ? (bn + s - 1) / s : -((-bn) / s);
    float *tile = sm;
    int *toff = reinterpret_cast<int *>(tile + a.tileRows * a.pitch);
    float *wk = reinterpret_cast<float *>(toff + a.KE);
    for (int e = tid; e < a.KE; e += blockDim.x) {
        const int i = c * a.KE + e;
        wk[e] = a.coef[i] * a.w[c * a.K + a.ek[i]];
    }
    const T *dy = static_cast<const T *>(a.dy) + (size_t)plane * a.P * a.Q;
    stage_tile<T>(tile, a.pitch, dy, a.P, a.Q, a0, a.tileRows, b0, a.tileCols);
    __syncthreads();
    T *dx = static_cast<T *>(a.dx) + (size_t)plane * a.H * a.W;
    // 32 consecutive dx outputs of a row per warp, 4 times 32 apart (conflict-free shared reads, see
    // stencil_generic_kernel)
    const int nch = (a.W + 127) >> 7;
    for (int g = tid; g < nrows * nch * 32; g += blockDim.x) {
        const int t = g >> 5, hr = t / nch, wc = (t - hr * nch) * 128 + (g & 31), h = hb + hr;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int e = 0; e < a.KE; ++e) {
            const int i = c * a.KE + e;
            const int num = h - a.oh[i] - s * a0;  // >= 0 inside the staged rows
            if (num < 0 || num % s) continue;
            const float *row = tile + (num / s) * a.pitch;
            const float wv = wk[e];
            const int ow = a.ow[i];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int cn = wc + 32 * j - ow - s * b0;
                if (cn >= 0 && cn % s == 0 && (cn / s) < a.tileCols) acc[j] = fmaf(row[cn / s], wv, acc[j]);
            }
        }
        T *drow = dx + (size_t)h * a.W;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (wc + 32 * j < a.W) drow[wc + 32 * j] = to_act<T>(acc[j]);
    }
}

struct BwdWArgs {
    const void *x, *dy;
    float *ws;
    const int16_t *oh, *ow;
    int C, H, W, P, Q, str, K;   // K here: expanded taps per channel (KE)
    int minOH, maxOH, minOW;
    int band, bands;
    int tileRows, tileCols, pitch;
    int rstep;  // Stencil::rstep of the forward geometry
};

// NV per-lane values -> lane L (< NV) ends with the warp sum of v[L] (NV a power of two <= 32)
template <int NV>
__device__ __forceinline__ float warp_reduce_scatter(float (&v)[NV]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int s = NV / 2; s >= 1; s >>= 1) {
        const bool upper = lane & s;
#pragma unroll
        for (int i = 0; i < s; ++i) {
            const float send = upper ? v[i] : v[i + s];
            const float keep = upper ? v[i + s] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
    }
    float r = v[0];
#pragma unroll
    for (int s = NV; s < 32; s <<= 1) r += __shfl_xor_sync(0xffffffffu, r, s);
    return r;
}

// ws[plane*bands + band][e] = sum over the band's outputs of dy[p][q] * x[str*p+oh_e][str*q+ow_e] (expanded taps);
// KC taps per round (8 for short kernels such as the stem's K=5, else 32)
template <typename T, int KC>
__global__ void __launch_bounds__(kThreads) bwd_weight_generic_kernel(BwdWArgs a) {
    extern __shared__ float sm[];
    __shared__ float red[kThreads / 32][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int plane = blockIdx.x / a.bands;
    const int bnd = blockIdx.x - plane * a.bands;
    const int c = plane % a.C;
    const int p0 = bnd * a.band;
    const int nrows = min(a.band, a.P - p0);
    float *tile = sm;
    float *sdy = tile + a.tileRows * a.pitch;
    int *toff = reinterpret_cast<int *>(sdy + a.band * a.Q);
    for (int k = tid; k < a.K; k += blockDim.x)
        toff[k] = (a.oh[c * a.K + k] - a.minOH) * a.pitch + (a.ow[c * a.K + k] - a.minOW);
    const T *x = static_cast<const T *>(a.x) + (size_t)plane * a.H * a.W;
    const T *dy = static_cast<const T *>(a.dy) + (size_t)plane * a.P * a.Q + (size_t)p0 * a.Q;
    const int h0 = a.str * p0 + a.minOH;
    const int rows = a.str * (nrows - 1) + 1 + (a.maxOH - a.minOH);
    stage_tile<T>(tile, a.pitch, x, a.H, a.W, h0, rows, a.minOW, a.tileCols, a.rstep);
    stage_tile<T>(sdy, a.Q, dy - (size_t)p0 * a.Q, a.P, a.Q, p0, nrows, 0, a.Q);
    __syncthreads();
    float *ws = a.ws + (size_t)blockIdx.x * a.K;
    for (int k0 = 0; k0 < a.K; k0 += KC) {
        float acc[KC];
#pragma unroll
        for (int j = 0; j < KC; ++j) acc[j] = 0.f;
        const int kn = min(KC, a.K - k0);
        for (int g = tid; g < nrows * a.Q; g += blockDim.x) {
            const int pr = g / a.Q, q = g - pr * a.Q;
            const float gv = sdy[g];
            const float *base = tile + pr * a.str * a.pitch + q * a.str;
#pragma unroll
            for (int j = 0; j < KC; ++j)
                if (j < kn) acc[j] = fmaf(gv, base[toff[k0 + j]], acc[j]);
        }
        const float r = warp_reduce_scatter<KC>(acc);
        red[warp][lane] = r;
        __syncthreads();
        if (tid < 32 && tid < kn) {
            float s = 0.f;
            for (int wi = 0; wi < (int)(blockDim.x >> 5); ++wi) s += red[wi][tid];
            ws[k0 + tid] = s;
        }
        __syncthreads();
    }
}

// dW[c][k] = sum_{e: k_e = k} coef_e * (sum_n sum_band ws[(n*C + c)*bands + band][e]), f64 accumulation,
// fixed order (rotation / shear: one e per k with coef 1).  One CTA per (c, k): thread t sums the
// entries t, t + 256, ... in order, then a fixed-shape tree over the threads -- deterministic.
__global__ void __launch_bounds__(256) bwd_weight_finalize_kernel(const float *ws, float *dW, const int16_t *ek,
                                                                  const float *coef, int N, int C, int K, int KE,
                                                                  int bands) {
    __shared__ double red[256];
    const int c = blockIdx.x / K, k = blockIdx.x - c * K, t = threadIdx.x;
    const int ne = N * bands;
    double acc = 0.0;
    for (int e = 0; e < KE; ++e) {
        if (ek[c * KE + e] != k || coef[c * KE + e] == 0.0f) continue;  // uniform over the block
        double s = 0.0;
        for (int i = t; i < ne; i += 256) {
            const int n = i / bands, b = i - n * bands;
            s += (double)ws[((size_t)(n * C + c) * bands + b) * KE + e];
        }
        red[t] = s;
        __syncthreads();
        for (int h = 128; h > 0; h >>= 1) {
            if (t < h) red[t] += red[t + h];
            __syncthreads();
        }
        if (t == 0) acc += (double)coef[c * KE + e] * red[0];
        __syncthreads();
    }
    if (t == 0) dW[blockIdx.x] = (float)acc;
}

o1d_status check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(O1D_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
    return O1D_OK;
}

template <typename F>
o1d_status dispatch_dtype(int dt, F &&f) {
    switch (dt) {
        case O1D_F32: return f(float());
        case O1D_BF16: return f(__nv_bfloat16());
        case O1D_F16: return f(__half());
    }
    return fail(O1D_UNSUPPORTED, "dtype");
}

void tile_geometry(const Stencil &st, int band, int *rows, int *cols, int *pitch) {
    *rows = st.str * (band - 1) + 1 + (st.maxDH - st.minDH);
    *cols = st.str * (st.Wo - 1) + 1 + (st.maxDW - st.minDW);
    int p = *cols;
    if ((p & 31) == 0) p += 1;  // avoid a power-of-two pitch
    *pitch = p;
}

size_t stencil_smem(const Stencil &st, int band, int extra_rows_per_out) {
    int rows, cols, pitch;
    tile_geometry(st, band, &rows, &cols, &pitch);
    return sizeof(float) * ((size_t)rows * pitch + 8 * st.str + pitch + 2 * st.KE +
                            (size_t)extra_rows_per_out * band * st.Wo);
}

}  // namespace

size_t dtype_size(int dt) { return dt == O1D_F32 ? 4 : 2; }

int generic_band_rows(const o1d_plan *, const Stencil &st, int extra) {
    return pick_band(st.Ho, [&](int b) { return stencil_smem(st, b, extra); });
}

o1d_status generic_stencil(const o1d_plan *pl, const Stencil &st, int band, const void *in, const float *w,
                           void *out, void *stream) {
    StencilArgs a;
    a.in = in; a.w = w; a.out = out; a.dh = st.d_dh; a.dw = st.d_dw; a.ek = pl->d_ek; a.coef = pl->d_coef;
    a.C = pl->d.C; a.Hi = st.Hi; a.Wi = st.Wi; a.Ho = st.Ho; a.Wo = st.Wo; a.str = st.str; a.K = pl->d.K; a.KE = st.KE;
    a.minDH = st.minDH; a.maxDH = st.maxDH; a.minDW = st.minDW;
    a.band = band; a.bands = (st.Ho + band - 1) / band; a.rstep = st.rstep;
    tile_geometry(st, band, &a.tileRows, &a.tileCols, &a.pitch);
    const size_t smem = stencil_smem(st, band, 0);
    const long grid = (long)pl->d.N * pl->d.C * a.bands;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return dispatch_dtype(pl->d.dtype, [&](auto tag) -> o1d_status {
        using T = decltype(tag);
        auto kern = a.KE <= 8 ? stencil_generic_kernel<T, 8> : stencil_generic_kernel<T, 0>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return check_launch("stencil_generic attr");
        kern<<<(unsigned)grid, kThreads, smem, s>>>(a);
        return check_launch("stencil_generic");
    });
}

o1d_status generic_bwd_input_strided(const o1d_plan *pl, const void *dy, const float *w, void *dx, void *stream) {
    const o1d_desc &d = pl->d;
    {
        // tiled path: the dy rows / columns a band of dx rows can reach, staged in shared memory
        BwdInArgs a;
        a.dy = dy; a.w = w; a.dx = dx; a.oh = pl->d_oh; a.ow = pl->d_ow; a.ek = pl->d_ek; a.coef = pl->d_coef;
        a.C = d.C; a.H = d.H; a.W = d.W; a.P = pl->P; a.Q = pl->Q; a.str = d.stride; a.K = d.K; a.KE = pl->KE;
        a.minOH = pl->minOH; a.maxOH = pl->maxOH; a.minOW = pl->minOW; a.maxOW = pl->maxOW;
        const int s = d.stride;
        a.tileCols = (d.W - 1 + a.maxOW - a.minOW) / s + 2;
        a.pitch = a.tileCols + ((a.tileCols & 31) == 0 ? 1 : 0);
        auto rows_for = [&](int b) { return (b - 1 + a.maxOH - a.minOH) / s + 2; };
        auto smem_for = [&](int b) { return sizeof(float) * ((size_t)rows_for(b) * a.pitch + 2 * a.KE); };
        const int band = pick_band(d.H, smem_for);
        if (band > 0) {
            a.band = band;
            a.bands = (d.H + band - 1) / band;
            a.tileRows = rows_for(band);
            const size_t smem = smem_for(band);
            const long grid = (long)d.N * d.C * a.bands;
            cudaStream_t st = static_cast<cudaStream_t>(stream);
            return dispatch_dtype(d.dtype, [&](auto tag) -> o1d_status {
                using T = decltype(tag);
                auto kern = s == 2 ? bwd_input_strided_tiled_kernel<T, 2> : bwd_input_strided_tiled_kernel<T, 0>;
                if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                    return check_launch("bwd_input_strided_tiled attr");
                kern<<<(unsigned)grid, kThreads, smem, st>>>(a);
                return check_launch("bwd_input_strided_tiled");
            });
        }
    }
    const long total = (long)d.N * d.C * d.H * d.W;
    const unsigned grid = (unsigned)((total + kThreads - 1) / kThreads);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return dispatch_dtype(d.dtype, [&](auto tag) -> o1d_status {
        using T = decltype(tag);
        bwd_input_strided_kernel<T><<<grid, kThreads, 0, s>>>(static_cast<const T *>(dy), w, static_cast<T *>(dx),
                                                              pl->d_oh, pl->d_ow, pl->d_ek, pl->d_coef, d.C, d.H,
                                                              d.W, pl->P, pl->Q, d.K, pl->KE, d.stride, total);
        return check_launch("bwd_input_strided");
    });
}

o1d_status generic_bwd_weight(const o1d_plan *pl, const void *x, const void *dy, float *dW, float *ws,
                              void *stream) {
    const o1d_desc &d = pl->d;
    const Stencil &st = pl->fwd;
    BwdWArgs a;
    a.x = x; a.dy = dy; a.ws = ws; a.oh = pl->d_oh; a.ow = pl->d_ow;
    a.C = d.C; a.H = d.H; a.W = d.W; a.P = pl->P; a.Q = pl->Q; a.str = d.stride; a.K = pl->KE;
    a.minOH = st.minDH; a.maxOH = st.maxDH; a.minOW = st.minDW;
    a.band = pl->bw_band; a.bands = pl->bw_bands; a.rstep = st.rstep;
    tile_geometry(st, a.band, &a.tileRows, &a.tileCols, &a.pitch);
    const size_t smem = sizeof(float) * ((size_t)a.tileRows * a.pitch + (size_t)a.band * a.Q + pl->KE);
    const long grid = (long)d.N * d.C * a.bands;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    o1d_status r = dispatch_dtype(d.dtype, [&](auto tag) -> o1d_status {
        using T = decltype(tag);
        auto kern = a.K <= 8 ? bwd_weight_generic_kernel<T, 8> : bwd_weight_generic_kernel<T, 32>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return check_launch("bwd_weight_generic attr");
        kern<<<(unsigned)grid, kThreads, smem, s>>>(a);
        return check_launch("bwd_weight_generic");
    });
    if (r != O1D_OK) return r;
    bwd_weight_finalize_kernel<<<d.C * d.K, 256, 0, s>>>(ws, dW, pl->d_ek, pl->d_coef, d.N, d.C, d.K, pl->KE, a.bands);
    return check_launch("bwd_weight_finalize");
}

}  // namespace o1d

// ----------------------------------------------------------------------------
// GPC topology probe.  The instruction cache is shared beyond one SM, so the
// specialised kernels give every GPC its own tap table ("home" table).  CTAs of
// one thread-block cluster always share a GPC; the probe launches many
// clusters and unions the %smid sets they land on.  Result: gpc id per smid
// (-1 for ids never observed).  Cached per device.
// ----------------------------------------------------------------------------
#include <map>
#include <mutex>
#include <numeric>

namespace o1d {
namespace {
__global__ void smid_probe_kernel(int *out) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
    const long long t0 = clock64();
    while (clock64() - t0 < 20000) {
    }
}

int uf_find(std::vector<int> &p, int x) {
    while (p[x] != x) x = p[x] = p[p[x]];
    return x;
}
}  // namespace

bool gpc_map(int device, std::vector<int> *gpc_of_smid) {
    static std::mutex mu;
    static std::map<int, std::vector<int>> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(device);
    if (it != cache.end()) {
        *gpc_of_smid = it->second;
        return !it->second.empty();
    }
    std::vector<int> result;
    int *d = nullptr;
    const int MAXS = 1024;
    if (cudaMalloc(&d, sizeof(int) * 16 * 256) == cudaSuccess) {
        cudaFuncSetAttribute(smid_probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        std::vector<int> par(MAXS), seen(MAXS, 0);
        std::iota(par.begin(), par.end(), 0);
        bool ok = false;
        for (int cs : {16, 8, 4, 2}) {
            for (int rep = 0; rep < 24; ++rep) {
                cudaLaunchConfig_t cfg = {};
                const int ncl = 160 / cs + rep % 5;
                cfg.gridDim = dim3(cs * ncl);
                cfg.blockDim = dim3(32);
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cs;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                if (cudaLaunchKernelEx(&cfg, smid_probe_kernel, d) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
                    cudaGetLastError();
                    break;
                }
                std::vector<int> c(cs * ncl);
                if (cudaMemcpy(c.data(), d, sizeof(int) * c.size(), cudaMemcpyDeviceToHost) != cudaSuccess) break;
                ok = true;
                for (int k = 0; k < ncl; ++k)
                    for (int j = 0; j < cs; ++j) {
                        const int s = c[k * cs + j], s0 = c[k * cs];
                        if (s < 0 || s >= MAXS || s0 < 0 || s0 >= MAXS) continue;
                        seen[s] = 1;
                        par[uf_find(par, s)] = uf_find(par, s0);
                    }
            }
        }
        cudaFree(d);
        if (ok) {
            int maxs = 0;
            for (int s = 0; s < MAXS; ++s)
                if (seen[s]) maxs = s;
            result.assign(maxs + 1, -1);
            std::map<int, int> ids;
            for (int s = 0; s <= maxs; ++s)
                if (seen[s]) {
                    const int r = uf_find(par, s);
                    auto f = ids.find(r);
                    if (f == ids.end()) f = ids.emplace(r, (int)ids.size()).first;
                    result[s] = f->second;
                }
        }
    }
    cudaGetLastError();
    cache[device] = result;
    *gpc_of_smid = result;
    return !result.empty();
}
}  // namespace o1d
