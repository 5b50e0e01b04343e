/*
 * oracle.c — plain, slow, obviously-correct CPU reference of the depthwise
 * oriented 1D convolution (arXiv 2309.15812).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with paper_2309_15812_b200/.
 *
 * Arithmetic: f64 accumulation over f64 inputs (the fp32 / bf16 activation
 * values upcast exactly).  Tap tables (oh, ow) are INPUTS: they come from
 * oracle/taps.py (exact floor of P:1263-1264).
 *
 * Layout: x[N][C][H][W], y[N][C][P][Q] with P = (H-1)/str + 1, Q = (W-1)/str + 1
 * (reading R2), w[C][K], taps oh/ow[C][K].
 *
 * Passages followed:
 *   forward          Def. 1, Eq. "definition" P:1261 + Eq. "coordinate" P:1263-1264:
 *                    y_npqc = sum_k x_{n,h,w,c} w_kc,  h = str*p + oh_ck, w = str*q + ow_ck
 *                    reads outside [0,H)x[0,W) contribute 0 (zero padding, reading R1).
 *   backward_input   the adjoint of that linear map in x (reading A5),
 *                    written in SCATTER form: every forward term x*w sends dy*w back to x.
 *   backward_weight  the adjoint in w: dW_kc = sum_{n,p,q} dy_npqc x_{n,h,w,c}.
 * Threads: OpenMP over independent (n,c) planes (forward, backward_input) or
 * channels (backward_weight) only; each output element is produced by one
 * thread in the order written, so results do not depend on the thread count.
 */
#include <stdint.h>
#include <stddef.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Accumulator type of forward / backward_weight: double (the oracle); the bench's
 * "f32acc" timing build compiles this file with -DORACLE_ACC=float (bench.py cpu_baseline
 * only; parity always uses the f64 build). */
#ifndef ORACLE_ACC
#define ORACLE_ACC double
#endif

static int out_dim(int L, int str) { return (L - 1) / str + 1; }

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* y = forward(x, w) */
void oracle_forward(int N, int C, int H, int W, int K, int str,
                    const int32_t *oh, const int32_t *ow,
                    const double *x, const double *w, double *y, int threads) {
    const int P = out_dim(H, str), Q = out_dim(W, str);
    const long planes = (long)N * C;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
#endif
    for (long nc = 0; nc < planes; ++nc) {
        const int c = (int)(nc % C);
        const double *xp = x + nc * H * W;
        double *yp = y + nc * P * Q;
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < Q; ++q) {
                ORACLE_ACC acc = 0.0;
                for (int k = 0; k < K; ++k) {
                    const int h = str * p + oh[c * K + k];
                    const int v = str * q + ow[c * K + k];
                    if (h >= 0 && h < H && v >= 0 && v < W)
                        acc += xp[h * W + v] * w[c * K + k];
                }
                yp[p * Q + q] = acc;
            }
    }
}

/* dx = backward_input(dy, w), scatter form */
void oracle_backward_input(int N, int C, int H, int W, int K, int str,
                           const int32_t *oh, const int32_t *ow,
                           const double *dy, const double *w, double *dx, int threads) {
    const int P = out_dim(H, str), Q = out_dim(W, str);
    const long planes = (long)N * C;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
#endif
    for (long nc = 0; nc < planes; ++nc) {
        const int c = (int)(nc % C);
        const double *gp = dy + nc * P * Q;
        double *dxp = dx + nc * H * W;
        for (long i = 0; i < (long)H * W; ++i) dxp[i] = 0.0;
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < Q; ++q)
                for (int k = 0; k < K; ++k) {
                    const int h = str * p + oh[c * K + k];
                    const int v = str * q + ow[c * K + k];
                    if (h >= 0 && h < H && v >= 0 && v < W)
                        dxp[h * W + v] += gp[p * Q + q] * w[c * K + k];
                }
    }
}

/* dW = backward_weight(x, dy), dW[C][K] */
void oracle_backward_weight(int N, int C, int H, int W, int K, int str,
                            const int32_t *oh, const int32_t *ow,
                            const double *x, const double *dy, double *dW, int threads) {
    const int P = out_dim(H, str), Q = out_dim(W, str);
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
#endif
    for (int c = 0; c < C; ++c)
        for (int k = 0; k < K; ++k) {
            ORACLE_ACC acc = 0.0;
            for (int n = 0; n < N; ++n) {
                const double *xp = x + ((long)n * C + c) * H * W;
                const double *gp = dy + ((long)n * C + c) * P * Q;
                for (int p = 0; p < P; ++p)
                    for (int q = 0; q < Q; ++q) {
                        const int h = str * p + oh[c * K + k];
                        const int v = str * q + ow[c * K + k];
                        if (h >= 0 && h < H && v >= 0 && v < W)
                            acc += gp[p * Q + q] * xp[h * W + v];
                    }
            }
            dW[c * K + k] = acc;
        }
}

/* ---------------------------------------------------------------------------
 * Bilinear discretisation (Sec. "Discretization and Interpolation";
 * Table "bilinear" P:322-334).  Tap k of channel c samples x at the REAL
 * coordinate (str*p + u_ck, str*q + v_ck) of Eq. coordinate2d; the tables give
 * its integer base corner (h0, w0) = (floor u, floor v) and fractional parts
 * (a, b) (oracle/taps.py bilinear_exact).  The sample is the bilinear
 * interpolation of the four neighbours, zero outside the image (reading R1):
 *     s = (1-a)(1-b) x[h][v] + (1-a) b x[h][v+1] + a (1-b) x[h+1][v] + a b x[h+1][v+1]
 * forward: y = sum_k w_k s_k; backward_input (scatter form): every term of s_k
 * sends dy * w_k * (its weight) back to its pixel; backward_weight: dW_k =
 * sum_{n,p,q} dy * s_k.
 * ------------------------------------------------------------------------- */
static double px_or_zero(const double *xp, int H, int W, int h, int v) {
    return (h >= 0 && h < H && v >= 0 && v < W) ? xp[(long)h * W + v] : 0.0;
}

static double bilinear_sample(const double *xp, int H, int W, int h, int v, double a, double b) {
    return (1.0 - a) * (1.0 - b) * px_or_zero(xp, H, W, h, v) + (1.0 - a) * b * px_or_zero(xp, H, W, h, v + 1) +
           a * (1.0 - b) * px_or_zero(xp, H, W, h + 1, v) + a * b * px_or_zero(xp, H, W, h + 1, v + 1);
}

void oracle_forward_bilinear(int N, int C, int H, int W, int K, int str, const int32_t *h0, const int32_t *w0,
                             const double *fa, const double *fb, const double *x, const double *w, double *y,
                             int threads) {
    const int P = out_dim(H, str), Q = out_dim(W, str);
    const long planes = (long)N * C;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
#endif
    for (long nc = 0; nc < planes; ++nc) {
        const int c = (int)(nc % C);
        const double *xp = x + nc * H * W;
        double *yp = y + nc * P * Q;
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < Q; ++q) {
                double acc = 0.0;
                for (int k = 0; k < K; ++k) {
                    const int i = c * K + k;
                    acc += w[i] * bilinear_sample(xp, H, W, str * p + h0[i], str * q + w0[i], fa[i], fb[i]);
                }
                yp[p * Q + q] = acc;
            }
    }
}

static void scatter_add(double *dxp, int H, int W, int h, int v, double g) {
    if (h >= 0 && h < H && v >= 0 && v < W) dxp[(long)h * W + v] += g;
}

void oracle_backward_input_bilinear(int N, int C, int H, int W, int K, int str, const int32_t *h0, const int32_t *w0,
                                    const double *fa, const double *fb, const double *dy, const double *w, double *dx,
                                    int threads) {
    const int P = out_dim(H, str), Q = out_dim(W, str);
    const long planes = (long)N * C;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
#endif
    for (long nc = 0; nc < planes; ++nc) {
        const int c = (int)(nc % C);
        const double *gp = dy + nc * P * Q;
        double *dxp = dx + nc * H * W;
        for (long i = 0; i < (long)H * W; ++i) dxp[i] = 0.0;
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < Q; ++q)
                for (int k = 0; k < K; ++k) {
                    const int i = c * K + k;
                    const double g = gp[p * Q + q] * w[i], a = fa[i], b = fb[i];
                    const int h = str * p + h0[i], v = str * q + w0[i];
                    scatter_add(dxp, H, W, h, v, g * ((1.0 - a) * (1.0 - b)));
                    scatter_add(dxp, H, W, h, v + 1, g * ((1.0 - a) * b));
                    scatter_add(dxp, H, W, h + 1, v, g * (a * (1.0 - b)));
                    scatter_add(dxp, H, W, h + 1, v + 1, g * (a * b));
                }
    }
}

void oracle_backward_weight_bilinear(int N, int C, int H, int W, int K, int str, const int32_t *h0, const int32_t *w0,
                                     const double *fa, const double *fb, const double *x, const double *dy, double *dW,
                                     int threads) {
    const int P = out_dim(H, str), Q = out_dim(W, str);
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
#endif
    for (int c = 0; c < C; ++c)
        for (int k = 0; k < K; ++k) {
            const int i = c * K + k;
            double acc = 0.0;
            for (int n = 0; n < N; ++n) {
                const double *xp = x + ((long)n * C + c) * H * W;
                const double *gp = dy + ((long)n * C + c) * P * Q;
                for (int p = 0; p < P; ++p)
                    for (int q = 0; q < Q; ++q)
                        acc += gp[p * Q + q] * bilinear_sample(xp, H, W, str * p + h0[i], str * q + w0[i], fa[i], fb[i]);
            }
            dW[i] = acc;
        }
}
