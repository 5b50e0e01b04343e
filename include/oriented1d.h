/*
 * oriented1d.h — C ABI of liboriented1d: the depthwise convolution of oriented
 * 1D kernels (arXiv 2309.15812, "Convolutional Networks with Oriented 1D
 * Kernels") on NVIDIA B200 (sm_100a).
 *
 * The operation (Def. 1):
 *     y[n][c][p][q] = sum_{k=0}^{K-1} x[n][c][h][w] * w[c][k]
 *     h = str*p + floor(-(k-pad) * sin(theta_c)),  w = str*q + floor((k-pad) * cos(theta_c))
 * with zero padding outside [0,H) x [0,W) (reading R1), output size
 * P = (H-1)/str + 1, Q = (W-1)/str + 1 (reading R2), floors of the exact real
 * value (reading R3).  The paper writes x in R^{N x H x W x C} as INDEX
 * notation; this library stores activations NCHW-contiguous (one plane per
 * (n,c), row-major), see DESIGN.md §Layout.
 *
 * Conventions for every call:
 *   - Every function returns o1d_status; nothing throws across the ABI.  On an
 *     error, o1d_last_error() returns a thread-local, NUL-terminated message that
 *     stays valid until the next call from the same thread.
 *   - Argument validation is host-side and happens BEFORE any launch; a failing
 *     call leaves every output untouched.
 *   - Device pointers are caller-owned (PyTorch allocates them).  They must be
 *     16-byte aligned, NCHW-contiguous, and must not alias each other.  The
 *     library never allocates device memory except inside o1d_plan_create (the
 *     plan's tap tables), and frees it in o1d_plan_destroy.
 *   - Compute calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *     default stream).  Outputs are OVERWRITTEN, never accumulated into.
 *   - Results are deterministic: the same plan and inputs give bitwise-identical
 *     outputs (no floating-point atomics anywhere).
 *   - Weights w and the weight gradient dW are fp32 [C][K] (k fastest).
 *     Activations x, y, dy, dx have the plan's dtype (fp32, bf16 or fp16);
 *     arithmetic is fp32 multiply-add with fp32 accumulation for every dtype.
 *   - A plan is immutable after creation and may be used from several host
 *     threads / streams concurrently (each launch of a specialised kernel takes
 *     its own work-queue slot; up to 64 launches per pass in flight), except
 *     o1d_step_host, which uses the plan's internal second stream.
 */
#ifndef ORIENTED1D_H_
#define ORIENTED1D_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define O1D_API __attribute__((visibility("default")))
#else
#define O1D_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    O1D_OK = 0,
    O1D_INVALID_ARG = 1,         /* NULL pointer / bad enum value                         */
    O1D_INVALID_SHAPE = 2,       /* a dimension < 1                                       */
    O1D_INVALID_CONFIG = 3,      /* K < 1, stride < 1, pad out of range, D does not divide C */
    O1D_SHAPE_MISMATCH = 4,      /* buffer sizes disagree with the plan                   */
    O1D_UNSUPPORTED = 5,         /* dtype / layout / shape the library does not implement */
    O1D_MISALIGNED = 6,          /* a device pointer is not 16-byte aligned               */
    O1D_WORKSPACE_TOO_SMALL = 7, /* ws_bytes < o1d_workspace_bytes(plan)                  */
    O1D_CUDA_ERROR = 8,          /* a CUDA runtime / driver call failed                   */
    O1D_JIT_ERROR = 9            /* runtime specialisation (NVRTC) failed                 */
} o1d_status;

typedef enum { O1D_F32 = 0, O1D_BF16 = 1, O1D_F16 = 2 } o1d_dtype;
typedef enum { O1D_NCHW = 0 } o1d_layout;
typedef enum { O1D_ASSIGN_CONTIGUOUS = 0, O1D_ASSIGN_CYCLED = 1 } o1d_assign;

/* Problem descriptor (Def. 1): N batch, C channels, H x W input, K taps, stride
 * `stride` on both axes, padding `pad` (a real number, Def. 1 / Eq. coordinate1d
 * P:346-351 write pad_w without restricting it to integers; pass any negative
 * value for the paper's default floor(K/2); otherwise 0 <= pad <= K-1),
 * activation dtype and layout.  `flags` selects the discretisation and
 * implementation options (O1D_FLAG_*), 0 = library default.  */
typedef struct {
    int32_t N, C, H, W, K;
    int32_t stride;
    double pad;
    int32_t dtype;   /* o1d_dtype  */
    int32_t layout;  /* o1d_layout */
    int32_t flags;
} o1d_desc;

/* Implementation selection (testing / tuning).  The default picks the fastest
 * kernel family that supports the problem. */
#define O1D_FLAG_FORCE_GENERIC 0x1  /* runtime-tap shared-memory kernels only (no JIT)  */
#define O1D_FLAG_NO_TMA        0x2  /* stage tiles with plain loads instead of TMA      */
/* Discretisation of the filter offsets (a property of the method, not a tuning option):
 * default = rotation (Def. 1); O1D_FLAG_SHEAR = the shear parameterisation of the
 * Appendix "Rotation vs Shearing", see o1d_make_taps_ex. */
#define O1D_FLAG_SHEAR         0x4
/* O1D_FLAG_BILINEAR = the bilinear-interpolation discretisation of P:309-311 (Sec.
 * "Discretization and Interpolation", Table "bilinear" P:322-334): each tap samples x at
 * the REAL coordinate of Eq. coordinate2d, (str*p - (k-pad) sin t, str*q + (k-pad) cos t),
 * interpolated from its four integer neighbours (zero outside the image).  See
 * o1d_make_bilinear.  Mutually exclusive with O1D_FLAG_SHEAR. */
#define O1D_FLAG_BILINEAR      0x8

typedef struct o1d_plan o1d_plan;

/* Tap-offset table (Eq. coordinate, Eq. coordinate1d):
 *   oh[c*K+k] = floor(-(k-pad) * sin(angles_deg[c])),  ow[c*K+k] = floor((k-pad) * cos(angles_deg[c]))
 * evaluated as the floor of the exact real value (reading R3): the angle is
 * reduced mod 360 deg exactly; at the Niven angles (sin or cos in {0,+-1/2,+-1})
 * the product is evaluated exactly, elsewhere it is irrational and its floor is
 * taken from f64 trig, re-evaluated in binary128 when within 1e-9 of an integer.
 * This is NOT SPEC's rule (f64 trig, snapped only at multiples of 90 deg): the two
 * differ on the 30-degree family, e.g. theta = 30, k - pad = -2 gives floor(2 * 0.49999999999999994)
 * = 0 under SPEC's rule and the exact floor(1) = 1 here (reading R3).
 * angles_deg: host [C] (degrees, any finite real).  oh, ow: host [C][K] outputs.
 * pad: any negative value => floor(K/2); otherwise a finite real |pad| <= 4096 (k - pad
 * is then a binary double, so the same exactness argument holds).  Pure host
 * function, no CUDA context needed.  Errors: INVALID_ARG (NULL, non-finite angle or
 * pad), INVALID_CONFIG (K < 1, |pad| > 4096), INVALID_SHAPE (C < 1). */
O1D_API o1d_status o1d_make_taps(int32_t K, double pad, int32_t C, const double *angles_deg,
                         int16_t *oh, int16_t *ow);

/* Tap-offset table for discretisation `mode`: O1D_TAPS_ROTATION (= o1d_make_taps) or
 * O1D_TAPS_SHEAR (Appendix "Rotation vs Shearing"): the offsets are sampled
 * where the filter axis crosses integer columns, (-(k-pad) tan t, k-pad) (S^x),
 * or integer rows, ((k-pad), -(k-pad) cot t) (S^y), keeping the direction of
 * the rotation form: offset = m (-sin t, cos t) / max(|sin t|, |cos t|), m = k - pad,
 * the column form when |cos t| >= |sin t| (reading R13); the non-integer
 * coordinate is floored exactly (tan t is rational only at t = 0, 45, 135 mod 180).
 * Same arguments, ownership and errors as o1d_make_taps; INVALID_ARG for a bad mode. */
#define O1D_TAPS_ROTATION 0
#define O1D_TAPS_SHEAR    1
#define O1D_TAPS_BILINEAR 2   /* the base (floor) corner of each bilinear tap = the rotation taps */
O1D_API o1d_status o1d_make_taps_ex(int32_t K, double pad, int32_t C, const double *angles_deg, int32_t mode,
                                    int16_t *oh, int16_t *ow);

/* Bilinear discretisation (O1D_FLAG_BILINEAR): tap k of channel c samples x at
 * the real offset (u, v) = (-(k-pad) sin t, (k-pad) cos t) from the output's anchor.  With
 * h0 = floor(u), w0 = floor(v) (exact floors, = o1d_make_taps) and the fractional parts
 * a = u - h0, b = v - w0 in [0, 1) (exact 0 / 1/2 at the Niven angles, else f64 trig), the
 * tap reads
 *     (1-a)(1-b) x[h0][w0] + (1-a) b x[h0][w0+1] + a (1-b) x[h0+1][w0] + a b x[h0+1][w0+1]
 * (zero outside the image; reading R14).  h0, w0: host int16 [C][K]; fa, fb: host f64 [C][K].
 * Arguments and errors as o1d_make_taps. */
O1D_API o1d_status o1d_make_bilinear(int32_t K, double pad, int32_t C, const double *angles_deg, int16_t *h0,
                                     int16_t *w0, double *fa, double *fb);

/* Per-channel angles from D directions: angle_i = i*180/D deg,
 * channels split into D equal groups; group(c) = floor(c*D/C) for
 * O1D_ASSIGN_CONTIGUOUS, c mod D for O1D_ASSIGN_CYCLED; D == C gives
 * c*180/C.  shift_deg != 0 adds the layer-wise rotation ("alternating
 * 90 deg"), result reduced mod 180 deg.  out: host [C].  Errors:
 * INVALID_CONFIG when D < 1 or (D does not divide C and D != C). */
O1D_API o1d_status o1d_direction_angles(int32_t D, int32_t C, int32_t assign, double shift_deg, double *out);

/* Create an immutable plan for descriptor `d` and per-channel angles
 * angles_deg (host [C], degrees).  Computes the tap tables (as
 * o1d_make_taps / o1d_make_bilinear), de-duplicates equal tables, derives halo
 * extents, selects (and, unless O1D_FLAG_FORCE_GENERIC, JIT-specialises) the kernels
 * and uploads the tables to the current CUDA device.  Specialised modules are cached
 * per process and device by their generated source, which does not depend on N: plans
 * that differ only in the batch size (or are re-created) share the compiled code.
 * *out receives the plan (NULL on error).  Must be called with the target device
 * current. */
O1D_API o1d_status o1d_plan_create(const o1d_desc *d, const double *angles_deg, o1d_plan **out);

/* Output size: P = (H-1)/stride + 1, Q = (W-1)/stride + 1. */
O1D_API o1d_status o1d_plan_out_shape(const o1d_plan *plan, int32_t *P, int32_t *Q);

/* Copy the plan's tap table to host oh, ow [C][K] (bilinear plans: the base corners). */
O1D_API o1d_status o1d_plan_get_taps(const o1d_plan *plan, int16_t *oh, int16_t *ow);

/* Plan-creation cost: host milliseconds spent in o1d_plan_create (tap tables, source
 * generation, NVRTC compile or module-cache hit, module load) and whether the
 * specialised modules came from the process-wide cache (1) or were compiled (0; -1 when
 * the plan has no specialised kernels). */
O1D_API o1d_status o1d_plan_stats(const o1d_plan *plan, double *create_ms, int32_t *jit_cache_hit);

/* Short NUL-terminated description of the kernels the plan selected
 * (family, tile shape, number of specialised tap tables). */
O1D_API const char *o1d_plan_describe(const o1d_plan *plan);

/* Bytes of device workspace o1d_backward_weight needs (fp32 partial sums). */
O1D_API size_t o1d_workspace_bytes(const o1d_plan *plan);

/* Forward (Def. 1).  x: device [N][C][H][W] (plan dtype), w: device fp32
 * [C][K], y: device [N][C][P][Q] (plan dtype), overwritten. */
O1D_API o1d_status o1d_forward(const o1d_plan *plan, const void *x, const float *w, void *y, void *stream);

/* backward_input: dx = adjoint of the forward map in x applied to dy
 *   dx[n][c][h][w] = sum_k sum_{p,q : str*p+oh_ck = h, str*q+ow_ck = w} dy[n][c][p][q] * w[c][k]
 * (reading A5).  dy: device [N][C][P][Q], w: device fp32 [C][K],
 * dx: device [N][C][H][W], overwritten. */
O1D_API o1d_status o1d_backward_input(const o1d_plan *plan, const void *dy, const float *w, void *dx, void *stream);

/* backward_weight: dW[c][k] = sum_{n,p,q} dy[n][c][p][q] * x[n][c][str*p+oh_ck][str*q+ow_ck]
 * (adjoint in w; out-of-range taps contribute 0).  x: device [N][C][H][W],
 * dy: device [N][C][P][Q], dW: device fp32 [C][K] (overwritten, never
 * accumulated), ws: device workspace of ws_bytes >= o1d_workspace_bytes(plan).
 * Deterministic: partial sums are reduced in a fixed order. */
O1D_API o1d_status o1d_backward_weight(const o1d_plan *plan, const void *x, const void *dy, float *dW,
                               void *ws, size_t ws_bytes, void *stream);

/* Fused backward: backward_input and backward_weight in ONE pass over x
 * and dy -- every (n, c) plane of x and dy is read from HBM once and both dx and the dW
 * partials are produced from the same shared-memory tiles (plus the fixed-order dW
 * finalize launch).  Same results as o1d_backward_input + o1d_backward_weight (dx
 * bitwise; dW bitwise, the same partial sums in the same order).  Buffers as for those
 * two calls; ws >= o1d_workspace_bytes(plan).  Plans without the fused kernel run the
 * two passes. */
O1D_API o1d_status o1d_backward(const o1d_plan *plan, const void *x, const void *dy, const float *w, void *dx,
                                float *dW, void *ws, size_t ws_bytes, void *stream);

/* One training step of the layer through HOST buffers (the end-to-end path):
 * copies x, w, dy host->device, runs forward, backward_input and
 * backward_weight, copies y, dx, dW device->host, then synchronises `stream`.
 * When all three passes run on the v2 specialised kernels the step is pipelined
 * over batch chunks (default 8, env O1D_E2E_CHUNKS): the plan's internal streams
 * copy chunk i+1 in and chunk i-1 out while chunk i is computed (the kernels
 * take a batch window; dW is finalised once, bitwise equal to the device path).
 * Otherwise the plan's second stream overlaps the two PCIe directions with each
 * other and with the kernels (forward + D2H y on `stream`; H2D dy,
 * backward_input, D2H dx, backward_weight, D2H dW on the second stream); calls
 * on one plan must not run concurrently.  Host buffers should be pinned.  dev_ws: device scratch of >= o1d_step_host_workspace_bytes(plan)
 * bytes (holds device copies of every tensor and the dW workspace). */
O1D_API size_t o1d_step_host_workspace_bytes(const o1d_plan *plan);
O1D_API o1d_status o1d_step_host(const o1d_plan *plan, const void *x_h, const float *w_h, const void *dy_h,
                         void *y_h, void *dx_h, float *dW_h, void *dev_ws, size_t dev_ws_bytes,
                         void *stream);

/* One training step of the layer on device buffers: forward (x -> y), backward_input
 * (dy -> dx) and backward_weight ((x, dy) -> dW), the same results as the three
 * calls in that order (bitwise).  The passes read only the step's inputs and write
 * disjoint outputs, so on the specialised kernels the second and third pass skip the
 * wait for the preceding pass and overlap its tail (programmatic dependent launch);
 * the first waits for the work before it on `stream`.  Buffers as for the three
 * calls; ws: >= o1d_workspace_bytes(plan).  Outputs must not alias inputs. */
O1D_API o1d_status o1d_step(const o1d_plan *plan, const void *x, const float *w, const void *dy, void *y, void *dx,
                            float *dW, void *ws, size_t ws_bytes, void *stream);

/* Number of kernel launches one call of each pass issues (for launch accounting);
 * pass 3 = o1d_backward. */
O1D_API int32_t o1d_launches_per_call(const o1d_plan *plan, int32_t pass /* 0 fwd, 1 bwd_in, 2 bwd_w, 3 fused bwd */);

/* Destroy a plan: makes the plan's device current, waits for the device's outstanding
 * work (a launch may still reference the plan's tables and scheduler counters), releases
 * its resources and restores the caller's current device.  NULL is a no-op. */
O1D_API void o1d_plan_destroy(o1d_plan *plan);

/* Diagnostics: the CUDA C++ source the plan's specialised kernels would be
 * compiled from (pass 0 forward, 1 backward_input, 2 backward_weight), built on
 * the host only (no GPU needed).  buf may be NULL to query the size; *len is
 * in/out (buffer size in, bytes incl. the NUL out).  UNSUPPORTED when the
 * problem is served by the generic kernels. */
O1D_API o1d_status o1d_spec_source(const o1d_desc *d, const double *angles_deg, int32_t pass, char *buf,
                                   size_t *len);
/* Diagnostics: with O1D_TRACE=1 in the environment at plan creation, the
 * specialised kernels append (globaltimer ns, tag) u64 pairs to a plan-owned
 * device buffer (first u64 = record count; tag = kind:4 | warp:4 | smid:8 |
 * block:16 | item:32).  Synchronises the device, copies up to `bytes` into
 * `host` and clears the buffer.  Returns the bytes copied (0: tracing off). */
O1D_API size_t o1d_debug_trace(const o1d_plan *plan, void *host, size_t bytes);
O1D_API const char *o1d_last_error(void);
O1D_API const char *o1d_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ORIENTED1D_H_ */
