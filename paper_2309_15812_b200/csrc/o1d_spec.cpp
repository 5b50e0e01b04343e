// o1d_spec.cpp — runtime-specialised ("spec") kernels of liboriented1d.
//
// Why: the tap loop of Def. 1 is a stencil whose offsets depend on the
// angle.  With the offsets known at compile time, each thread keeps a 7x7 block
// of outputs in registers and loads every input pixel its block needs from
// shared memory ONCE, feeding all (output, tap) pairs that use it (~6 shared
// loads per output at K=31 instead of 31).  The paper reached the same
// conclusion on its hardware ("a specific CUDA kernel for every input size",
// P:694); here the specialisation is done at plan time with NVRTC for sm_100a,
// one `case` per distinct tap table of the plan.
//
// Pipeline (one persistent CTA per SM):
//   * P consumer "pairs" (wpg warps each, 4 block rows x 8 block columns per warp)
//     and NPROD producer warps; every pair owns NB tile slots (mbarriers full /
//     empty); producers take planes from per-table atomic counters (every SM
//     has a "home" table; when it is exhausted the CTA steals from the others,
//     so completion never depends on where CTAs land), stage the channel's
//     weights and issue one TMA 4-D load per plane (image rows only, columns
//     past the image zero-filled by the TMA unit, zero rows shared between
//     consecutive slots serve as the vertical halo, reading R1).
//   * forward / backward_input (negated taps): packed FP32 (fma.rn.f32x2) with
//     the tap weight as the broadcast operand; outputs -> per-warp staging band
//     -> TMA bulk store.
//   * backward_weight: the dy plane is TMA-loaded into a per-pair slot; every
//     lane keeps its 7x7 dy block in registers, accumulates one partial per
//     distinct tap offset (pixel pairs, FFMA2), folds them into per-tap sums
//     v[k] (weighted for bilinear taps), reduces over the warp and writes
//     ws[c][n][band][k]; a second launch sums the partials in f64, fixed order.
//   * fused backward (NEXT-2): x and dy planes of one item land in the same
//     slot; the pair computes the weight-gradient partials and the
//     backward_input band from the same tiles (x and dy read from HBM once).
// The generated source does not depend on the batch size N (a kernel
// parameter), so a process-wide cache keyed by (device, source) lets plans
// that differ only in N share one compiled module.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "o1d_spec.h"

namespace o1d {
namespace {

// ---------------------------------------------------------------- driver API
struct Driver {
    PFN_cuModuleLoadData_v2000 moduleLoadData = nullptr;
    PFN_cuModuleUnload_v2000 moduleUnload = nullptr;
    PFN_cuModuleGetFunction_v2000 moduleGetFunction = nullptr;
    PFN_cuFuncSetAttribute_v9000 funcSetAttribute = nullptr;
    PFN_cuLaunchKernelEx_v11060 launchKernelEx = nullptr;
    PFN_cuTensorMapEncodeTiled_v12000 encodeTiled = nullptr;
    PFN_cuGetErrorString_v6000 getErrorString = nullptr;
    PFN_cuCtxGetCurrent_v4000 ctxGetCurrent = nullptr;
    PFN_cuCtxPushCurrent_v4000 ctxPush = nullptr;
    PFN_cuCtxPopCurrent_v4000 ctxPop = nullptr;
    PFN_cuOccupancyMaxActiveBlocksPerMultiprocessor_v6050 occupancy = nullptr;
    std::string err;
};

template <typename T>
bool entry(const char *name, T *fn, std::string *err) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) {
        *err = std::string("driver entry point not found: ") + name;
        return false;
    }
    *fn = reinterpret_cast<T>(p);
    return true;
}

Driver &drv() {
    static Driver d;
    static std::once_flag once;
    std::call_once(once, [] {
        std::string e;
        bool ok = entry("cuModuleLoadData", &d.moduleLoadData, &e) && entry("cuModuleUnload", &d.moduleUnload, &e) &&
                  entry("cuModuleGetFunction", &d.moduleGetFunction, &e) &&
                  entry("cuFuncSetAttribute", &d.funcSetAttribute, &e) &&
                  entry("cuTensorMapEncodeTiled", &d.encodeTiled, &e) && entry("cuGetErrorString", &d.getErrorString, &e) &&
                  entry("cuLaunchKernelEx", &d.launchKernelEx, &e) && entry("cuCtxGetCurrent", &d.ctxGetCurrent, &e) &&
                  entry("cuCtxPushCurrent", &d.ctxPush, &e) && entry("cuCtxPopCurrent", &d.ctxPop, &e) &&
                  entry("cuOccupancyMaxActiveBlocksPerMultiprocessor", &d.occupancy, &e);
        if (!ok) d.err = e;
    });
    return d;
}

std::string cu_err(CUresult r) {
    const char *s = nullptr;
    if (drv().getErrorString) drv().getErrorString(r, &s);
    return s ? s : ("CUresult " + std::to_string((int)r));
}

// --------------------------------------------------------------------- NVRTC
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram *nvrtcProgram_t;
struct Nvrtc {
    nvrtcResult_t (*create)(nvrtcProgram_t *, const char *, const char *, int, const char *const *, const char *const *) = nullptr;
    nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char *const *) = nullptr;
    nvrtcResult_t (*logSize)(nvrtcProgram_t, size_t *) = nullptr;
    nvrtcResult_t (*log)(nvrtcProgram_t, char *) = nullptr;
    nvrtcResult_t (*cubinSize)(nvrtcProgram_t, size_t *) = nullptr;
    nvrtcResult_t (*cubin)(nvrtcProgram_t, char *) = nullptr;
    nvrtcResult_t (*destroy)(nvrtcProgram_t *) = nullptr;
    std::string err;
};

Nvrtc &nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *cands[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                               "/usr/local/cuda/lib64/libnvrtc.so"};
        void *h = nullptr;
        for (const char *c : cands)
            if ((h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) {
            n.err = "cannot dlopen libnvrtc.so.12";
            return;
        }
        n.create = reinterpret_cast<decltype(n.create)>(dlsym(h, "nvrtcCreateProgram"));
        n.compile = reinterpret_cast<decltype(n.compile)>(dlsym(h, "nvrtcCompileProgram"));
        n.logSize = reinterpret_cast<decltype(n.logSize)>(dlsym(h, "nvrtcGetProgramLogSize"));
        n.log = reinterpret_cast<decltype(n.log)>(dlsym(h, "nvrtcGetProgramLog"));
        n.cubinSize = reinterpret_cast<decltype(n.cubinSize)>(dlsym(h, "nvrtcGetCUBINSize"));
        n.cubin = reinterpret_cast<decltype(n.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
        if (!n.create || !n.compile || !n.logSize || !n.log || !n.cubinSize || !n.cubin || !n.destroy)
            n.err = "libnvrtc is missing symbols";
    });
    return n;
}

bool compile_cubin(const std::string &src, const std::string &name, std::vector<char> *out, std::string *log) {
    Nvrtc &nv = nvrtc();
    if (!nv.err.empty()) {
        *log = nv.err;
        return false;
    }
    nvrtcProgram_t prog = nullptr;
    if (nv.create(&prog, src.c_str(), name.c_str(), 0, nullptr, nullptr) != 0) {
        *log = "nvrtcCreateProgram failed";
        return false;
    }
    const char *opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--ptxas-options=-v", "-DNDEBUG"};
    const nvrtcResult_t rc = nv.compile(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
    size_t ls = 0;
    nv.logSize(prog, &ls);
    std::string lg(ls, '\0');
    if (ls) nv.log(prog, &lg[0]);
    *log = lg;
    bool ok = rc == 0;
    if (ok) {
        size_t cs = 0;
        nv.cubinSize(prog, &cs);
        out->resize(cs);
        nv.cubin(prog, out->data());
    }
    nv.destroy(&prog);
    return ok;
}

int env_int(const char *n, int dflt) {
    const char *v = getenv(n);
    return (v && *v) ? atoi(v) : dflt;
}

// ------------------------------------------------------------ plan geometry
constexpr int R = 7, S = 7;  // per-thread output block (rows x cols)

struct Tap {
    int dh, dw;
    std::vector<std::pair<int, float>> ks;  // (tap index k, coefficient) sharing this offset (R7; bilinear R14)
};

struct Geo {  // one distinct (weighted) tap table, one pass
    std::vector<Tap> taps;
    int minDH, maxDH, minDW, maxDW;
    int pitch;  // smem row pitch (elements) this table needs
};

int pitch_for(int cols) {
    int p = cols;
    while (p % 16 != 8) ++p;  // 7*pitch = 8 or 24 mod 32 -> conflict-free LDS.32
    return p;
}

// Distinct offsets of one channel's expanded taps.  The tile starts at image column 0 and is
// `pitch` wide, so columns past the image are zero-filled by TMA; reads left of column 0
// wrap into the previous row's zero columns (pitch >= Win - minDW).
Geo make_geo(const int16_t *dh_, const int16_t *dw_, const int16_t *k_, const float *coef, int KE, bool negate, int BC,
             int Win) {
    Geo g;
    std::map<std::pair<int, int>, int> idx;
    g.minDH = g.minDW = 1 << 20;
    g.maxDH = g.maxDW = -(1 << 20);
    for (int e = 0; e < KE; ++e) {
        if (coef[e] == 0.0f) continue;  // padding entries
        const int dh = negate ? -dh_[e] : dh_[e], dw = negate ? -dw_[e] : dw_[e];
        auto it = idx.find({dh, dw});
        if (it == idx.end()) {
            it = idx.emplace(std::make_pair(dh, dw), (int)g.taps.size()).first;
            g.taps.push_back(Tap{dh, dw, {}});
        }
        g.taps[it->second].ks.push_back({k_[e], coef[e]});
        g.minDH = std::min(g.minDH, dh);
        g.maxDH = std::max(g.maxDH, dh);
        g.minDW = std::min(g.minDW, dw);
        g.maxDW = std::max(g.maxDW, dw);
    }
    if (g.taps.empty()) {  // all-zero table (cannot happen for K >= 1): one dummy offset
        g.taps.push_back(Tap{0, 0, {{0, 0.0f}}});
        g.minDH = g.maxDH = g.minDW = g.maxDW = 0;
    }
    g.pitch = pitch_for(std::max(Win - std::min(g.minDW, 0), S * BC + std::max(g.maxDW, 0)));
    return g;
}

std::string flit(float v) {  // exact float literal
    char b[48];
    snprintf(b, sizeof b, "%.9ef", (double)v);
    return b;
}

}  // namespace

constexpr int kSlots = 64;  // concurrent launches per pass that can be in flight on one plan
constexpr int kCS = 32;     // scheduler counter stride (unsigned): one 128-byte line per counter
constexpr size_t kTraceBytes = 8 + ((size_t)32 << 20);  // count + 2^21 (time, tag) records
constexpr int kPasses = 4;  // 0 forward, 1 backward_input, 2 backward_weight, 3 fused backward

// one compiled module (shared by every plan whose generated source is identical)
struct Mod {
    CUmodule mod = nullptr;
    CUcontext ctx = nullptr;
    CUfunction fn = nullptr, fin = nullptr;
    std::string regs;
    ~Mod() {
        if (!mod) return;
        Driver &d = drv();
        if (ctx && d.ctxPush(ctx) == CUDA_SUCCESS) {
            d.moduleUnload(mod);
            CUcontext dummy;
            d.ctxPop(&dummy);
        }
    }
};

// launch geometry of one pass
struct Lay {
    int P = 1, NB = 2, NS = 2, NPROD = 1, wpg = 1;
    bool early = true;  // stencil outputs stored to the staging band row by row inside the tap code
    int pitch = 0, zrows = 0, hin = 0;    // ring 1: x (passes 0, 2, 3) or dy (pass 1)
    int pitch2 = 0, zrows2 = 0, hin2 = 0; // ring 2 (fused): dy with the negated tables' halo
    int dyp = 0, dyrows = 0;              // backward_weight: dense dy box per pair
    size_t zb = 0, tb = 0, zb2 = 0, tb2 = 0, db = 0, sb = 0;
    size_t off_item = 0, off_w = 0, off_stg = 0, off_dy = 0, off_t = 0, off_t2 = 0, total = 0;
    // 16-bit ring-1 planes: staged = one TMA box of the raw plane into a per-pair staging buffer,
    // widened to the fp32 slot by the pair's producer (else: per-lane 16-byte loads, see emit_producer)
    bool staged = false;
    size_t stb = 0, off_st = 0;
    // 16-bit planes whose rows are not 16-byte multiples (ConvNeXt stage 2: 28 x 2 B): every TMA box views
    // a plane as rows of 8 elements (the plane itself is a 16-byte multiple), so only dense whole-row boxes
    // are used (raw input plane, dy block, output band) and the widening maps elements to (row, column)
    bool flat = false;
    int ncw() const { return P * wpg; }
    size_t ring1() const { return zb + (size_t)NS * (zb + tb); }
    size_t ring2() const { return tb2 ? zb2 + (size_t)NS * (zb2 + tb2) : 0; }
};

// small-plane kernels (H, W <= 14): launch geometry of one pass (see gen_small_pass)
struct SmallLay {
    int BRs = 1, BCs = 1, QW = 1;  // 7x7 block positions per plane = warps per quad
    int NQ = 1, NB = 2, G = 1;     // quads, input slots per quad, 32-plane groups per channel
    int UB = 8;                    // bytes per unit (UPu pixels) of the LDGSTS slots and the output staging
    int UPu = 2, es = 4;           // pixels per unit (1 for odd H*W), activation bytes
    bool sync_copy = false;        // 16-bit odd planes: 2-byte units copied by plain loads (cp.async moves >= 4 B)
    bool tma = false;              // inputs by one TMA box per item, plane-major, 4-pixel (16-byte) units
    int UPi = 2;                   // pixels per input unit
    int ustr = 0, lstr = 0;        // input slots: bytes between units of one plane / between planes (lanes)
    bool tma_out = false;          // stencil outputs staged plane-major and written by one TMA box store
    int hp_in = 0, hp_dy = 0, hp_out = 0;  // units per plane: input, dy (backward_weight), output
    size_t slotb = 0, dyb = 0, outb = 0;
    size_t off_item = 0, off_w = 0, off_slot = 0, off_out = 0, total = 0;
    int NS() const { return NQ * NB; }
    int threads() const { return 32 * (NQ + NQ * QW); }
};

struct SpecSet {
    int BR = 0, BC = 0, wpg = 1, nt = 0, nsm = 0, K = 0;
    bool small = false;                  // small-plane kernels (gen_small_pass) instead of gen_pass
    long small_items = 0;                // small: work items (C x 32-plane groups)
    SmallLay sl[3];
    bool has[kPasses] = {false, false, false, false};
    bool fused_step = false;             // o1d_step uses pass 3 (O1D_FUSED at plan creation)
    Lay lay[kPasses];
    std::vector<Geo> fwd, bwd;           // per distinct table
    std::shared_ptr<Mod> mod[kPasses];
    size_t smem[kPasses] = {0, 0, 0, 0};
    int grid[kPasses] = {0, 0, 0, 0}, threads[kPasses] = {0, 0, 0, 0};
    bool pdl = true;                     // programmatic dependent launch (O1D_PDL at plan creation)
    std::string src3;                    // fused backward source, compiled on first use
    std::mutex mu3;
    // work-queue counters: kPasses x kSlots launch slots x (NT next counters + 1 done counter);
    // every launch takes the next slot (host atomic), so concurrent launches on different
    // streams never share counters; a slot is reset by the last producer warp of its launch
    unsigned *d_sched = nullptr;
    unsigned long long *d_trace = nullptr;  // diagnostics (O1D_TRACE=1)
    std::atomic<unsigned> launch_seq{0};
};

namespace {

// ------------------------------------------------------------- code emission
const char *kPrelude = R"(
typedef unsigned long long u64;
typedef unsigned int u32;
struct __align__(64) TmaDesc { u64 v[16]; };
struct Params {
  TmaDesc in_map;    // ring-1 planes: x (forward, backward_weight, fused) or dy (backward_input)
  TmaDesc out_map;   // stencil: y / dx band box; backward_weight: dense dy box; fused: dx band box
  TmaDesc aux_map;   // fused: dy planes for ring 2
  const float* w;
  void* io;
  float* ws;
  unsigned* sched;   // [NT] next-plane counters (CS apart), [NT * CS] = done counter
  float* dW;
  u64* trace;        // diagnostics (O1D_TRACE): [0] = record count, then (globaltimer, tag) pairs
  int N, n0, nlen;   // batch size; batch window [n0, n0 + nlen) (nlen = 0: all)
  int nowait;        // 1: no griddepcontrol.wait before the loads (o1d_step: inputs not from the predecessor)
  const void* cvt1;  // 16-bit plans: ring-1 planes (x or dy) widened to fp32 by the producers
  const void* cvt2;  // 16-bit fused plans: ring-2 planes (dy)
  const void* src1;  // small-plane kernels: input planes (x, or dy for backward_input)
  const void* src2;  // small-plane backward_weight: dy planes
  void* dst;         // small-plane stencil: output planes (y or dx)
};
// streaming 16-byte load (read once: no L1 allocation, evict-first in L2)
__device__ __forceinline__ uint4 ldg_stream(const void* ptr, u64 pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ u32 sa(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* b, u32 n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(n));
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(u64* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* b, u32 bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_test(u64* b, u32 ph) {  // non-blocking: phase with parity ph completed?
  u32 r;
  asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(r) : "r"(sa(b)), "r"(ph) : "memory");
  return r != 0;
}
__device__ __forceinline__ void mbar_wait(u64* b, u32 ph) {
  // try_wait with a suspend-time hint: the warp sleeps until the phase completes
  // instead of spinning (spin loops steal issue slots from the compute warps)
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n @!p bra W_%=;\n}\n"
               :: "r"(sa(b)), "r"(ph), "r"(0x100000u) : "memory");
}
// streaming TMA load: every plane is read once, so it is marked evict-first in L2 (the
// kernel's code, constants and scheduler counters then stay L2-resident across launches)
__device__ __forceinline__ u64 policy_evict_first() {
  u64 p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ void tma_load(void* dst, const TmaDesc* m, int x, int y, int z, int w, u64* b, u64 pol) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;"
               :: "r"(sa(dst)), "l"(m), "r"(x), "r"(y), "r"(z), "r"(w), "r"(sa(b)), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_store_band(const TmaDesc* m, const void* src, int row0, int c, int n, u64 pol) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%2, %3, %4, %5}], [%1], %6;"
               :: "l"(m), "r"(sa(src)), "r"(0), "r"(row0), "r"(c), "r"(n), "l"(pol) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ u64 f2pack(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float f2lo(u64 v) { float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); return lo; }
__device__ __forceinline__ float f2hi(u64 v) { float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); return hi; }
// packed fp32 FMA (two lanes per instruction, each fma.rn): d = a * b + c
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
// programmatic dependent launch: wait for the preceding grid (and its memory) before
// touching global memory; allow the next grid to start launching when we run dry
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ u32 smid() { u32 r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
__device__ __forceinline__ u64 gtimer() { u64 r; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(r)); return r; }
// diagnostics: one (time, tag) record in this warp's private region (256 records
// per warp, no atomics); tag = kind:4 | warp:4 | smid:8 | block:16 | item:32
__device__ __forceinline__ void trace_ev(u64* tr, u32 kind, int item, int& n) {
  if (!tr) return;
  const u64 i = ((u64)blockIdx.x * 32 + (threadIdx.x >> 5)) * 256 + (n++ & 255);
  if (i >= (1ull << 21)) return;
  tr[1 + 2 * i] = gtimer();
  tr[2 + 2 * i] = ((u64)kind << 60) | ((u64)((threadIdx.x >> 5) & 15) << 56) | ((u64)(smid() & 255) << 48) |
                  ((u64)(blockIdx.x & 0xffff) << 32) | (u32)item;
}
// NV per-lane values -> lane L ends with the warp sum of v[L % NV]
template <int NV> __device__ __forceinline__ float reduce_scatter(float (&v)[NV], int lane) {
#pragma unroll
  for (int s = NV / 2; s >= 1; s >>= 1) {
    const bool up = lane & s;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = up ? v[i] : v[i + s];
      const float keep = up ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  float r = v[0];
#pragma unroll
  for (int s = NV; s < 32; s <<= 1) r += __shfl_xor_sync(0xffffffffu, r, s);
  return r;
}
// ------------------------------------------------------------------- scheduler
// Planes of table t: its channels (CHLIST[CHOFF[t] ..]) x the batch (window); item i of a
// table is channel index i mod nch, sample i / nch (consecutive items walk the channels
// first: the planes in flight form a compact address range).  Producer lane 0 takes items
// from per-table counters; when its table is exhausted it moves on to the next one (every
// table is visited once), so every item is taken exactly once whatever SMs the CTAs land on.
__device__ __forceinline__ int nch_of(int t) { return CHOFF[t + 1] - CHOFF[t]; }
__device__ __forceinline__ int sched_resolve(unsigned* sched, int& tcur, unsigned raw, int& tried, int nper) {
  while (tcur >= 0) {
    if (raw < (unsigned)(nch_of(tcur) * nper)) return (tcur << 22) | (int)raw;
    if (++tried >= NT) { tcur = -1; break; }
    tcur = tcur + 1 == NT ? 0 : tcur + 1;
    raw = atomicAdd(sched + tcur * CS, 1u);
  }
  return -1;
}
__device__ __forceinline__ void item_cn(int item, int& t, int& c, int& n, int n0) {
  t = (item >> 22) & 31;
  const int i = item & 0x3FFFFF;
  const int nch = nch_of(t);
  n = i / nch;
  c = CHLIST[CHOFF[t] + (i - n * nch)];
  n += n0;
}
// the launch's last producer warp resets the slot's counters for its next use
__device__ __forceinline__ void sched_exit(unsigned* sched, unsigned per_cta) {
  __threadfence();
  if (atomicAdd(sched + NT * CS, 1u) == gridDim.x * per_cta - 1) {
    for (int t = 0; t < NT; ++t) sched[t * CS] = 0u;
    sched[NT * CS] = 0u;
    __threadfence();
  }
}
)";

struct Ctx {
    int C, K, Ho, Wo, BR, BC, nt, nsm;
    int Wi = 0;                    // input width (x)
    int act = 0;                   // activation dtype (o1d_dtype)
    bool flat = false;             // planes viewed as rows of 8 elements by the TMA maps (Lay::flat)
    std::vector<int> home;         // home table per %smid (empty: TPC-pair fallback)
    std::vector<int> table_of;
};

void emit_header(std::ostringstream &os, const Ctx &x) {
    os << "#define NT " << x.nt << "\n#define CS " << kCS << "\n";
    if (x.act == O1D_F32)
        os << "typedef float act_t;\n#define LD(v) (v)\n"
              "__device__ __forceinline__ float to_act(float v) { return v; }\n";
    else if (x.act == O1D_BF16)
        os << "typedef unsigned short act_t;\n#define LD(v) __uint_as_float(((unsigned)(v)) << 16)\n"
              "__device__ __forceinline__ act_t to_act(float v) { unsigned short r; asm(\"cvt.rn.bf16.f32 %0, %1;\" : \"=h\"(r) : \"f\"(v)); return r; }\n";
    else
        os << "typedef unsigned short act_t;\n"
              "__device__ __forceinline__ float h2f(unsigned short h) { float f; asm(\"cvt.f32.f16 %0, %1;\" : \"=f\"(f) : \"h\"(h)); return f; }\n"
              "#define LD(v) h2f(v)\n"
              "__device__ __forceinline__ act_t to_act(float v) { unsigned short r; asm(\"cvt.rn.f16.f32 %0, %1;\" : \"=h\"(r) : \"f\"(v)); return r; }\n";
    // tiles in shared memory are fp32 for every dtype: 16-bit planes are widened by the
    // producer warps on the way in (LDG -> convert -> STS), so the tap loops never convert
    os << "typedef float tile_t;\n#define LDT(v) (v)\n";
    if (x.act == O1D_BF16)
        os << "__device__ __forceinline__ float4 w4(unsigned a, unsigned b) {\n"
              "  return make_float4(__uint_as_float(a << 16), __uint_as_float(a & 0xffff0000u), __uint_as_float(b << 16),\n"
              "                     __uint_as_float(b & 0xffff0000u));\n}\n";
    else if (x.act == O1D_F16)
        os << "__device__ __forceinline__ float4 w4(unsigned a, unsigned b) {\n"
              "  return make_float4(h2f((unsigned short)(a & 0xffffu)), h2f((unsigned short)(a >> 16)), h2f((unsigned short)(b & 0xffffu)),\n"
              "                     h2f((unsigned short)(b >> 16)));\n}\n";
    std::vector<int> choff(x.nt + 1, 0), chlist;
    for (int t = 0; t < x.nt; ++t) {
        choff[t] = (int)chlist.size();
        for (int c = 0; c < x.C; ++c)
            if (x.table_of[c] == t) chlist.push_back(c);
    }
    choff[x.nt] = (int)chlist.size();
    os << "__constant__ int CHOFF[" << x.nt + 1 << "] = {";
    for (int t = 0; t <= x.nt; ++t) os << (t ? "," : "") << choff[t];
    os << "};\n__constant__ short CHLIST[" << x.C << "] = {";
    for (int c = 0; c < x.C; ++c) os << (c ? "," : "") << chlist[c];
    os << "};\n";
    // home table per SM (see home_tables()); fallback without a topology probe:
    // (smid / 2) mod NT, i.e. TPC pairs share a table
    const int nh = x.home.empty() ? x.nsm : (int)x.home.size();
    os << "#define NHOME " << nh << "\n__constant__ unsigned char HOME[" << nh << "] = {";
    for (int s = 0; s < nh; ++s) os << (s ? "," : "") << (x.home.empty() ? (s / 2) % x.nt : x.home[s]);
    os << "};\n" << kPrelude;
}

// List schedule of independent accumulator updates: repeatedly emit the update whose
// accumulator was used least recently (ties: original order), so dependent FMAs on one
// accumulator are spread out (measured: near-horizontal tables otherwise chain every
// second FFMA2 on one accumulator -> fixed-latency "wait" stalls).
void emit_lru(std::ostringstream &os, const char *ind, std::vector<std::pair<std::string, std::string>> &fm,
              std::map<std::string, long> &last_use, long &clock) {
    std::vector<bool> done(fm.size(), false);
    for (size_t n = 0; n < fm.size(); ++n) {
        long best = -1, bt = 0;
        for (size_t i = 0; i < fm.size(); ++i) {
            if (done[i]) continue;
            auto it = last_use.find(fm[i].first);
            const long t = it == last_use.end() ? -1000000 : it->second;
            if (best < 0 || t < bt) best = (long)i, bt = t;
            if (t == -1000000) break;
        }
        done[best] = true;
        last_use[fm[best].first] = clock++;
        os << ind << fm[best].second << "\n";
    }
}

std::string cn(int v) { return v < 0 ? "m" + std::to_string(-v) : std::to_string(v); }

// merged weight of one distinct offset: sum over its (k, coef) of coef * w[k] (R7, R14)
std::string merged_weight(const Tap &t) {
    std::string e;
    for (size_t q = 0; q < t.ks.size(); ++q) {
        if (q) e += " + ";
        if (t.ks[q].second == 1.0f) e += "wv[" + std::to_string(t.ks[q].first) + "]";
        else e += flit(t.ks[q].second) + " * wv[" + std::to_string(t.ks[q].first) + "]";
    }
    return e;
}

// Stencil taps of one table with packed FFMA2 (assigns a<r>_<s>): output columns are
// paired so that the pixel pair starts at an even column relative to the block: taps with
// even dw accumulate into pairs (0,1),(2,3),(4,5) + scalar 6 (set A), taps with odd dw into
// pairs (1,2),(3,4),(5,6) + scalar 0 (set B).  Every pixel pair is then an even-aligned
// (v_j, v_j+1) register pair; a_rs = A_rs + B_rs at the end.  Footprint rows are walked
// top to bottom, the loads of row k+1 emitted before the FMAs of row k.  Returns the
// issue-cost estimate (FMA instructions + loads).
// `store_row` (optional): called with r once output row r is final (after the last footprint row that
// reaches it), with const float a<r>_<s> declared in scope -- the caller emits its stores there, so the
// epilogue's shared-memory stores overlap the remaining FMAs.  Without it the outputs are assigned to
// a<r>_<s> variables declared by the caller.
long emit_stencil_taps(std::ostringstream &os, const Geo &g, int pitch, const char *ind,
                       const std::function<void(int)> &store_row = nullptr) {
    long cost = 0;
    const int nd = (int)g.taps.size();
    for (int d = 0; d < nd; ++d)
        os << ind << "const float m" << d << " = " << merged_weight(g.taps[d]) << ";\n"
           << ind << "const u64 M" << d << " = f2pack(m" << d << ", m" << d << ");\n";
    for (int r = 0; r < R; ++r)
        os << ind << "u64 A" << r << "_0 = 0ull, A" << r << "_2 = 0ull, A" << r << "_4 = 0ull; float A" << r << "_6 = 0.f;\n"
           << ind << "u64 B" << r << "_1 = 0ull, B" << r << "_3 = 0ull, B" << r << "_5 = 0ull; float B" << r << "_0 = 0.f;\n";
    struct Row {
        int i;
        std::vector<std::pair<int, int>> pairs;  // (r, distinct tap)
        std::set<int> need, pr;
    };
    std::vector<Row> rows;
    for (int i = g.minDH; i <= g.maxDH + R - 1; ++i) {
        Row rw{i, {}, {}, {}};
        for (int r = 0; r < R; ++r)
            for (int d = 0; d < nd; ++d)
                if (g.taps[d].dh == i - r) rw.pairs.push_back({r, d});
        if (rw.pairs.empty()) continue;
        std::set<int> scal;
        for (auto &p : rw.pairs) {
            const int dw = g.taps[p.second].dw;
            if (((dw % 2) + 2) % 2 == 0) {
                for (int s = 0; s < 6; s += 2) rw.pr.insert(dw + s);
                scal.insert(dw + 6);
            } else {
                for (int s = 1; s < 7; s += 2) rw.pr.insert(dw + s);
                scal.insert(dw);
            }
        }
        rw.need = scal;
        for (int j : rw.pr) rw.need.insert(j), rw.need.insert(j + 1);
        rows.push_back(rw);
    }
    auto vname = [&](int i, int j) { return "v" + cn(i) + "_" + cn(j); };
    auto pname = [&](int i, int j) { return "P" + cn(i) + "_" + cn(j); };
    auto loads = [&](const Row &rw) {
        for (int j : rw.need) {
            os << ind << "const float " << vname(rw.i, j) << " = LDT(tb[" << rw.i * pitch + j << "]);\n";
            ++cost;
        }
        for (int j : rw.pr)
            os << ind << "const u64 " << pname(rw.i, j) << " = f2pack(" << vname(rw.i, j) << ", " << vname(rw.i, j + 1) << ");\n";
    };
    const int nrows = (int)rows.size();
    std::map<std::string, long> last_use;
    long clock = 0;
    int next_store = 0;
    auto emit_final = [&](int r) {  // a_rs = A_rs + B_rs (the two column-parity sets)
        const std::string t = store_row ? "const float a" : "a";
        os << ind << t << r << "_0 = f2lo(A" << r << "_0) + B" << r << "_0;\n"
           << ind << t << r << "_1 = f2hi(A" << r << "_0) + f2lo(B" << r << "_1);\n"
           << ind << t << r << "_2 = f2lo(A" << r << "_2) + f2hi(B" << r << "_1);\n"
           << ind << t << r << "_3 = f2hi(A" << r << "_2) + f2lo(B" << r << "_3);\n"
           << ind << t << r << "_4 = f2lo(A" << r << "_4) + f2hi(B" << r << "_3);\n"
           << ind << t << r << "_5 = f2hi(A" << r << "_4) + f2lo(B" << r << "_5);\n"
           << ind << t << r << "_6 = A" << r << "_6 + f2hi(B" << r << "_5);\n";
        if (store_row) store_row(r);
    };
    for (int k = 0; k < nrows; ++k) {
        if (k == 0) {
            loads(rows[0]);
            if (nrows > 1) loads(rows[1]);
        } else if (k + 1 < nrows) {
            loads(rows[k + 1]);
        }
        const Row &rw = rows[k];
        std::vector<std::pair<std::string, std::string>> fm;  // (accumulator, statement)
        for (int q = 0; q < 4; ++q)
            for (auto &p : rw.pairs) {
                const int r = p.first, d = p.second, dw = g.taps[d].dw;
                std::ostringstream st;
                std::string acc;
                if (((dw % 2) + 2) % 2 == 0) {
                    if (q < 3) {
                        const int s = 2 * q;
                        acc = "A" + std::to_string(r) + "_" + std::to_string(s);
                        st << acc << " = ffma2(" << pname(rw.i, dw + s) << ", M" << d << ", " << acc << ");";
                    } else {
                        acc = "A" + std::to_string(r) + "_6";
                        st << acc << " = fmaf(" << vname(rw.i, dw + 6) << ", m" << d << ", " << acc << ");";
                    }
                } else {
                    if (q < 3) {
                        const int s = 2 * q + 1;
                        acc = "B" + std::to_string(r) + "_" + std::to_string(s);
                        st << acc << " = ffma2(" << pname(rw.i, dw + s) << ", M" << d << ", " << acc << ");";
                    } else {
                        acc = "B" + std::to_string(r) + "_0";
                        st << acc << " = fmaf(" << vname(rw.i, dw) << ", m" << d << ", " << acc << ");";
                    }
                }
                fm.push_back({acc, st.str()});
                ++cost;
            }
        emit_lru(os, ind, fm, last_use, clock);
        if (store_row)  // output rows no later footprint row reaches are final: store them now
            while (next_store < R && next_store + g.maxDH <= rw.i) emit_final(next_store++);
    }
    while (next_store < R) emit_final(next_store++);
    return cost;
}


// backward_weight partials of the distinct offsets `ds` with packed FP32, pixel pairs: the
// dy value g(r,s) is the broadcast operand, the pixel pair (p(u), p(u+step)) an aligned
// register pair (every pixel in exactly one pair: two LDS.32, no copies) and the
// accumulator pair holds two offsets one `step` apart; uses with no partner are scalar
// FMAs.  Declares float q<d> for every d in ds.  Returns the issue-cost estimate.
long emit_wgrad_pp(std::ostringstream &os, const Geo &g, const std::vector<int> &ds, int pitch, const char *ind) {
    long cost = 0;
    auto par = [](int v) { return ((v % 2) + 2) % 2; };
    struct Op {
        int lo, hi, r, s, i, j;  // hi < 0: scalar use of tap lo
    };
    std::map<std::pair<int, int>, int> at;  // (dh, dw) -> distinct tap
    for (int d : ds) at[{g.taps[d].dh, g.taps[d].dw}] = d;
    // Packed uses for pair step (sh, sw): pixels are partitioned into register pairs (p(u), p(u + step))
    // -- lo = even column for odd sw, else even row for odd sh -- and tap pairs (d, d + step) take one
    // FFMA2 where the pixel of d is a lo; the rest are scalar FMAs.  Every step is tried and the one
    // with the fewest FMA instructions is kept: near-22.5 deg lines alternate (0,1) and (-1,1) steps
    // between taps and pair best at (-1,3) / (-2,1) / (2,1) / (1,2) (e.g. 1050 -> 980 FMA
    // instructions per lane-item at 22.5 deg, K=31; same 1519 FMAs).
    auto gen_ops = [&](int sh, int sw) {
        auto is_lo = [&](int i, int j) { return (sw % 2) ? par(j) == 0 : par(i) == 0; };
        auto next_of = [&](int d) {
            auto it = at.find({g.taps[d].dh + sh, g.taps[d].dw + sw});
            return it == at.end() ? -1 : it->second;
        };
        std::vector<Op> ops;
        std::vector<int> order(ds);
        auto proj = [&](int d) { return g.taps[d].dh * sh + g.taps[d].dw * sw; };
        std::sort(order.begin(), order.end(), [&](int a, int b) { return proj(a) != proj(b) ? proj(a) < proj(b) : a < b; });
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s) {
                std::set<int> used;
                for (int d : order) {
                    if (used.count(d)) continue;
                    const int i = r + g.taps[d].dh, j = s + g.taps[d].dw;
                    const int nx = next_of(d);
                    if (nx >= 0 && !used.count(nx) && is_lo(i, j)) {
                        ops.push_back({d, nx, r, s, i, j});
                        used.insert(d), used.insert(nx);
                    } else {
                        ops.push_back({d, -1, r, s, i, j});
                        used.insert(d);
                    }
                }
            }
        return ops;
    };
    const std::pair<int, int> cand[] = {{0, 1}, {1, 0}, {-1, 1}, {1, 1}, {-1, 2}, {1, 2}, {-2, 1}, {2, 1},
                                        {-1, 3}, {1, 3}, {-3, 1}, {3, 1}, {-2, 3}, {2, 3}, {-3, 2}, {3, 2}};
    int sh = 0, sw = 1;
    std::vector<Op> ops;
    const int ncand = env_int("O1D_PPSTEPS", 16);  // 4: the round-1 candidate set
    for (int ci = 0; ci < ncand && ci < 16; ++ci) {
        std::vector<Op> o = gen_ops(cand[ci].first, cand[ci].second);
        if (ops.empty() || o.size() < ops.size()) ops.swap(o), sh = cand[ci].first, sw = cand[ci].second;
    }
    // pixel rows in order: bounded pixel liveness
    std::stable_sort(ops.begin(), ops.end(), [&](const Op &a, const Op &b) {
        return std::min(a.i, a.i + (a.hi >= 0 ? sh : 0)) < std::min(b.i, b.i + (b.hi >= 0 ? sh : 0));
    });
    std::set<int> pair_lo, lone;
    for (auto &o : ops) (o.hi >= 0 ? pair_lo : lone).insert(o.lo);
    for (int d : pair_lo) os << ind << "u64 QP" << d << " = 0ull;\n";
    for (int d : lone) os << ind << "float QL" << d << " = 0.f;\n";
    std::set<std::pair<int, int>> loaded, packed;
    auto px = [&](int i, int j) {
        const std::string n = "x" + cn(i) + "_" + cn(j);
        if (loaded.insert({i, j}).second) {
            os << ind << "const float " << n << " = LDT(tb[" << i * pitch + j << "]);\n";
            ++cost;
        }
        return n;
    };
    std::map<std::string, long> last_use;
    long clock = 0;
    std::vector<std::pair<std::string, std::string>> fm;  // the current pixel-row group's FMAs
    int gkey = 1 << 30;
    for (auto &o : ops) {
        const int key = std::min(o.i, o.i + (o.hi >= 0 ? sh : 0));
        if (key != gkey) {  // the previous group's FMAs go out before a new group
            emit_lru(os, ind, fm, last_use, clock);
            fm.clear();
            gkey = key;
        }
        const std::string gn = "g" + std::to_string(o.r) + "_" + std::to_string(o.s);
        if (o.hi >= 0) {
            const std::string a = px(o.i, o.j), b = px(o.i + sh, o.j + sw), pn = "pp" + cn(o.i) + "_" + cn(o.j);
            if (packed.insert({o.i, o.j}).second) os << ind << "const u64 " << pn << " = f2pack(" << a << ", " << b << ");\n";
            const std::string acc = "QP" + std::to_string(o.lo);
            fm.push_back({acc, acc + " = ffma2(" + pn + ", f2pack(" + gn + ", " + gn + "), " + acc + ");"});
        } else {
            const std::string a = px(o.i, o.j);
            const std::string acc = "QL" + std::to_string(o.lo);
            fm.push_back({acc, acc + " = fmaf(" + gn + ", " + a + ", " + acc + ");"});
        }
        ++cost;
    }
    emit_lru(os, ind, fm, last_use, clock);
    std::map<int, int> hi_of;  // tap -> the pair in which it is the high half
    for (auto &o : ops)
        if (o.hi >= 0) hi_of[o.hi] = o.lo;
    for (int d : ds) {
        std::vector<std::string> t;
        if (pair_lo.count(d)) t.push_back("f2lo(QP" + std::to_string(d) + ")");
        if (hi_of.count(d)) t.push_back("f2hi(QP" + std::to_string(hi_of[d]) + ")");
        if (lone.count(d)) t.push_back("QL" + std::to_string(d));
        os << ind << "const float q" << d << " = ";
        if (t.empty()) os << "0.f";
        for (size_t q = 0; q < t.size(); ++q) os << (q ? " + " : "") << t[q];
        os << ";\n";
    }
    return cost;
}

// backward_weight of one table: rounds of <= 32 distinct offsets (register budget), each
// folded into the per-tap sums v[k] += coef * q_d (rotation: v[k] = q_{d(k)}; duplicate taps
// get equal sums, reading R7; bilinear taps the weighted sum of their neighbours, R14).
long emit_wgrad_taps(std::ostringstream &os, const Geo &g, int pitch, int K, const char *ind) {
    long cost = 0;
    const int nd = (int)g.taps.size();
    std::vector<int> all(nd);
    for (int d = 0; d < nd; ++d) all[d] = d;
    std::stable_sort(all.begin(), all.end(), [&](int a, int b) {
        return g.taps[a].dh != g.taps[b].dh ? g.taps[a].dh < g.taps[b].dh : g.taps[a].dw < g.taps[b].dw;
    });
    std::vector<bool> written(K, false);
    const int nr = (nd + 31) / 32;
    for (int rd = 0; rd < nr; ++rd) {
        std::vector<int> ds(all.begin() + (size_t)nd * rd / nr, all.begin() + (size_t)nd * (rd + 1) / nr);
        std::sort(ds.begin(), ds.end());
        os << ind << "{\n";
        const std::string ind2 = std::string(ind) + "  ";
        cost += emit_wgrad_pp(os, g, ds, pitch, ind2.c_str());
        for (int d : ds)
            for (auto &kc : g.taps[d].ks) {
                os << ind2 << "v[" << kc.first << "] " << (written[kc.first] ? "+= " : "= ");
                written[kc.first] = true;
                if (kc.second == 1.0f) os << "q" << d << ";\n";
                else os << flit(kc.second) << " * q" << d << ";\n";
            }
        os << ind << "}\n";
    }
    for (int k = 0; k < K; ++k)
        if (!written[k]) os << ind << "v[" << k << "] = 0.f;\n";
    return cost;
}

// ------------------------------------------------------------------- layout
// ring layout: [zero rows][slot 0][zero rows][slot 1]...[zero rows]; a slot holds the
// image rows of one plane (TMA box from row 0, `pitch` columns); the zero rows between
// slots are the vertical halo of both neighbours (>= the tables' reach, reading R1)
void ring_geom(const std::vector<Geo> &geo, int Hin, int BR, int es, int *pitch, int *zrows, size_t *zb, size_t *tb) {
    *pitch = 0, *zrows = 0;
    for (auto &g : geo) {
        *pitch = std::max(*pitch, g.pitch);
        *zrows = std::max(*zrows, std::max(-g.minDH, R * BR - Hin + g.maxDH) + 1);
    }
    *zb = ((size_t)*zrows * *pitch * es + 127) & ~(size_t)127;
    *tb = ((size_t)Hin * *pitch * es + 127) & ~(size_t)127;
}

bool make_lay(Lay *Lp, int pass, int wpg, const std::vector<Geo> &fwd, const std::vector<Geo> &bwd, int H, int Ho, int Wo,
              int BR, int BC, int es, int P_req, int NB_req) {
    Lay L;
    L.wpg = wpg;
    const bool stencil = pass <= 1, wgrad = pass == 2, fused = pass == 3;
    // rings hold fp32 tiles for every dtype (16-bit planes are widened by the producers)
    ring_geom(pass == 1 ? bwd : fwd, pass == 1 ? Ho : H, BR, 4, &L.pitch, &L.zrows, &L.zb, &L.tb);
    L.hin = pass == 1 ? Ho : H;
    if (fused) {
        ring_geom(bwd, Ho, BR, 4, &L.pitch2, &L.zrows2, &L.zb2, &L.tb2);
        L.hin2 = Ho;
    }
    L.flat = (Wo * es) % 16 != 0;
    if (wgrad) {
        const int vec = 16 / es;
        L.dyp = L.flat ? Wo : (S * BC + vec - 1) & ~(vec - 1);
        L.dyrows = R * BR;
        while (L.flat && (L.dyrows * Wo) % 8 != 0) ++L.dyrows;  // whole 8-element rows of the flat view (zero-filled past P)
        L.db = ((size_t)L.dyp * L.dyrows * es + 127) & ~(size_t)127;
    }
    const size_t budget = (size_t)227 * 1024 - 64;
    const int NSmax = 16;
    // staged 16-bit loads for the stencil passes (measured: forward 50.8 -> 49.1 us at S1 bf16; the
    // weight gradient was slower staged, 52.4 -> 55.0 us, and keeps the per-lane loads)
    bool stage = es != 4 && stencil && env_int("O1D_STAGE", 1) != 0;
    auto fit = [&](int P, int NB) {
        L.P = P, L.NB = NB, L.NS = P * NB;
        if (L.NS > NSmax || P * wpg > 15) return false;
        // more than 4 pairs: 2 producers poll theirs round-robin (4 when they widen 16-bit planes)
        L.NPROD = P <= 4 ? P : es != 4 ? 4 : 2;
        // header: full[16], empty[16], dyempty[8] mbarriers | s_item[16] | weights | bands | dy slots | rings
        L.off_item = 8 * (2 * (size_t)NSmax + 16);  // + stfull[8]
        L.off_w = (L.off_item + 4 * (size_t)NSmax + 15) & ~(size_t)15;
        L.off_stg = (L.off_w + (wgrad ? 0 : (size_t)L.NS * 64 * 4) + 127) & ~(size_t)127;
        L.sb = (stencil || fused) ? (((size_t)4 * R * Wo * es + 127) & ~(size_t)127) : 0;
        L.off_dy = L.off_stg + (size_t)L.ncw() * L.sb;
        L.off_t = (L.off_dy + (size_t)P * L.db + 1023) & ~(size_t)1023;
        L.off_t2 = L.off_t + L.ring1();
        L.off_st = L.off_t2 + L.ring2();
        L.staged = stage && P <= 4;
        L.stb = L.staged ? (((size_t)L.hin * Wo * es + 127) & ~(size_t)127) : 0;
        L.total = L.off_st + (size_t)P * L.stb;
        return L.total + 16 <= budget;
    };
    bool ok = false;
    for (int attempt = 0; attempt < 2 && !ok; ++attempt, stage = false) {
        if (P_req > 0) {
            ok = fit(P_req, std::max(1, NB_req > 0 ? NB_req : 2));
        } else {
            // default: 8 consumer warps (4 pairs at 56x56), two slots per pair; fewer pairs when the
            // slots do not fit (the fused kernel's x + dy slots)
            for (int P = std::max(1, std::min(8, 8 / wpg)); P >= 1 && !ok; --P) ok = fit(P, NB_req > 0 ? NB_req : 2);
        }
        if (ok && stage && L.P < 4 && es != 4) ok = false;  // staging must not cost consumer pairs: retry without
    }
    if (!ok) return false;
    *Lp = L;
    return true;
}

// prologue zeroing of a ring: only what no TMA load ever writes -- the zero-row regions and
// each slot's tail past its box
void emit_zero_ring(std::ostringstream &os, size_t off, size_t zb, size_t tb, size_t box, int NS, int nthreads,
                    const std::string &tid = "tid") {
    const size_t tail = tb - box, stride = zb + tb;
    if (box % 16 || zb % 16 || tail % 16) {
        os << "  for (int i = " << tid << "; i < " << (zb + NS * stride) / 16 << "; i += " << nthreads << ")\n"
           << "    reinterpret_cast<uint4*>(smem + " << off << ")[i] = make_uint4(0u, 0u, 0u, 0u);\n";
        return;
    }
    const size_t per = (zb + tail) / 16;
    os << "  for (int i = " << tid << "; i < " << (NS + 1) * per << "; i += " << nthreads << ") {  // zero rows + slot tails\n"
       << "    const int s = i / " << per << ", k = i - s * " << per << ";\n"
       << "    const int off = s * " << stride << " + (k < " << zb / 16 << " ? k * 16 : " << zb + box << " + (k - " << zb / 16
       << ") * 16);\n"
       << "    if (s < " << NS << " || k < " << zb / 16 << ") *reinterpret_cast<uint4*>(smem + " << off << " + off) = make_uint4(0u, 0u, 0u, 0u);\n"
       << "  }\n";
}

void emit_prologue(std::ostringstream &os, const Lay &L, int pass, int es) {
    const int nthreads = 32 * (L.ncw() + L.NPROD);
    os << "  extern __shared__ __align__(1024) unsigned char smem[];\n"
       << "  u64* const full = reinterpret_cast<u64*>(smem);\n"
       << "  u64* const empty = full + 16;\n"
       << "  u64* const dyempty = full + 32;\n"
       << "  int* const s_item = reinterpret_cast<int*>(smem + " << L.off_item << ");\n"
       << "  float* const wsm = reinterpret_cast<float*>(smem + " << L.off_w << ");\n"
       << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n"
       << "  int trn = 0;\n";
    (void)nthreads;
    (void)es;
    os << "  if (tid == 0) {\n"
       << "    for (int s = 0; s < " << L.NS << "; ++s) { mbar_init(full + s, 32); mbar_init(empty + s, " << L.wpg << "); }\n";
    if (pass == 2) os << "    for (int q = 0; q < " << L.P << "; ++q) mbar_init(dyempty + q, " << L.wpg << ");\n";
    if (L.staged) os << "    for (int q = 0; q < " << L.P << "; ++q) mbar_init(full + 40 + q, 1);   // stfull: raw plane staged\n";
    os << "    fence_mbar_init();\n"
       << "  }\n"
       << "  __syncthreads();\n";
}

// Widening of one 16-bit plane (Hin rows of Win elements, dense, at `src`) into an fp32 slot (`dst`, rows
// `pitch` floats apart) by one warp: lane -> (row wr of a group of RPI rows, 16-byte chunk wc of the row),
// computed once per plane, then one fully unrolled LDS/LDG.128 -> 8 x widen -> 2 x STS.128 per row group
// with immediate offsets (the chunk index division of the round-2 loop cost ~45 instructions per chunk in a
// kernel whose SM sub-partitions are issue-bound).  All loads of the plane are in flight before the first
// store.  The pad columns [Win, pitch) are zeroed once in the consumer prologue (never written here).
void emit_widen(std::ostringstream &os, const std::string &src, bool global, int Hin, int Win, const std::string &dst, int pitch,
                const char *ind) {
    if (Win % 8 != 0) {
        // rows of 4-element units that straddle 16-byte chunks (flat planes, Lay::flat): chunk k holds
        // elements 8k .. 8k+7, each half (4 elements) lies in one row
        const int nch = Hin * Win / 8, iters = (nch + 31) / 32;
        os << ind << "{\n"
           << ind << "  const uint4* const s0 = reinterpret_cast<const uint4*>(" << src << ") + lane;\n"
           << ind << "  float* const d0 = " << dst << ";\n"
           << ind << "  uint4 v[" << iters << "];\n";
        for (int it = 0; it < iters; ++it)
            os << ind << "  if (lane + " << 32 * it << " < " << nch << ") v[" << it << "] = "
               << (global ? "ldg_stream(s0 + " + std::to_string(32 * it) + ", pol)" : "s0[" + std::to_string(32 * it) + "]") << ";\n";
        for (int it = 0; it < iters; ++it)
            os << ind << "  if (lane + " << 32 * it << " < " << nch << ") {\n"
               << ind << "    const int e0 = 8 * (lane + " << 32 * it << "), r0 = e0 / " << Win << ", c0 = e0 - r0 * " << Win << ";\n"
               << ind << "    const int e1 = e0 + 4, r1 = e1 / " << Win << ", c1 = e1 - r1 * " << Win << ";\n"
               << ind << "    *reinterpret_cast<float4*>(d0 + r0 * " << pitch << " + c0) = w4(v[" << it << "].x, v[" << it << "].y);\n"
               << ind << "    *reinterpret_cast<float4*>(d0 + r1 * " << pitch << " + c1) = w4(v[" << it << "].z, v[" << it << "].w);\n"
               << ind << "  }\n";
        os << ind << "}\n";
        return;
    }
    const int cpr = Win / 8, rpi = 32 / cpr, iters = (Hin + rpi - 1) / rpi;
    os << ind << "{\n"
       << ind << "  const int wr = lane / " << cpr << ", wc = lane - wr * " << cpr << ";\n"
       << ind << "  if (wr < " << rpi << ") {\n"
       << ind << "    const uint4* const s0 = reinterpret_cast<const uint4*>(" << src << ") + wr * " << cpr << " + wc;\n"
       << ind << "    float* const d0 = " << dst << " + wr * " << pitch << " + wc * 8;\n"
       << ind << "    uint4 v[" << iters << "];\n";
    for (int it = 0; it < iters; ++it) {
        const bool guard = (it + 1) * rpi > Hin;
        os << ind << "    " << (guard ? "if (wr + " + std::to_string(it * rpi) + " < " + std::to_string(Hin) + ") " : "") << "v[" << it
           << "] = " << (global ? "ldg_stream(s0 + " + std::to_string(it * rpi * cpr) + ", pol)" : "s0[" + std::to_string(it * rpi * cpr) + "]")
           << ";\n";
    }
    for (int it = 0; it < iters; ++it) {
        const bool guard = (it + 1) * rpi > Hin;
        os << ind << "    " << (guard ? "if (wr + " + std::to_string(it * rpi) + " < " + std::to_string(Hin) + ") " : "") << "{ float4* d = reinterpret_cast<float4*>(d0 + "
           << it * rpi * pitch << "); d[0] = w4(v[" << it << "].x, v[" << it << "].y); d[1] = w4(v[" << it << "].z, v[" << it << "].w); }\n";
    }
    os << ind << "  }\n" << ind << "}\n";
}

// Producer warps.  Pair q owns slots q*NB .. q*NB+NB-1; its j-th item goes to slot
// q*NB + j % NB.  One producer per pair (P <= 4) sleeps in try_wait until the pair frees a
// slot; with more pairs two producers poll theirs round-robin so a slow pair never holds up
// another pair's loads.  After the scheduler runs dry every pair gets an end marker (-1).
void emit_producer_staged(std::ostringstream &os, const Ctx &x, const Lay &L, int pass, int es);

void emit_producer(std::ostringstream &os, const Ctx &x, const Lay &L, int pass, int es) {
    if (L.staged) {
        emit_producer_staged(os, x, L, pass, es);
        return;
    }
    const int NB = L.NB, P = L.P;
    const bool wgrad = pass == 2, fused = pass == 3, cvt = es != 4;
    // TMA bytes the slot's full barrier expects (the widened 16-bit rings arrive by STS)
    const size_t bytes = (cvt ? 0 : (size_t)L.hin * L.pitch * 4) + (wgrad ? (size_t)L.dyp * L.dyrows * es : 0) +
                         (fused && !cvt ? (size_t)L.hin2 * L.pitch2 * 4 : 0);
    const int PQ = (P + L.NPROD - 1) / L.NPROD;  // pairs per producer warp
    // single-item scheduler atomics in flight (0: claim when a slot frees)
    const int PREF = std::max(0, env_int("O1D_PREF", 0)), PA = std::max(1, PREF);
    os << "  if (warp < " << L.NPROD << ") {\n"
       << "    const int pw = warp;\n"
       << "    int tcur = 0, tried = 0;\n"
       << "    const u64 pol = policy_evict_first();\n"
       << "    const int nper = p.nlen > 0 ? p.nlen : p.N;\n"
       << "    unsigned lo = 0, pf[" << PA << "];   // the first P_NB items come in one batch (fills the ring without round trips)\n"
       << "    // the scheduler counters of this launch slot were last touched 64 launches ago: the\n"
       << "    // first atomics run before griddepcontrol.wait (only x / dy / w may come from the predecessor)\n"
       << "    if (lane == 0) {\n"
       << "      trace_ev(p.trace, 0, -1, trn);\n"
       << "      tcur = HOME[smid() % NHOME];\n"
       << "      lo = atomicAdd(p.sched + tcur * CS, " << PQ * NB << "u);\n"
       << "#pragma unroll\n"
       << "      for (int k = 0; k < " << PREF << "; ++k) pf[k] = atomicAdd(p.sched + tcur * CS, 1u);\n"
       << "      (void)pf;\n"
       << "    }\n"
       << "    if (!p.nowait) pdl_wait();\n"
       << "    int jq[" << PQ << "];   // items issued per served pair (-1: end marker sent)\n"
       << "    for (int qi = 0; qi < " << PQ << "; ++qi) jq[qi] = pw + qi * " << L.NPROD << " < " << P << " ? 0 : -1;\n"
       << "    int bat = 0, live = (" << P + L.NPROD - 1 << " - pw) / " << L.NPROD << ", idle = 0;\n"
       << "    while (live > 0) {\n"
       << "      bool any = false;\n"
       << "#pragma unroll 1\n"
       << "      for (int qi = 0; qi < " << PQ << "; ++qi) {\n"
       << "        const int q = pw + qi * " << L.NPROD << ";\n"
       << "        const int j = jq[qi];\n"
       << "        if (j < 0) continue;\n"
       << "        const int s = q * " << NB << " + j % " << NB << ";\n"
       << (PQ == 1 ? "        if (j >= " + std::to_string(NB) + ") mbar_wait(empty + s, ((j / " + std::to_string(NB) + ") & 1) ^ 1);\n"
                   : "        if (j >= " + std::to_string(NB) + " && !mbar_test(empty + s, ((j / " + std::to_string(NB) +
                         ") & 1) ^ 1)) continue;   // slot still in use\n");
    if (wgrad && PQ != 1)  // the pair's dy slot is free once it copied the dy block of its previous item
        os << "        if (j >= 1 && !mbar_test(dyempty + q, ((j - 1) & 1))) continue;\n";
    os << "        int item = -1;\n"
       << "        if (lane == 0) {\n"
       << "          if (bat < " << PQ * NB << " && lo + bat < (unsigned)(nch_of(tcur) * nper)) {\n"
       << "            item = (tcur << 22) | (int)(lo + bat++);\n"
       << "          } else {\n"
       << "            bat = " << PQ * NB << ";   // the batch is exhausted: every later item comes from pf\n"
       // (tcur < 0: every table is exhausted -- no atomic on a counter before the slot's array)
       << (PREF == 0 ? "            item = tcur >= 0 ? sched_resolve(p.sched, tcur, atomicAdd(p.sched + tcur * CS, 1u), tried, nper) : -1;\n"
                       : "            const unsigned v = pf[0];\n"
                         "#pragma unroll\n"
                         "            for (int k = 0; k + 1 < " + std::to_string(PREF) + "; ++k) pf[k] = pf[k + 1];\n"
                         "            const int t0 = tcur;\n"
                         "            item = sched_resolve(p.sched, tcur, v, tried, nper);\n"
                         "            if (tcur != t0) {   // moved to another table: the prefetched indices belong to the old one\n"
                         "#pragma unroll\n"
                         "              for (int k = 0; k < " + std::to_string(PREF) + "; ++k) pf[k] = tcur >= 0 ? atomicAdd(p.sched + tcur * CS, 1u) : 0xffffffffu;\n"
                         "            } else {\n"
                         "              pf[" + std::to_string(PREF - 1) + "] = tcur >= 0 ? atomicAdd(p.sched + tcur * CS, 1u) : 0xffffffffu;\n"
                         "            }\n")
       << "          }\n"
       << "        }\n"
       << "        item = __shfl_sync(0xffffffffu, item, 0);\n"
       << "        int t2 = 0, c2 = 0, n2 = 0;\n"
       << "        if (item >= 0) item_cn(item, t2, c2, n2, p.n0);\n"
       << "        if (lane == 0) {\n"
       << "          s_item[s] = item;\n"
       << "          if (item >= 0) {\n"
       << "            trace_ev(p.trace, 1, item, trn);\n";
    if (bytes) os << "            mbar_expect_tx(full + s, " << bytes << "u);\n";
    if (!cvt) os << "            tma_load(smem + " << L.off_t + L.zb << " + s * " << L.zb + L.tb << ", &p.in_map, 0, 0, c2, n2, full + s, pol);\n";
    if (wgrad) {
        // one producer per pair: the x plane goes out as soon as its slot is free; the dy plane
        // waits (lane 0 only) until the pair has copied its previous dy block to registers
        if (PQ == 1) os << "            if (j >= 1) mbar_wait(dyempty + q, ((j - 1) & 1));\n";
        os << "            tma_load(smem + " << L.off_dy << " + q * " << L.db << ", &p.out_map, 0, 0, c2, n2, full + s, pol);\n";
    }
    if (fused && !cvt)
        os << "            tma_load(smem + " << L.off_t2 + L.zb2 << " + s * " << L.zb2 + L.tb2 << ", &p.aux_map, 0, 0, c2, n2, full + s, pol);\n";
    os << "          }\n"
       << "        }\n";
    if (cvt) {
        // 16-bit planes: every lane loads 16-byte chunks (8 elements) of the plane, all loads in
        // flight before the first use, widens them to fp32 and stores them into the slot's
        // image columns; the arrive below releases them to the consumers (mbarrier release)
        auto widen = [&](const char *srcp, int Hin, int Win, size_t slot_off, size_t slot_stride, int pitch) {
            os << "        if (item >= 0)\n";
            emit_widen(os, "reinterpret_cast<const act_t*>(" + std::string(srcp) + ") + ((u64)n2 * " + std::to_string(x.C) + " + c2) * " +
                               std::to_string((long)Hin * Win),
                       true, Hin, Win, "reinterpret_cast<float*>(smem + " + std::to_string(slot_off) + " + s * " + std::to_string(slot_stride) + ")",
                       pitch, "        ");
        };
        widen("p.cvt1", L.hin, pass == 1 ? x.Wo : x.Wi, L.off_t + L.zb, L.zb + L.tb, L.pitch);
        if (fused) widen("p.cvt2", L.hin2, x.Wo, L.off_t2 + L.zb2, L.zb2 + L.tb2, L.pitch2);
    }
    if (!wgrad)
        os << "        if (item >= 0)\n"
           << "          for (int k = lane; k < " << x.K << "; k += 32) wsm[s * 64 + k] = __ldg(p.w + c2 * " << x.K << " + k);\n";
    os << "        mbar_arrive(full + s);   // 32 producer arrivals (+ the bytes) complete the phase\n"
       << "        if (item < 0) { jq[qi] = -1; --live; } else { jq[qi] = j + 1; }\n"
       << "        any = true;\n"
       << "      }\n"
       << "      if (!any) { if (++idle > 1) __nanosleep(256); } else idle = 0;\n"
       << "    }\n"
       << "    // a kernel that skipped griddepcontrol.wait (o1d_step) still completes only after its\n"
       << "    // predecessor: whatever waits for this grid then also sees the predecessor done\n"
       << "    if (p.nowait) pdl_wait();\n"
       << "    pdl_trigger();\n"
       << "    if (lane == 0) sched_exit(p.sched, " << L.NPROD << "u);\n"
       << "    return;\n"
       << "  }\n";
}

// consumer set-up after the producer branch: zeroing of what no producer writes, then the warp's
// pair / band / lane block
void emit_consumer_prologue(std::ostringstream &os, const Ctx &x, const Lay &L, int pass) {
    const bool fused = pass == 3;
    // the warps of a pair are P warp ids apart: they sit on the same SM sub-partition as
    // their producer and run the same code a few instructions apart (shared L0 I-cache)
    os << "  // consumers zero what no producer ever writes (the zero rows between slots and the slot\n"
       << "  // tails) while the producers' first loads are in flight; the regions are disjoint\n";
    {
        const int nc = 32 * L.ncw();
        emit_zero_ring(os, L.off_t, L.zb, L.tb, (size_t)L.hin * L.pitch * 4, L.NS, nc, "(tid - " + std::to_string(32 * L.NPROD) + ")");
        auto zero_pad = [&](size_t off, size_t zb, size_t tb, int hin, int pitch, int win) {
            // columns [W, pitch) of every slot row: the widening producers write only [0, W)
            const int ppr = (pitch - win) / 4;
            os << "  for (int i = tid - " << 32 * L.NPROD << "; i < " << L.NS * hin * ppr << "; i += " << nc << ") {\n"
               << "    const int s = i / " << hin * ppr << ", k = i - s * " << hin * ppr << ", r = k / " << ppr << ", cc = k - r * " << ppr << ";\n"
               << "    *reinterpret_cast<float4*>(smem + " << off + zb << " + s * " << zb + tb << " + (r * " << pitch << " + "
               << win << " + cc * 4) * 4) = make_float4(0.f, 0.f, 0.f, 0.f);\n"
               << "  }\n";
        };
        if (x.act != O1D_F32) {  // 16-bit planes are widened into the fp32 rings (staged or per lane)
            zero_pad(L.off_t, L.zb, L.tb, L.hin, L.pitch, pass == 0 || pass == 2 || fused ? x.Wi : x.Wo);
            if (fused) zero_pad(L.off_t2, L.zb2, L.tb2, L.hin2, L.pitch2, x.Wo);
        }
        if (fused) emit_zero_ring(os, L.off_t2, L.zb2, L.tb2, (size_t)L.hin2 * L.pitch2 * 4, L.NS, nc, "(tid - " + std::to_string(32 * L.NPROD) + ")");
        os << "  asm volatile(\"bar.sync 1, " << nc << ";\" ::: \"memory\");\n";
    }
    os << "  const int cw = warp - " << L.NPROD << ", q = cw % " << L.P << ", wg = cw / " << L.P << ";\n"
       << "  int bc = lane & 7, br = (lane >> 3) + 4 * wg;\n"
       << "  const bool active = bc < " << x.BC << " && br < " << x.BR << ";\n"
       << "  if (!active) { bc = 0; br = 0; }\n"
       << "  const int row0 = " << 4 * R << " * wg;   // first output row of this warp's band\n";
}


// 16-bit planes, staged: the pair's producer (one per pair) keeps one raw plane in flight in its
// staging buffer (one TMA box, async), widens the previous one into the pair's fp32 slot
// (LDS.128 -> 2 x STS.128) and claims + issues the next plane right after, so the load latency
// overlaps the pair's tap loop instead of stalling the producer on its own loads.
void emit_producer_staged(std::ostringstream &os, const Ctx &x, const Lay &L, int pass, int es) {
    const int NB = L.NB, P = L.P;
    const bool wgrad = pass == 2;
    const int Win = x.Wo;  // stride 1: input width = output width
    const size_t raw = (size_t)L.hin * Win * es;
    (void)es;
    const int PREF = std::max(0, std::min(2, env_int("O1D_PREF", 0))), PA = std::max(1, PREF);  // see emit_producer
    auto claim = [&](const char *var) {
        os << "      {\n"
           << "        int it_ = -1;\n"
           << "        if (lane == 0) {\n"
           << "          if (bat < " << NB << " && lo + bat < (unsigned)(nch_of(tcur) * nper)) {\n"
           << "            it_ = (tcur << 22) | (int)(lo + bat++);\n"
           << "          } else {\n"
           << "            bat = " << NB << ";\n";
        if (PREF == 0) {
            os << "            it_ = tcur >= 0 ? sched_resolve(p.sched, tcur, atomicAdd(p.sched + tcur * CS, 1u), tried, nper) : -1;\n";
        } else {
            os << "            const unsigned v = pf[0];\n"
               << "            for (int k = 0; k + 1 < " << PREF << "; ++k) pf[k] = pf[k + 1];\n"
               << "            const int t0 = tcur;\n"
               << "            it_ = sched_resolve(p.sched, tcur, v, tried, nper);\n"
               << "            if (tcur != t0) {\n"
               << "              for (int k = 0; k < " << PREF << "; ++k) pf[k] = tcur >= 0 ? atomicAdd(p.sched + tcur * CS, 1u) : 0xffffffffu;\n"
               << "            } else {\n"
               << "              pf[" << PREF - 1 << "] = tcur >= 0 ? atomicAdd(p.sched + tcur * CS, 1u) : 0xffffffffu;\n"
               << "            }\n";
        }
        os << "          }\n"
           << "        }\n"
           << "        " << var << " = __shfl_sync(0xffffffffu, it_, 0);\n"
           << "      }\n";
    };
    auto issue = [&](const char *var) {  // lane 0: raw plane of item `var` into the staging buffer
        os << "      if (lane == 0 && " << var << " >= 0) {\n"
           << "        int t3, c3, n3; item_cn(" << var << ", t3, c3, n3, p.n0);\n"
           << "        asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\" :: \"r\"(sa(stfull)), \"r\"(" << raw << "u) : \"memory\");\n"
           << "        tma_load(stage, &p.in_map, 0, 0, c3, n3, stfull, pol);\n"
           << "      }\n";
    };
    os << "  if (warp < " << L.NPROD << ") {\n"
       << "    const int q = warp;\n"
       << "    int tcur = 0, tried = 0, bat = 0;\n"
       << "    const u64 pol = policy_evict_first();\n"
       << "    const int nper = p.nlen > 0 ? p.nlen : p.N;\n"
       << "    u64* const stfull = full + 40 + q;\n"
       << "    unsigned char* const stage = smem + " << L.off_st << " + q * " << L.stb << ";\n"
       << "    unsigned lo = 0, pf[" << PA << "];\n"
       << "    if (lane == 0) {\n"
       << "      trace_ev(p.trace, 0, -1, trn);\n"
       << "      tcur = HOME[smid() % NHOME];\n"
       << "      lo = atomicAdd(p.sched + tcur * CS, " << NB << "u);\n"
       << "      for (int k = 0; k < " << PREF << "; ++k) pf[k] = atomicAdd(p.sched + tcur * CS, 1u);\n"
       << "      (void)pf;\n"
       << "    }\n"
       << "    if (!p.nowait) pdl_wait();\n"
       << "    int nxt;\n";
    claim("nxt");
    issue("nxt");
    os << "    for (int j = 0;; ++j) {\n"
       << "      const int s = q * " << NB << " + j % " << NB << ";\n"
       << "      const int item = nxt;\n"
       << "      if (j >= " << NB << ") mbar_wait(empty + s, ((j / " << NB << ") & 1) ^ 1);\n";
    if (wgrad) os << "      if (j >= 1) mbar_wait(dyempty + q, ((j - 1) & 1));\n";
    os << "      int t2 = 0, c2 = 0, n2 = 0;\n"
       << "      if (item >= 0) item_cn(item, t2, c2, n2, p.n0);\n"
       << "      if (lane == 0) {\n"
       << "        s_item[s] = item;\n";
    if (wgrad)
        os << "        if (item >= 0) {\n"
           << "          mbar_expect_tx(full + s, " << (size_t)L.dyp * L.dyrows * es << "u);\n"
           << "          tma_load(smem + " << L.off_dy << " + q * " << L.db << ", &p.out_map, 0, 0, c2, n2, full + s, pol);\n"
           << "        }\n";
    os << "      }\n"
       << "      if (item >= 0) {\n"
       << "        mbar_wait(stfull, j & 1);\n"
       ;
    emit_widen(os, "stage", false, L.hin, Win, "reinterpret_cast<float*>(smem + " + std::to_string(L.off_t + L.zb) + " + s * " + std::to_string(L.zb + L.tb) + ")",
               L.pitch, "        ");
    if (!wgrad)
        os << "        for (int k = lane; k < " << x.K << "; k += 32) wsm[s * 64 + k] = __ldg(p.w + c2 * " << x.K << " + k);\n";
    os << "      }\n"
       << "      __syncwarp();\n"
       << "      asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");   // staging reads before the next TMA write\n"
       << "      if (item >= 0) {\n";
    claim("nxt");
    issue("nxt");
    os << "      } else {\n"
       << "        nxt = -1;\n"
       << "      }\n"
       << "      mbar_arrive(full + s);\n"
       << "      if (item < 0) break;\n"
       << "    }\n"
       << "    if (p.nowait) pdl_wait();\n"
       << "    pdl_trigger();\n"
       << "    if (lane == 0) sched_exit(p.sched, " << L.NPROD << "u);\n"
       << "    return;\n"
       << "  }\n";
    (void)P;
}

void emit_loop_head(std::ostringstream &os, const Lay &L) {
    os << "  for (int it = 0;; ++it) {   // it: this pair's item index\n"
       << "    const int s = q * " << L.NB << " + it % " << L.NB << ";\n"
       << "    if (lane == 0) trace_ev(p.trace, 2, it, trn);\n"
       << "    mbar_wait(full + s, (it / " << L.NB << ") & 1);\n"
       << "    const int item = s_item[s];\n"
       << "    if (lane == 0) trace_ev(p.trace, 3, item, trn);\n"
       << "    if (item < 0) break;\n"
       << "    int t, c, n; item_cn(item, t, c, n, p.n0);\n";
}

// early stores (Lay::early): before the tap loop, wait until the previous band store has read the
// staging band and point `sto` at this lane's block in it; the tap code stores each output row as
// soon as it is final; emit_band_tail then publishes the band with one TMA store
void emit_band_head(std::ostringstream &os, const Ctx &x, const char *ind) {
    os << ind << "if (lane == 0) asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\");  // previous band store has read stg\n"
       << ind << "__syncwarp();\n"
       << ind << "act_t* const sto = reinterpret_cast<act_t*>(stg) + (" << R << " * br - row0) * " << x.Wo << " + " << S << " * bc;\n";
}
void emit_band_tail(std::ostringstream &os, const Ctx &x, const char *ind) {
    os << ind << "asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
       << ind << "__syncwarp();\n"
       << ind << "if (lane == 0 && row0 < " << x.Ho << ") tma_store_band(&p.out_map, stg, " << (x.flat ? "row0 * " + std::to_string(x.Wo / 2) + " / 4" : "row0")
       << ", c, n, policy_evict_first());\n";
}

// stencil outputs: registers -> this warp's staging band -> TMA bulk store (evict-first)
void emit_band_store(std::ostringstream &os, const Ctx &x, const Lay &L) {
    const bool ragged = (R * x.BR != x.Ho) || (S * x.BC != x.Wo);
    os << "    if (lane == 0) asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\");  // previous band store has read stg\n"
       << "    __syncwarp();\n"
       << "    if (active) {\n"
       << "      act_t* const sto = reinterpret_cast<act_t*>(stg) + (" << R << " * br - row0) * " << x.Wo << " + " << S << " * bc;\n";
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) {
            os << "      ";
            if (ragged) os << "if (" << R << " * br + " << r << " < " << x.Ho << " && " << S << " * bc + " << s << " < " << x.Wo << ") ";
            os << "sto[" << r * x.Wo + s << "] = to_act(a" << r << "_" << s << ");\n";
        }
    os << "    }\n"
       << "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
       << "    __syncwarp();\n"
       << "    if (lane == 0 && row0 < " << x.Ho << ") tma_store_band(&p.out_map, stg, " << (x.flat ? "row0 * " + std::to_string(x.Wo / 2) + " / 4" : "row0")
       << ", c, n, policy_evict_first());\n";
}

void emit_wgrad_write(std::ostringstream &os, const Ctx &x, const Lay &L, int NV) {
    os << "    {\n"
       << "      const float part = reduce_scatter<" << NV << ">(v, lane);\n"
       << "      if (lane < " << x.K << ") p.ws[((u64)(c * p.N + n) * " << L.wpg << " + wg) * " << x.K << " + lane] = part;\n"
       << "    }\n";
}

void emit_finalize(std::ostringstream &os, const Ctx &x, int wpg) {
    // dW[c][k] = sum over (n, band) of the partials, f64, fixed order.  One CTA per channel:
    // thread (j, k) sums entries j, j+8, ... of column k (all loads in flight), then a
    // fixed-order f64 sum over j.
    os << "extern \"C\" __global__ void __launch_bounds__(256) o1d_wgrad_finalize(const float* __restrict__ ws, float* __restrict__ dW, int N) {\n"
       << "  __shared__ double part[8][64];\n"
       << "  pdl_wait();\n"
       << "  pdl_trigger();   // the next kernel may start its set-up (it waits for our completion)\n"
       << "  const int c = blockIdx.x, j = threadIdx.x >> 5 /* 0..7 */, lane = threadIdx.x & 31;\n"
       << "  const int NE = N * " << wpg << ";\n"
       << "  const float* base = ws + (u64)c * NE * " << x.K << ";\n"
       << "  for (int k = lane; k < " << x.K << "; k += 32) {\n"
       << "    double s = 0.0;\n"
       << "#pragma unroll 16\n"
       << "    for (int e = j; e < NE; e += 8) s += (double)__ldcg(base + (u64)e * " << x.K << " + k);\n"
       << "    part[j][k] = s;\n"
       << "  }\n"
       << "  __syncthreads();\n"
       << "  if (threadIdx.x < " << x.K << ") {\n"
       << "    double s = 0.0;\n"
       << "    for (int q = 0; q < 8; ++q) s += part[q][threadIdx.x];\n"
       << "    dW[c * " << x.K << " + threadIdx.x] = (float)s;\n"
       << "  }\n"
       << "}\n";
}

int nv_of(int K) {
    int NV = 1;
    while (NV < K) NV *= 2;
    return NV;
}

// Generated kernel of one pass.  The per-table case bodies are emitted first (their issue
// costs set the SM placement, see home_tables), then assembled.
struct Cases {
    std::vector<std::string> body;   // per table
    std::vector<long> cost;
};

// stores of one final output row into this warp's staging band (`sto`, see emit_band_head)
void emit_store_row(std::ostringstream &os, const Ctx &x, int r, const char *ind) {
    const bool ragged = (R * x.BR != x.Ho) || (S * x.BC != x.Wo);
    os << ind << "if (active" << (R * x.BR != x.Ho ? " && " + std::to_string(R) + " * br + " + std::to_string(r) + " < " + std::to_string(x.Ho) : "")
       << ") {\n";
    for (int s = 0; s < S; ++s) {
        os << ind << "  ";
        if (ragged && S * x.BC != x.Wo) os << "if (" << S << " * bc + " << s << " < " << x.Wo << ") ";
        os << "sto[" << r * x.Wo + s << "] = to_act(a" << r << "_" << s << ");\n";
    }
    os << ind << "}\n";
}

Cases stencil_cases(const std::vector<Geo> &geo, int pitch, const Ctx *early) {
    Cases cs;
    for (size_t t = 0; t < geo.size(); ++t) {
        std::ostringstream os;
        std::function<void(int)> st;
        if (early) st = [&os, early](int r) { emit_store_row(os, *early, r, "      "); };
        const long c = emit_stencil_taps(os, geo[t], pitch, "      ", st);
        cs.body.push_back(os.str());
        cs.cost.push_back(c);
    }
    return cs;
}

Cases wgrad_cases(const std::vector<Geo> &geo, int pitch, int K) {
    Cases cs;
    for (size_t t = 0; t < geo.size(); ++t) {
        std::ostringstream os;
        const long c = emit_wgrad_taps(os, geo[t], pitch, K, "      ");
        cs.body.push_back(os.str());
        cs.cost.push_back(c);
    }
    return cs;
}

void emit_switch(std::ostringstream &os, const Cases &cs, const std::string &tb_base, int pitch, const std::string &elem) {
    os << "    switch (t) {\n";
    for (size_t t = 0; t < cs.body.size(); ++t)
        os << "    case " << t << ": {\n"
           << "      const " << elem << "* tb = " << tb_base << " + (" << R << " * br) * " << pitch << " + " << S << " * bc;\n"
           << cs.body[t] << "      break;\n    }\n";
    os << "    }\n";
}

std::string gen_pass(const Ctx &x, const Lay &L, int pass, const Cases &st, const Cases &wg) {
    std::ostringstream os;
    emit_header(os, x);
    const int es = x.act == O1D_F32 ? 4 : 2;
    const int nthreads = 32 * (L.ncw() + L.NPROD);
    const int NV = nv_of(x.K);
    const char *name = pass <= 1 ? "o1d_stencil" : pass == 2 ? "o1d_wgrad" : "o1d_bwd_fused";
    if (pass == 3) {
        // phase 1: weight-gradient partials of one item (dy block from ring 2, pixels from ring 1)
        os << "__device__ __noinline__ void fused_wgrad(const Params& p, const tile_t* xt, const tile_t* dyt, int t, int c, int n,\n"
           << "                                         int wg, int lane, bool active, int bc, int br) {\n"
           << "  const tile_t* const dys = dyt + (" << R << " * br) * " << L.pitch2 << " + " << S << " * bc;\n";
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s)
                os << "  const float g" << r << "_" << s << " = active ? LDT(dys[" << r * L.pitch2 + s << "]) : 0.f;\n";
        os << "  float v[" << NV << "];   // v[k], k < K: assigned by the table's case\n"
           << "#pragma unroll\n"
           << "  for (int k = " << x.K << "; k < " << NV << "; ++k) v[k] = 0.f;\n"
           << "  {\n";
        emit_switch(os, wg, "xt", L.pitch, "tile_t");
        emit_wgrad_write(os, x, L, NV);
        os << "  }\n}\n";
        // phase 2: backward_input band of the item from the dy tile, slot release, band store
        os << "__device__ __noinline__ void fused_dx(const Params& p, const tile_t* dyt, const float* wv, unsigned char* stg,\n"
           << "                                      u64* empty_s, int t, int c, int n, int row0, int lane, bool active,\n"
           << "                                      int bc, int br) {\n";
        if (L.early) emit_band_head(os, x, "  ");
        else
            for (int r = 0; r < R; ++r)
                for (int s = 0; s < S; ++s) os << "  float a" << r << "_" << s << ";\n";
        os << "  {\n";
        emit_switch(os, st, "dyt", L.pitch2, "tile_t");
        os << "    __syncwarp();\n"
           << "    if (lane == 0) mbar_arrive(empty_s);   // x + dy slot released\n";
        if (L.early) emit_band_tail(os, x, "    ");
        else emit_band_store(os, x, L);
        os << "  }\n}\n";
    }
    os << "extern \"C\" __global__ void __launch_bounds__(" << nthreads << ", 1) " << name << "(const __grid_constant__ Params p) {\n";
    emit_prologue(os, L, pass, es);
    emit_producer(os, x, L, pass, es);
    emit_consumer_prologue(os, x, L, pass);
    os << "  // -------------------------------------------------------------- consumers\n";
    const std::string ring1 = "reinterpret_cast<const tile_t*>(smem + " + std::to_string(L.off_t + L.zb) + " + s * " +
                              std::to_string(L.zb + L.tb) + ")";
    if (pass != 2) os << "  unsigned char* const stg = smem + " << L.off_stg << " + cw * " << L.sb << ";   // this warp's output band\n";
    if (pass == 2)
        os << "  const act_t* const dys = reinterpret_cast<const act_t*>(smem + " << L.off_dy << " + q * " << L.db << ") + (" << R
           << " * br) * " << L.dyp << " + " << S << " * bc;\n";
    emit_loop_head(os, L);
    if (pass <= 1) {
        os << "    const float* wv = wsm + s * 64;\n";
        if (L.early) emit_band_head(os, x, "    ");
        else
            for (int r = 0; r < R; ++r)
                for (int s = 0; s < S; ++s) os << "    float a" << r << "_" << s << ";\n";
        emit_switch(os, st, ring1, L.pitch, "tile_t");
        os << "    __syncwarp();\n"
           << "    if (lane == 0) { mbar_arrive(empty + s); trace_ev(p.trace, 4, item, trn); }   // done with the slot\n";
        if (L.early) emit_band_tail(os, x, "    ");
        else emit_band_store(os, x, L);
    } else if (pass == 2) {
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s)
                os << "    const float g" << r << "_" << s << " = active"
                   // flat dy rows are dense: columns past the plane (ragged last block) belong to the next row
                   << (L.flat && S * x.BC > x.Wo ? " && " + std::to_string(S) + " * bc + " + std::to_string(s) + " < " + std::to_string(x.Wo) : std::string())
                   << " ? LD(dys[" << r * L.dyp + s << "]) : 0.f;\n";
        os << "    __syncwarp();\n"
           << "    if (lane == 0) mbar_arrive(dyempty + q);   // dy block in registers: the pair's dy slot is free\n"
           << "    float v[" << NV << "];   // v[k], k < K: assigned by the table's case\n"
           << "#pragma unroll\n"
           << "    for (int k = " << x.K << "; k < " << NV << "; ++k) v[k] = 0.f;\n";
        emit_switch(os, wg, ring1, L.pitch, "tile_t");
        os << "    __syncwarp();\n"
           << "    if (lane == 0) { mbar_arrive(empty + s); trace_ev(p.trace, 4, item, trn); }  // x slot released\n";
        emit_wgrad_write(os, x, L, NV);
    } else {
        // fused backward: the weight-gradient partials (x ring 1, dy ring 2), then the
        // backward_input band from the same dy tile; the slot is released after both.  The two
        // phases are separate non-inlined functions (they share no live registers; one function
        // holding both switches took ptxas ~10x longer to compile)
        const std::string ring2 = "reinterpret_cast<const tile_t*>(smem + " + std::to_string(L.off_t2 + L.zb2) + " + s * " +
                                  std::to_string(L.zb2 + L.tb2) + ")";
        os << "    fused_wgrad(p, " << ring1 << ", " << ring2 << ", t, c, n, wg, lane, active, bc, br);\n"
           << "    fused_dx(p, " << ring2 << ", wsm + s * 64, stg, empty + s, t, c, n, row0, lane, active, bc, br);\n";
    }
    os << "    if (lane == 0) trace_ev(p.trace, 5, item, trn);\n"
       << "  }\n";
    if (pass != 2) os << "  if (lane == 0) asm volatile(\"cp.async.bulk.wait_group 0;\" ::: \"memory\");\n";
    os << "}\n";
    if (pass >= 2) emit_finalize(os, x, L.wpg);
    return os.str();
}

// ------------------------------------------------------------- small planes
// Planes of at most 14 x 14 (the K-sweep's 14 x 14, ConvNeXt stage 3) do not fit the
// warp-per-band kernels (a 7x7-block lane map covers 56 x 28 outputs) and their rows are not
// TMA-legal (14 floats = 56 B).  Here a unit of work is 32 planes of one channel (batch samples
// 32g .. 32g+31): lane j owns plane j, and a "quad" of BRs x BCs warps owns the item, warp bp
// computing the 7x7 block at block position bp of all 32 planes.  The block position is a
// compile-time constant of the warp's code, so every (output, tap) pair that falls outside the
// image is dropped at compile time -- no zero halo in shared memory and exactly the in-bounds
// FMAs (SURVEY 8(a1) pruning).  Shared memory holds the 32 planes unit-major: unit u (pixels
// 2u, 2u+1 of the row-major plane) of plane j at [(u * 33 + j) * UB], so the 32 lanes reading the
// same unit of their planes hit 32 (fp32: 16 x 8-byte) distinct banks, and a producer lane
// copying unit u of one plane writes them with one cp.async (LDGSTS) per unit: no conversion
// pass, no registers, completion tracked by the slot's mbarrier.
constexpr int kSmallLanes = 33;  // unit stride in a slot: 32 planes + 1 (bank skew)

// unit loads / stores of the unit-major slots (fp32: float2, 16-bit: packed u32)
void emit_small_header(std::ostringstream &os, int act, int UPu) {
    os << "__device__ __forceinline__ void cp_async_unit(void* dst, const void* src, u64 pol) {\n";
    if (UPu == 1 && act != O1D_F32)
        os << "  *reinterpret_cast<unsigned short*>(dst) = __ldg(reinterpret_cast<const unsigned short*>(src)); (void)pol;\n";
    else if (UPu == 1 || act != O1D_F32)
        os << "  asm volatile(\"cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;\" :: \"r\"(sa(dst)), \"l\"(src), \"l\"(pol) : \"memory\");\n";
    else
        os << "  asm volatile(\"cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\" :: \"r\"(sa(dst)), \"l\"(src), \"l\"(pol) : \"memory\");\n";
    os << "}\n"
       << "__device__ __forceinline__ void cp_async_w(void* dst, const void* src) {\n"
       << "  asm volatile(\"cp.async.ca.shared.global [%0], [%1], 4;\" :: \"r\"(sa(dst)), \"l\"(src) : \"memory\");\n"
       << "}\n"
       << "__device__ __forceinline__ void cp_async_arrive(u64* b) {\n"
       << "  asm volatile(\"cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\" :: \"r\"(sa(b)) : \"memory\");\n"
       << "}\n";
    if (UPu == 1 && act == O1D_F32)
        os << "typedef float unit_t;\n"
              "__device__ __forceinline__ float ulo(unit_t v) { return v; }\n"
              "__device__ __forceinline__ float uhi(unit_t v) { return 0.f; }\n";
    else if (UPu == 1)
        os << "typedef unsigned short unit_t;\n"
              "__device__ __forceinline__ float ulo(unit_t v) { return LD(v); }\n"
              "__device__ __forceinline__ float uhi(unit_t v) { return 0.f; }\n";
    else if (act == O1D_F32)
        os << "typedef float2 unit_t;\n"
              "__device__ __forceinline__ float ulo(unit_t v) { return v.x; }\n"
              "__device__ __forceinline__ float uhi(unit_t v) { return v.y; }\n"
              "__device__ __forceinline__ unit_t upack(float lo, float hi) { return make_float2(lo, hi); }\n";
    else if (act == O1D_BF16)
        os << "typedef unsigned unit_t;\n"
              "__device__ __forceinline__ float ulo(unit_t v) { return __uint_as_float(v << 16); }\n"
              "__device__ __forceinline__ float uhi(unit_t v) { return __uint_as_float(v & 0xffff0000u); }\n"
              "__device__ __forceinline__ unit_t upack(float lo, float hi) { unit_t r; asm(\"cvt.rn.bf16x2.f32 %0, %1, %2;\" : \"=r\"(r) : \"f\"(hi), \"f\"(lo)); return r; }\n";
    else
        os << "typedef unsigned unit_t;\n"
              "__device__ __forceinline__ float ulo(unit_t v) { return h2f((unsigned short)(v & 0xffffu)); }\n"
              "__device__ __forceinline__ float uhi(unit_t v) { return h2f((unsigned short)(v >> 16)); }\n"
              "__device__ __forceinline__ unit_t upack(float lo, float hi) { unit_t r; asm(\"cvt.rn.f16x2.f32 %0, %1, %2;\" : \"=r\"(r) : \"f\"(hi), \"f\"(lo)); return r; }\n";
}

struct SmallOut {
    int r, s, oy, ox;
};

std::vector<SmallOut> small_outs(int br, int bc, int Ho, int Wo) {
    std::vector<SmallOut> o;
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s)
            if (R * br + r < Ho && S * bc + s < Wo) o.push_back({r, s, R * br + r, S * bc + s});
    return o;
}

// pixel (h, w) of the unit-major input slot `base` (a per-lane pointer): loads each unit once,
// row of units by row of units, the next row's loads ahead of the current row's FMAs.
// `fmas[u]` = FMA statements (accumulator, text with X as the pixel placeholder) per input unit half.
struct UnitFma {
    std::string acc, text;  // text: statement with "@" replaced by the pixel value
    int width = 1;          // 2: "@" is the pixel pair (i, i+1) of the unit as a packed u64
};

long emit_unit_stream(std::ostringstream &os, const std::map<int, std::vector<std::pair<int, UnitFma>>> &fm, int Win,
                      const std::string &base, int ustr, int UP, const char *ind) {
    long cost = 0;
    std::vector<std::vector<int>> rows;  // units grouped by the image row of their first pixel
    int lastrow = -1 << 30;
    for (auto &kv : fm) {
        const int row = (UP * kv.first) / Win;
        if (row != lastrow) rows.push_back({}), lastrow = row;
        rows.back().push_back(kv.first);
    }
    auto load = [&](const std::vector<int> &us) {
        for (int u : us) {
            os << ind << "const uin_t U" << u << " = *reinterpret_cast<const uin_t*>(" << base << " + " << (size_t)u * ustr
               << ");\n";
            ++cost;
            std::set<int> comp;
            for (auto &e : fm.at(u))
                for (int w = 0; w < e.second.width; ++w) comp.insert(e.first + w);
            for (int i : comp) os << ind << "const float P" << u << "_" << i << " = UPX(U" << u << ", " << i << ");\n";
        }
    };
    std::map<std::string, long> last_use;
    long clock = 0;
    for (size_t k = 0; k < rows.size(); ++k) {
        if (k == 0) {
            load(rows[0]);
            if (rows.size() > 1) load(rows[1]);
        } else if (k + 1 < rows.size()) {
            load(rows[k + 1]);
        }
        std::vector<std::pair<std::string, std::string>> st;
        for (int u : rows[k])
            for (auto &e : fm.at(u)) {
                std::string t = e.second.text;
                const std::string pu = "P" + std::to_string(u) + "_";
                const std::string pv = e.second.width == 2 ? "f2pack(" + pu + std::to_string(e.first) + ", " + pu +
                                                                 std::to_string(e.first + 1) + ")"
                                                           : pu + std::to_string(e.first);
                for (size_t pos; (pos = t.find('@')) != std::string::npos;) t.replace(pos, 1, pv);
                st.push_back({e.second.acc, t});
                ++cost;
            }
        emit_lru(os, ind, st, last_use, clock);
    }
    return cost;
}

// stencil code of one (table, block position): outputs a<r>_<s> of this lane's plane, stored
// into the quad's output staging (`ob`, unit-major like the input slots) when complete
long emit_small_stencil(std::ostringstream &os, const Geo &g, int br, int bc, int Hin, int Win, int Ho, int Wo, int UB,
                        int ustr, int UP, bool pm_out, int UPo, const char *ind) {
    long cost = 0;
    const int nd = (int)g.taps.size();
    const auto outs = small_outs(br, bc, Ho, Wo);
    std::vector<bool> used(nd, false);
    std::map<int, std::vector<std::pair<int, UnitFma>>> fm;
    // Packed FP32 (even Win: a pixel pair (e, e+1) with e even is an aligned register pair of its
    // unit): the outputs (ox, ox+1) of one row take tap d with one FFMA2 when ox + dw is even and
    // both are in the image -- accumulator pairs at even ox ("A") for even dw, at odd ox ("B") for
    // odd dw; every other in-image (output, tap) is a scalar FMA into S_r_s.  a = A + B + S.
    const bool packed = Win % 2 == 0 && UP >= 2;
    std::map<std::pair<int, int>, const SmallOut *> at;  // (r, ox) -> output
    for (auto &o : outs) at[{o.r, o.ox}] = &o;
    auto inimg = [&](const SmallOut &o, int d) {
        const int h = o.oy + g.taps[d].dh, w = o.ox + g.taps[d].dw;
        return h >= 0 && h < Hin && w >= 0 && w < Win;
    };
    std::set<std::string> pairs_used;
    std::set<std::pair<int, int>> scal_used;
    for (auto &o : outs)
        for (int d = 0; d < nd; ++d) {
            if (!inimg(o, d)) continue;  // zero padding: dropped at compile time
            used[d] = true;
            const int h = o.oy + g.taps[d].dh, w = o.ox + g.taps[d].dw;
            const int e = h * Win + w;
            if (packed) {
                const bool lo = (w % 2 + 2) % 2 == 0;  // this output is the low half of its pair
                const SmallOut *mate = nullptr;
                auto it = at.find({o.r, lo ? o.ox + 1 : o.ox - 1});
                if (it != at.end() && inimg(*it->second, d)) mate = it->second;
                if (mate) {
                    if (!lo) continue;  // the pair is issued from its low half
                    const std::string acc = std::string((o.ox % 2 == 0) ? "A" : "B") + std::to_string(o.r) + "_" + std::to_string(o.ox);
                    pairs_used.insert(acc);
                    UnitFma f{acc, acc + " = ffma2(@, M" + std::to_string(d) + ", " + acc + ");", 2};
                    fm[e / UP].push_back({e % UP, f});
                    continue;
                }
            }
            scal_used.insert({o.r, o.s});
            const std::string acc = "S" + std::to_string(o.r) + "_" + std::to_string(o.s);
            fm[e / UP].push_back({e % UP, UnitFma{acc, acc + " = fmaf(@, m" + std::to_string(d) + ", " + acc + ");", 1}});
        }
    for (int d = 0; d < nd; ++d)
        if (used[d]) {
            os << ind << "const float m" << d << " = " << merged_weight(g.taps[d]) << ";\n";
            if (packed) os << ind << "const u64 M" << d << " = f2pack(m" << d << ", m" << d << ");\n";
        }
    for (auto &a : pairs_used) os << ind << "u64 " << a << " = 0ull;\n";
    for (auto &rs : scal_used) os << ind << "float S" << rs.first << "_" << rs.second << " = 0.f;\n";
    cost += emit_unit_stream(os, fm, Win, "xb", ustr, UP, ind);
    for (auto &o : outs) {  // a = A + B + S
        std::vector<std::string> t;
        for (const char *X : {"A", "B"}) {
            const std::string lo = X + std::to_string(o.r) + "_" + std::to_string(o.ox);
            const std::string hi = X + std::to_string(o.r) + "_" + std::to_string(o.ox - 1);
            if (pairs_used.count(lo)) t.push_back("f2lo(" + lo + ")");
            if (pairs_used.count(hi)) t.push_back("f2hi(" + hi + ")");
        }
        if (scal_used.count({o.r, o.s})) t.push_back("S" + std::to_string(o.r) + "_" + std::to_string(o.s));
        os << ind << "const float a" << o.r << "_" << o.s << " = ";
        if (t.empty()) os << "0.f";
        for (size_t q = 0; q < t.size(); ++q) os << (q ? " + " : "") << t[q];
        os << ";\n";
    }
    if (pm_out) {  // plane-major staging (this lane's plane at ob): one fp32 store per output
        for (auto &o : outs) {
            os << ind << "*reinterpret_cast<float*>(ob + " << (o.oy * Wo + o.ox) * 4 << ") = a" << o.r << "_" << o.s << ";\n";
            ++cost;
        }
        return cost;
    }
    // outputs -> staging: pairs of one output unit held by this lane go out as one store
    std::map<int, std::pair<std::string, std::string>> ou;  // output unit -> (lo, hi) value names
    for (auto &o : outs) {
        const int e = o.oy * Wo + o.ox;
        auto &slot = ou[e / UPo];
        (e % UPo ? slot.second : slot.first) = "a" + std::to_string(o.r) + "_" + std::to_string(o.s);
    }
    for (auto &kv : ou) {
        const size_t off = (size_t)kv.first * kSmallLanes * UB;
        const auto &lo = kv.second.first, &hi = kv.second.second;
        if (!lo.empty() && !hi.empty()) {
            os << ind << "*reinterpret_cast<unit_t*>(ob + " << off << ") = upack(" << lo << ", " << hi << ");\n";
        } else {
            const int es = UB / UPo;
            const size_t o2 = off + (lo.empty() ? es : 0);
            os << ind << "*reinterpret_cast<act_t*>(ob + " << o2 << ") = to_act(" << (lo.empty() ? hi : lo) << ");\n";
        }
        ++cost;
    }
    return cost;
}

// backward_weight partials of one (table, block position): q_d = sum over this lane's in-image
// (output, tap) pairs of dy * x, folded into v[k] (coefficients as emit_wgrad_taps)
long emit_small_wgrad(std::ostringstream &os, const Geo &g, int br, int bc, int Hin, int Win, int Ho, int Wo, int K,
                      int ustr, int UP, const char *ind) {
    long cost = 0;
    const int nd = (int)g.taps.size();
    const auto outs = small_outs(br, bc, Ho, Wo);
    // dy values of this lane's block
    std::set<int> du;
    for (auto &o : outs) du.insert((o.oy * Wo + o.ox) / UP);
    for (int u : du) {
        os << ind << "const uin_t D" << u << " = *reinterpret_cast<const uin_t*>(db + " << (size_t)u * ustr << ");\n";
        ++cost;
    }
    for (auto &o : outs) {
        const int e = o.oy * Wo + o.ox;
        os << ind << "const float g" << o.r << "_" << o.s << " = UPX(D" << e / UP << ", " << e % UP << ");\n";
    }
    std::vector<bool> used(nd, false), upair(nd, false), uscal(nd, false);
    std::map<int, std::vector<std::pair<int, UnitFma>>> fm;
    // packed FP32 (even Win): outputs (ox, ox+1) of one row whose pixels (e, e+1) start at an even
    // e take tap d with one FFMA2 (dy pair x pixel pair) into the pair accumulator Q<d>; the rest
    // are scalar FMAs into q<d>
    const bool packed = Win % 2 == 0 && UP >= 2;
    std::map<std::pair<int, int>, const SmallOut *> at;
    for (auto &o : outs) at[{o.r, o.ox}] = &o;
    auto inimg = [&](const SmallOut &o, int d) {
        const int h = o.oy + g.taps[d].dh, w = o.ox + g.taps[d].dw;
        return h >= 0 && h < Hin && w >= 0 && w < Win;
    };
    auto gn = [](const SmallOut &o) { return "g" + std::to_string(o.r) + "_" + std::to_string(o.s); };
    std::set<std::pair<int, int>> gpairs;  // (r, s): dy pair (s, s+1) packed once per item
    std::set<std::pair<int, int>> gbcast;  // (r, s): dy value broadcast to both halves (tap pairs)
    std::map<std::pair<int, int>, int> tap_at;  // (dh, dw) -> distinct tap
    for (int d = 0; d < nd; ++d) tap_at[{g.taps[d].dh, g.taps[d].dw}] = d;
    std::set<std::pair<int, int>> tpairs;  // (d, d2): tap pair accumulators QT<d>_<d2>
    std::set<std::pair<const SmallOut *, int>> covered;
    auto pix = [&](const SmallOut &o, int d) {
        return (o.oy + g.taps[d].dh) * Win + o.ox + g.taps[d].dw;
    };
    // 1: output pairs (ox, ox+1), even dw: dy pair x pixel pair into Q<d>
    for (auto &o : outs)
        for (int d = 0; d < nd && packed && Wo % 2 == 0; ++d) {
            if (!inimg(o, d) || ((g.taps[d].dw % 2) + 2) % 2 != 0 || covered.count({&o, d})) continue;
            const int e = pix(o, d);
            if (e % 2 != 0) continue;
            auto it = at.find({o.r, o.ox + 1});
            if (it == at.end() || !inimg(*it->second, d)) continue;
            covered.insert({&o, d}), covered.insert({it->second, d});
            used[d] = upair[d] = true;
            gpairs.insert({o.r, o.s});
            const std::string acc = "Q" + std::to_string(d);
            fm[e / UP].push_back({e % UP, UnitFma{acc, acc + " = ffma2(@, GP" + std::to_string(o.r) + "_" + std::to_string(o.s) + ", " + acc + ");", 2}});
        }
    // 2: tap pairs (d, d2 = d + (0, 1)) of one output: pixel pair x broadcast dy into QT<d>_<d2>
    std::map<int, std::vector<std::pair<std::string, bool>>> tpart;  // d -> (QT name, hi half?)
    for (auto &o : outs)
        for (int d = 0; d < nd && packed; ++d) {
            if (!inimg(o, d) || covered.count({&o, d})) continue;
            const int e = pix(o, d);
            if (e % 2 != 0) continue;
            auto it = tap_at.find({g.taps[d].dh, g.taps[d].dw + 1});
            if (it == tap_at.end()) continue;
            const int d2 = it->second;
            if (!inimg(o, d2) || covered.count({&o, d2})) continue;
            covered.insert({&o, d}), covered.insert({&o, d2});
            used[d] = used[d2] = true;
            gbcast.insert({o.r, o.s});
            const std::string acc = "QT" + std::to_string(d) + "_" + std::to_string(d2);
            if (tpairs.insert({d, d2}).second) {
                tpart[d].push_back({acc, false});
                tpart[d2].push_back({acc, true});
            }
            fm[e / UP].push_back({e % UP, UnitFma{acc, acc + " = ffma2(@, GB" + std::to_string(o.r) + "_" + std::to_string(o.s) + ", " + acc + ");", 2}});
        }
    // 3: the rest, scalar FMAs into q<d>
    for (auto &o : outs)
        for (int d = 0; d < nd; ++d) {
            if (!inimg(o, d) || covered.count({&o, d})) continue;
            used[d] = uscal[d] = true;
            const int e = pix(o, d);
            const std::string acc = "q" + std::to_string(d);
            fm[e / UP].push_back({e % UP, UnitFma{acc, acc + " = fmaf(" + gn(o) + ", @, " + acc + ");", 1}});
        }
    for (auto &rs : gpairs)
        os << ind << "const u64 GP" << rs.first << "_" << rs.second << " = f2pack(g" << rs.first << "_" << rs.second << ", g"
           << rs.first << "_" << rs.second + 1 << ");\n";
    for (auto &rs : gbcast)
        os << ind << "const u64 GB" << rs.first << "_" << rs.second << " = f2pack(g" << rs.first << "_" << rs.second << ", g"
           << rs.first << "_" << rs.second << ");\n";
    for (int d = 0; d < nd; ++d) {
        if (upair[d]) os << ind << "u64 Q" << d << " = 0ull;\n";
        if (uscal[d]) os << ind << "float q" << d << " = 0.f;\n";
    }
    for (auto &tp : tpairs) os << ind << "u64 QT" << tp.first << "_" << tp.second << " = 0ull;\n";
    cost += emit_unit_stream(os, fm, Win, "xb", ustr, UP, ind);
    for (int d = 0; d < nd; ++d) {
        if (!used[d]) continue;
        std::vector<std::string> t;
        if (uscal[d]) t.push_back("q" + std::to_string(d));
        if (upair[d]) t.push_back("f2lo(Q" + std::to_string(d) + ") + f2hi(Q" + std::to_string(d) + ")");
        for (auto &tp : tpart[d]) t.push_back((tp.second ? "f2hi(" : "f2lo(") + tp.first + ")");
        os << ind << "const float qs" << d << " = ";
        for (size_t i = 0; i < t.size(); ++i) os << (i ? " + " : "") << t[i];
        os << ";\n";
    }
    std::vector<bool> written(K, false);
    for (int d = 0; d < nd; ++d) {
        if (!used[d]) continue;
        for (auto &kc : g.taps[d].ks) {
            os << ind << "v[" << kc.first << "] " << (written[kc.first] ? "+= " : "= ");
            written[kc.first] = true;
            if (kc.second == 1.0f) os << "qs" << d << ";\n";
            else os << flit(kc.second) << " * qs" << d << ";\n";
        }
    }
    for (int k = 0; k < K; ++k)
        if (!written[k]) os << ind << "v[" << k << "] = 0.f;\n";
    return cost;
}

// layout of one small-plane pass; false if it does not fit shared memory
bool make_small_lay(SmallLay *out, int pass, int H, int W, int Ho, int Wo, int N, int es) {
    SmallLay L;
    L.BRs = (Ho + R - 1) / R;
    L.BCs = (Wo + S - 1) / S;
    L.QW = L.BRs * L.BCs;
    L.es = es;
    L.UPu = (H * W) % 2 == 0 && (Ho * Wo) % 2 == 0 ? 2 : 1;
    L.UB = L.UPu * es;
    L.sync_copy = L.UPu == 1 && es == 2;
    L.G = (N + 31) / 32;
    const int Hin = pass == 1 ? Ho : H, Win = pass == 1 ? Wo : W;
    // fp32 planes whose byte size is a multiple of 16 (and at most 256 elements, one TMA box row)
    // arrive by one TMA box per item; others by per-unit cp.async (LDGSTS)
    L.tma = es == 4 && (Hin * Win) % 4 == 0 && Hin * Win <= 256 && (pass != 2 || (Ho * Wo) % 4 == 0) && env_int("O1D_SMALL_TMA", 1);
    L.UPi = L.tma ? 4 : L.UPu;
    L.ustr = L.tma ? 16 : kSmallLanes * L.UB;
    L.lstr = L.tma ? Hin * Win * 4 : L.UB;
    L.hp_in = Hin * Win / L.UPu;
    L.hp_dy = pass == 2 ? Ho * Wo / L.UPu : 0;
    L.hp_out = pass <= 1 ? (pass == 0 ? Ho * Wo : H * W) / L.UPu : 0;
    auto rnd = [](size_t b) { return (b + 127) & ~(size_t)127; };
    L.slotb = rnd(L.tma ? (size_t)32 * Hin * Win * 4 : (size_t)L.hp_in * kSmallLanes * L.UB);
    L.dyb = L.hp_dy ? rnd(L.tma ? (size_t)32 * Ho * Wo * 4 : (size_t)L.hp_dy * kSmallLanes * L.UB) : 0;
    const int hwo = L.hp_out * L.UPu;
    L.tma_out = pass <= 1 && es == 4 && hwo % 4 == 0 && hwo <= 256 && env_int("O1D_SMALL_TMA", 1);
    L.outb = L.hp_out ? rnd(L.tma_out ? (size_t)32 * hwo * 4 : (size_t)L.hp_out * kSmallLanes * L.UB) : 0;
    const size_t budget = (size_t)227 * 1024 - 64;
    for (int NQ = std::max(1, 8 / L.QW); NQ >= 1; --NQ) {
        for (int NB = 3; NB >= 2; --NB) {
            if (NQ * NB > 16) continue;
            L.NQ = NQ, L.NB = NB;
            L.off_item = 8 * 32;  // full[16], empty[16]
            L.off_w = L.off_item + 4 * 16;
            L.off_slot = (L.off_w + (size_t)L.NS() * 64 * 4 + 127) & ~(size_t)127;
            L.off_out = L.off_slot + (size_t)L.NS() * (L.slotb + L.dyb);
            L.total = L.off_out + (size_t)NQ * L.outb;
            // at least two quads (or 8 warps) unless a single quad is all that fits
            if (L.total + 16 <= budget && (NB == 2 || NQ * L.QW >= 8)) {
                *out = L;
                return true;
            }
        }
    }
    return false;
}

void emit_finalize_ne(std::ostringstream &os, int K, const std::string &ne) {
    os << "extern \"C\" __global__ void __launch_bounds__(256) o1d_wgrad_finalize(const float* __restrict__ ws, float* __restrict__ dW, int N) {\n"
       << "  __shared__ double part[8][64];\n"
       << "  pdl_wait();\n"
       << "  pdl_trigger();\n"
       << "  const int c = blockIdx.x, j = threadIdx.x >> 5, lane = threadIdx.x & 31;\n"
       << "  const int NE = " << ne << ";\n"
       << "  const float* base = ws + (u64)c * NE * " << K << ";\n"
       << "  for (int k = lane; k < " << K << "; k += 32) {\n"
       << "    double s = 0.0;\n"
       << "#pragma unroll 16\n"
       << "    for (int e = j; e < NE; e += 8) s += (double)__ldcg(base + (u64)e * " << K << " + k);\n"
       << "    part[j][k] = s;\n"
       << "  }\n"
       << "  __syncthreads();\n"
       << "  for (int k = threadIdx.x; k < " << K << "; k += 256) {\n"
       << "    double s = 0.0;\n"
       << "    for (int q = 0; q < 8; ++q) s += part[q][k];\n"
       << "    dW[c * " << K << " + k] = (float)s;\n"
       << "  }\n"
       << "}\n";
}

std::string gen_small_pass(const Ctx &x, const SmallLay &L, int pass, const std::vector<Geo> &geo, int Hx, int Wx,
                           std::vector<long> *cost_out) {
    std::ostringstream os;
    const bool pref = env_int("O1D_PREF", 0) != 0;  // claimed group indices kept in flight (round 2: two)
    emit_header(os, x);
    emit_small_header(os, x.act, L.UPu);
    if (L.tma)
        os << "typedef float4 uin_t;\n#define UPX(v, i) ((i) == 0 ? (v).x : (i) == 1 ? (v).y : (i) == 2 ? (v).z : (v).w)\n";
    else
        os << "typedef unit_t uin_t;\n#define UPX(v, i) ((i) == 0 ? ulo(v) : uhi(v))\n";
    const int nthreads = L.threads();
    const int NB = L.NB, QW = L.QW, NQ = L.NQ;
    const int K = x.K;
    const int Hin = pass == 1 ? x.Ho : Hx, Win = pass == 1 ? x.Wo : Wx;
    const int Hout = pass == 1 ? Hx : x.Ho, Wout = pass == 1 ? Wx : x.Wo;
    const int NV32 = (K + 31) / 32;  // backward_weight: rounds of 32 taps per warp reduction
    // per (table, block position) case bodies
    std::vector<std::string> body;
    cost_out->assign(geo.size(), 0);
    for (size_t t = 0; t < geo.size(); ++t)
        for (int bp = 0; bp < QW; ++bp) {
            std::ostringstream b;
            const int br = bp / L.BCs, bc = bp % L.BCs;
            long c = pass <= 1 ? emit_small_stencil(b, geo[t], br, bc, Hin, Win, Hout, Wout, L.UB, L.ustr, L.UPi, L.tma_out, L.UPu, "      ")
                               : emit_small_wgrad(b, geo[t], br, bc, Hin, Win, x.Ho, x.Wo, K, L.ustr, L.UPi, "      ");
            (*cost_out)[t] += c;
            body.push_back(b.str());
        }
    os << "extern \"C\" __global__ void __launch_bounds__(" << nthreads << ", 1) o1d_small(const __grid_constant__ Params p) {\n"
       << "  extern __shared__ __align__(1024) unsigned char smem[];\n"
       << "  u64* const full = reinterpret_cast<u64*>(smem);\n"
       << "  u64* const empty = full + 16;\n"
       << "  int* const s_item = reinterpret_cast<int*>(smem + " << L.off_item << ");\n"
       << "  float* const wsm = reinterpret_cast<float*>(smem + " << L.off_w << ");\n"
       << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n"
       << "  int trn = 0;\n"
       << "  if (tid == 0) {\n"
       << "    for (int s = 0; s < " << L.NS() << "; ++s) { mbar_init(full + s, 32); mbar_init(empty + s, " << QW << "); }\n"
       << "    fence_mbar_init();\n"
       << "  }\n"
       << "  __syncthreads();\n"
       << "  const int G = (p.N + 31) / 32;   // 32-plane groups per channel\n"
       // ------------------------------------------------------------------ producers
       << "  if (warp < " << NQ << ") {\n"
       << "    const int q = warp;\n"
       << "    int tcur = 0, tried = 0;\n"
       << "    unsigned pf0 = 0u, pf1 = 0u;\n"
       << "    const u64 pol = policy_evict_first();\n"
       << "    if (lane == 0) {\n"
       << "      trace_ev(p.trace, 0, -1, trn);\n"
       << "      tcur = HOME[smid() % NHOME];\n"
       << (pref ? "      pf0 = atomicAdd(p.sched + tcur * CS, 1u);\n"
                  "      pf1 = atomicAdd(p.sched + tcur * CS, 1u);\n" : "")
       << "    }\n"
       << "    (void)pf0; (void)pf1;\n"
       << "    if (!p.nowait) pdl_wait();\n"
       << "    for (int j = 0;; ++j) {\n"
       << "      const int s = q * " << NB << " + j % " << NB << ";\n"
       << "      if (j >= " << NB << ") mbar_wait(empty + s, ((j / " << NB << ") & 1) ^ 1);\n"
       << "      int item = -1;\n"
       << "      if (lane == 0) {\n"
       << (pref ? "        const unsigned v = pf0;\n"
                  "        pf0 = pf1;\n"
                  "        const int t0 = tcur;\n"
                  "        item = sched_resolve(p.sched, tcur, v, tried, G);\n"
                  "        if (tcur != t0) {\n"
                  "          pf0 = tcur >= 0 ? atomicAdd(p.sched + tcur * CS, 1u) : 0xffffffffu;\n"
                  "          pf1 = tcur >= 0 ? atomicAdd(p.sched + tcur * CS, 1u) : 0xffffffffu;\n"
                  "        } else {\n"
                  "          pf1 = tcur >= 0 ? atomicAdd(p.sched + tcur * CS, 1u) : 0xffffffffu;\n"
                  "        }\n"
                  // claim on demand (O1D_PREF=0, see emit_producer): no claimed-but-unstarted groups at the end
                : "        item = tcur >= 0 ? sched_resolve(p.sched, tcur, atomicAdd(p.sched + tcur * CS, 1u), tried, G) : -1;\n")
       << "        s_item[s] = item;\n"
       << "        if (item >= 0) trace_ev(p.trace, 1, item, trn);\n"
       << "      }\n"
       << "      item = __shfl_sync(0xffffffffu, item, 0);\n"
       << "      if (item >= 0) {\n"
       << "        int t, c, g; item_cn(item, t, c, g, 0);\n"
       << "        unsigned char* const dst = smem + " << L.off_slot << " + s * " << L.slotb + L.dyb << ";\n";
    auto copy_planes = [&](const char *src, int HW, int hp, size_t dst_off) {
        const int nk = (hp + 31) / 32;
        os << "        {\n"
           << "          const unsigned char* const src = reinterpret_cast<const unsigned char*>(" << src << ") + ((u64)(32 * g) * "
           << x.C << " + c) * " << (long)HW * L.es << ";\n"
           << "#pragma unroll 1\n"
           << "          for (int jj = 0; jj < 32; ++jj) {\n"
           << "            if (32 * g + jj >= p.N) break;\n"
           << "            const unsigned char* const pl = src + (u64)jj * " << (long)x.C * HW * L.es << ";\n"
           << "#pragma unroll\n"
           << "            for (int k = 0; k < " << nk << "; ++k) {\n"
           << "              const int u = lane + 32 * k;\n"
           << "              if (u < " << hp << ") cp_async_unit(dst + " << dst_off << " + (u * " << kSmallLanes << " + jj) * " << L.UB
           << ", pl + u * " << L.UB << ", pol);\n"
           << "            }\n"
           << "          }\n"
           << "        }\n";
    };
    if (L.tma) {  // one box (all pixels, this channel, 32 samples; samples past the batch zero-filled)
        os << "        if (lane == 0) {\n"
           << "          mbar_expect_tx(full + s, " << L.slotb + L.dyb << "u);\n"
           << "          tma_load(dst, &p.in_map, 0, 0, c, 32 * g, full + s, pol);\n";
        if (pass == 2) os << "          tma_load(dst + " << L.slotb << ", &p.aux_map, 0, 0, c, 32 * g, full + s, pol);\n";
        os << "        }\n";
    } else {
        copy_planes("p.src1", Hin * Win, L.hp_in, 0);
        if (pass == 2) copy_planes("p.src2", x.Ho * x.Wo, L.hp_dy, L.slotb);
    }
    if (pass <= 1) {
        if (L.sync_copy)
            os << "        for (int k = lane; k < " << K << "; k += 32) wsm[s * 64 + k] = __ldg(p.w + c * " << K << " + k);\n";
        else
            os << "        for (int k = lane; k < " << K << "; k += 32) cp_async_w(wsm + s * 64 + k, p.w + c * " << K << " + k);\n";
    }
    os << "      }\n"
       << (L.sync_copy ? "      mbar_arrive(full + s);   // plain copies: the arrive releases them\n"
                       : "      cp_async_arrive(full + s);   // 32 lanes: each arrival fires when the lane's copies have landed\n")
       << "      if (item < 0) break;\n"
       << "    }\n"
       << "    if (p.nowait) pdl_wait();\n"
       << "    pdl_trigger();\n"
       << "    if (lane == 0) sched_exit(p.sched, " << NQ << "u);\n"
       << "    return;\n"
       << "  }\n"
       // ------------------------------------------------------------------ consumers
       << "  const int cw = warp - " << NQ << ", q = cw / " << QW << ", bp = cw % " << QW << ";\n";
    if (pass <= 1)
        os << "  unsigned char* const ob = smem + " << L.off_out << " + q * " << L.outb << " + lane * "
           << (L.tma_out ? Hout * Wout * 4 : L.UB) << ";\n";
    os << "  for (int it = 0;; ++it) {\n"
       << "    const int s = q * " << NB << " + it % " << NB << ";\n"
       << "    if (lane == 0) trace_ev(p.trace, 2, it, trn);\n"
       << "    mbar_wait(full + s, (it / " << NB << ") & 1);\n"
       << "    const int item = s_item[s];\n"
       << "    if (lane == 0) trace_ev(p.trace, 3, item, trn);\n"
       << "    if (item < 0) break;\n"
       << "    int t, c, g; item_cn(item, t, c, g, 0);\n"
       << "    const unsigned char* const xb = smem + " << L.off_slot << " + s * " << L.slotb + L.dyb << " + lane * " << L.lstr << ";\n";
    if (pass <= 1) {
        os << "    const float* const wv = wsm + s * 64;\n"
           << (L.tma_out ? "    if (bp == 0 && lane == 0) asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\");   // previous box store has read the staging\n" : "")
           << "    asm volatile(\"bar.sync %0, %1;\" :: \"r\"(1 + q), \"r\"(" << 32 * QW << ") : \"memory\");   // previous write-back done\n"
           << "    switch (t * " << QW << " + bp) {\n";
        for (size_t i = 0; i < body.size(); ++i) os << "    case " << i << ": {\n" << body[i] << "      break;\n    }\n";
        os << "    }\n"
           << "    __syncwarp();\n"
           << "    if (lane == 0) { mbar_arrive(empty + s); trace_ev(p.trace, 4, item, trn); }   // input slot free\n"
           << (L.tma_out ? "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");   // staging writes -> the TMA store\n" : "")
           << "    asm volatile(\"bar.sync %0, %1;\" :: \"r\"(1 + q), \"r\"(" << 32 * QW << ") : \"memory\");   // all blocks staged\n";
    if (pass <= 1 && L.tma_out) {
        // one box store: all pixels of the 32 planes (samples past the batch are clipped by the TMA unit)
        os << "    if (bp == 0 && lane == 0) tma_store_band(&p.out_map, smem + " << L.off_out << " + q * " << L.outb
           << ", 0, c, 32 * g, policy_evict_first());\n";
    } else if (pass <= 1) {
        // write-back: warp bp stores planes bp, bp + QW, ... (coalesced along each plane)
        os << "    {\n"
           << "      const int HWo = " << Hout * Wout << ";\n"
           << "      unsigned char* const dbase = reinterpret_cast<unsigned char*>(p.dst) + ((u64)(32 * g) * " << x.C
           << " + c) * (u64)HWo * " << L.es << ";\n"
           << "      const unsigned char* const obq = smem + " << L.off_out << " + q * " << L.outb << ";\n"
           << "#pragma unroll 1\n"
           << "      for (int jj = bp; jj < 32; jj += " << QW << ") {\n"
           << "        if (32 * g + jj >= p.N) break;\n"
           << "        unsigned char* const pl = dbase + (u64)jj * " << (long)x.C * Hout * Wout * L.es << ";\n"
           << "#pragma unroll\n"
           << "        for (int k = 0; k < " << (L.hp_out + 31) / 32 << "; ++k) {\n"
           << "          const int u = lane + 32 * k;\n"
           << "          if (u < " << L.hp_out << ") {\n"
           << "            const unit_t v = *reinterpret_cast<const unit_t*>(obq + (u * " << kSmallLanes << " + jj) * " << L.UB << ");\n"
           << "            __stcs(reinterpret_cast<unit_t*>(pl) + u, v);\n"
           << "          }\n"
           << "        }\n"
           << "      }\n"
           << "    }\n";
    }
    } else {
        os << "    const unsigned char* const db = xb + " << L.slotb << ";\n"
           << "    float v[" << 32 * NV32 << "];\n"
           << "#pragma unroll\n"
           << "    for (int k = " << K << "; k < " << 32 * NV32 << "; ++k) v[k] = 0.f;\n"
           << "    switch (t * " << QW << " + bp) {\n";
        for (size_t i = 0; i < body.size(); ++i) os << "    case " << i << ": {\n" << body[i] << "      break;\n    }\n";
        os << "    }\n"
           << "    __syncwarp();\n"
           << "    if (lane == 0) { mbar_arrive(empty + s); trace_ev(p.trace, 4, item, trn); }   // input slot free\n"
           << "    if (32 * g + lane >= p.N) {   // lanes past the batch hold stale planes\n"
           << "#pragma unroll\n"
           << "      for (int k = 0; k < " << 32 * NV32 << "; ++k) v[k] = 0.f;\n"
           << "    }\n";
        for (int rd = 0; rd < NV32; ++rd) {
            os << "    {\n"
               << "      float vv[32];\n"
               << "#pragma unroll\n"
               << "      for (int k = 0; k < 32; ++k) vv[k] = v[" << 32 * rd << " + k];\n"
               << "      const float part = reduce_scatter<32>(vv, lane);\n"
               << "      if (" << 32 * rd << " + lane < " << K << ") p.ws[(((u64)c * G + g) * " << QW << " + bp) * " << K << " + "
               << 32 * rd << " + lane] = part;\n"
               << "    }\n";
        }
    }
    os << "    if (lane == 0) trace_ev(p.trace, 5, item, trn);\n"
       << "  }\n";
    if (pass <= 1 && L.tma_out) os << "  if (bp == 0 && lane == 0) asm volatile(\"cp.async.bulk.wait_group 0;\" ::: \"memory\");\n";
    os << "}\n";
    if (pass == 2) emit_finalize_ne(os, K, "((N + 31) / 32) * " + std::to_string(QW));
    return os.str();
}

o1d_status encode(CUtensorMap *m, const void *ptr, int dtype, int W, int H, int C, int N, int boxW, int boxH, int boxN = 1) {
    const size_t es = dtype_size(dtype);
    cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)W * es, (cuuint64_t)W * H * es, (cuuint64_t)W * H * C * es};
    cuuint32_t box[4] = {(cuuint32_t)boxW, (cuuint32_t)boxH, 1, (cuuint32_t)boxN};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUtensorMapDataType dt = dtype == O1D_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : dtype == O1D_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    CUresult r = drv().encodeTiled(m, dt, 4, const_cast<void *>(ptr), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(O1D_CUDA_ERROR, "cuTensorMapEncodeTiled: " + cu_err(r));
    return O1D_OK;
}

// Home tap table of every SM.  Measured (profiles/r1/icache.md): the SM instruction cache
// is shared by the two SMs of a TPC (splitting TPC mates across tables costs 35%), and
// every extra distinct table running on the GPU costs instruction-cache hits.  SMs are
// ordered GPC by GPC (gpc_map probe) and each table gets a contiguous run of TPC pairs
// proportional to its work (planes x issue cost of its case).
std::vector<int> home_tables(const std::vector<int> &gpc_of_smid, const std::vector<long> &work, int nt) {
    const int n = (int)gpc_of_smid.size();
    std::vector<int> home(n, 0);
    std::map<int, std::vector<int>> groups;  // gpc -> smids (unknown ids: own group)
    for (int s = 0; s < n; ++s) groups[gpc_of_smid[s] >= 0 ? gpc_of_smid[s] : 100000 + s].push_back(s);
    double total = 0;
    for (int t = 0; t < nt; ++t) total += (double)work[t];
    std::vector<int> ordered;
    for (auto &g : groups) ordered.insert(ordered.end(), g.second.begin(), g.second.end());
    double acc = 0;
    int t = 0;
    const int m = (int)ordered.size();
    for (int i = 0; i < m; i += 2) {  // TPC pairs stay together
        const double pos = (i + 1.0) * total / m;
        while (t < nt - 1 && pos >= acc + (double)work[t]) acc += (double)work[t], ++t;
        home[ordered[i]] = t;
        if (i + 1 < m) home[ordered[i + 1]] = t;
    }
    return home;
}

// process-wide module cache: (device, source) -> module.  Plans hold shared_ptrs; the cache
// keeps weak references plus strong references to the most recent modules, so a plan that
// is destroyed and re-created (or another batch size) reuses the compiled code.
std::mutex g_cache_mu;
std::map<std::pair<int, std::string>, std::weak_ptr<Mod>> g_cache;
std::deque<std::shared_ptr<Mod>> g_recent;

std::shared_ptr<Mod> cache_get(int dev, const std::string &src) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find({dev, src});
    if (it == g_cache.end()) return nullptr;
    return it->second.lock();
}

void cache_put(int dev, const std::string &src, const std::shared_ptr<Mod> &m) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache[{dev, src}] = m;
    g_recent.push_back(m);
    while (g_recent.size() > 24) g_recent.pop_front();
    for (auto it = g_cache.begin(); it != g_cache.end();)  // drop dead entries
        it = it->second.expired() ? g_cache.erase(it) : std::next(it);
}

const char *kFnName[kPasses] = {"o1d_stencil", "o1d_stencil", "o1d_wgrad", "o1d_bwd_fused"};

// small planes (H, W <= 14): passes 0-2 on gen_small_pass, no fused backward
bool small_prepare(const o1d_plan *pl, SpecSet *sp, std::string src[kPasses], int nsm, const std::vector<int> *gpc) {
    const o1d_desc &d = pl->d;
    const int es = (int)dtype_size(d.dtype);
    sp->small = true;
    sp->small_items = (long)d.C * ((d.N + 31) / 32);
    sp->nt = pl->n_distinct;
    sp->nsm = nsm;
    sp->K = d.K;
    std::vector<int> rep(sp->nt, -1);
    std::vector<long> count(sp->nt, 0);
    for (int c = 0; c < d.C; ++c) {
        if (rep[pl->table_of[c]] < 0) rep[pl->table_of[c]] = c;
        count[pl->table_of[c]] += 1;
    }
    for (int t = 0; t < sp->nt; ++t) {
        const size_t o = (size_t)rep[t] * pl->KE;
        sp->fwd.push_back(make_geo(&pl->eoh[o], &pl->eow[o], &pl->ek[o], &pl->ecoef[o], pl->KE, false, 1, d.W));
        sp->bwd.push_back(make_geo(&pl->eoh[o], &pl->eow[o], &pl->ek[o], &pl->ecoef[o], pl->KE, true, 1, pl->Q));
    }
    Ctx x{d.C, d.K, pl->P, pl->Q, 1, 1, sp->nt, nsm};
    x.act = d.dtype;
    x.Wi = d.W;
    x.table_of.assign(pl->table_of.begin(), pl->table_of.end());
    for (int i = 0; i < 3; ++i) {
        sp->has[i] = make_small_lay(&sp->sl[i], i, d.H, d.W, pl->P, pl->Q, d.N, es);
        if (!sp->has[i]) continue;
        std::vector<long> cost;
        Ctx xi = x;
        // the case costs are only known after generation: generate once for the costs, then
        // again with the SM placement they imply (the source text differs only in HOME)
        src[i] = gen_small_pass(xi, sp->sl[i], i, i == 1 ? sp->bwd : sp->fwd, d.H, d.W, &cost);
        if (gpc && !gpc->empty()) {
            std::vector<long> work(sp->nt);
            for (int t = 0; t < sp->nt; ++t) work[t] = count[t] * (100 + cost[t]);
            xi.home = home_tables(*gpc, work, sp->nt);
            src[i] = gen_small_pass(xi, sp->sl[i], i, i == 1 ? sp->bwd : sp->fwd, d.H, d.W, &cost);
        }
    }
    return sp->has[0] || sp->has[1] || sp->has[2];
}

// Host-only part: eligibility, geometry and generated sources (no CUDA calls).
// Returns false (and no sources) when the plan is not eligible for any pass.
bool spec_prepare(const o1d_plan *pl, SpecSet *sp, std::string src[kPasses], int nsm, const std::vector<int> *gpc) {
    const o1d_desc &d = pl->d;
    const int es = (int)dtype_size(d.dtype);
    if (d.stride != 1) return false;  // stride 2 runs on the generic kernels
    if (d.K > 64 || pl->n_distinct > 16) return false;
    if (d.H <= 2 * R && d.W <= 2 * S && env_int("O1D_SMALL", 1) != 0)
        return small_prepare(pl, sp, src, nsm, gpc);
    if ((d.W * es) % 16 != 0) {
        // 16-bit rows that are not 16-byte multiples: flat TMA views (Lay::flat) need whole planes of
        // 16-byte multiples, rows of 4-element (8-byte) units, band starts on 8-element boundaries
        // (28-row bands, W even) and boxes of <= 256 eight-element rows
        if (es != 2 || d.W % 4 != 0 || ((long)d.H * d.W) % 8 != 0 || (long)d.H * d.W / 8 > 256) return false;
    }
    if (pl->n_distinct > 16 || (long)d.N * d.C >= (1L << 22)) return false;
    if (d.W > 256 || d.H > 256) return false;
    sp->BR = (pl->P + R - 1) / R;
    sp->BC = (pl->Q + S - 1) / S;
    if (sp->BC > 8) return false;  // one 8-block column group per band (W <= 56)
    sp->wpg = (sp->BR + 3) / 4;
    sp->nt = pl->n_distinct;
    sp->nsm = nsm;
    sp->K = d.K;
    std::vector<int> rep(sp->nt, -1);  // one representative channel per distinct table
    std::vector<long> count(sp->nt, 0);
    for (int c = 0; c < d.C; ++c) {
        if (rep[pl->table_of[c]] < 0) rep[pl->table_of[c]] = c;
        count[pl->table_of[c]] += 1;
    }
    const int KE = pl->KE;
    for (int t = 0; t < sp->nt; ++t) {
        const size_t o = (size_t)rep[t] * KE;
        sp->fwd.push_back(make_geo(&pl->eoh[o], &pl->eow[o], &pl->ek[o], &pl->ecoef[o], KE, false, sp->BC, d.W));
        sp->bwd.push_back(make_geo(&pl->eoh[o], &pl->eow[o], &pl->ek[o], &pl->ecoef[o], KE, true, sp->BC, pl->Q));
        for (const Geo *g : {&sp->fwd.back(), &sp->bwd.back()})
            if (g->pitch > 256 || g->maxDH - g->minDH > 128) return false;
    }
    Ctx x{d.C, d.K, pl->P, pl->Q, sp->BR, sp->BC, sp->nt, nsm};
    x.act = d.dtype;
    x.Wi = d.W;
    x.table_of.assign(pl->table_of.begin(), pl->table_of.end());
    const int P_req = env_int("O1D_P", 0), NB_req = env_int("O1D_NBUF", 0);
    const int P3_req = env_int("O1D_P3", 0);
    const bool early = env_int("O1D_EARLY", 1) != 0;
    bool any = false;
    for (int i = 0; i < kPasses; ++i) {
        if ((i >= 2) && d.K > 32) continue;  // per-tap reduction over one warp (v[k], k < 32)
        sp->has[i] = make_lay(&sp->lay[i], i, sp->wpg, sp->fwd, sp->bwd, d.H, pl->P, pl->Q, sp->BR, sp->BC, es,
                              i == 3 ? P3_req : P_req, NB_req) &&
                     sp->lay[i].NB >= 2;
        sp->lay[i].early = early;
        any = any || sp->has[i];
    }
    if (!any) return false;
    for (int i = 0; i < kPasses; ++i) {
        if (!sp->has[i]) continue;
        const Lay &L = sp->lay[i];
        const Cases st = i == 2 ? Cases{} : stencil_cases(i == 0 ? sp->fwd : sp->bwd, i == 0 ? L.pitch : i == 1 ? L.pitch : L.pitch2,
                                                          L.early ? &x : nullptr);
        const Cases wg = i >= 2 ? wgrad_cases(sp->fwd, L.pitch, d.K) : Cases{};
        Ctx xi = x;
        xi.flat = L.flat;
        if (gpc && !gpc->empty()) {
            // SMs per table in proportion to planes x the issue count of the table's case(s) in
            // THIS pass (+100: per-item cost outside the case; the wgrad's per-table costs differ
            // from the stencil's, pairing varies by angle)
            std::vector<long> work(sp->nt);
            for (int t = 0; t < sp->nt; ++t) {
                long c = 100;
                if (!st.cost.empty()) c += st.cost[t];
                if (!wg.cost.empty()) c += wg.cost[t];
                work[t] = count[t] * c;
            }
            xi.home = home_tables(*gpc, work, sp->nt);
        }
        src[i] = gen_pass(xi, L, i, st, wg);
    }
    return true;
}

}  // namespace

namespace {
const char *kSrcName[kPasses] = {"o1d_fwd.cu", "o1d_bwd_in.cu", "o1d_wgrad.cu", "o1d_bwd_fused.cu"};

// compile (or take from the module cache) and load the modules of passes `which`; sets
// launch geometry.  *all_hit: every module came from the cache.
// On-disk cubin cache (across processes): NVRTC takes seconds per generated pass, and a model builds
// one plan per distinct layer shape.  Key = FNV-1a 64 of (source, compile options); files
// <dir>/o1d_<key>.cubin (+ .log: the ptxas report).  dir = $O1D_CACHE_DIR, else $HOME/.cache/oriented1d;
// O1D_DISK_CACHE=0 disables it.  Writes go to a temporary name and are renamed into place, so readers
// never see a partial file; an entry that fails to load is recompiled.
std::string disk_cache_path(const std::string &src) {
    if (env_int("O1D_DISK_CACHE", 1) == 0) return std::string();
    std::string dir;
    if (const char *d = getenv("O1D_CACHE_DIR")) dir = d;
    else if (const char *h = getenv("HOME")) dir = std::string(h) + "/.cache/oriented1d";
    if (dir.empty()) return std::string();
    mkdir((dir.substr(0, dir.rfind('/'))).c_str(), 0755);
    mkdir(dir.c_str(), 0755);
    unsigned long long h = 1469598103934665603ull;
    const std::string key = src + "\n// sm_100a -std=c++17 -lineinfo -DNDEBUG v1";
    for (unsigned char ch : key) h = (h ^ ch) * 1099511628211ull;
    char name[64];
    snprintf(name, sizeof name, "/o1d_%016llx", h);
    return dir + name;
}
bool read_file(const std::string &path, std::string *out) {
    FILE *f = fopen(path.c_str(), "rb");
    if (!f) return false;
    std::string d;
    char buf[1 << 16];
    size_t n;
    while ((n = fread(buf, 1, sizeof buf, f)) > 0) d.append(buf, n);
    fclose(f);
    *out = d;
    return !d.empty();
}
void write_file_atomic(const std::string &path, const char *data, size_t n) {
    const std::string tmp = path + ".tmp" + std::to_string((long)getpid()) + "_" +
                            std::to_string((unsigned long)std::hash<std::thread::id>()(std::this_thread::get_id()));
    FILE *f = fopen(tmp.c_str(), "wb");
    if (!f) return;
    const bool ok = fwrite(data, 1, n, f) == n;
    if (fclose(f) == 0 && ok) rename(tmp.c_str(), path.c_str());
    else unlink(tmp.c_str());
}

o1d_status load_passes(SpecSet *sp, const std::vector<int> &which, const std::string *src, int device, long planes,
                       bool *all_hit) {
    Driver &dr = drv();
    std::vector<char> cubin[kPasses];
    std::string logs[kPasses];
    bool ok[kPasses] = {true, true, true, true}, need[kPasses] = {false, false, false, false};
    *all_hit = true;
    for (int i : which) {
        if (i == 1 && sp->has[0] && src[1] == src[0]) continue;  // identical sources: shares pass 0's module
        sp->mod[i] = cache_get(device, src[i]);
        if (!sp->mod[i]) need[i] = true, *all_hit = false;
    }
    std::string dpath[kPasses];
    bool from_disk[kPasses] = {false, false, false, false};
    for (int i = 0; i < kPasses; ++i) {
        if (!need[i]) continue;
        dpath[i] = disk_cache_path(src[i]);
        std::string cb, lg;
        if (!dpath[i].empty() && read_file(dpath[i] + ".cubin", &cb) && read_file(dpath[i] + ".log", &lg)) {
            cubin[i].assign(cb.begin(), cb.end());
            logs[i] = lg;
            from_disk[i] = true;
        }
    }
    auto compile = [&](int i) {
        ok[i] = compile_cubin(src[i], kSrcName[i], &cubin[i], &logs[i]);
        if (ok[i] && !dpath[i].empty()) {
            write_file_atomic(dpath[i] + ".cubin", cubin[i].data(), cubin[i].size());
            write_file_atomic(dpath[i] + ".log", logs[i].data(), logs[i].size());
        }
    };
    {
        std::vector<std::thread> th;
        for (int i = 0; i < kPasses; ++i)
            if (need[i] && !from_disk[i]) th.emplace_back([&, i] { compile(i); });
        for (auto &t : th) t.join();
    }
    for (int i = 0; i < kPasses; ++i)
        if (need[i] && !ok[i]) return fail(O1D_JIT_ERROR, std::string("NVRTC failed for ") + kSrcName[i] + ":\n" + logs[i].substr(0, 4000));
    for (int i = 0; i < kPasses; ++i) {
        if (!need[i]) continue;
        auto m = std::make_shared<Mod>();
        CUresult r = dr.ctxGetCurrent(&m->ctx);
        if (r == CUDA_SUCCESS) r = dr.moduleLoadData(&m->mod, cubin[i].data());
        if (r != CUDA_SUCCESS && from_disk[i]) {  // a stale or damaged cache entry: compile afresh
            from_disk[i] = false;
            compile(i);
            if (!ok[i]) return fail(O1D_JIT_ERROR, std::string("NVRTC failed for ") + kSrcName[i] + ":\n" + logs[i].substr(0, 4000));
            r = dr.moduleLoadData(&m->mod, cubin[i].data());
        }
        if (r == CUDA_SUCCESS) r = dr.moduleGetFunction(&m->fn, m->mod, sp->small ? "o1d_small" : kFnName[i]);
        if (r == CUDA_SUCCESS && i >= 2) r = dr.moduleGetFunction(&m->fin, m->mod, "o1d_wgrad_finalize");
        if (r != CUDA_SUCCESS) return fail(O1D_CUDA_ERROR, std::string("loading specialised kernel: ") + cu_err(r));
        const std::string &lg = logs[i];
        size_t fpos = lg.find(std::string("Compiling entry function '") + (sp->small ? "o1d_small" : kFnName[i]) + "'");
        size_t pos = lg.find("Used ", fpos == std::string::npos ? 0 : fpos);
        m->regs = pos == std::string::npos ? "?" : lg.substr(pos, lg.find('\n', pos) - pos);
        cache_put(device, src[i], m);
        sp->mod[i] = m;
    }
    for (int i : which) {
        if (i == 1 && sp->has[0] && src[1] == src[0]) sp->mod[1] = sp->mod[0];
        if (sp->small) {
            sp->smem[i] = sp->sl[i].total + 16;
            sp->threads[i] = sp->sl[i].threads();
        } else {
            const Lay &L = sp->lay[i];
            sp->smem[i] = L.total + 16;
            sp->threads[i] = 32 * (L.ncw() + L.NPROD);
        }
        CUresult r = dr.funcSetAttribute(sp->mod[i]->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)sp->smem[i]);
        int blocks = 0;
        if (r == CUDA_SUCCESS) r = dr.occupancy(&blocks, sp->mod[i]->fn, sp->threads[i], sp->smem[i]);
        if (r != CUDA_SUCCESS || blocks < 1)
            return fail(O1D_CUDA_ERROR, std::string("specialised kernel: ") + (r != CUDA_SUCCESS ? cu_err(r) : "zero occupancy"));
        sp->grid[i] = (int)std::min<long>(sp->small ? sp->small_items : planes, (long)blocks * sp->nsm);
    }
    return O1D_OK;
}

std::string describe_of(const o1d_plan *pl, const SpecSet *sp, bool all_hit) {
    char buf[1200];
    if (sp->small) {
        int len = snprintf(buf, sizeof buf,
                           "spec-small(32-plane items, 7x7 blocks at compile-time positions, %d tap tables, module cache %s",
                           sp->nt, all_hit ? "hit" : "miss");
        const char *pn[3] = {"fwd", "bwd_in", "wgrad"};
        for (int i = 0; i < 3 && len < (int)sizeof buf; ++i) {
            const SmallLay &L = sp->sl[i];
            if (sp->has[i] && sp->mod[i])
                len += snprintf(buf + len, sizeof buf - len, "; %s: %d quads x %d warps, %d slots, grid %d, smem %zu [%s]", pn[i],
                                L.NQ, L.QW, L.NS(), sp->grid[i], sp->smem[i], sp->mod[i]->regs.c_str());
            else
                len += snprintf(buf + len, sizeof buf - len, "; %s: generic", pn[i]);
        }
        if (len < (int)sizeof buf) snprintf(buf + len, sizeof buf - len, "; bwd_fused: generic)");
        return buf;
    }
    int len = snprintf(buf, sizeof buf,
                       "spec-v2(persistent warp-specialised, 7x7 blocks, %d tap tables, %d expanded taps/channel, module cache %s",
                       sp->nt, pl->KE, all_hit ? "hit" : "miss");
    const char *pn[kPasses] = {"fwd", "bwd_in", "wgrad", "bwd_fused"};
    for (int i = 0; i < kPasses && len < (int)sizeof buf; ++i) {
        if (sp->has[i] && sp->mod[i])
            len += snprintf(buf + len, sizeof buf - len, "; %s: %d pairs x %d warps, %d slots, grid %d, smem %zu [%s]", pn[i],
                            sp->lay[i].P, sp->lay[i].wpg, sp->lay[i].NS, sp->grid[i], sp->smem[i], sp->mod[i]->regs.c_str());
        else if (sp->has[i])
            len += snprintf(buf + len, sizeof buf - len, "; %s: compiled on first use", pn[i]);
        else
            len += snprintf(buf + len, sizeof buf - len, "; %s: generic", pn[i]);
    }
    if (len < (int)sizeof buf) snprintf(buf + len, sizeof buf - len, ")%s", sp->fused_step ? " step=fused" : "");
    return buf;
}
}  // namespace

o1d_status spec_create(o1d_plan *pl) {
    pl->spec = nullptr;
    const o1d_desc &d = pl->d;
    Driver &dr = drv();
    if (!dr.err.empty()) return O1D_OK;  // no driver entry points: generic path
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pl->device) != cudaSuccess || nsm < 1)
        return fail(O1D_CUDA_ERROR, "cannot query the SM count");
    std::unique_ptr<SpecSet> sp(new SpecSet());
    std::string src[kPasses];
    std::vector<int> gpc;
    if (!gpc_map(pl->device, &gpc)) gpc.clear();
    if (!spec_prepare(pl, sp.get(), src, nsm, &gpc)) return O1D_OK;
    if (const char *dir = getenv("O1D_DUMP_SOURCE")) {
        for (int i = 0; i < kPasses; ++i) {
            if (!sp->has[i]) continue;
            FILE *f = fopen((std::string(dir) + "/" + kSrcName[i]).c_str(), "w");
            if (f) {
                fputs(src[i].c_str(), f);
                fclose(f);
            }
        }
    }
    sp->pdl = env_int("O1D_PDL", 1) != 0;
    sp->fused_step = sp->has[3] && env_int("O1D_FUSED", 0) != 0;
    // the fused backward is compiled on its first use unless the step uses it (its code is the
    // backward_input and backward_weight cases together: the longest compile of the plan)
    std::vector<int> which;
    for (int i = 0; i < 3; ++i)
        if (sp->has[i]) which.push_back(i);
    if (sp->fused_step) which.push_back(3);
    else if (sp->has[3]) sp->src3 = src[3];
    bool all_hit = true;
    if (o1d_status st = load_passes(sp.get(), which, src, pl->device, (long)d.N * d.C, &all_hit)) return st;
    pl->jit_cache_hit = all_hit;
    const size_t nsched = (size_t)kPasses * kSlots * (sp->nt + 1) * kCS;
    if (cudaMalloc(&sp->d_sched, sizeof(unsigned) * nsched) != cudaSuccess ||
        cudaMemset(sp->d_sched, 0, sizeof(unsigned) * nsched) != cudaSuccess) {
        if (sp->d_sched) cudaFree(sp->d_sched);
        return fail(O1D_CUDA_ERROR, "scheduler counter allocation failed");
    }
    const char *tr = getenv("O1D_TRACE");
    if (tr && *tr && strcmp(tr, "0") != 0 && cudaMalloc(&sp->d_trace, kTraceBytes) == cudaSuccess)
        cudaMemset(sp->d_trace, 0, kTraceBytes);
    pl->describe = describe_of(pl, sp.get(), all_hit);
    if (getenv("O1D_VERBOSE")) fprintf(stderr, "[o1d] %s\n", pl->describe.c_str());
    pl->spec = sp.release();
    return O1D_OK;
}

// lazy load of the fused backward (pass 3), thread-safe
static o1d_status ensure_fused(const o1d_plan *pl) {
    SpecSet *sp = pl->spec;
    std::lock_guard<std::mutex> lk(sp->mu3);
    if (sp->mod[3]) return O1D_OK;
    std::string src[kPasses];
    src[3] = sp->src3;
    bool hit = true;
    if (o1d_status st = load_passes(sp, {3}, src, pl->device, (long)pl->d.N * pl->d.C, &hit)) return st;
    const_cast<o1d_plan *>(pl)->describe = describe_of(pl, sp, pl->jit_cache_hit);
    return O1D_OK;
}

void spec_destroy(o1d_plan *pl) {
    SpecSet *sp = pl->spec;
    if (!sp) return;
    if (sp->d_sched) cudaFree(sp->d_sched);
    if (sp->d_trace) cudaFree(sp->d_trace);
    delete sp;  // module references (unloaded when no plan and no cache slot holds them)
    pl->spec = nullptr;
}

bool spec_has(const o1d_plan *pl, int pass) { return pl->spec && pass >= 0 && pass < kPasses && pl->spec->has[pass]; }
bool spec_step_fused(const o1d_plan *pl) { return pl->spec && pl->spec->fused_step; }
// batch windows (o1d_step_host pipelining): every pass of the step on the specialised kernels
bool spec_window_ok(const o1d_plan *pl) {
    const SpecSet *sp = pl->spec;
    return sp && !sp->small && sp->has[0] && ((sp->has[1] && sp->has[2]) || sp->fused_step);
}
o1d_status spec_finalize(const o1d_plan *pl, int pass, float *dW, const float *ws, void *stream) {
    const SpecSet *sp = pl->spec;
    const void *wsp = ws;
    int N = pl->d.N;
    void *fargs[] = {&wsp, &dW, &N};
    CUlaunchAttribute attr[1];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[0].value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig fc{};
    fc.gridDimX = (unsigned)pl->d.C;
    fc.gridDimY = fc.gridDimZ = 1;
    fc.blockDimX = 256;
    fc.blockDimY = fc.blockDimZ = 1;
    fc.hStream = static_cast<CUstream>(stream);
    fc.attrs = attr;
    fc.numAttrs = sp->pdl ? 1 : 0;
    const CUresult r = drv().launchKernelEx(&fc, sp->mod[pass]->fin, fargs, nullptr);
    if (r != CUDA_SUCCESS) return fail(O1D_CUDA_ERROR, "launch of wgrad finalize: " + cu_err(r));
    return O1D_OK;
}
int spec_launches(const o1d_plan *, int pass) { return pass >= 2 ? 2 : 1; }
size_t spec_workspace_bytes(const o1d_plan *pl) {
    if (!pl->spec) return 0;
    if (pl->spec->small) return sizeof(float) * (size_t)pl->d.C * pl->spec->sl[2].G * pl->spec->sl[2].QW * pl->d.K;
    return sizeof(float) * (size_t)pl->d.N * pl->d.C * pl->spec->wpg * pl->d.K;
}

// kernel parameters (mirrors the generated `Params`)
struct alignas(64) HostParams {
    CUtensorMap in_map, out_map, aux_map;
    const float *w;
    void *io;
    float *ws;
    unsigned *sched;
    float *dW;
    unsigned long long *trace;
    int N, n0, nlen, nowait;
    const void *cvt1, *cvt2;
    const void *src1, *src2;
    void *dst;
};

// tensor maps / pointers of a small-plane launch: planes as rows of H*W elements, one box = the 32
// samples of one channel (TMA paths); raw pointers for the cp.async paths
static o1d_status small_maps(const o1d_plan *pl, int pass, const RunArgs &a, HostParams *hp) {
    const SpecSet *sp = pl->spec;
    const o1d_desc &d = pl->d;
    hp->src1 = pass == 1 ? a.dy : a.x;
    hp->src2 = a.dy;
    hp->dst = pass == 0 ? a.y : a.dx;
    if (sp->sl[pass].tma_out) {
        const int hwo = pass == 0 ? pl->P * pl->Q : d.H * d.W;
        if (o1d_status st = encode(&hp->out_map, hp->dst, d.dtype, hwo, 1, d.C, d.N, hwo, 1, 32)) return st;
    }
    if (sp->sl[pass].tma) {
        const int hwi = pass == 1 ? pl->P * pl->Q : d.H * d.W;
        if (o1d_status st = encode(&hp->in_map, hp->src1, d.dtype, hwi, 1, d.C, d.N, hwi, 1, 32)) return st;
        if (pass == 2)
            if (o1d_status st = encode(&hp->aux_map, a.dy, d.dtype, pl->P * pl->Q, 1, d.C, d.N, pl->P * pl->Q, 1, 32))
                return st;
    }
    return O1D_OK;
}

// tensor maps of a spec-v2 launch: ring-1 planes x (passes 0, 2, 3) or dy (pass 1), the output band
// (stencil) or dense dy box (backward_weight), ring-2 dy planes (fused)
static o1d_status ring_maps(const o1d_plan *pl, int pass, const RunArgs &a, HostParams *hp) {
    const SpecSet *sp = pl->spec;
    const o1d_desc &d = pl->d;
    const Lay &L = sp->lay[pass];
    const void *in = pass == 1 ? a.dy : a.x;
    const int inW = pass == 1 ? pl->Q : d.W, inH = pass == 1 ? pl->P : d.H;
    const bool cvt = d.dtype != O1D_F32;  // 16-bit rings are widened by the producers
    if (L.staged) {  // raw 16-bit plane, dense box (widened by the producer from its staging buffer)
        if (o1d_status st = L.flat ? encode(&hp->in_map, in, d.dtype, 8, inH * inW / 8, d.C, d.N, 8, L.hin * inW / 8)
                                   : encode(&hp->in_map, in, d.dtype, inW, inH, d.C, d.N, inW, L.hin))
            return st;
    } else if (cvt) {
        hp->cvt1 = in;
        hp->cvt2 = a.dy;
    } else if (o1d_status st = encode(&hp->in_map, in, d.dtype, inW, inH, d.C, d.N, L.pitch, L.hin)) {
        return st;
    }
    if (pass == 0 || pass == 1 || pass == 3) {  // dense output band box for the TMA store
        void *out = pass == 0 ? a.y : a.dx;
        const int oW = pass == 0 ? pl->Q : d.W, oH = pass == 0 ? pl->P : d.H;
        if (o1d_status st = L.flat ? encode(&hp->out_map, out, d.dtype, 8, oH * oW / 8, d.C, d.N, 8, std::min(oH, 4 * R) * oW / 8)
                                   : encode(&hp->out_map, out, d.dtype, oW, oH, d.C, d.N, oW, std::min(oH, 4 * R)))
            return st;
    }
    if (pass == 2)  // dy plane, rows padded to whole 7-row blocks (zero-filled)
        if (o1d_status st = L.flat ? encode(&hp->out_map, a.dy, d.dtype, 8, pl->P * pl->Q / 8, d.C, d.N, 8, L.dyrows * pl->Q / 8)
                                   : encode(&hp->out_map, a.dy, d.dtype, pl->Q, pl->P, d.C, d.N, L.dyp, L.dyrows))
            return st;
    if (pass == 3 && !cvt)  // dy planes for ring 2 (the dx stencil's input, the dy block of the partials)
        if (o1d_status st = encode(&hp->aux_map, a.dy, d.dtype, pl->Q, pl->P, d.C, d.N, L.pitch2, L.hin2)) return st;
    return O1D_OK;
}

o1d_status spec_run(const o1d_plan *pl, int pass, const RunArgs &a, void *stream, int n0, int nlen, bool finalize,
                    bool nowait) {
    if (nlen > 0 && !spec_window_ok(pl)) return fail(O1D_UNSUPPORTED, "batch windows need the specialised kernels");
    if (pass == 3)
        if (o1d_status st = ensure_fused(pl)) return st;
    const SpecSet *sp = pl->spec;
    const o1d_desc &d = pl->d;
    HostParams hp;
    std::memset(&hp, 0, sizeof hp);
    if (o1d_status st = sp->small ? small_maps(pl, pass, a, &hp) : ring_maps(pl, pass, a, &hp)) return st;
    hp.w = a.w;
    hp.ws = a.ws;
    hp.dW = a.dW;
    const unsigned slot = const_cast<SpecSet *>(sp)->launch_seq.fetch_add(1) % kSlots;
    hp.sched = sp->d_sched + ((size_t)pass * kSlots + slot) * (sp->nt + 1) * kCS;
    hp.trace = sp->d_trace;
    hp.N = d.N;
    hp.n0 = nlen > 0 ? n0 : 0;
    hp.nlen = nlen > 0 ? nlen : 0;
    hp.nowait = nowait ? 1 : 0;
    void *args[] = {&hp};
    CUlaunchAttribute attr[1];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[0].value.programmaticStreamSerializationAllowed = 1;
    CUlaunchConfig cfg{};
    cfg.gridDimX = (unsigned)sp->grid[pass];
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = (unsigned)sp->threads[pass];
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.sharedMemBytes = (unsigned)sp->smem[pass];
    cfg.hStream = static_cast<CUstream>(stream);
    cfg.attrs = attr;
    cfg.numAttrs = sp->pdl ? 1 : 0;
    CUresult r = drv().launchKernelEx(&cfg, sp->mod[pass]->fn, args, nullptr);
    if (r != CUDA_SUCCESS) return fail(O1D_CUDA_ERROR, "launch of specialised kernel: " + cu_err(r));
    if (pass >= 2 && finalize) return spec_finalize(pl, pass, a.dW, a.ws, stream);
    return O1D_OK;
}

size_t spec_trace(const o1d_plan *pl, void *host, size_t bytes) {
    const SpecSet *sp = pl->spec;
    if (!sp || !sp->d_trace) return 0;
    const size_t n = std::min(bytes, kTraceBytes);
    if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpy(host, sp->d_trace, n, cudaMemcpyDeviceToHost) != cudaSuccess)
        return 0;
    cudaMemset(sp->d_trace, 0, kTraceBytes);
    return n;
}

o1d_status spec_source(const o1d_plan *pl, int pass, std::string *out) {
    SpecSet sp;
    std::string src[kPasses];
    if (pass < 0 || pass >= kPasses) return fail(O1D_INVALID_ARG, "pass must be 0, 1, 2 or 3");
    if (!spec_prepare(pl, &sp, src, 148, nullptr) || !sp.has[pass])
        return fail(O1D_UNSUPPORTED, "plan is not eligible for a specialised kernel for this pass");
    *out = src[pass];
    return O1D_OK;
}

}  // namespace o1d
