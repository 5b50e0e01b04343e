// o1d_spec.cpp — runtime-specialised ("spec") kernels of liboriented1d.
//
// Why: the tap loop of Def. 1 is a stencil whose offsets depend on
// the angle.  With the offsets known at compile time, each thread can keep an
// R x S block of outputs in registers and load every input pixel its block
// needs from shared memory ONCE, feeding all (output, tap) pairs that use it
// (~6 shared loads per output at K=31 instead of 31).  The paper reached the
// same conclusion on its hardware ("a specific CUDA kernel for every input
// size"); here the specialisation is done at plan time with NVRTC for
// sm_100a, one case per distinct tap table of the plan.
//
// Per CTA: one (n, c) plane.  TMA (cp.async.bulk.tensor, 4-D map over
// W,H,C,N) stages the plane plus the table's halo into shared memory in one
// copy, the out-of-image part zero-filled by the TMA unit (reading R1); 64
// threads each own a 7x7 output block; the thread->block map and the smem
// pitch (= 8 mod 16 floats) make every LDS.32 of a warp conflict-free; outputs
// go registers -> smem -> TMA store.  backward_input is the same kernel with
// negated taps (stride 1).  backward_weight keeps the block's 49 dy values in
// registers, accumulates one partial per distinct tap, reduces them with a
// 31-shuffle reduce-scatter and a fixed-order CTA sum, and the last CTA of
// each channel (epoch counter) sums the N plane partials in f64, in n order:
// deterministic, one launch.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <atomic>
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
    PFN_cuLaunchKernel_v4000 launchKernel = nullptr;
    PFN_cuLaunchKernelEx_v11060 launchKernelEx = nullptr;
    PFN_cuTensorMapEncodeTiled_v12000 encodeTiled = nullptr;
    PFN_cuGetErrorString_v6000 getErrorString = nullptr;
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
                  entry("cuFuncSetAttribute", &d.funcSetAttribute, &e) && entry("cuLaunchKernel", &d.launchKernel, &e) &&
                  entry("cuTensorMapEncodeTiled", &d.encodeTiled, &e) && entry("cuGetErrorString", &d.getErrorString, &e) &&
                  entry("cuLaunchKernelEx", &d.launchKernelEx, &e);
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
    const char *opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--ptxas-options=-v",
                          "-DNDEBUG"};
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

// ------------------------------------------------------------ plan geometry
constexpr int R = 7, S = 7;  // per-thread output block (rows x cols)

struct Tap {
    int dh, dw;
    std::vector<int> ks;  // tap indices k sharing this offset (duplicates, reading R7)
};

struct Geo {  // one distinct tap table, one pass
    std::vector<Tap> taps;
    std::vector<int> k2d;  // k -> distinct index
    int minDH, maxDH, minDW, maxDW;
    int rows, pitch;       // TMA box (rows x pitch elements) = shared-memory tile
    int x0;                // first tile column in image coordinates (0: see make_geo)
    int guard;             // bytes of zeros in front of the tile (>= one pitch, 128-aligned)
    uint32_t bytes;        // TMA box bytes
};

int pitch_for(int cols) {
    int p = cols;
    while (p % 16 != 8) ++p;  // 7*pitch = 8 or 24 mod 32 -> conflict-free LDS.32
    return p;
}

// Tile geometry.  The box starts at image column 0 and is `pitch` wide, so the
// columns past the image edge are zero-filled by the TMA unit; a read left of
// column 0 wraps to the previous row's zero columns (pitch >= Win - minDW), and
// a zero guard row in front of the tile serves the first row.  The left halo
// therefore costs no shared memory, and the innermost TMA start coordinate is
// always 0 (TMA needs a 16-byte-aligned innermost start).
Geo make_geo(const int16_t *oh, const int16_t *ow, int K, bool negate, int BR, int BC, int es, int Win) {
    Geo g;
    std::map<std::pair<int, int>, int> idx;
    g.k2d.resize(K);
    g.minDH = g.minDW = 1 << 20;
    g.maxDH = g.maxDW = -(1 << 20);
    for (int k = 0; k < K; ++k) {
        const int dh = negate ? -oh[k] : oh[k], dw = negate ? -ow[k] : ow[k];
        auto it = idx.find({dh, dw});
        if (it == idx.end()) {
            it = idx.emplace(std::make_pair(dh, dw), (int)g.taps.size()).first;
            g.taps.push_back(Tap{dh, dw, {}});
        }
        g.taps[it->second].ks.push_back(k);
        g.k2d[k] = it->second;
        g.minDH = std::min(g.minDH, dh);
        g.maxDH = std::max(g.maxDH, dh);
        g.minDW = std::min(g.minDW, dw);
        g.maxDW = std::max(g.maxDW, dw);
    }
    g.x0 = 0;
    g.rows = R * BR + (g.maxDH - g.minDH);
    g.pitch = pitch_for(std::max(Win - std::min(g.minDW, 0), S * BC + std::max(g.maxDW, 0)));
    g.bytes = (uint32_t)(g.rows * g.pitch * es);
    g.guard = ((g.pitch * es) + 127) & ~127;
    return g;
}

}  // namespace

constexpr int kSlots = 64;  // concurrent launches per pass that can be in flight on one plan
constexpr int kCS = 32;     // scheduler counter stride (unsigned): one 128-byte line per counter
constexpr size_t kBalBytes = 2048;  // >= sizeof(Bal) in the generated prelude (1288 B)
constexpr size_t kTraceBytes = 8 + ((size_t)32 << 20);  // count + 2^21 (time, tag) records

struct SpecSet {
    int BR = 0, BC = 0, nthreads = 0, wpg = 0, G = 1, nt = 0, nsm = 0, gw = 1;
    bool v2 = false;                      // any pass on the v2 pipeline (one tap group, NS-slot ring, shared zero rows)
    bool v2p[3] = {false, false, false};  // per pass
    int pitch2[3] = {0, 0, 0}, rows2[3] = {0, 0, 0}, ns2 = 0;
    std::vector<Geo> fwd, bwd;  // per distinct table
    std::vector<int> count;     // planes per table
    CUmodule mod[3] = {nullptr, nullptr, nullptr};
    CUfunction fn[3] = {nullptr, nullptr, nullptr};
    CUfunction fin = nullptr;  // wgrad finalize
    size_t smem[3] = {0, 0, 0};
    int grid[3] = {0, 0, 0};
    int threads[3] = {0, 0, 0};
    // work-queue counters: 3 passes x kSlots launch slots x (NT next counters + 1 done counter);
    // every launch takes the next slot (host atomic), so concurrent launches on
    // different streams never share counters; a slot is reset by its last CTA
    unsigned *d_sched = nullptr;
    unsigned long long *d_trace = nullptr;  // diagnostics (O1D_TRACE=1): event records of the next launches
    unsigned char *d_bal = nullptr;         // adaptive placement state, kBalBytes per pass (v2)
    std::vector<int> home2[3];              // initial SM -> home table per pass (v2)
    std::atomic<unsigned> launch_seq{0};
    std::string regs[3];
};

namespace {

// ------------------------------------------------------------- code emission
const char *kPrelude = R"(
typedef unsigned long long u64;
typedef unsigned int u32;
struct __align__(64) TmaDesc { u64 v[16]; };
struct Params {
  TmaDesc in_map[NT];
  TmaDesc out_map;   // y / dx dense box (stencil TMA store)
  const float* w;
  void* io;          // y (forward) / dx (backward_input) / dy (wgrad)
  float* ws;
  unsigned* sched;   // [NT] next-plane counters, [NT] = done counter
  unsigned* cnt;     // [C] per-channel epoch counters (wgrad)
  float* dW;
  int only;          // >= 0: this launch processes table `only` alone (table-sequential mode)
  int adapt;         // 1: this launch measures per-table costs and updates the placement (every K-th launch)
  u64* trace;        // diagnostics (O1D_TRACE): [0] = record count, then (globaltimer, tag) pairs
  void* bal;         // v2 adaptive balance state (Bal) or null
  int n0, nlen;      // v2 batch window: planes with n in [n0, n0 + nlen) (nlen = 0: the whole batch)
  int nowait;        // 1: no griddepcontrol.wait (the inputs do not come from the preceding kernel, o1d_step)
};
// Adaptive placement (v2): consumers add their per-item busy cycles per table; the
// last consumer warp of a launch turns them into per-table costs (blended with the
// previous estimate) and rewrites the SM -> home-table map the next launch of the
// pass starts from: SMs per table in proportion to planes x measured cost, TPC pairs
// kept together, along the GPC-ordered SM list.  Placement only: results do not
// depend on which SM processes a plane.
struct Bal { u64 tsum[16]; unsigned tcnt[16]; float ema[16]; unsigned done; unsigned pad; unsigned home[256]; };
__device__ __forceinline__ void bal_flush(void* bv, int t, u64 busy, unsigned items) {
  Bal* b = reinterpret_cast<Bal*>(bv);
  if (b && t >= 0 && items) { atomicAdd(&b->tsum[t], busy); atomicAdd(&b->tcnt[t], items); }
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
__device__ __forceinline__ void mbar_expect(u64* b, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(b)), "r"(bytes) : "memory");
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
// streaming TMA load: the tile is read once, so it is marked evict-first in L2 (the
// kernel's code, constants and scheduler counters then stay L2-resident across launches)
__device__ __forceinline__ u64 policy_evict_first() {
  u64 p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ void tma_load_ef(void* dst, const TmaDesc* m, int x, int y, int z, int w, u64* b, u64 pol) {
  if (!pol) {
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 :: "r"(sa(dst)), "l"(m), "r"(x), "r"(y), "r"(z), "r"(w), "r"(sa(b)) : "memory");
    return;
  }
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;"
               :: "r"(sa(dst)), "l"(m), "r"(x), "r"(y), "r"(z), "r"(w), "r"(sa(b)), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const TmaDesc* m, int x, int y, int z, int w, u64* b) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
               :: "r"(sa(dst)), "l"(m), "r"(x), "r"(y), "r"(z), "r"(w), "r"(sa(b)) : "memory");
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
// 32 values per lane -> lane L returns the warp sum of v[L] (31 shuffles)
__device__ __forceinline__ float reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = lane & s;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = up ? v[i] : v[i + s];
      const float keep = up ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}
// Work scheduler (producer lane 0): per-table atomic counters handing out
// planes; a CTA starts on its SM's home table (so co-resident warps share one
// specialised code path in the instruction cache) and moves on to the next
// table when it is exhausted.  `raw` is a counter value fetched one plane
// ahead, so the atomic's latency is hidden behind a whole plane of compute.
// items of table t in this launch: all of it, or (CMAJOR item order) the planes of the
// batch window -- a contiguous item range nch * [0, nlen), shifted by n0 in item_cn
__device__ __forceinline__ int cnt_w(int t, int nlen) { return nlen > 0 ? (CHOFF[t + 1] - CHOFF[t]) * nlen : COUNT[t]; }
__device__ __forceinline__ int sched_resolve(unsigned* sched, int& tcur, unsigned& raw, int& tried, bool steal, int nlen = 0) {
  while (tcur >= 0) {
    if (raw < (unsigned)cnt_w(tcur, nlen)) return (tcur << 22) | (int)raw;
    if (++tried >= NT || !STEAL || !steal) { tcur = -1; break; }
    tcur = tcur + 1 == NT ? 0 : tcur + 1;
    raw = atomicAdd(sched + tcur * CS, 1u);
  }
  return -1;
}
// v2 scheduler (producer lane 0): items are taken in batches of GB consecutive
// indices of the current table with the next batch's atomic always in flight, so
// a producer serving several consumer pairs is not limited to one item per
// atomic round trip (~1 us under load)
__device__ __forceinline__ int sched2_next(unsigned* sched, int& tcur, unsigned& lo, unsigned& hi, unsigned& nxt,
                                           int& tried, bool steal) {
  while (tcur >= 0) {
    if (lo < hi && lo < (unsigned)COUNT[tcur]) return (tcur << 22) | (int)(lo++);
    if (nxt < (unsigned)COUNT[tcur]) { lo = nxt; hi = nxt + GB; nxt = atomicAdd(sched + tcur * CS, (unsigned)GB); continue; }
    if (++tried >= NT || !STEAL || !steal) { tcur = -1; break; }
    tcur = tcur + 1 == NT ? 0 : tcur + 1;
    lo = hi = 0;
    nxt = atomicAdd(sched + tcur * CS, (unsigned)GB);
  }
  return -1;
}
__device__ __forceinline__ void sched_prefetch(unsigned* sched, int tcur, unsigned& raw) {
  if (tcur >= 0) raw = atomicAdd(sched + tcur * CS, 1u);
}
__device__ __forceinline__ void item_cn(int item, int& t, int& c, int& n, int n0 = 0) {
  t = (item >> 22) & 31;   // bits 27..29: batch flags (v2 wgrad)
  const int i = item & 0x3FFFFF;
#if CMAJOR
  // consecutive items walk the table's channels first: the planes in flight on the GPU
  // form a compact address range (n-major walks stride C*H*W apart)
  const int nch = CHOFF[t + 1] - CHOFF[t];
  n = i / nch;
  c = CHLIST[CHOFF[t] + (i - n * nch)];
  n += n0;
#else
  c = CHLIST[CHOFF[t] + i / NB];
  n = i - (i / NB) * NB;
#endif
}
// Called by all 32 lanes of the last consumer warp of the launch: per-table costs in
// parallel (lane t), then every lane places its share of the TPC pairs (prefix-sum
// search over the table works) -- no serial chain of global-memory round trips.
__device__ void bal_exit(void* bv, int lane) {
#if NORD > 0
  Bal* b = reinterpret_cast<Bal*>(bv);
  float wk = 0.f;
  if (lane < NT) {
    const unsigned n = *((volatile unsigned*)&b->tcnt[lane]);
    const float ema = *((volatile float*)&b->ema[lane]);
    const float m = n ? (float)(*((volatile u64*)&b->tsum[lane])) / (float)n : ema;
    const float e = ema > 0.f ? 0.5f * (ema + m) : m;
    wk = (float)COUNT[lane] * (e > 0.f ? e : 1.f);
    b->ema[lane] = e;
    b->tsum[lane] = 0ull;
    b->tcnt[lane] = 0u;
  }
  float pre[NT + 1];
  pre[0] = 0.f;
#pragma unroll
  for (int q = 0; q < NT; ++q) pre[q + 1] = pre[q] + __shfl_sync(0xffffffffu, wk, q);
  const float tot = pre[NT];
  unsigned have = 0u;   // tables this lane assigned at least one pair to
  int mine[(NORD / 2 + 31) / 32];
#pragma unroll
  for (int k = 0; k < (NORD / 2 + 31) / 32; ++k) {
    const int i = 2 * (lane + 32 * k);
    mine[k] = -1;
    if (i < NORD) {
      const float pos = (i + 1.f) * tot / NORD;
      int t = 0;
      while (t < NT - 1 && pos >= pre[t + 1]) ++t;
      mine[k] = t;
      have |= 1u << t;
    }
  }
  unsigned all_t = __reduce_or_sync(0xffffffffu, have);
  bool cover = true;
#pragma unroll
  for (int q = 0; q < NT; ++q) cover = cover && (((all_t >> q) & 1u) || COUNT[q] == 0);
  if (cover) {
#pragma unroll
    for (int k = 0; k < (NORD / 2 + 31) / 32; ++k) {
      const int i = 2 * (lane + 32 * k);
      if (i < NORD) {
        b->home[ORDER[i]] = (unsigned)mine[k];
        if (i + 1 < NORD) b->home[ORDER[i + 1]] = (unsigned)mine[k];
      }
    }
  }
  if (lane == 0) b->done = 0u;
  __threadfence();
#endif
}
// CTA-level accounting in shared memory: [16] u64 busy cycles, [16] u32 items, u32 warps done
__device__ __forceinline__ void bal_flush_cta(unsigned char* sb, int t, u64 busy, unsigned items) {
  if (t < 0 || !items) return;
  atomicAdd(reinterpret_cast<u64*>(sb) + t, busy);
  atomicAdd(reinterpret_cast<unsigned*>(sb + 128) + t, items);
}
// the last consumer warp of the CTA moves the CTA's totals to the global state (one set of
// atomics per CTA, not per warp: per-warp global atomics serialised ~1200 warps at kernel end)
__device__ void bal_warp_exit(void* bv, unsigned char* sb, int t, u64 busy, unsigned items, unsigned ncw, int lane) {
  // (all lanes) lane 0 adds the warp's totals to the CTA's; the CTA's last consumer warp adds
  // the CTA's totals to the launch's (one set of global atomics per CTA); the launch's last
  // CTA recomputes the placement
  int last = 0;
  if (lane == 0) {
    bal_flush_cta(sb, t, busy, items);
    __threadfence_block();
    if (atomicAdd(reinterpret_cast<unsigned*>(sb + 192), 1u) == ncw - 1) {
      __threadfence_block();
      for (int q = 0; q < NT; ++q) {
        const unsigned n = *((volatile unsigned*)(sb + 128) + q);
        if (n) bal_flush(bv, q, *((volatile u64*)sb + q), n);
      }
      __threadfence();
      last = atomicAdd(&reinterpret_cast<Bal*>(bv)->done, 1u) == gridDim.x - 1;
      __threadfence();
    }
  }
  if (__shfl_sync(0xffffffffu, last, 0)) bal_exit(bv, lane);
}
__device__ __forceinline__ void sched_exit(unsigned* sched, unsigned per_cta = 1) {
  __threadfence();
  if (atomicAdd(sched + NT * CS, 1u) == gridDim.x * per_cta - 1) {
    for (int t = 0; t < NT; ++t) sched[t * CS] = 0u;
    sched[NT * CS] = 0u;
    __threadfence();
  }
}
)";

bool env_flag(const char *n) {
    const char *v = getenv(n);
    return v && *v && strcmp(v, "0") != 0;
}

int env_int(const char *n, int dflt) {
    const char *v = getenv(n);
    return (v && *v) ? atoi(v) : dflt;
}

struct Ctx {
    int N, C, K, Ho, Wo, BR, BC, wpg, G, nt, nsm;  // wpg: warps (bands) per tap group; G: tap groups
    bool ffma2 = false;                                  // packed fp32 FMA in the stencil
    bool ffma2_w = false;                                // packed fp32 FMA in wgrad (measured slower: 74 vs 64 us)
    int minb = 1;                                        // __launch_bounds__ min blocks per SM (stencil)
    int gw = 2;                                          // tap groups of the wgrad kernel
    int act = 0;                                         // activation dtype (o1d_dtype)
    std::vector<int> home;                               // home table per %smid (empty: TPC-pair fallback)
    std::vector<int> order;                              // SMs in GPC order (adaptive placement; empty: off)
    bool steal = true;                                   // CTAs move to other tables once theirs is done
    bool convert = false;                                // 16-bit tiles widened to an fp32 smem copy
    bool v2 = false;                                     // v2 pipeline (see gen_stencil2)
    int nthreads() const { return 32 * wpg * G; }
};

void emit_header(std::ostringstream &os, const Ctx &x, const std::vector<int> &table_of, const std::vector<int> &count) {
    os << "#define NT " << x.nt << "\n#define NB " << x.N << "\n#define STEAL " << (x.steal ? 1 : 0) << "\n"
       << "#define GB " << std::max(1, env_int("O1D_GRAB", 1)) << "\n"
       << "#define CS " << kCS << "   // scheduler counters 128 bytes apart (one L2 line each: no atomic contention between tables)\n"
       << "#define CMAJOR " << env_int("O1D_CMAJOR", 1) << "\n";
    // tile reads: fp32 copy (convert path) or the raw activation tile
    os << (x.convert ? "#define LDT(v) (v)\n" : "#define LDT(v) LD(v)\n");
    // activation element type in shared memory / HBM; arithmetic is fp32 throughout
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
    os << "__constant__ int COUNT[" << x.nt << "] = {";
    for (int t = 0; t < x.nt; ++t) os << (t ? "," : "") << count[t];
    os << "};\n";
    std::vector<int> choff(x.nt + 1, 0), chlist;
    for (int t = 0; t < x.nt; ++t) {
        choff[t] = (int)chlist.size();
        for (int c = 0; c < x.C; ++c)
            if (table_of[c] == t) chlist.push_back(c);
    }
    choff[x.nt] = (int)chlist.size();
    os << "__constant__ int CHOFF[" << x.nt + 1 << "] = {";
    for (int t = 0; t <= x.nt; ++t) os << (t ? "," : "") << choff[t];
    os << "};\n__constant__ short CHLIST[" << x.C << "] = {";
    for (int c = 0; c < x.C; ++c) os << (c ? "," : "") << chlist[c];
    os << "};\n";
    // home table per SM (see home_tables()); fallback without a topology probe:
    // (smid / 2) mod NT, i.e. TPC pairs share a table
    os << "#define NORD " << x.order.size() << "\n";
    if (!x.order.empty()) {
        os << "__constant__ unsigned char ORDER[" << x.order.size() << "] = {";
        for (size_t i = 0; i < x.order.size(); ++i) os << (i ? "," : "") << x.order[i];
        os << "};\n";
    }
    const int nh = x.home.empty() ? x.nsm : (int)x.home.size();
    os << "#define NHOME " << nh << "\n__constant__ unsigned char HOME[" << nh << "] = {";
    for (int s = 0; s < nh; ++s) os << (s ? "," : "") << (x.home.empty() ? (s / 2) % x.nt : x.home[s]);
    os << "};\n" << kPrelude;
}

// Estimated issue cost of a contiguous range of distinct taps for one 7x7 block:
// 4 packed/scalar FMA instructions per (row, tap) + one LDS per footprint pixel.
int range_cost(const Geo &g, int lo, int hi) {
    std::set<std::pair<int, int>> px;
    for (int d = lo; d < hi; ++d)
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s) px.insert({r + g.taps[d].dh, s + g.taps[d].dw});
    return 4 * R * (hi - lo) + (int)px.size();
}

// Distinct taps of tap group gi: contiguous ranges of the distinct-tap list whose
// boundaries balance the estimated cost (groups run on different warps that
// meet at the output combine, so the slowest group sets the pace).
int pair_axis(const Geo &g);
int parity_of(int v);
thread_local bool g_parity_groups = true;  // set per plan (O1D_PARITY)

std::vector<int> group_taps(const Geo &g, int gi, int G) {
    const int nd = (int)g.taps.size();
    if (G == 2 && g_parity_groups) {  // parity of the offset along the table's pair axis
        const int axis = pair_axis(g);
        std::vector<int> v;
        for (int d = 0; d < nd; ++d)
            if (parity_of(axis == 0 ? g.taps[d].dh : g.taps[d].dw) == gi) v.push_back(d);
        if (!v.empty() || gi == 1) return v;
    }
    std::vector<int> cut(G + 1, 0);
    cut[G] = nd;
    for (int q = 1; q < G; ++q) cut[q] = (q * nd) / G;
    if (G == 2) {  // exact search of the single cut point
        int best = 1 << 30;
        for (int c = 1; c < nd; ++c) {
            const int m = std::max(range_cost(g, 0, c), range_cost(g, c, nd));
            if (m < best) best = m, cut[1] = c;
        }
    }
    std::vector<int> v;
    for (int d = cut[gi]; d < cut[gi + 1]; ++d) v.push_back(d);
    return v;
}

// For each footprint pixel (row i, col j relative to the block's top-left) of the
// taps `ds`, the (distinct tap, r, s) uses: one LDS per needed input pixel, then
// the FMAs that consume it (the register-blocked form of Def. 1's sum over k).
template <typename F>
void for_each_pixel(const Geo &g, const std::vector<int> &ds, F &&f) {
    int lo_h = 1 << 20, hi_h = -(1 << 20);
    for (int d : ds) lo_h = std::min(lo_h, g.taps[d].dh), hi_h = std::max(hi_h, g.taps[d].dh);
    for (int i = lo_h; i <= hi_h + R - 1; ++i) {
        std::vector<std::pair<int, int>> pairs;  // (r, distinct tap)
        for (int r = 0; r < R; ++r)
            for (int d : ds)
                if (g.taps[d].dh == i - r) pairs.push_back({r, d});
        if (pairs.empty()) continue;
        int lo = 1 << 20, hi = -(1 << 20);
        for (auto &p : pairs) {
            lo = std::min(lo, g.taps[p.second].dw);
            hi = std::max(hi, g.taps[p.second].dw + S - 1);
        }
        for (int j = lo; j <= hi; ++j) {
            std::vector<std::pair<int, std::pair<int, int>>> uses;  // (d, (r, s))
            for (auto &p : pairs) {
                const int s = j - g.taps[p.second].dw;
                if (s >= 0 && s < S) uses.push_back({p.second, {p.first, s}});
            }
            if (uses.empty()) continue;
            f(i, j, uses);
        }
    }
}

// I-cache warm-up chunks (v2): the straight-line tap code of a table is split into
// g_chunks guarded chunks `if (wm & bit) { ... }`; a real item runs them all
// (wm = ~0), the warm-up pass at kernel start runs one chunk per consumer warp so
// the cold code is fetched by all warps in parallel (measured: the first tap loop
// of a table otherwise takes ~10 us of instruction fetch instead of ~1.6 us).
thread_local int g_chunks = 0;  // (generator state: plans may be created from several threads)
#define EFH (env_int("O1D_EF", 1) != 0)  // evict-first L2 hints on the streaming TMA traffic (v2)
#define YST (env_int("O1D_YSTORE", 0) != 0)  // stencil outputs by warp copy instead of TMA band store
#define YSTG (env_int("O1D_YSTG", 0) != 0)   // stencil outputs stored from registers (no staging band)
// stencil outputs staged in the consumed tile slot (v2).  Off: measured 48.1 vs 45.2 us forward at
// P = 4 (pair barrier + deferred slot release), and the extra pair it makes room for (P = 5) was slower still
#define INSLOT (env_int("O1D_INSLOT", 0) != 0)
struct Chunker {
    std::ostringstream &os;
    const char *ind;
    int total, n, cur = -1;
    void at(int idx) {
        if (n <= 1 || total <= 0) return;
        const int k = (int)((long)idx * n / total);
        if (k == cur) return;
        if (cur >= 0) os << ind << "}\n";
        os << ind << "if (wm & " << (1u << k) << "u) {\n";
        cur = k;
    }
    void end() {
        if (n > 1 && cur >= 0) os << ind << "}\n";
    }
};

size_t tile_bytes_of(const std::vector<Geo> &geo) {
    size_t b = 0;
    for (auto &g : geo) b = std::max(b, (size_t)g.guard + g.bytes);
    return (b + 1023) & ~(size_t)1023;
}

// fp32 copy of a 16-bit tile (convert path): same pitch/rows, fp32 guard
int guard32(const Geo &g) { return ((g.pitch * 4) + 127) & ~127; }
size_t tile32_bytes_of(const std::vector<Geo> &geo) {
    size_t b = 0;
    for (auto &g : geo) b = std::max(b, (size_t)guard32(g) + (size_t)g.rows * g.pitch * 4);
    return (b + 1023) & ~(size_t)1023;
}

// emitted by the consumer warps of a converted (16-bit) plan right after the tile
// of ring buffer b landed: widen it to fp32 once (conflict-free sequential
// LDS.32 -> STS.64), release the 16-bit buffer to the producer, and compute from
// the fp32 copy with the conflict-free fp32 lane map.
void emit_convert(std::ostringstream &os, const Ctx &x, const std::vector<Geo> &geo, size_t TB, size_t OFF32,
                  int ncw) {
    const int nc = 32 * ncw;
    os << "    asm volatile(\"bar.sync 13, " << nc << ";\" ::: \"memory\");  // previous fp32 tile fully consumed\n"
       << "    {\n      const int ctid = tid - 32;\n      switch (t) {\n";
    for (int q = 0; q < x.nt; ++q) {
        const Geo &g = geo[q];
        const int npairs = g.rows * g.pitch / 2;
        os << "      case " << q << ": {\n"
           << "        const unsigned* src = reinterpret_cast<const unsigned*>(smem + b * " << TB << " + " << g.guard << ");\n"
           << "        float2* dst = reinterpret_cast<float2*>(smem + " << OFF32 + guard32(g) << ");\n"
           << "        for (int e = ctid; e < " << npairs << "; e += " << nc << ") { const unsigned v = src[e]; dst[e] = "
           << (x.act == O1D_BF16 ? "make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xffff0000u));"
                                 : "make_float2(h2f((unsigned short)(v & 0xffffu)), h2f((unsigned short)(v >> 16)));")
           << " }\n        break;\n      }\n";
    }
    os << "      }\n    }\n"
       << "    asm volatile(\"bar.arrive %0, %1;\" :: \"r\"(14 + b), \"r\"(" << 32 * (ncw + 1) << ") : \"memory\");  // 16-bit buffer free\n"
       << "    asm volatile(\"bar.sync 13, " << nc << ";\" ::: \"memory\");  // fp32 tile complete\n";
}

size_t stage_bytes_of(const Ctx &x) {
    const int rows = ((x.BR * R + 4 * R - 1) / (4 * R)) * (4 * R);  // whole 4*7-row bands
    return ((size_t)rows * x.Wo * 4 + 1023) & ~(size_t)1023;
}

// List schedule of independent accumulator updates: repeatedly emit the update whose
// accumulator was used least recently (ties: original order), so dependent FMAs on one
// accumulator are spread out (O1D_LRU=0: keep the given order).
void emit_lru(std::ostringstream &os, const char *ind, std::vector<std::pair<std::string, std::string>> &fm,
              std::map<std::string, long> &last_use, long &clock) {
    if (!env_int("O1D_LRU", 1)) {
        for (auto &f : fm) os << ind << f.second << "\n";
        return;
    }
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

// Stencil taps of group `ds` with packed FFMA2: output columns are paired
// (s, s+1) so that the pixel pair starts at an even column relative to the
// block: taps with even dw accumulate into pairs (0,1),(2,3),(4,5) + scalar 6
// (set A), taps with odd dw into pairs (1,2),(3,4),(5,6) + scalar 0 (set B).
// Every pixel pair is then an even-aligned (v_j, v_j+1) register pair.  The
// two sets are added at the end: a_rs = A_rs + B_rs.
void emit_stencil_compute_ffma2(std::ostringstream &os, const Geo &g, const std::vector<int> &ds, const char *ind) {
    for (int d : ds) {
        os << ind << "const float m" << d << " = ";
        for (size_t q = 0; q < g.taps[d].ks.size(); ++q) os << (q ? " + " : "") << "wv[" << g.taps[d].ks[q] << "]";
        os << ";\n" << ind << "const u64 M" << d << " = f2pack(m" << d << ", m" << d << ");\n";
    }
    for (int r = 0; r < R; ++r)
        os << ind << "u64 A" << r << "_0 = 0ull, A" << r << "_2 = 0ull, A" << r << "_4 = 0ull; float A" << r
           << "_6 = 0.f;\n"
           << ind << "u64 B" << r << "_1 = 0ull, B" << r << "_3 = 0ull, B" << r << "_5 = 0ull; float B" << r
           << "_0 = 0.f;\n";
    int lo_h = 1 << 20, hi_h = -(1 << 20);
    for (int d : ds) lo_h = std::min(lo_h, g.taps[d].dh), hi_h = std::max(hi_h, g.taps[d].dh);
    // rows of the block footprint: (i, (r, d) uses, pixels to load, even-aligned pairs)
    struct Row {
        int i;
        std::vector<std::pair<int, int>> pairs;
        std::set<int> need, pr;
    };
    std::vector<Row> rows;
    for (int i = lo_h; i <= hi_h + R - 1; ++i) {
        Row rw{i, {}, {}, {}};
        for (int r = 0; r < R; ++r)
            for (int d : ds)
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
    auto cn = [](int v) { return v < 0 ? "m" + std::to_string(-v) : std::to_string(v); };
    auto vname = [&](int i, int j) { return "v" + cn(i) + "_" + cn(j); };
    auto pname = [&](int i, int j) { return "P" + cn(i) + "_" + cn(j); };
    // loads of footprint row k are emitted LA rows ahead of its FMAs (software pipelining:
    // with two consumer warps per SM sub-partition the LDS latency is otherwise exposed)
    // (the look-ahead stays inside one warm-up chunk: values never cross a chunk guard)
    const int LA = std::max(0, env_int("O1D_LA", 1));
    auto loads = [&](const Row &rw) {
        for (int j : rw.need)
            os << ind << "const float " << vname(rw.i, j) << " = LDT(tb[" << (rw.i - g.minDH) * g.pitch + (j - g.x0) << "]);\n";
        for (int j : rw.pr)
            os << ind << "const u64 " << pname(rw.i, j) << " = f2pack(" << vname(rw.i, j) << ", " << vname(rw.i, j + 1) << ");\n";
    };
    const int nrows = (int)rows.size();
    auto chunk_of = [&](int k) { return g_chunks > 1 ? (int)((long)k * g_chunks / nrows) : 0; };
    Chunker ch{os, ind, nrows, g_chunks};
    std::map<std::string, long> last_use;
    long clock = 0;
    for (int k = 0; k < nrows; ++k) {
        ch.at(k);
        const bool first = k == 0 || chunk_of(k - 1) != chunk_of(k);
        if (first)  // chunk start: this row and the look-ahead rows of the chunk
            for (int k2 = k; k2 <= k + LA && k2 < nrows && chunk_of(k2) == chunk_of(k); ++k2) loads(rows[k2]);
        else if (k + LA < nrows && chunk_of(k + LA) == chunk_of(k))
            loads(rows[k + LA]);
        const Row &rw = rows[k];
        // the row's FMAs, then a list schedule that keeps updates of one accumulator as far
        // apart as possible (measured: near-horizontal tables put all taps of a footprint
        // row on the same output row, and a slot-major order then chained every second
        // FFMA2 on one accumulator: fixed-latency "wait" stalls)
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
            }
        emit_lru(os, ind, fm, last_use, clock);
    }
    ch.end();
    for (int r = 0; r < R; ++r) {
        os << ind << "a" << r << "_0 = f2lo(A" << r << "_0) + B" << r << "_0;\n"
           << ind << "a" << r << "_1 = f2hi(A" << r << "_0) + f2lo(B" << r << "_1);\n"
           << ind << "a" << r << "_2 = f2lo(A" << r << "_2) + f2hi(B" << r << "_1);\n"
           << ind << "a" << r << "_3 = f2hi(A" << r << "_2) + f2lo(B" << r << "_3);\n"
           << ind << "a" << r << "_4 = f2lo(A" << r << "_4) + f2hi(B" << r << "_3);\n"
           << ind << "a" << r << "_5 = f2hi(A" << r << "_4) + f2lo(B" << r << "_5);\n"
           << ind << "a" << r << "_6 = A" << r << "_6 + f2hi(B" << r << "_5);\n";
    }
}

// O1D_W8 (v2 stencils, fp32): every lane computes an 8-column block that starts at
// an even column -- 7*bc for even bc, 7*bc - 1 for odd bc -- and keeps 7 of its 8
// outputs.  All pixel pairs are then 8-byte aligned and load with one LDS.64 each
// (with 7-column blocks half the lanes start at an odd column and every pair is
// two LDS.32); even-dw taps run as 4 FFMA2 per row, odd-dw taps as 3 FFMA2 + 2 FFMA.
// Off: parity-green but measured 62 vs 44 us forward (166 registers; the 8-byte
// loads of a half-warp hit 2-way bank conflicts for every pitch with this lane map,
// and the eighth column adds 14% FMAs)
#define W8 (env_int("O1D_W8", 0) != 0)
void emit_stencil_compute_w8(std::ostringstream &os, const Geo &g, const std::vector<int> &ds, const char *ind) {
    for (int d : ds) {
        os << ind << "const float m" << d << " = ";
        for (size_t q = 0; q < g.taps[d].ks.size(); ++q) os << (q ? " + " : "") << "wv[" << g.taps[d].ks[q] << "]";
        os << ";\n" << ind << "const u64 M" << d << " = f2pack(m" << d << ", m" << d << ");\n";
    }
    for (int r = 0; r < R; ++r)
        os << ind << "u64 A" << r << "_0 = 0ull, A" << r << "_2 = 0ull, A" << r << "_4 = 0ull, A" << r << "_6 = 0ull;\n"
           << ind << "u64 B" << r << "_1 = 0ull, B" << r << "_3 = 0ull, B" << r << "_5 = 0ull; float B" << r << "_0 = 0.f, B" << r
           << "_7 = 0.f;\n";
    int lo_h = 1 << 20, hi_h = -(1 << 20);
    for (int d : ds) lo_h = std::min(lo_h, g.taps[d].dh), hi_h = std::max(hi_h, g.taps[d].dh);
    struct Row {
        int i;
        std::vector<std::pair<int, int>> pairs;
        std::set<int> even;   // aligned pairs (e, e + 1) to load
    };
    std::vector<Row> rows;
    for (int i = lo_h; i <= hi_h + R - 1; ++i) {
        Row rw{i, {}, {}};
        for (int r = 0; r < R; ++r)
            for (int d : ds)
                if (g.taps[d].dh == i - r) rw.pairs.push_back({r, d});
        if (rw.pairs.empty()) continue;
        for (auto &p : rw.pairs) {
            const int dw = g.taps[p.second].dw;
            for (int s = 0; s < 8; ++s) rw.even.insert((dw + s) & ~1);   // (v & ~1: floor to even, also for v < 0)
        }
        rows.push_back(rw);
    }
    auto cn = [](int v) { return v < 0 ? "m" + std::to_string(-v) : std::to_string(v); };
    auto qname = [&](int i, int e) { return "Q" + cn(i) + "_" + cn(e); };
    auto scal = [&](int i, int j) {  // pixel j of row i as a float (half of its aligned pair)
        return std::string("f2") + ((j & 1) ? "hi(" : "lo(") + qname(i, j & ~1) + ")";
    };
    const int LA = std::max(0, env_int("O1D_LA", 1));
    auto loads = [&](const Row &rw) {
        for (int e : rw.even) {
            const int off = rw.i * g.pitch + e;   // even: pitch is even and the lane base is even
            os << ind << "const u64 " << qname(rw.i, e) << " = *reinterpret_cast<const u64*>(tb + " << off << ");\n";
        }
    };
    const int nrows = (int)rows.size();
    auto chunk_of = [&](int k) { return g_chunks > 1 ? (int)((long)k * g_chunks / nrows) : 0; };
    Chunker ch{os, ind, nrows, g_chunks};
    std::map<std::string, long> last_use;
    long clock = 0;
    for (int k = 0; k < nrows; ++k) {
        ch.at(k);
        const bool first = k == 0 || chunk_of(k - 1) != chunk_of(k);
        if (first)
            for (int k2 = k; k2 <= k + LA && k2 < nrows && chunk_of(k2) == chunk_of(k); ++k2) loads(rows[k2]);
        else if (k + LA < nrows && chunk_of(k + LA) == chunk_of(k))
            loads(rows[k + LA]);
        const Row &rw = rows[k];
        std::vector<std::pair<std::string, std::string>> fm;
        for (int q = 0; q < 5; ++q)
            for (auto &p : rw.pairs) {
                const int r = p.first, d = p.second, dw = g.taps[d].dw;
                const std::string rs = std::to_string(r);
                std::ostringstream st;
                std::string acc;
                if (((dw % 2) + 2) % 2 == 0) {
                    if (q == 4) continue;
                    acc = "A" + rs + "_" + std::to_string(2 * q);
                    st << acc << " = ffma2(" << qname(rw.i, dw + 2 * q) << ", M" << d << ", " << acc << ");";
                } else if (q < 3) {
                    acc = "B" + rs + "_" + std::to_string(2 * q + 1);
                    st << acc << " = ffma2(" << qname(rw.i, dw + 2 * q + 1) << ", M" << d << ", " << acc << ");";
                } else {
                    const int s = q == 3 ? 0 : 7;
                    acc = "B" + rs + "_" + std::to_string(s);
                    st << acc << " = fmaf(" << scal(rw.i, dw + s) << ", m" << d << ", " << acc << ");";
                }
                fm.push_back({acc, st.str()});
            }
        emit_lru(os, ind, fm, last_use, clock);
    }
    ch.end();
    os << ind << "const bool oddb = bc & 1;   // odd lanes keep outputs 1..7 of their block, even lanes 0..6\n";
    for (int r = 0; r < R; ++r) {
        const std::string rs = std::to_string(r);
        os << ind << "{\n"
           << ind << "  const float o0 = f2lo(A" << rs << "_0) + B" << rs << "_0, o1 = f2hi(A" << rs << "_0) + f2lo(B" << rs << "_1);\n"
           << ind << "  const float o2 = f2lo(A" << rs << "_2) + f2hi(B" << rs << "_1), o3 = f2hi(A" << rs << "_2) + f2lo(B" << rs << "_3);\n"
           << ind << "  const float o4 = f2lo(A" << rs << "_4) + f2hi(B" << rs << "_3), o5 = f2hi(A" << rs << "_4) + f2lo(B" << rs << "_5);\n"
           << ind << "  const float o6 = f2lo(A" << rs << "_6) + f2hi(B" << rs << "_5), o7 = f2hi(A" << rs << "_6) + B" << rs << "_7;\n";
        for (int c = 0; c < 7; ++c)
            os << ind << "  a" << rs << "_" << c << " = oddb ? o" << c + 1 << " : o" << c << ";\n";
        os << ind << "}\n";
    }
}

// Warp-specialised stencil kernel (forward / backward_input):
//   warp 0        producer: schedules planes, stages weights, issues TMA loads
//                 into a 2-deep ring of tiles (mbarriers full[2] / empty[2])
//   warps 1..     consumers: 7x7 register blocks, G tap groups; after the tap
//                 loop each warp releases the tile (empty arrive) and the
//                 groups combine through the staging tile with pairwise named
//                 barriers; group 0 warps TMA-store their own 4*7-row band.
// No CTA-wide barrier in the steady state.
// ---------------------------------------------------------------------------
// Parity tap groups + packed FP32 (FFMA2) along one axis.
//
// With two tap groups, taps are split by the parity of their offset along the
// table's "pair axis" (rows if the dh parities are balanced, else columns).
// Outputs (stencil) or dy values (wgrad) are paired along that axis — rows
// (0,1),(2,3),(4,5) + row 6, or columns likewise — so the pixel pair of every
// FFMA2 starts at a coordinate of the group's parity: each loaded pixel sits in
// exactly one register pair and no copies are needed.
// ---------------------------------------------------------------------------
int parity_of(int v) { return ((v % 2) + 2) % 2; }

// 0: pair along rows (uses dh parity), 1: along columns (dw parity)
int pair_axis(const Geo &g) {
    int ev = 0, od = 0, ew = 0, ow = 0;
    for (auto &t : g.taps) (parity_of(t.dh) ? od : ev)++, (parity_of(t.dw) ? ow : ew)++;
    return std::abs(ev - od) <= std::abs(ew - ow) ? 0 : 1;
}

std::string coord(int v) { return v < 0 ? "m" + std::to_string(-v) : std::to_string(v); }

// One FMA of the paired formulation: accumulator `acc` (pair or scalar),
// pixel (i, j) [pair: with its partner one step along the axis], tap d, and
// the (r, s) of the output (stencil) / dy value (wgrad) it multiplies.
struct PairOp {
    bool pair;
    int d, r, s, i, j;
};

// ops for taps `ds` of table g along `axis`, ordered by footprint row (liveness)
// and slot-major within a row (independent accumulators back to back)
std::vector<PairOp> pair_ops(const Geo &g, const std::vector<int> &ds, int axis) {
    std::vector<PairOp> ops;
    for (int d : ds) {
        const int dh = g.taps[d].dh, dw = g.taps[d].dw;
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s) {
                const int u = axis == 0 ? r : s;  // coordinate along the pair axis
                if (u == 6) ops.push_back({false, d, r, s, r + dh, s + dw});
                else if (u % 2 == 0) ops.push_back({true, d, r, s, r + dh, s + dw});
            }
    }
    std::stable_sort(ops.begin(), ops.end(), [](const PairOp &a, const PairOp &b) {
        if (a.i != b.i) return a.i < b.i;
        return a.r * S + a.s < b.r * S + b.s;
    });
    return ops;
}

// emits loads of pixel (i, j) [and the pair partner] on first use; returns the operand name
struct PixelCache {
    const Geo &g;
    std::ostringstream &os;
    const char *ind;
    int axis;
    std::set<std::pair<int, int>> loaded, packed;
    std::string px(int i, int j) {
        if (loaded.insert({i, j}).second)
            os << ind << "const float px" << coord(i) << "_" << coord(j) << " = LDT(tb[" << (i - g.minDH) * g.pitch + (j - g.x0)
               << "]);\n";
        return "px" + coord(i) + "_" + coord(j);
    }
    std::string pair(int i, int j) {
        const int i2 = axis == 0 ? i + 1 : i, j2 = axis == 0 ? j : j + 1;
        const std::string a = px(i, j), b = px(i2, j2);
        const std::string name = "pp" + coord(i) + "_" + coord(j);
        if (packed.insert({i, j}).second) os << ind << "const u64 " << name << " = f2pack(" << a << ", " << b << ");\n";
        return name;
    }
};

// stencil: a_rs += Σ_d w_d · px(r+dh, s+dw) for the taps `ds` (assigns a_rs)
void emit_stencil_compute_paired(std::ostringstream &os, const Geo &g, const std::vector<int> &ds, int axis,
                                 const char *ind) {
    for (int d : ds) {
        os << ind << "const float m" << d << " = ";
        for (size_t q = 0; q < g.taps[d].ks.size(); ++q) os << (q ? " + " : "") << "wv[" << g.taps[d].ks[q] << "]";
        os << ";\n" << ind << "const u64 M" << d << " = f2pack(m" << d << ", m" << d << ");\n";
    }
    // accumulators: pairs keyed by the first (r, s) of the pair, scalars on the last row/column
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) {
            const int u = axis == 0 ? r : s;
            if (u == 6) os << ind << "float AS" << r << "_" << s << " = 0.f;\n";
            else if (u % 2 == 0) os << ind << "u64 AP" << r << "_" << s << " = 0ull;\n";
        }
    PixelCache pc{g, os, ind, axis, {}, {}};
    for (const PairOp &o : pair_ops(g, ds, axis)) {
        if (o.pair) {
            const std::string p = pc.pair(o.i, o.j);
            os << ind << "AP" << o.r << "_" << o.s << " = ffma2(" << p << ", M" << o.d << ", AP" << o.r << "_" << o.s << ");\n";
        } else {
            const std::string p = pc.px(o.i, o.j);
            os << ind << "AS" << o.r << "_" << o.s << " = fmaf(" << p << ", m" << o.d << ", AS" << o.r << "_" << o.s << ");\n";
        }
    }
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) {
            const int u = axis == 0 ? r : s;
            if (u == 6) {
                os << ind << "a" << r << "_" << s << " = AS" << r << "_" << s << ";\n";
            } else if (u % 2 == 0) {
                const int r2 = axis == 0 ? r + 1 : r, s2 = axis == 0 ? s : s + 1;
                os << ind << "a" << r << "_" << s << " = f2lo(AP" << r << "_" << s << "); a" << r2 << "_" << s2
                   << " = f2hi(AP" << r << "_" << s << ");\n";
            }
        }
}

// wgrad: q_d = Σ_{r,s} g_rs · px(r+dh, s+dw) for the taps `ds` (declares float q<d>)
void emit_wgrad_compute_paired(std::ostringstream &os, const Geo &g, const std::vector<int> &ds, int axis,
                               const char *ind) {
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) {
            const int u = axis == 0 ? r : s;
            if (u % 2 == 0 && u < 6) {
                const int r2 = axis == 0 ? r + 1 : r, s2 = axis == 0 ? s : s + 1;
                os << ind << "const u64 G" << r << "_" << s << " = f2pack(g" << r << "_" << s << ", g" << r2 << "_" << s2
                   << ");\n";
            }
        }
    for (int d : ds) os << ind << "u64 QP" << d << " = 0ull; float QS" << d << " = 0.f;\n";
    PixelCache pc{g, os, ind, axis, {}, {}};
    for (const PairOp &o : pair_ops(g, ds, axis)) {
        if (o.pair) {
            const std::string p = pc.pair(o.i, o.j);
            os << ind << "QP" << o.d << " = ffma2(" << p << ", G" << o.r << "_" << o.s << ", QP" << o.d << ");\n";
        } else {
            const std::string p = pc.px(o.i, o.j);
            os << ind << "QS" << o.d << " = fmaf(" << p << ", g" << o.r << "_" << o.s << ", QS" << o.d << ");\n";
        }
    }
    for (int d : ds) os << ind << "const float q" << d << " = (f2lo(QP" << d << ") + f2hi(QP" << d << ")) + QS" << d << ";\n";
}

std::string gen_stencil(const Ctx &x, const std::vector<Geo> &geo, const std::vector<int> &table_of,
                        const std::vector<int> &count) {
    std::ostringstream os;
    emit_header(os, x, table_of, count);
    const size_t TB = tile_bytes_of(geo);
    const size_t SB = stage_bytes_of(x);
    const size_t T32 = x.convert ? tile32_bytes_of(geo) : 0, OFF32 = 2 * TB;
    const size_t off_stage = 2 * TB + T32, off_wsm = off_stage + SB, off_bar = off_wsm + 3 * 64 * 4,
                 off_item = off_bar + 32;  // wsm: [2] producer-staged + [1] consumer copy (convert path)
    const int ncw = x.wpg * x.G;  // consumer warps
    const bool ragged = (R * x.BR != x.Ho) || (S * x.BC != x.Wo);
    const int band = 4 * R;       // output rows per consumer warp
    const int bcg = (x.BC + 7) / 8;
    os << "extern \"C\" __global__ void __launch_bounds__(" << 32 * (ncw + 1) << ", " << x.minb
       << ") o1d_stencil(const __grid_constant__ Params p) {\n"
       << "  extern __shared__ __align__(1024) unsigned char smem[];\n"
       << "  float* const wsm = reinterpret_cast<float*>(smem + " << off_wsm << ");\n"
       << "  u64* const full = reinterpret_cast<u64*>(smem + " << off_bar << ");\n"
       << "  u64* const empty = full + 2;\n"
       << "  int* const s_item = reinterpret_cast<int*>(smem + " << off_item << ");\n"
       << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n"
       << "  int trn = 0;\n"
       << "  for (int i = threadIdx.x; i < " << (2 * TB + T32) / 16 << "; i += blockDim.x) {  // zero guards (and tiles)\n"
       << "    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0u, 0u, 0u, 0u);\n"
       << "  }\n"
       << "  if (tid == 0) {\n"
       << "    mbar_init(full, 32); mbar_init(full + 1, 32);\n"

       << "    fence_mbar_init();\n  }\n"
       << "  __syncthreads();\n"
       << "  if (warp == 0) {\n"
       << "    // ------------------------------------------------------------ producer\n"
       << "    int tcur = 0, tried = 0; unsigned raw = 0;\n"
       << "    pdl_wait();\n"
       << "    if (lane == 0) { trace_ev(p.trace, 0, -1, trn); tcur = p.only >= 0 ? p.only : HOME[smid() % NHOME]; raw = atomicAdd(p.sched + tcur * CS, 1u); }\n"
       << "    for (int it = 0;; ++it) {\n"
       << "      const int b = it & 1;\n"
       << "      // buffer b is free once every consumer warp released item it-2: a named\n"
       << "      // barrier per buffer parity (the producer blocks in hardware, no spinning)\n"
       << "      if (it >= 2) asm volatile(\"bar.sync %0, %1;\" :: \"r\"(14 + b), \"r\"(" << 32 * (ncw + 1) << ") : \"memory\");\n"
       << "      int item = -1;\n"
       << "      if (lane == 0) { item = sched_resolve(p.sched, tcur, raw, tried, p.only < 0); sched_prefetch(p.sched, tcur, raw); }\n"
       << "      item = __shfl_sync(0xffffffffu, item, 0);\n"
       << "      int t2 = 0, c2 = 0, n2 = 0;\n"
       << "      if (item >= 0) item_cn(item, t2, c2, n2);\n"
       << "      if (lane == 0 && item >= 0) {   // issue the tile load first: it is the long pole\n"
       << "        trace_ev(p.trace, 1, item, trn);\n"
       << "        unsigned char* dst = smem + b * " << TB << ";\n"
       << "        switch (t2) {\n";
    for (int t = 0; t < x.nt; ++t)
        os << "        case " << t << ": mbar_expect_tx(full + b, " << geo[t].bytes << "u); tma_load(dst + " << geo[t].guard
           << ", &p.in_map[" << t << "], " << geo[t].x0 << ", " << geo[t].minDH << ", c2, n2, full + b); break;\n";
    os << "        }\n"
       << "      }\n"
       << "      if (item >= 0)\n"
       << "        for (int k = lane; k < " << x.K << "; k += 32) wsm[b * 64 + k] = __ldg(p.w + c2 * " << x.K << " + k);\n"
       << "      if (lane == 0) s_item[b] = item;\n"
       << "      mbar_arrive(full + b);   // 32 producer arrivals (+ the tile bytes) complete the phase\n"
       << "      if (item < 0) { pdl_trigger(); break; }\n"
       << "    }\n"
       << "    if (lane == 0) sched_exit(p.sched);\n"
       << "    return;\n"
       << "  }\n"
       << "  // -------------------------------------------------------------- consumers\n"
       << "  const int cw = warp - 1, grp = cw / " << x.wpg << ", wg = cw - grp * " << x.wpg << ";\n"
       << "  int bc = (lane & 7) + 8 * (wg % " << bcg << "), br = (lane >> 3) + 4 * (wg / " << bcg << ");\n"
       << "  const bool active = bc < " << x.BC << " && br < " << x.BR << ";\n"
       << "  if (!active) { bc = 0; br = 0; }\n"
       << "  const int row0 = " << band << " * (wg / " << bcg << ");   // first output row of this warp's band\n"
       << "  float* const stg = reinterpret_cast<float*>(smem + " << off_stage << ");\n"
       << "  float* const sto = stg + (" << R << " * br) * " << x.Wo << " + " << S << " * bc;\n";
    if (bcg != 1) os << "  // (several warps per band: bands are stored by the warp with wg % bcg == 0)\n";
    os << "  for (int it = 0;; ++it) {\n"
       << "    const int b = it & 1;\n"
       << "    if (lane == 0) trace_ev(p.trace, 2, it, trn);\n"
       << "    mbar_wait(full + b, (it >> 1) & 1);\n"
       << "    const int item = s_item[b];\n"
       << "    if (lane == 0) trace_ev(p.trace, 3, item, trn);\n"
       << "    if (item < 0) break;\n"
       << "    int t, c, n; item_cn(item, t, c, n);\n"
       << "    const unsigned char* tile = " << (x.convert ? "smem + " + std::to_string(OFF32) : "smem + b * " + std::to_string(TB)) << ";\n"
       << "    const float* wv = wsm + " << (x.convert ? "128" : "b * 64") << ";\n";
    if (x.convert) {
        // the 16-bit buffer (and its weight slot) is released before the tap loop:
        // keep this plane's weights in the consumer-owned slot wsm[2]
        os << "    asm volatile(\"bar.sync 13, " << 32 * ncw << ";\" ::: \"memory\");  // previous plane's weights consumed\n"
           << "    if (tid - 32 < " << x.K << ") wsm[128 + tid - 32] = wsm[b * 64 + tid - 32];\n";
        emit_convert(os, x, geo, TB, OFF32, ncw);
    }
    if (x.G > 1)  // the previous band store has long finished reading the staging area: free it now
        os << "    if (grp == 0) {\n"
           << "      if (lane == 0) asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\");\n"
           << "      __syncwarp();\n"
           << "      asm volatile(\"bar.arrive %0, %1;\" :: \"r\"(1 + wg), \"r\"(64) : \"memory\");\n"
           << "    }\n";
    os << "";
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) os << "    float a" << r << "_" << s << ";\n";
    os << "    switch (t) {\n";
    for (int t = 0; t < x.nt; ++t) {
        const Geo &g = geo[t];
        os << "    case " << t << ": {\n"
           << "      const " << (x.convert ? "float" : "act_t") << "* tb = reinterpret_cast<const " << (x.convert ? "float" : "act_t")
           << "*>(tile + " << (x.convert ? guard32(g) : g.guard) << ") + (" << R << " * br) * " << g.pitch << " + " << S << " * bc;\n";
        for (int gi = 0; gi < x.G; ++gi) {
            const std::vector<int> ds = group_taps(g, gi, x.G);
            os << "      " << (gi ? "else " : "") << (gi + 1 < x.G ? "if (grp == " + std::to_string(gi) + ") " : "")
               << "{\n";
            if (x.ffma2 && g_parity_groups && x.G == 2) {
                emit_stencil_compute_paired(os, g, ds, pair_axis(g), "        ");
            } else if (x.ffma2) {
                emit_stencil_compute_ffma2(os, g, ds, "        ");
            } else {
                for (int r = 0; r < R; ++r)
                    for (int s = 0; s < S; ++s) os << "        a" << r << "_" << s << " = 0.f;\n";
                for (int d : ds) {
                    os << "        const float m" << d << " = ";
                    for (size_t q = 0; q < g.taps[d].ks.size(); ++q) os << (q ? " + " : "") << "wv[" << g.taps[d].ks[q] << "]";
                    os << ";\n";
                }
                for_each_pixel(g, ds, [&](int i, int j, const std::vector<std::pair<int, std::pair<int, int>>> &uses) {
                    os << "        { const float v = LDT(tb[" << (i - g.minDH) * g.pitch + (j - g.x0) << "]);";
                    for (auto &u : uses) {
                        const int r = u.second.first, s = u.second.second;
                        os << " a" << r << "_" << s << " = fmaf(v, m" << u.first << ", a" << r << "_" << s << ");";
                    }
                    os << " }\n";
                });
            }
            os << "      }\n";
        }
        os << "      break;\n    }\n";
    }
    os << "    }\n"
       << "    __syncwarp();\n"
       << "    if (lane == 0) trace_ev(p.trace, 4, item, trn);\n"
       << (x.convert ? std::string("")
                     : "    asm volatile(\"bar.arrive %0, %1;\" :: \"r\"(14 + b), \"r\"(" + std::to_string(32 * (ncw + 1)) +
                           ") : \"memory\");  // done with the tile\n");
    auto store_pred = [&](int r, int s) {
        std::ostringstream q;
        if (ragged) q << "if (" << R << " * br + " << r << " < " << x.Ho << " && " << S << " * bc + " << s << " < " << x.Wo << ") ";
        return q.str();
    };
    // partial (fp32) or final write of the block into the band's staging area;
    // final 16-bit outputs are packed in place (pitch Wo) once the warp has read
    // its fp32 partials, so the TMA store reads a dense act_t band
    auto emit_sts = [&](bool add, bool final_) {
        if (!final_ || x.act == O1D_F32) {
            os << "      if (active) {\n";
            for (int r = 0; r < R; ++r)
                for (int s = 0; s < S; ++s) {
                    os << "        " << store_pred(r, s) << "sto[" << r * x.Wo + s << "] = ";
                    if (add) os << "sto[" << r * x.Wo + s << "] + ";
                    os << "a" << r << "_" << s << ";\n";
                }
            os << "      }\n";
            return;
        }
        if (add) {
            os << "      if (active) {\n";
            for (int r = 0; r < R; ++r)
                for (int s = 0; s < S; ++s)
                    os << "        " << store_pred(r, s) << "a" << r << "_" << s << " = sto[" << r * x.Wo + s << "] + a"
                       << r << "_" << s << ";\n";
            os << "      }\n";
        }
        os << "      __syncwarp();\n"
           << "      if (active) {\n"
           << "        act_t* stb = reinterpret_cast<act_t*>(stg + row0 * " << x.Wo << ") + (" << R << " * br - row0) * "
           << x.Wo << " + " << S << " * bc;\n";
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s)
                os << "        " << store_pred(r, s) << "stb[" << r * x.Wo + s << "] = to_act(a" << r << "_" << s << ");\n";
        os << "      }\n";
    };
    // named barriers per band (warp wg of every group): id 1+wg "free" (group 0 -> others), id 1+wpg+wg chain
    const int nb = 64;  // every named barrier pairs two warps (one arrives, one syncs)
    if (x.G == 1) {
        os << "    if (lane == 0) asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\");\n"
           << "    __syncwarp();\n";
        emit_sts(false, true);
    } else {
        // group G-1 writes first, then G-2 adds, ..., group 0 adds and stores.
        // ("staging free" is signalled by group 0 at the top of the iteration, see below)
        for (int gi = x.G - 1; gi >= 0; --gi) {
            os << "    if (grp == " << gi << ") {\n";
            if (gi == x.G - 1)
                os << "      asm volatile(\"bar.sync %0, %1;\" :: \"r\"(1 + wg), \"r\"(" << nb << ") : \"memory\");\n";
            else
                os << "      asm volatile(\"bar.sync %0, %1;\" :: \"r\"(" << 1 + x.wpg << " + " << gi << " * " << x.wpg
                   << " + wg), \"r\"(64) : \"memory\");\n";
            emit_sts(gi != x.G - 1, gi == 0);
            if (gi > 0)
                os << "      asm volatile(\"bar.arrive %0, %1;\" :: \"r\"(" << 1 + x.wpg << " + " << gi - 1 << " * "
                   << x.wpg << " + wg), \"r\"(64) : \"memory\");\n";
            os << "    }\n";
        }
    }
    // group 0 warps store their band: rows [row0, row0 + band) of the plane
    os << "    if (grp == 0" << (bcg != 1 ? " && (wg % " + std::to_string(bcg) + ") == 0" : std::string()) << ") {\n"
       << "      asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
       << "      __syncwarp();\n"
       << "      if (lane == 0 && row0 < " << x.Ho << ") {\n"
       << "        asm volatile(\"cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];\"\n"
       << "                     :: \"l\"(&p.out_map), \"r\"(sa(stg + row0 * " << x.Wo << ")), \"r\"(0), \"r\"(row0), \"r\"(c), \"r\"(n) : \"memory\");\n"
       << "        asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n"
       << "      }\n"
       << "    }\n"
       << "    if (lane == 0) trace_ev(p.trace, 5, item, trn);\n"
       << "  }\n"
       << "  if (lane == 0) asm volatile(\"cp.async.bulk.wait_group 0;\" ::: \"memory\");\n"
       << "}\n";
    return os.str();
}

// ===========================================================================
// v2 pipeline (default): one tap group per warp, one persistent CTA per SM.
//
// Measured on the v1 design (tools/trace_pass.py, O1D_TRACE): with the taps
// split over two warp groups, the per-plane group combine (pairwise named
// barriers + a second partial pass through shared memory) took ~30% of every
// consumer warp's time; with one group the warps computed ~2x faster per FMA
// but waited for tiles most of the time (a 2-slot ring = one plane of
// lookahead), and the v1 wgrad's per-plane reductions stalled the same way.
//
// v2: one CTA per SM = a producer warp + P consumer "pairs" (wpg warps each,
// one band of 4 block rows per warp, ALL taps).  Items (planes) go round-robin
// to the pairs (item it -> pair it % P) and to an NS-slot ring (slot it % NS),
// so NS - P planes are in flight while P are computed.  A slot holds only the
// image rows (TMA box from row 0, OOB columns zero-filled by the TMA unit);
// consecutive slots share zero rows that serve as the vertical halo (reading
// R1), so a slot is ~35% smaller than a v1 tile with its halo.  Stencil
// outputs are staged in the consumed slot; the PRODUCER issues the TMA store
// (consumers never wait for it) before it reloads the slot.  backward_weight
// also TMA-loads the dy plane into a per-pair slot that the pair releases as
// soon as its dy block is in registers.
// ---------------------------------------------------------------------------
struct Lay2 {
    int NS = 3, NB = 2, P = 1, NPROD = 1, wpg = 1, pitch = 0, zrows = 0, dyp = 0, dyrows = 0, hin = 0, BW = 1;
    bool inslot = false;   // stencil output bands staged in the consumed slot (no staging area)
    size_t sbi = 0;        // bytes per warp band inside the slot
    size_t zb = 0, tb = 0, db = 0, sb = 0, off_item = 0, off_bal = 0, off_w = 0, off_scr = 0, off_stg = 0, off_dy = 0, off_t = 0,
           total = 0;
    int ncw() const { return P * wpg; }
    size_t slot(int s) const { return off_t + zb + (size_t)s * (zb + tb); }
};

Lay2 lay2(const Ctx &x, const std::vector<Geo> &geo, int es, int Hin, bool wgrad, bool allow_inslot = true) {
    Lay2 L;
    L.wpg = x.wpg;
    L.hin = Hin;
    // backward_weight: a consumer pair takes BW consecutive planes (n) of one channel and
    // reduces its tap partials once per batch (fixed order: deterministic)
    L.BW = wgrad ? std::max(1, std::min(x.N, env_int("O1D_WB", 1))) : 1;  // (measured: 4 -> 58 us vs 51 us, register pressure)
    L.P = std::max(1, std::min(8, env_int("O1D_P", std::max(1, 8 / x.wpg))));
    while (L.P * L.wpg > 15) --L.P;
    // producer pw serves pairs pw, pw + NPROD, ...  Default: one producer per pair up to 4 pairs
    // (it then sleeps in try_wait; measured +1.8% over two polling producers), else 2
    L.NPROD = std::max(1, std::min(L.P, env_int("O1D_NPROD", L.P <= 4 ? L.P : 2)));
    for (auto &g : geo) {
        L.pitch = std::max(L.pitch, g.pitch);
        L.zrows = std::max(L.zrows, std::max(-g.minDH, R * x.BR - Hin + g.maxDH) + 1);
    }
    L.zb = ((size_t)L.zrows * L.pitch * es + 127) & ~(size_t)127;
    L.tb = ((size_t)Hin * L.pitch * es + 127) & ~(size_t)127;
    if (wgrad) {
        const int vec = 16 / es;
        L.dyp = (S * x.BC + vec - 1) & ~(vec - 1);
        L.dyrows = R * x.BR;
        L.db = ((size_t)L.dyp * L.dyrows * es + 127) & ~(size_t)127;
    }
    // header: full[NSmax], empty[NSmax], dyempty[8] mbarriers | s_item | weights | scratch | dy slots | zero rows + slots
    const int NSmax = 16;
    L.off_item = 8 * (2 * (size_t)NSmax + 8);
    L.off_bal = (L.off_item + 4 * (size_t)NSmax + 15) & ~(size_t)15;  // CTA placement accounting (adaptive)
    L.off_w = L.off_bal + 16 * 8 + 16 * 4 + 16;
    L.off_scr = L.off_w + (wgrad ? 0 : (size_t)NSmax * 64 * 4);
    L.off_stg = (L.off_scr + (wgrad ? (size_t)L.ncw() * 32 * 4 : 0) + 127) & ~(size_t)127;
    L.sbi = ((size_t)4 * R * x.Wo * es + 127) & ~(size_t)127;
    // O1D_INSLOT: a pair writes its output bands into the slot it just consumed (the slot is
    // released once the band stores have read it), so the staging area becomes tile slots
    L.inslot = allow_inslot && INSLOT && !wgrad && !YSTG && !YST && (size_t)L.wpg * L.sbi <= (size_t)Hin * L.pitch * es;
    L.sb = (wgrad || YSTG || L.inslot) ? 0 : L.sbi;  // per-warp output staging band
    L.off_dy = L.off_stg + (size_t)L.ncw() * L.sb;
    L.off_t = (L.off_dy + (size_t)L.P * L.db + 1023) & ~(size_t)1023;
    const size_t budget = (size_t)env_int("O1D_SMEM_KB", 227) * 1024 - 64;
    const int fit = budget > L.off_t + L.zb ? (int)((budget - L.off_t - L.zb) / (L.zb + L.tb)) : 0;
    L.NB = std::max(1, std::min(env_int("O1D_NBUF", 2), std::min(fit, NSmax) / L.P));  // slots per pair
    L.NS = L.P * L.NB;
    L.total = L.off_t + (size_t)L.NS * (L.zb + L.tb) + L.zb;
    if (L.inslot && L.NB < 2) return lay2(x, geo, es, Hin, wgrad, false);  // the deferred release needs a second slot
    return L;
}

// geometry as the v2 emitters see it: tile row 0 = image row 0, uniform pitch
std::vector<Geo> geo2(const std::vector<Geo> &geo, const Lay2 &L) {
    std::vector<Geo> v = geo;
    for (auto &g : v) g.minDH = 0, g.x0 = 0, g.pitch = L.pitch;
    return v;
}

// prologue zeroing of the tile area: only what no TMA load ever writes -- the zero-row
// regions between the slots and each slot's tail past its box -- unless O1D_ZALL=1
// (every slot byte; ~1 us of stores per CTA at the start of a launch)
std::string zero_v2(const Lay2 &L, int es, int nthreads) {
    std::ostringstream os;
    const size_t box = (size_t)L.hin * L.pitch * es, tail = L.tb - box, stride = L.zb + L.tb;
    if (env_int("O1D_ZALL", 0) || box % 16 || L.zb % 16) {
        os << "  for (int i = tid; i < " << (L.total - L.off_t) / 16 << "; i += " << nthreads << ")  // zero rows + slots\n"
           << "    reinterpret_cast<uint4*>(tiles)[i] = make_uint4(0u, 0u, 0u, 0u);\n";
        return os.str();
    }
    // region s (0..NS): zero rows at s * stride, then (s < NS) the tail of slot s after its box
    const size_t per = (L.zb + tail) / 16;
    os << "  for (int i = tid; i < " << (L.NS + 1) * per << "; i += " << nthreads << ") {  // zero rows + slot tails\n"
       << "    const int s = i / " << per << ", k = i - s * " << per << ";\n"
       << "    const int off = s * " << stride << " + (k < " << L.zb / 16 << " ? k * 16 : " << L.zb + box << " + (k - " << L.zb / 16
       << ") * 16);\n"
       << "    if (s < " << L.NS << " || k < " << L.zb / 16 << ") *reinterpret_cast<uint4*>(tiles + off) = make_uint4(0u, 0u, 0u, 0u);\n"
       << "  }\n";
    return os.str();
}

void emit_v2_prologue(std::ostringstream &os, const Lay2 &L, int nthreads, bool wgrad, int es) {
    os << "  extern __shared__ __align__(1024) unsigned char smem[];\n"
       << "  u64* const full = reinterpret_cast<u64*>(smem);\n"
       << "  u64* const empty = full + 16;\n"
       << "  u64* const dyempty = full + 32;\n"
       << "  int* const s_item = reinterpret_cast<int*>(smem + " << L.off_item << ");\n"
       << "  float* const wsm = reinterpret_cast<float*>(smem + " << L.off_w << ");\n"
       << "  unsigned char* const tiles = smem + " << L.off_t << ";\n"
       << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n"
       << "  int trn = 0;\n"
       << zero_v2(L, es, nthreads)
       << "  if (tid < " << (16 * 8 + 16 * 4 + 16) / 4 << ") reinterpret_cast<unsigned*>(smem + " << L.off_bal << ")[tid] = 0u;\n"
       << "  if (tid == 0) {\n"
       << "    for (int s = 0; s < " << L.NS << "; ++s) { mbar_init(full + s, 32); mbar_init(empty + s, " << L.wpg << "); }\n";
    if (wgrad) os << "    for (int q = 0; q < " << L.P << "; ++q) mbar_init(dyempty + q, " << L.wpg << ");\n";
    os << "    fence_mbar_init();\n"
       << "  }\n"
       << "  __syncthreads();\n";
}

// producer warp.  Each consumer pair q owns NB slots (q * NB .. q * NB + NB - 1);
// its j-th item goes to slot q * NB + j % NB.  The producer serves the pairs
// round-robin and never blocks on one pair: a pair whose next slot is still
// busy (test_wait on its empty barrier) is skipped until later, so a slow pair
// cannot hold up the loads of the others (measured with a single FIFO ring:
// head-of-line blocking left consumers waiting ~20% of the time).  After the
// scheduler runs dry every pair gets an end marker (-1).
void emit_v2_producer(std::ostringstream &os, const Ctx &x, const Lay2 &L, bool wgrad, int es) {
    const int NB = L.NB, P = L.P;
    const size_t bytes = (size_t)L.hin * L.pitch * es + (wgrad ? (size_t)L.dyp * L.dyrows * es : 0);  // exact box bytes
    const int PQ = (P + L.NPROD - 1) / L.NPROD;  // pairs per producer warp, at most (producer pw serves pairs pw, pw + NPROD, ...)
    os << "#define P_NB " << PQ * NB << "\n#define PREF " << std::max(1, env_int("O1D_PREF", 2)) << "\n"
       << "  if (warp < " << L.NPROD << ") {\n"
       << "    const int pw = warp;\n"
       << "    int tcur = 0, tried = 0; unsigned raw = 0;\n"
       << "    // the scheduler counters of this launch slot were last touched 64 launches ago: the\n"
       << "    // first atomics run before griddepcontrol.wait, overlapping the preceding kernel's tail\n"
       << "    // (only the data -- x / dy / w -- may be produced by it)\n"
       << "    const bool early = " << (env_int("O1D_EARLY", 1) ? "p.bal == nullptr" : "false") << ";\n"
       << "    if (!early && !p.nowait) pdl_wait();\n"
       << "    const u64 pol = " << (EFH ? "policy_evict_first()" : "0ull") << ";\n"
       << "    unsigned lo = 0, hi = 0, nxt = 0;   // the first P*NB items come in one batch (fills the ring without round trips)\n"
       << "    unsigned pf[PREF];\n"
       << "    if (lane == 0) {\n"
       << "      trace_ev(p.trace, 0, -1, trn);\n"
       << "      tcur = p.only >= 0 ? p.only : (p.bal ? (int)reinterpret_cast<const Bal*>(p.bal)->home[smid() % NHOME] : (int)HOME[smid() % NHOME]);\n"
       << "      lo = atomicAdd(p.sched + tcur * CS, " << PQ * NB << "u); hi = lo + " << PQ * NB << ";\n"
       << (env_int("O1D_SCHED2", 0) ? "      nxt = atomicAdd(p.sched + tcur * CS, (unsigned)GB);\n"
           : env_int("O1D_PREF", 2) > 1 ? "#pragma unroll\n      for (int k = 0; k < PREF; ++k) pf[k] = atomicAdd(p.sched + tcur * CS, 1u);\n"
                                        : "      nxt = atomicAdd(p.sched + tcur * CS, 1u);\n")
       << "    }\n"
       << "    (void)raw;\n"
       << (env_int("O1D_L2PF", 0)
               ? "    if (early && lane == 0) {\n"
                 "      // L2 prefetch of the first planes while the preceding kernel drains: a prefetch only\n"
                 "      // warms L2 (coherent), the shared-memory loads still wait for griddepcontrol.wait\n"
                 "      for (int k = 0; k < P_NB; ++k) {\n"
                 "        if (lo + k >= (unsigned)cnt_w(tcur, p.nlen)) break;\n"
                 "        int t3, c3, n3; item_cn((tcur << 22) | (int)(lo + k), t3, c3, n3, p.n0);\n"
                 "        asm volatile(\"cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];\"\n"
                 "                     :: \"l\"(&p.in_map[0]), \"r\"(0), \"r\"(0), \"r\"(c3), \"r\"(n3) : \"memory\");\n" +
                     std::string(wgrad ? "        asm volatile(\"cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];\"\n"
                                         "                     :: \"l\"(&p.out_map), \"r\"(0), \"r\"(0), \"r\"(c3), \"r\"(n3) : \"memory\");\n"
                                       : "") +
                 "      }\n"
                 "    }\n"
               : "")
       << "    if (early && !p.nowait) pdl_wait();\n"
       << "    int jq[" << PQ << "];   // items issued per served pair (-1: end marker sent)\n"
       << "    for (int qi = 0; qi < " << PQ << "; ++qi) jq[qi] = pw + qi * " << L.NPROD << " < " << P << " ? 0 : -1;\n"
       << (L.BW > 1 ? "    int bq[" + std::to_string(PQ) + "], eq[" + std::to_string(PQ) + "], nq[" + std::to_string(PQ) +
                          "];   // current batch item / next plane / planes, per served pair\n"
                          "    for (int qi = 0; qi < " + std::to_string(PQ) + "; ++qi) { bq[qi] = -1; eq[qi] = 0; nq[qi] = 0; }\n"
                    : "")
       << "    int issued = 0, fetched = 0, live = (" << P + L.NPROD - 1 << " - pw) / " << L.NPROD << ", idle = 0;   // planes issued / scheduler items taken (lane 0)\n"
       << "    while (live > 0) {\n"
       << "      bool any = false;\n"
       << "#pragma unroll 1\n"
       << "      for (int qi = 0; qi < " << PQ << "; ++qi) {\n"
       << "        const int q = pw + qi * " << L.NPROD << ";\n"
       << "        const int j = jq[qi];\n"
       << "        if (j < 0) continue;\n"
       << "        const int s = q * " << NB << " + j % " << NB << ";\n"
       << (PQ == 1
               // one pair per producer: nothing else to serve, so the producer sleeps in
               // try_wait instead of polling (no issue slots taken from its SM sub-partition)
               ? "        if (j >= " + std::to_string(NB) + ") mbar_wait(empty + s, ((j / " + std::to_string(NB) + ") & 1) ^ 1);\n"
               : "        if (j >= " + std::to_string(NB) + " && !mbar_test(empty + s, ((j / " + std::to_string(NB) +
                     ") & 1) ^ 1)) continue;   // slot still in use\n");
    if (wgrad)  // the pair's dy slot is free once it copied the dy block of its previous item
        os << (PQ == 1 ? "        if (j >= 1) mbar_wait(dyempty + q, ((j - 1) & 1));\n"
                       : "        if (j >= 1 && !mbar_test(dyempty + q, ((j - 1) & 1))) continue;\n");
    os << "        if (lane == 0) trace_ev(p.trace, 6, q * 65536 + j, trn);   // slot found free\n"
       << "        int item = -1;\n";
    if (L.BW > 1) {
        // batches: the scheduler hands out (channel, n-batch) items; the pair gets the batch's
        // planes one by one, flagged first (bit 27) / last (bit 28)
        os << "        if (bq[qi] >= 0 && eq[qi] < nq[qi]) {\n"
           << "          item = bq[qi];\n"
           << "        } else {\n";
    }
    os << ""
       << (env_int("O1D_PREF", 2) > 1 && !env_int("O1D_SCHED2", 0)
               ? "        if (lane == 0) {\n"
                 "          // PREF single-item atomics in flight: each issue consumes the oldest one\n"
                 "          if (fetched < P_NB && lo + fetched < (unsigned)cnt_w(tcur, p.nlen)) item = (tcur << 22) | (int)(lo + fetched);\n"
                 "          else {\n"
                 "            unsigned v = pf[0];\n"
                 "#pragma unroll\n"
                 "            for (int k = 0; k + 1 < PREF; ++k) pf[k] = pf[k + 1];\n"
                 "            const int t0 = tcur;\n"
                 "            item = sched_resolve(p.sched, tcur, v, tried, p.only < 0, p.nlen);\n"
                 "            if (tcur != t0) {   // moved to another table: the prefetched indices belong to the old one\n"
                 "#pragma unroll\n"
                 "              for (int k = 0; k < PREF; ++k) pf[k] = tcur >= 0 ? atomicAdd(p.sched + tcur * CS, 1u) : 0xffffffffu;\n"
                 "            } else {\n"
                 "              pf[PREF - 1] = tcur >= 0 ? atomicAdd(p.sched + tcur * CS, 1u) : 0xffffffffu;   // (tcur < 0: table exhausted)\n"
                 "            }\n"
                 "          }\n"
                 "          ++fetched;\n"
                 "        }\n"
               : env_int("O1D_SCHED2", 0)
               ? "        if (lane == 0) item = sched2_next(p.sched, tcur, lo, hi, nxt, tried, p.only < 0);\n"
               : "        if (lane == 0) {\n"
                 "          if (fetched < P_NB && lo + fetched < (unsigned)cnt_w(tcur, p.nlen)) item = (tcur << 22) | (int)(lo + fetched);\n"
                 "          else { item = sched_resolve(p.sched, tcur, nxt, tried, p.only < 0, p.nlen); sched_prefetch(p.sched, tcur, nxt); }\n"
                 "          ++fetched;\n"
                 "        }\n")
       << (L.BW > 1 ? "          bq[qi] = __shfl_sync(0xffffffffu, item, 0); eq[qi] = 0;\n"
                      "          if (bq[qi] >= 0) {\n"
                      "            const int tb = bq[qi] >> 22, b = bq[qi] & 0x3FFFFF, nch = CHOFF[tb + 1] - CHOFF[tb];\n"
                      "            nq[qi] = min(" + std::to_string(L.BW) + ", NB - (b / nch) * " + std::to_string(L.BW) + ");\n"
                      "          }\n"
                      "          item = bq[qi];\n"
                      "        }\n"
                      "        if (item >= 0) {   // plane eq of batch item: CMAJOR plane index c_idx + nch * n\n"
                      "          const int tb = item >> 22, b = item & 0x3FFFFF, nch = CHOFF[tb + 1] - CHOFF[tb];\n"
                      "          const int n0 = (b / nch) * " + std::to_string(L.BW) + ";\n"
                      "          item = (tb << 22) | ((b % nch) + nch * (n0 + eq[qi])) | (eq[qi] == 0 ? (1 << 27) : 0) |\n"
                      "                 (eq[qi] == nq[qi] - 1 ? (1 << 28) : 0);\n"
                      "          ++eq[qi];\n"
                      "        }\n"
                    : "")
       << "        item = __shfl_sync(0xffffffffu, item, 0);\n"
       << "        ++issued;\n"
       << "        int t2 = 0, c2 = 0, n2 = 0;\n"
       << "        if (item >= 0) item_cn(item, t2, c2, n2, p.n0);\n"
       << "        if (lane == 0) {\n"
       << "          s_item[s] = item;\n"
       << "          if (item >= 0) {\n"
       << "            trace_ev(p.trace, 1, item, trn);\n"
       << "            mbar_expect_tx(full + s, " << bytes << "u);\n"
       << "            tma_load_ef(tiles + " << L.zb << " + s * " << L.zb + L.tb << ", &p.in_map[0], 0, 0, c2, n2, full + s" << (EFH ? ", pol);\n" : ", 0ull);\n");
    if (wgrad)
        os << "            tma_load_ef(smem + " << L.off_dy << " + q * " << L.db << ", &p.out_map, 0, 0, c2, n2, full + s" << (EFH ? ", pol);\n" : ", 0ull);\n");
    os << "          }\n"
       << "        }\n";
    if (!wgrad && !env_int("O1D_WASYNC", 0)) {
        os << "        if (item >= 0)\n"
           << "          for (int k = lane; k < " << x.K << "; k += 32) wsm[s * 64 + k] = __ldg(p.w + c2 * " << x.K << " + k);\n"
           << "        mbar_arrive(full + s);   // 32 producer arrivals (+ the bytes) complete the phase\n";
    } else if (!wgrad) {
        // weights: asynchronous 4-byte copies whose completion arrives on the slot's barrier
        // (the producer never waits for them: a synchronous load here serialised the producer
        // on one L2 round trip per item)
        os << "        if (item >= 0) {\n"
           << "          for (int k = lane; k < " << x.K << "; k += 32)\n"
           << "            asm volatile(\"cp.async.ca.shared.global [%0], [%1], 4;\" :: \"r\"(sa(wsm + s * 64 + k)), \"l\"(p.w + c2 * " << x.K << " + k) : \"memory\");\n"
           << "          asm volatile(\"cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\" :: \"r\"(sa(full + s)) : \"memory\");\n"
           << "        } else {\n"
           << "          mbar_arrive(full + s);\n"
           << "        }\n";
    } else {
        os << "        mbar_arrive(full + s);   // 32 producer arrivals (+ the bytes) complete the phase\n";
    }
    os << ""
       << "        if (item < 0) { jq[qi] = -1; --live; } else { jq[qi] = j + 1; }\n"
       << "        any = true;\n"
       << "      }\n"
       << "      if (!any) { if (++idle > " << env_int("O1D_IDLE", 1) << ") __nanosleep(" << env_int("O1D_SLEEP", 256) << "); } else idle = 0;\n"
       << "    }\n"
       << "    // a kernel that skipped griddepcontrol.wait (o1d_step) still completes only after its\n"
       << "    // predecessor: whatever waits for this grid then also sees the predecessor done\n"
       << "    if (p.nowait) pdl_wait();\n"
       << "    pdl_trigger();\n"
       << "    if (lane == 0) sched_exit(p.sched, " << L.NPROD << "u);\n"
       << "    return;\n"
       << "  }\n"
       << (env_int("O1D_PAIRSMSP", 1)
               // the warps of a pair are P warp ids apart: with P = 4 they sit on the same SM
               // sub-partition and run the same code a few instructions apart (shared L0 I-cache)
               ? "  const int cw = warp - " + std::to_string(L.NPROD) + ", q = cw % " + std::to_string(L.P) + ", wg = cw / " +
                     std::to_string(L.P) + ";\n"
               : "  const int cw = warp - " + std::to_string(L.NPROD) + ", q = cw / " + std::to_string(L.wpg) + ", wg = cw - q * " +
                     std::to_string(L.wpg) + ";\n")
       << "  int bc = lane & 7, br = (lane >> 3) + 4 * wg;\n"
       << "  const bool active = bc < " << x.BC << " && br < " << x.BR << ";\n"
       << "  if (!active) { bc = 0; br = 0; }\n";
}

// consumer item-loop head (v2): j is the pair's item index; j < 0 is the optional
// I-cache warm-up pass over the CTA's home table (one code chunk per warp)
#define V2_LOOP_HEAD \
    "    const bool warm = it < 0;\n" \
    "    const int s = warm ? 0 : q * " << L.NB << " + it % " << L.NB << ";\n" \
    "    int item = 0, t = 0, c = 0, n = 0;\n" \
    "    unsigned wm = 0xffffffffu;\n" \
    "    if (warm) {\n" \
    "      t = p.only >= 0 ? p.only : HOME[smid() % NHOME];\n" \
    "      wm = " << (g_chunks > 1 ? "1u << (cw % " + std::to_string(g_chunks) + ")" : std::string("0xffffffffu")) << ";\n" \
    "    } else {\n" \
    "      if (lane == 0) trace_ev(p.trace, 2, it, trn);\n" \
    "      mbar_wait(full + s, (it / " << L.NB << ") & 1);\n" \
    << (L.inslot ? "      if (ps >= 0) {   // previous slot: free once our band store has read it\n" \
                   "        if (lane == 0) { asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\"); mbar_arrive(empty + ps); }\n" \
                   "        ps = -1;\n" \
                   "      }\n" : "") << \
    "      item = s_item[s];\n" \
    "      if (lane == 0) trace_ev(p.trace, 3, item, trn);\n" \
    "      if (item < 0) break;\n" \
    "      item_cn(item, t, c, n, p.n0);\n" \
    "    }\n"

// adaptive placement accounting (per consumer warp): busy cycles per item of table t
#define BAL_ITEM_END \
    (x.order.empty() ? "" : \
    "    if (t != bt) { if (lane == 0) bal_flush_cta(smem + " + std::to_string(L.off_bal) + ", bt, busy, nbusy); bt = t; busy = 0; nbusy = 0; }\n" \
    "    busy += (u64)(clock64() - tb0); ++nbusy;\n")
#define BAL_EXIT \
    (x.order.empty() ? std::string() : \
    "  if (p.bal && p.adapt) bal_warp_exit(p.bal, smem + " + std::to_string(L.off_bal) + ", bt, busy, nbusy, " + std::to_string(L.ncw()) + "u, lane);\n")

std::string gen_stencil2(const Ctx &x, const std::vector<Geo> &geo_in, const std::vector<int> &table_of,
                         const std::vector<int> &count, int Hin, const Lay2 &L) {
    std::ostringstream os;
    emit_header(os, x, table_of, count);
    const std::vector<Geo> geo = geo2(geo_in, L);
    const int nthreads = 32 * (L.ncw() + L.NPROD);
    // O1D_WARM bit 1: chunked I-cache warm-up for the stencils.  Off by default: with the
    // evict-first TMA traffic the code stays L2-resident and the chunk guards cost ~9% issue
    g_chunks = (env_int("O1D_WARM", 0) & 1) ? std::min(32, L.ncw()) : 0;
    const bool ragged = (R * x.BR != x.Ho) || (S * x.BC != x.Wo);
    const int es = x.act == O1D_F32 ? 4 : 2;
    os << "extern \"C\" __global__ void __launch_bounds__(" << nthreads << ", 1) o1d_stencil(const __grid_constant__ Params p) {\n";
    emit_v2_prologue(os, L, nthreads, false, es);
    emit_v2_producer(os, x, L, false, es);
    os << "  // -------------------------------------------------------------- consumers\n"
       << (L.inslot ? "" : "  unsigned char* const stg = smem + " + std::to_string(L.off_stg) + " + cw * " + std::to_string(L.sb) + ";   // this warp's output band\n")
       << "  const int row0 = " << 4 * R << " * wg;\n"
       << (L.inslot ? "  int ps = -1;   // slot whose release waits for this warp's band store\n" : "")
       << (x.order.empty() ? "" : "  int bt = -1; u64 busy = 0; unsigned nbusy = 0;   // adaptive placement accounting\n")
       // O1D_PREWARM bit 1 (bit 2: wgrad): one unguarded pass over the home table's code before
       // the first tile arrives.  Off: the first plane is then hot, but the cold fetch still
       // ends at ~7.5 us on the cold tables and the steady tap loop measured 2.56 vs 2.37 us
       << "  for (int it = " << (g_chunks > 1 || (env_int("O1D_PREWARM", 0) & 1) ? -1 : 0) << ";; ++it) {   // it: this pair's item index\n"
       << V2_LOOP_HEAD
       << (x.order.empty() ? "" : "    const long long tb0 = clock64();\n")
       << "    unsigned char* const tile = tiles + " << L.zb << " + s * " << L.zb + L.tb << ";\n"
       << "    const float* wv = wsm + s * 64;\n";
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) os << "    float a" << r << "_" << s << ";\n";
    os << "    switch (t) {\n";
    for (int t0 = 0; t0 < x.nt; ++t0) {
        // O1D_CASE_REV=1: cases emitted in reverse order (code-layout experiment)
        const int t = env_int("O1D_CASE_REV", 0) ? x.nt - 1 - t0 : t0;
        const Geo &g = geo[t];
        const bool w8 = W8 && x.ffma2 && x.act == O1D_F32 && L.pitch % 2 == 0;
        os << "    case " << t << ": {\n"
           << "      const act_t* tb = reinterpret_cast<const act_t*>(tile) + (" << R << " * br) * " << L.pitch << " + " << S
           << " * bc" << (w8 ? " - (bc & 1)" : "") << ";\n";
        const std::vector<int> ds = group_taps(g, 0, 1);
        if (w8) {
            emit_stencil_compute_w8(os, g, ds, "      ");
        } else if (x.ffma2) {
            emit_stencil_compute_ffma2(os, g, ds, "      ");
        } else {
            for (int r = 0; r < R; ++r)
                for (int s = 0; s < S; ++s) os << "      a" << r << "_" << s << " = 0.f;\n";
            for (int d : ds) {
                os << "      const float m" << d << " = ";
                for (size_t k = 0; k < g.taps[d].ks.size(); ++k) os << (k ? " + " : "") << "wv[" << g.taps[d].ks[k] << "]";
                os << ";\n";
            }
            for_each_pixel(g, ds, [&](int i, int j, const std::vector<std::pair<int, std::pair<int, int>>> &uses) {
                os << "      { const float v = LD(tb[" << i * L.pitch + j << "]);";
                for (auto &u : uses) {
                    const int r = u.second.first, s = u.second.second;
                    os << " a" << r << "_" << s << " = fmaf(v, m" << u.first << ", a" << r << "_" << s << ");";
                }
                os << " }\n";
            });
        }
        os << "      break;\n    }\n";
    }
    os << "    }\n"
       << "    if (warm) continue;\n"
       << "    __syncwarp();\n";
    if (L.inslot) {
        // both warps of the pair are done reading the slot before either overwrites it
        if (L.wpg > 1) os << "    asm volatile(\"bar.sync %0, %1;\" :: \"r\"(1 + q), \"r\"(" << 32 * L.wpg << ") : \"memory\");\n";
        os << "    unsigned char* const stg = tile + wg * " << L.sbi << ";   // this warp's output band, in the slot\n"
           << "    ps = s;\n";
    } else {
        os << "    if (lane == 0) { mbar_arrive(empty + s); trace_ev(p.trace, 4, item, trn); }   // done with the slot\n";
    }
    if (YSTG) {  // O1D_YSTG=1: outputs straight from registers (streaming stores), no staging band
        os << "    if (active) {\n"
           << "      act_t* const yo = reinterpret_cast<act_t*>(p.io) + ((u64)(n * " << x.C << " + c) * " << x.Ho << " + " << R
           << " * br) * " << x.Wo << " + " << S << " * bc;\n";
        for (int r = 0; r < R; ++r)
            for (int s2 = 0; s2 < S; ++s2) {
                os << "      ";
                if (ragged) os << "if (" << R << " * br + " << r << " < " << x.Ho << " && " << S << " * bc + " << s2 << " < " << x.Wo << ") ";
                os << "__stcs(yo + " << r * x.Wo + s2 << ", to_act(a" << r << "_" << s2 << "));\n";
            }
        os << "    }\n"
           << "    if (lane == 0) trace_ev(p.trace, 5, item, trn);\n"
           << BAL_ITEM_END
           << "  }\n"
           << BAL_EXIT
           << "}\n";
        g_chunks = 0;
        return os.str();
    }
    os << ""
       << (YST || L.inslot ? "" : "    if (lane == 0) asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\");  // previous band store has read stg\n")
       << "    __syncwarp();\n"
       << "    if (active) {\n"
       << "      act_t* const sto = reinterpret_cast<act_t*>(stg) + (" << R << " * br - row0) * " << x.Wo << " + " << S << " * bc;\n";
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) {
            os << "      ";
            if (ragged) os << "if (" << R << " * br + " << r << " < " << x.Ho << " && " << S << " * bc + " << s << " < " << x.Wo << ") ";
            os << "sto[" << r * x.Wo + s << "] = to_act(a" << r << "_" << s << ");\n";
        }
    os << "    }\n";
    if (YST) {
        // O1D_YSTORE=1: the warp copies its staged band with 16-byte loads/stores (no async-proxy
        // fence, no wait for a previous bulk store); rows are contiguous in stg and in y
        const int band = 4 * R;
        os << "    __syncwarp();\n"
           << "    {\n"
           << "      const int nr = min(" << band << ", " << x.Ho << " - row0);\n"
           << "      const uint4* src = reinterpret_cast<const uint4*>(stg);\n"
           << "      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<act_t*>(p.io) + ((u64)(n * " << x.C << " + c) * " << x.Ho
           << " + row0) * " << x.Wo << ");\n"
           << "      for (int i = lane; i < nr * " << x.Wo * es / 16 << "; i += 32) __stcs(dst + i, src[i]);\n"
           << "    }\n"
           << "    __syncwarp();\n";
    }
    os << (YST ? "    if (false) {\n" : "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n    __syncwarp();\n    if (lane == 0 && row0 < " + std::to_string(x.Ho) + ") {\n")
       << (EFH ? "      asm volatile(\"cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%2, %3, %4, %5}], [%1], %6;\"\n"
                 "                   :: \"l\"(&p.out_map), \"r\"(sa(stg)), \"r\"(0), \"r\"(row0), \"r\"(c), \"r\"(n), \"l\"(policy_evict_first()) : \"memory\");\n"
               : "      asm volatile(\"cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];\"\n"
                 "                   :: \"l\"(&p.out_map), \"r\"(sa(stg)), \"r\"(0), \"r\"(row0), \"r\"(c), \"r\"(n) : \"memory\");\n")
       << "      asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n"
       << "    }\n"
       << "    if (lane == 0) trace_ev(p.trace, 5, item, trn);\n"
       << BAL_ITEM_END
       << "  }\n"
       << "  if (lane == 0) asm volatile(\"cp.async.bulk.wait_group 0;\" ::: \"memory\");\n"
       << BAL_EXIT
       << "}\n";
    g_chunks = 0;
    return os.str();
}

// backward_weight taps with packed FP32 (v2).  Taps adjacent along the table's
// run axis (axis 0: same dh, dw and dw-1; axis 1: same dw, dh and dh-1) share
// the pixel: for pixel px and dy values g(u), g(u+1) one step apart along that
// axis, q[tap a] += g(u) px and q[tap a-1] += g(u+1) px is one fma.rn.f32x2 with
// px as the broadcast operand and (g(u), g(u+1)) an aligned dy register pair
// (u even).  Which tap pair that is depends on the pixel's parity along the
// axis, so each tap has two accumulator halves (set E for even pixel
// coordinates, set O for odd), summed at the end; uses without a partner are
// scalar FMAs into the tap's half of the matching set.
void emit_wgrad_compute_runs(std::ostringstream &os, const Geo &g, const std::vector<int> &ds, int axis,
                             const char *ind, int chunks) {
    auto cn = [](int v) { return v < 0 ? "m" + std::to_string(-v) : std::to_string(v); };
    std::map<std::pair<int, int>, int> at;  // (dh, dw) -> distinct tap
    for (int d : ds) at[{g.taps[d].dh, g.taps[d].dw}] = d;
    auto A = [&](int d) { return axis == 0 ? g.taps[d].dw : g.taps[d].dh; };
    auto Bc = [&](int d) { return axis == 0 ? g.taps[d].dh : g.taps[d].dw; };
    auto tap_at = [&](int b, int a) {  // tap with pair-axis coordinate a, other b
        auto it = at.find(axis == 0 ? std::make_pair(b, a) : std::make_pair(a, b));
        return it == at.end() ? -1 : it->second;
    };
    auto par = [](int v) { return ((v % 2) + 2) % 2; };
    // accumulators: set P (0 = E, 1 = O) pair keyed by its lo tap (coordinate a with par(a) == P)
    // and hi tap (a - 1); a tap whose partner is absent keeps a scalar.
    auto acc_of = [&](int P, int d, bool *is_pair, bool *is_lo, int *lo_tap) {
        const int a = A(d), b = Bc(d);
        const int lo = par(a) == P ? d : tap_at(b, a + 1);
        const int hi = par(a) == P ? tap_at(b, a - 1) : d;
        *is_pair = lo >= 0 && hi >= 0;
        *is_lo = lo == d;
        *lo_tap = lo >= 0 ? lo : d;
        return std::string(*is_pair ? "QP" : "QS") + std::to_string(P) + "_" + std::to_string(*is_pair ? lo : d);
    };
    // lone uses of a paired accumulator: a separate scalar per tap (O1D_WG_LONE=1) or
    // the pair half (=0)
    const bool lone_sep = env_int("O1D_WG_LONE", 1) != 0;
    if (lone_sep)
        for (int d : ds) os << ind << "float QL" << d << " = 0.f;\n";
    // declarations
    std::set<std::string> decl;
    for (int P = 0; P < 2; ++P)
        for (int d : ds) {
            bool ip, il;
            int lt;
            const std::string n = acc_of(P, d, &ip, &il, &lt);
            if (decl.insert(n).second) os << ind << (ip ? "u64 " : "float ") << n << (ip ? " = 0ull;\n" : " = 0.f;\n");
        }
    // dy register pairs along the axis: (g(u), g(u+1)) for even u in 0..5
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) {
            const int u = axis == 0 ? s : r;
            if (u % 2 == 0 && u < 6) {
                const int r2 = axis == 0 ? r : r + 1, s2 = axis == 0 ? s + 1 : s;
                os << ind << "const u64 GP" << r << "_" << s << " = f2pack(g" << r << "_" << s << ", g" << r2 << "_" << s2 << ");\n";
            }
        }
    int npx = 0, ipx = 0;
    for_each_pixel(g, ds, [&](int, int, const std::vector<std::pair<int, std::pair<int, int>>> &) { ++npx; });
    Chunker ch{os, ind, npx, chunks};
    for_each_pixel(g, ds, [&](int i, int j, const std::vector<std::pair<int, std::pair<int, int>>> &uses) {
        ch.at(ipx++);
        os << ind << "{ const float px = LD(tb[" << i * g.pitch + j << "]); const u64 PX = f2pack(px, px);";
        const int P = par(axis == 0 ? j : i);
        // uses keyed by (other block coordinate, coordinate along the axis)
        std::map<std::pair<int, int>, int> u2d;
        for (auto &u : uses) {
            const int r = u.second.first, s = u.second.second;
            u2d[axis == 0 ? std::make_pair(r, s) : std::make_pair(s, r)] = u.first;
        }
        std::set<std::pair<int, int>> done;
        for (auto &kv : u2d) {
            const int o = kv.first.first, uu = kv.first.second, d = kv.second;
            if (done.count(kv.first)) continue;
            const int r = axis == 0 ? o : uu, s = axis == 0 ? uu : o;
            auto nx = u2d.find({o, uu + 1});
            bool ip, il;
            int lt;
            const std::string acc = acc_of(P, d, &ip, &il, &lt);
            if (uu % 2 == 0 && uu < 6 && nx != u2d.end() && ip && il) {
                // lo: tap d (coordinate a = pixel - u), hi: tap at a - 1 == the tap of use u + 1
                os << " " << acc << " = ffma2(GP" << r << "_" << s << ", PX, " << acc << ");";
                done.insert(kv.first);
                done.insert(nx->first);
            } else {
                done.insert(kv.first);
                if (ip && lone_sep) {
                    os << " QL" << d << " = fmaf(g" << r << "_" << s << ", px, QL" << d << ");";
                } else if (ip) {
                    os << " " << acc << " = " << (il ? "f2pack(fmaf(g" : "f2pack(f2lo(" + acc + "), fmaf(g") << r << "_" << s
                       << ", px, " << (il ? "f2lo(" : "f2hi(") << acc << "))" << (il ? ", f2hi(" + acc + "));" : "));");
                } else {
                    os << " " << acc << " = fmaf(g" << r << "_" << s << ", px, " << acc << ");";
                }
            }
        }
        os << " }\n";
    });
    ch.end();
    for (int d : ds) {
        std::string term[2];
        for (int P = 0; P < 2; ++P) {
            bool ip, il;
            int lt;
            const std::string n = acc_of(P, d, &ip, &il, &lt);
            term[P] = ip ? (il ? "f2lo(" + n + ")" : "f2hi(" + n + ")") : n;
        }
        os << ind << "const float q" << d << " = " << term[0] << " + " << term[1] << (lone_sep ? " + QL" + std::to_string(d) : std::string()) << ";\n";
    }
    (void)cn;
}

// backward_weight taps with packed FP32, pixel pairs (v2, default).  Mirror of the
// stencil's A/B scheme: the dy value g(r,s) is the broadcast operand (a plain
// register), the pixel pair (p(u), p(u+1)) one step apart along the table's run
// axis is an aligned register pair (u even, block-relative: every pixel sits in
// exactly one pair, loaded with two LDS.32, no copies), and the accumulator pair
// holds two taps adjacent along that axis: (q[d], q[d + step]).  A tap is the
// low half of one pair and the high half of another (its partners on either
// side), so both are summed at the end; uses with no partner are scalar FMAs.
void emit_wgrad_compute_pp(std::ostringstream &os, const Geo &g, const std::vector<int> &ds, int sh, int sw,
                           const char *ind, int chunks) {
    // (sh, sw): pair step = tap displacement of the two halves; the low pixel of a pair is the
    // one with an even column (sw != 0) or an even row (sw == 0): a partition of the pixels
    auto cn = [](int v) { return v < 0 ? "m" + std::to_string(-v) : std::to_string(v); };
    auto par = [](int v) { return ((v % 2) + 2) % 2; };
    auto is_lo = [&](int i, int j) { return sw != 0 ? par(j) == 0 : par(i) == 0; };
    std::map<std::pair<int, int>, int> at;  // (dh, dw) -> distinct tap
    for (int d : ds) at[{g.taps[d].dh, g.taps[d].dw}] = d;
    auto next_of = [&](int d) {
        auto it = at.find({g.taps[d].dh + sh, g.taps[d].dw + sw});
        return it == at.end() ? -1 : it->second;
    };
    struct Op {
        int lo, hi, r, s, i, j;  // hi < 0: scalar use of tap lo
    };
    std::vector<Op> ops;
    // greedy pairing walks the taps in the step direction (a chain d, d+step, d+2 step, ...)
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
        if (loaded.insert({i, j}).second) os << ind << "const float " << n << " = LD(tb[" << i * g.pitch + j << "]);\n";
        return n;
    };
    Chunker ch{os, ind, (int)ops.size(), chunks};
    std::map<std::string, long> last_use;
    long clock = 0;
    std::vector<std::pair<std::string, std::string>> fm;  // the current pixel-row group's FMAs
    int gkey = 1 << 30;
    auto flush = [&]() {
        emit_lru(os, ind, fm, last_use, clock);
        fm.clear();
    };
    int k = 0;
    const int nops = (int)ops.size();
    for (auto &o : ops) {
        const int key = std::min(o.i, o.i + (o.hi >= 0 ? sh : 0));
        const bool new_chunk = chunks > 1 && (k == 0 || (long)k * chunks / nops != (long)(k - 1) * chunks / nops);
        if (key != gkey || new_chunk) {  // the previous group's FMAs go out before a new group / chunk
            flush();
            gkey = key;
        }
        ch.at(k++);
        if (new_chunk) loaded.clear(), packed.clear();  // values do not cross chunk scopes
        if (o.hi >= 0) {
            const std::string a = px(o.i, o.j), b = px(o.i + sh, o.j + sw), pn = "pp" + cn(o.i) + "_" + cn(o.j);
            if (packed.insert({o.i, o.j}).second) os << ind << "const u64 " << pn << " = f2pack(" << a << ", " << b << ");\n";
            const std::string acc = "QP" + std::to_string(o.lo);
            fm.push_back({acc, acc + " = ffma2(" + pn + ", f2pack(g" + std::to_string(o.r) + "_" + std::to_string(o.s) + ", g" +
                                   std::to_string(o.r) + "_" + std::to_string(o.s) + "), " + acc + ");"});
        } else {
            const std::string a = px(o.i, o.j);
            const std::string acc = "QL" + std::to_string(o.lo);
            fm.push_back({acc, acc + " = fmaf(g" + std::to_string(o.r) + "_" + std::to_string(o.s) + ", " + a + ", " + acc + ");"});
        }
    }
    flush();
    ch.end();
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
}

// pair step for the packed wgrad: the displacement with the most paired products
std::pair<int, int> pp_step(const Geo &g, const std::vector<int> &ds) {
    const std::pair<int, int> cand[] = {{0, 1}, {1, 0}, {-1, 1}, {1, 1}};
    std::pair<int, int> best = cand[0];
    long bestn = -1;
    std::set<std::pair<int, int>> o;
    for (int d : ds) o.insert({g.taps[d].dh, g.taps[d].dw});
    for (auto c : cand) {
        long n = 0;  // adjacent pairs along c (the greedy pairs ~ half of the uses of each adjacent pair)
        for (int d : ds) n += o.count({g.taps[d].dh + c.first, g.taps[d].dw + c.second});
        if (n > bestn) bestn = n, best = c;
    }
    return best;
}

// pair axis of a table for the packed wgrad: the axis with more adjacent tap pairs
int run_axis(const Geo &g) {
    std::set<std::pair<int, int>> o;
    for (auto &t : g.taps) o.insert({t.dh, t.dw});
    int h = 0, v = 0;
    for (auto &t : g.taps) h += o.count({t.dh, t.dw - 1}), v += o.count({t.dh - 1, t.dw});
    return h >= v ? 0 : 1;
}

// backward_weight, v2: x tiles through the slot ring, dy planes through one slot
// per pair (released right after the pair copied its dy blocks to registers).
std::string gen_wgrad2(const Ctx &x, const std::vector<Geo> &geo_in, const std::vector<int> &table_of,
                       const std::vector<int> &count, int Hin, const Lay2 &L) {
    std::ostringstream os;
    std::vector<int> count_b(count);  // scheduler items: (channel, batch of BW planes)
    const int NBATCH = (x.N + L.BW - 1) / L.BW;
    for (int t = 0; t < x.nt; ++t) count_b[t] = count[t] / x.N * NBATCH;
    emit_header(os, x, table_of, count_b);
    const std::vector<Geo> geo = geo2(geo_in, L);
    const int nthreads = 32 * (L.ncw() + L.NPROD);
    g_chunks = (env_int("O1D_WARM", 0) & 2) ? std::min(32, L.ncw()) : 0;  // bit 2: wgrad warm-up (off: see stencil)
    const int es = x.act == O1D_F32 ? 4 : 2;
    int maxd = 0;
    for (int t = 0; t < x.nt; ++t) maxd = std::max(maxd, (int)geo[t].taps.size());
    int NV = 1;
    while (NV < maxd) NV *= 2;  // reduce-scatter width (<= 32 distinct taps)
    // tap -> distinct-tap slot.  In global memory (read through L1): the lanes read 31
    // different entries at once, which the constant cache would serialise
    os << (env_int("O1D_K2S_CONST", 0) ? "__constant__" : "__device__ const") << " unsigned char K2S[" << x.nt << "][" << x.K << "] = {";
    for (int t = 0; t < x.nt; ++t) {
        os << (t ? "," : "") << "{";
        for (int k = 0; k < x.K; ++k) os << (k ? "," : "") << geo[t].k2d[k];
        os << "}";
    }
    os << "};\n"
       << "__device__ __forceinline__ float reduce_scatter_nv(float (&v)[" << NV << "], int lane) {\n"
       << "#pragma unroll\n"
       << "  for (int s = " << NV / 2 << "; s >= 1; s >>= 1) {\n"
       << "    const bool up = lane & s;\n"
       << "#pragma unroll\n"
       << "    for (int i = 0; i < s; ++i) {\n"
       << "      const float send = up ? v[i] : v[i + s];\n"
       << "      const float keep = up ? v[i + s] : v[i];\n"
       << "      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);\n"
       << "    }\n  }\n"
       << "  float r = v[0];\n"
       << "#pragma unroll\n"
       << "  for (int s = " << NV << "; s < 32; s <<= 1) r += __shfl_xor_sync(0xffffffffu, r, s);\n"
       << "  return r;\n}\n";
    os << "extern \"C\" __global__ void __launch_bounds__(" << nthreads << ", 1) o1d_wgrad(const __grid_constant__ Params p) {\n";
    emit_v2_prologue(os, L, nthreads, true, es);
    emit_v2_producer(os, x, L, true, es);
    os << "  float* const scr = reinterpret_cast<float*>(smem + " << L.off_scr << ");\n"
       << "  const act_t* const dys = reinterpret_cast<const act_t*>(smem + " << L.off_dy << " + q * " << L.db << ") + (" << R
       << " * br) * " << L.dyp << " + " << S << " * bc;\n"
       << "  float v[" << NV << "];\n"
       << (x.order.empty() ? "" : "  int bt = -1; u64 busy = 0; unsigned nbusy = 0;   // adaptive placement accounting\n")
       << "  for (int it = " << (g_chunks > 1 || (env_int("O1D_PREWARM", 0) & 2) ? -1 : 0) << ";; ++it) {   // it: this pair's item index\n"
       << V2_LOOP_HEAD
       << (x.order.empty() ? "" : "    const long long tb0 = clock64();\n");
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s)
            os << "    const float g" << r << "_" << s << " = active ? LD(dys[" << r * L.dyp + s << "]) : 0.f;\n";
    os << "    __syncwarp();\n"
       << "    if (lane == 0 && !warm) mbar_arrive(dyempty + q);   // dy block in registers: the pair's dy slot is free\n"
       << "    const unsigned char* const tile = tiles + " << L.zb << " + s * " << L.zb + L.tb << ";\n"
       << (L.BW > 1 ? "    if (item & (1 << 27)) for (int k = 0; k < " + std::to_string(NV) + "; ++k) v[k] = 0.f;   // first plane of the batch\n"
                      : "    for (int k = 0; k < " + std::to_string(NV) + "; ++k) v[k] = 0.f;\n")
       << "    switch (t) {\n";
    for (int t = 0; t < x.nt; ++t) {
        const Geo &g = geo[t];
        os << "    case " << t << ": {\n"
           << "      const act_t* tb = reinterpret_cast<const act_t*>(tile) + (" << R << " * br) * " << L.pitch << " + " << S
           << " * bc;\n";
        const std::vector<int> ds = group_taps(g, 0, 1);
        const int wgm = env_int("O1D_WG_FFMA2", 2);  // 2: pixel pairs (default), 1: dy pairs, 0: scalar
        if (wgm) {
            if (wgm == 2) {
                std::pair<int, int> st = pp_step(g, ds);
                if (env_int("O1D_PPSTEP", -1) >= 0) {  // experiment: force one pairing step for every table
                    const int f = env_int("O1D_PPSTEP", 0);
                    st = f == 0 ? std::make_pair(0, 1) : f == 1 ? std::make_pair(1, 0) : f == 2 ? std::make_pair(-1, 1) : std::make_pair(1, 1);
                }
                emit_wgrad_compute_pp(os, g, ds, st.first, st.second, "      ", g_chunks);
            }
            else emit_wgrad_compute_runs(os, g, ds, run_axis(g), "      ", g_chunks);
            for (size_t k = 0; k < ds.size(); ++k) os << "      v[" << k << "] " << (L.BW > 1 ? "+=" : "=") << " q" << ds[k] << ";\n";
            os << "      break;\n    }\n";
            continue;
        }
        for (int d : ds) os << "      float q" << d << " = 0.f;\n";
        int npx = 0, ipx = 0;
        for_each_pixel(g, ds, [&](int, int, const std::vector<std::pair<int, std::pair<int, int>>> &) { ++npx; });
        Chunker ch{os, "      ", npx, g_chunks};
        for_each_pixel(g, ds, [&](int i, int j, const std::vector<std::pair<int, std::pair<int, int>>> &uses) {
            ch.at(ipx++);
            os << "      { const float px = LD(tb[" << i * L.pitch + j << "]);";
            for (auto &u : uses)
                os << " q" << u.first << " = fmaf(g" << u.second.first << "_" << u.second.second << ", px, q" << u.first << ");";
            os << " }\n";
        });
        ch.end();
        for (size_t k = 0; k < ds.size(); ++k) os << "      v[" << k << "] " << (L.BW > 1 ? "+=" : "=") << " q" << ds[k] << ";\n";
        os << "      break;\n    }\n";
    }
    os << "    }\n"
       << "    if (warm) continue;\n"
       << "    __syncwarp();\n"
       << "    if (lane == 0) { mbar_arrive(empty + s); trace_ev(p.trace, 4, item, trn); }  // x slot released\n"
       << (L.BW > 1 ? "    if (!(item & (1 << 28))) continue;   // reduce once per batch\n" : "")
       << "    const float part = reduce_scatter_nv(v, lane);\n"
       << "    if (lane < " << NV << ") scr[cw * 32 + lane] = part;\n"
       << "    __syncwarp();\n"
       << "    float* wsp = p.ws + ((u64)(c * " << NBATCH << " + n / " << L.BW << ") * " << L.wpg << " + wg) * " << x.K << ";\n"
       << "    for (int k = lane; k < " << x.K << "; k += 32) wsp[k] = scr[cw * 32 + " << (env_int("O1D_K2S_CONST", 0) ? "K2S[t][k]" : "__ldg(&K2S[t][k])") << "];\n"
       << "    __syncwarp();\n"
       << "    if (lane == 0) trace_ev(p.trace, 5, item, trn);\n"
       << BAL_ITEM_END
       << "  }\n"
       << BAL_EXIT
       << "}\n";
    const int NE = NBATCH * L.wpg;
    os << "extern \"C\" __global__ void __launch_bounds__(256) o1d_wgrad_finalize(const float* __restrict__ ws, float* __restrict__ dW) {\n"
       << "  __shared__ double part[8][64];\n"
       << "  pdl_wait();\n"
       << (env_int("O1D_FIN_TRIGGER", 1) ? "  pdl_trigger();   // the next kernel may start its set-up (it waits for our completion)\n" : "")
       << "  const int c = blockIdx.x, j = threadIdx.x >> 5 /* 0..7 */, lane = threadIdx.x & 31;\n"
       << "  const float* base = ws + (u64)c * " << NE << " * " << x.K << ";\n"
       << "  for (int k = lane; k < " << x.K << "; k += 32) {\n"
       << "    double s = 0.0;\n"
       << "#pragma unroll 16\n"
       << "    for (int e = j; e < " << NE << "; e += 8) s += (double)__ldcg(base + (u64)e * " << x.K << " + k);\n"
       << "    part[j][k] = s;\n"
       << "  }\n"
       << "  __syncthreads();\n"
       << "  if (threadIdx.x < " << x.K << ") {\n"
       << "    double s = 0.0;\n"
       << "    for (int k = 0; k < 8; ++k) s += part[k][threadIdx.x];\n"
       << "    dW[c * " << x.K << " + threadIdx.x] = (float)s;\n"
       << "  }\n"
       << "}\n";
    g_chunks = 0;
    return os.str();
}

size_t stencil_smem(const Ctx &x, const std::vector<Geo> &geo) {
    return 2 * tile_bytes_of(geo) + (x.convert ? tile32_bytes_of(geo) : 0) + stage_bytes_of(x) + 3 * 64 * 4 + 32 + 16;
}

// Warp-specialised backward_weight kernel:
//   warp 0      producer: schedules planes, TMA-loads the x tile (per-table box,
//               zero halo) and the dy plane (dense box) into a 2-deep ring
//   warps 1..   consumers: GW tap groups x wpg bands; each thread keeps its 7x7
//               block of dy in registers and accumulates one partial per
//               distinct tap of its group; a warp reduce-scatter leaves the
//               warp's partial of tap L in lane L; partials go to
//               ws[plane][band][k]; the warp that completes a channel (epoch
//               counter) sums them in f64 in (n, band) order into dW.
// backward_weight taps of group `ds` with packed FFMA2 along block ROWS: the
// dy values of rows (0,1), (2,3), (4,5) are register pairs (g pair, one
// alignment for every tap), the pixel pair is the vertical pair
// (px(i,j), px(i+1,j)) with i = r + dh, and each tap accumulates into one
// register pair QP_d; row 6 adds into the low half.  q_d = lo + hi at the end.
void emit_wgrad_compute_ffma2(std::ostringstream &os, const Geo &g, const std::vector<int> &ds, const char *ind) {
    // g pairs (rows 0..5); row 6 stays scalar
    for (int r = 0; r < 6; r += 2)
        for (int s = 0; s < S; ++s)
            os << ind << "const u64 G" << r << "_" << s << " = f2pack(g" << r << "_" << s << ", g" << r + 1 << "_" << s
               << ");\n";
    for (int d : ds) os << ind << "u64 QP" << d << " = 0ull;\n";
    int lo_h = 1 << 20, hi_h = -(1 << 20);
    for (int d : ds) lo_h = std::min(lo_h, g.taps[d].dh), hi_h = std::max(hi_h, g.taps[d].dh);
    std::set<std::pair<int, int>> loaded;
    auto pxn = [](int i, int j) {
        return std::string("px") + (i < 0 ? "m" + std::to_string(-i) : std::to_string(i)) + "_" +
               (j < 0 ? "m" + std::to_string(-j) : std::to_string(j));
    };
    auto load = [&](int i, int j) {
        if (loaded.insert({i, j}).second)
            os << ind << "const float " << pxn(i, j) << " = LDT(tb[" << (i - g.minDH) * g.pitch + (j - g.x0) << "]);\n";
    };
    for (int i = lo_h; i <= hi_h + R - 1; ++i) {
        // pairs starting at footprint row i: taps with r = i - dh in {0, 2, 4}
        std::vector<std::pair<int, int>> pr;  // (d, r)
        std::vector<int> single;              // d with i - dh == 6
        for (int d : ds) {
            const int r = i - g.taps[d].dh;
            if (r == 0 || r == 2 || r == 4) pr.push_back({d, r});
            if (r == 6) single.push_back(d);
        }
        if (pr.empty() && single.empty()) continue;
        std::set<int> pj;
        for (auto &q : pr)
            for (int s = 0; s < S; ++s) pj.insert(g.taps[q.first].dw + s);
        for (int j : pj) load(i, j), load(i + 1, j);
        for (int d : single)
            for (int s = 0; s < S; ++s) load(i, g.taps[d].dw + s);
        for (int j : pj)
            os << ind << "const u64 PV" << (i < 0 ? "m" + std::to_string(-i) : std::to_string(i)) << "_"
               << (j < 0 ? "m" + std::to_string(-j) : std::to_string(j)) << " = f2pack(" << pxn(i, j) << ", "
               << pxn(i + 1, j) << ");\n";
        // slot-major emission: consecutive instructions hit different accumulators
        for (int s = 0; s < S; ++s)
            for (auto &q : pr) {
                const int d = q.first, r = q.second, j = g.taps[d].dw + s;
                os << ind << "QP" << d << " = ffma2(PV" << (i < 0 ? "m" + std::to_string(-i) : std::to_string(i)) << "_"
                   << (j < 0 ? "m" + std::to_string(-j) : std::to_string(j)) << ", G" << r << "_" << s << ", QP" << d
                   << ");\n";
            }
        for (int s = 0; s < S; ++s)
            for (int d : single)
                os << ind << "QP" << d << " = f2pack(fmaf(" << pxn(i, g.taps[d].dw + s) << ", g6_" << s << ", f2lo(QP" << d
                   << ")), f2hi(QP" << d << "));\n";
    }
    for (int d : ds) os << ind << "const float q" << d << " = f2lo(QP" << d << ") + f2hi(QP" << d << ");\n";
}

std::string gen_wgrad(const Ctx &x, const std::vector<Geo> &geo, const std::vector<int> &table_of,
                      const std::vector<int> &count) {
    std::ostringstream os;
    emit_header(os, x, table_of, count);
    const int G = x.G;
    const size_t TB = tile_bytes_of(geo);
    const int es = x.act == O1D_F32 ? 4 : 2, vec = 16 / es;
    const int dyp = (S * x.BC + vec - 1) & ~(vec - 1);  // dy box pitch: whole 7-col blocks, 16-byte rows (zero-filled past Wo)
    const int dyrows = R * x.BR;             // padded rows, zero-filled by TMA
    const size_t DB = ((size_t)dyp * dyrows * es + 1023) & ~(size_t)1023;
    const int ncw = x.wpg * G;
    const size_t T32 = x.convert ? tile32_bytes_of(geo) : 0, OFF32 = 2 * TB;
    const size_t off_dy = 2 * TB + T32, off_scr = off_dy + 2 * DB, off_bar = off_scr + (size_t)ncw * 32 * 4,
                 off_item = off_bar + 32;
    int maxd = 0;
    std::vector<std::vector<int>> k2g(x.nt, std::vector<int>(x.K)), k2s(x.nt, std::vector<int>(x.K));
    for (int t = 0; t < x.nt; ++t)
        for (int gi = 0; gi < G; ++gi) {
            const std::vector<int> ds = group_taps(geo[t], gi, G);
            maxd = std::max(maxd, (int)ds.size());
            for (int k = 0; k < x.K; ++k)
                for (size_t q = 0; q < ds.size(); ++q)
                    if (geo[t].k2d[k] == ds[q]) k2g[t][k] = gi, k2s[t][k] = (int)q;
        }
    int NV = 1;
    while (NV < maxd) NV *= 2;  // reduce-scatter width (<= 32: K <= 64 and G >= 2, or K <= 32)
    os << "__device__ const unsigned char K2G[" << x.nt << "][" << x.K << "] = {";   // global, read via L1 (see gen_wgrad2)
    for (int t = 0; t < x.nt; ++t) {
        os << (t ? "," : "") << "{";
        for (int k = 0; k < x.K; ++k) os << (k ? "," : "") << k2g[t][k];
        os << "}";
    }
    os << "};\n__device__ const unsigned char K2S[" << x.nt << "][" << x.K << "] = {";
    for (int t = 0; t < x.nt; ++t) {
        os << (t ? "," : "") << "{";
        for (int k = 0; k < x.K; ++k) os << (k ? "," : "") << k2s[t][k];
        os << "}";
    }
    os << "};\n";
    // reduce-scatter of NV values over the warp: lane L ends with the warp sum of v[L % NV]
    os << "__device__ __forceinline__ float reduce_scatter_nv(float (&v)[" << NV << "], int lane) {\n"
       << "#pragma unroll\n"
       << "  for (int s = " << NV / 2 << "; s >= 1; s >>= 1) {\n"
       << "    const bool up = lane & s;\n"
       << "#pragma unroll\n"
       << "    for (int i = 0; i < s; ++i) {\n"
       << "      const float send = up ? v[i] : v[i + s];\n"
       << "      const float keep = up ? v[i + s] : v[i];\n"
       << "      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);\n"
       << "    }\n  }\n"
       << "  float r = v[0];\n"
       << "#pragma unroll\n"
       << "  for (int s = " << NV << "; s < 32; s <<= 1) r += __shfl_xor_sync(0xffffffffu, r, s);\n"
       << "  return r;\n}\n";
    const int bcg = (x.BC + 7) / 8;
    const unsigned target = (unsigned)(x.N * ncw);
    os << "extern \"C\" __global__ void __launch_bounds__(" << 32 * (ncw + 1) << ", " << x.minb
       << ") o1d_wgrad(const __grid_constant__ Params p) {\n"
       << "  extern __shared__ __align__(1024) unsigned char smem[];\n"
       << "  float* const scr = reinterpret_cast<float*>(smem + " << off_scr << ");\n"
       << "  u64* const full = reinterpret_cast<u64*>(smem + " << off_bar << ");\n"
       << "  int* const s_item = reinterpret_cast<int*>(smem + " << off_item << ");\n"
       << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n"
       << "  int trn = 0;\n"
       << "  for (int i = threadIdx.x; i < " << (2 * TB + T32) / 16 << "; i += blockDim.x)  // zero guards (and tiles)\n"
       << "    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0u, 0u, 0u, 0u);\n"
       << "  if (tid == 0) { mbar_init(full, 32); mbar_init(full + 1, 32); fence_mbar_init(); }\n"
       << "  __syncthreads();\n"
       << "  if (warp == 0) {\n"
       << "    int tcur = 0, tried = 0; unsigned raw = 0;\n"
       << "    pdl_wait();\n"
       << "    if (lane == 0) { trace_ev(p.trace, 0, -1, trn); tcur = p.only >= 0 ? p.only : HOME[smid() % NHOME]; raw = atomicAdd(p.sched + tcur * CS, 1u); }\n"
       << "    for (int it = 0;; ++it) {\n"
       << "      const int b = it & 1;\n"
       << "      if (it >= 2) asm volatile(\"bar.sync %0, %1;\" :: \"r\"(14 + b), \"r\"(" << 32 * (ncw + 1) << ") : \"memory\");\n"
       << "      int item = -1;\n"
       << "      if (lane == 0) { item = sched_resolve(p.sched, tcur, raw, tried, p.only < 0); sched_prefetch(p.sched, tcur, raw); }\n"
       << "      item = __shfl_sync(0xffffffffu, item, 0);\n"
       << "      if (lane == 0) {\n"
       << "        s_item[b] = item;\n"
       << "        if (item >= 0) {\n"
       << "          int t2, c2, n2; item_cn(item, t2, c2, n2);\n"
       << "          trace_ev(p.trace, 1, item, trn);\n"
       << "          unsigned char* dst = smem + b * " << TB << ";\n"
       << "          switch (t2) {\n";
    for (int t = 0; t < x.nt; ++t)
        os << "          case " << t << ": mbar_expect_tx(full + b, " << geo[t].bytes + (uint32_t)(dyp * dyrows * es)
           << "u); tma_load(dst + " << geo[t].guard << ", &p.in_map[" << t << "], " << geo[t].x0 << ", " << geo[t].minDH
           << ", c2, n2, full + b); break;\n";
    os << "          }\n"
       << "          tma_load(smem + " << off_dy << " + b * " << DB << ", &p.out_map, 0, 0, c2, n2, full + b);\n"
       << "        }\n"
       << "      }\n"
       << "      mbar_arrive(full + b);\n"
       << "      if (item < 0) { pdl_trigger(); break; }\n"
       << "    }\n"
       << "    if (lane == 0) sched_exit(p.sched);\n"
       << "    return;\n"
       << "  }\n"
       << "  const int cw = warp - 1, grp = cw / " << x.wpg << ", wg = cw - grp * " << x.wpg << ";\n"
       << "  int bc = (lane & 7) + 8 * (wg % " << bcg << "), br = (lane >> 3) + 4 * (wg / " << bcg << ");\n"
       << "  const bool active = bc < " << x.BC << " && br < " << x.BR << ";\n"
       << "  if (!active) { bc = 0; br = 0; }\n"
       << "  float v[" << NV << "];\n"
       << "  for (int it = 0;; ++it) {\n"
       << "    const int b = it & 1;\n"
       << "    if (lane == 0) trace_ev(p.trace, 2, it, trn);\n"
       << "    mbar_wait(full + b, (it >> 1) & 1);\n"
       << "    const int item = s_item[b];\n"
       << "    if (lane == 0) trace_ev(p.trace, 3, item, trn);\n"
       << "    if (item < 0) break;\n"
       << "    int t, c, n; item_cn(item, t, c, n);\n"
       << "    const unsigned char* tile = " << (x.convert ? "smem + " + std::to_string(OFF32) : "smem + b * " + std::to_string(TB)) << ";\n"
       << "    const act_t* gb = reinterpret_cast<const act_t*>(smem + " << off_dy << " + b * " << DB << ") + (" << R
       << " * br) * " << dyp << " + " << S << " * bc;\n";
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s)
            os << "    const float g" << r << "_" << s << " = active ? LD(gb[" << r * dyp + s << "]) : 0.f;\n";
    if (x.convert) emit_convert(os, x, geo, TB, OFF32, ncw);  // also releases the dy buffer (g is in registers)
    os << "    for (int q = 0; q < " << NV << "; ++q) v[q] = 0.f;\n"
       << "    switch (t) {\n";
    for (int t = 0; t < x.nt; ++t) {
        const Geo &g = geo[t];
        os << "    case " << t << ": {\n"
           << "      const " << (x.convert ? "float" : "act_t") << "* tb = reinterpret_cast<const " << (x.convert ? "float" : "act_t")
           << "*>(tile + " << (x.convert ? guard32(g) : g.guard) << ") + (" << R << " * br) * " << g.pitch << " + " << S << " * bc;\n";
        for (int gi = 0; gi < G; ++gi) {
            const std::vector<int> ds = group_taps(g, gi, G);
            os << "      " << (gi ? "else " : "") << (gi + 1 < G ? "if (grp == " + std::to_string(gi) + ") " : "") << "{\n";
            if (x.ffma2_w && g_parity_groups && G == 2) {
                emit_wgrad_compute_paired(os, g, ds, pair_axis(g), "        ");
            } else if (x.ffma2_w) {
                emit_wgrad_compute_ffma2(os, g, ds, "        ");
            } else {
                for (int d : ds) os << "        float q" << d << " = 0.f;\n";
                for_each_pixel(g, ds, [&](int i, int j, const std::vector<std::pair<int, std::pair<int, int>>> &uses) {
                    os << "        { const float px = LDT(tb[" << (i - g.minDH) * g.pitch + (j - g.x0) << "]);";
                    for (auto &u : uses)
                        os << " q" << u.first << " = fmaf(g" << u.second.first << "_" << u.second.second << ", px, q"
                           << u.first << ");";
                    os << " }\n";
                });
            }
            for (size_t q = 0; q < ds.size(); ++q) os << "        v[" << q << "] = q" << ds[q] << ";\n";
            os << "      }\n";
        }
        os << "      break;\n    }\n";
    }
    os << "    }\n"
       << (x.convert ? std::string("")
                     : "    asm volatile(\"bar.arrive %0, %1;\" :: \"r\"(14 + b), \"r\"(" + std::to_string(32 * (ncw + 1)) +
                           ") : \"memory\");  // tile + dy released\n")
       << "    if (lane == 0) trace_ev(p.trace, 4, item, trn);\n"
       << "    const float part = reduce_scatter_nv(v, lane);\n"
       << "    if (lane < " << NV << ") scr[cw * 32 + lane] = part;\n"
       << "    __syncwarp();\n"
       << "    float* wsp = p.ws + ((u64)(c * " << x.N << " + n) * " << x.wpg << " + wg) * " << x.K << ";\n"
       << "    for (int k = lane; k < " << x.K << "; k += 32)\n"
       << "      if (__ldg(&K2G[t][k]) == grp) wsp[k] = scr[cw * 32 + __ldg(&K2S[t][k])];\n"
       << "    if (lane == 0) trace_ev(p.trace, 5, item, trn);\n"
       << "  }\n"
       << "}\n";
    // finalize (second launch; the kernel boundary orders the partial writes):
    // dW[c][k] = sum over (n, band) of the partials, f64, fixed order
    // One CTA per channel: thread (j, k) sums entries j, j+8, ... of column k
    // (all loads in flight), then a fixed-order f64 sum over j.
    const int NE = x.N * x.wpg;
    os << "extern \"C\" __global__ void __launch_bounds__(256) o1d_wgrad_finalize(const float* __restrict__ ws, float* __restrict__ dW) {\n"
       << "  __shared__ double part[8][64];\n"
       << "  pdl_wait();\n"
       << (env_int("O1D_FIN_TRIGGER", 1) ? "  pdl_trigger();   // the next kernel may start its set-up (it waits for our completion)\n" : "")
       << "  const int c = blockIdx.x, j = threadIdx.x >> 5 /* 0..7 */, lane = threadIdx.x & 31;\n"
       << "  const float* base = ws + (u64)c * " << NE << " * " << x.K << ";\n"
       << "  for (int k = lane; k < " << x.K << "; k += 32) {\n"
       << "    double s = 0.0;\n"
       << "#pragma unroll 16\n"
       << "    for (int e = j; e < " << NE << "; e += 8) s += (double)__ldcg(base + (u64)e * " << x.K << " + k);\n"
       << "    part[j][k] = s;\n"
       << "  }\n"
       << "  __syncthreads();\n"
       << "  if (threadIdx.x < " << x.K << ") {\n"
       << "    double s = 0.0;\n"
       << "    for (int q = 0; q < 8; ++q) s += part[q][threadIdx.x];\n"
       << "    dW[c * " << x.K << " + threadIdx.x] = (float)s;\n"
       << "  }\n"
       << "}\n";
    return os.str();
}

size_t wgrad_smem(const Ctx &x, const std::vector<Geo> &geo) {
    const size_t TB = tile_bytes_of(geo);
    const int es = x.act == O1D_F32 ? 4 : 2, vec = 16 / es;
    const size_t DB = ((size_t)((S * x.BC + vec - 1) & ~(vec - 1)) * R * x.BR * es + 1023) & ~(size_t)1023;
    return 2 * TB + (x.convert ? tile32_bytes_of(geo) : 0) + 2 * DB + (size_t)x.wpg * x.G * 32 * 4 + 32 + 16;
}

o1d_status encode(CUtensorMap *m, const void *ptr, int dtype, int W, int H, int C, int N, int boxW, int boxH) {
    const size_t es = dtype_size(dtype);
    cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)W * es, (cuuint64_t)W * H * es, (cuuint64_t)W * H * C * es};
    cuuint32_t box[4] = {(cuuint32_t)boxW, (cuuint32_t)boxH, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUtensorMapDataType dt = dtype == O1D_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : dtype == O1D_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    CUresult r = drv().encodeTiled(m, dt, 4, const_cast<void *>(ptr), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (env_flag("O1D_TMA_DEBUG"))
        fprintf(stderr, "[o1d] tensor map dims %d %d %d %d box %d %d -> %d\n", W, H, C, N, boxW, boxH, (int)r);
    if (r != CUDA_SUCCESS) return fail(O1D_CUDA_ERROR, "cuTensorMapEncodeTiled: " + cu_err(r));
    return O1D_OK;
}

}  // namespace

// Home tap table of every SM.  Measured (profiles/r1/icache.md): the SM
// instruction cache is shared by the two SMs of a TPC (splitting TPC mates
// across tables costs 35%), and every extra distinct table running on the GPU
// costs instruction-cache hits (D=1: 40.7 us, 2: 41.1, 4: 45.7, 8: 52.0 forward).
// SMs are ordered GPC by GPC (gpc_map probe) and each table gets a contiguous
// run of TPC pairs proportional to its planes.  mode 1: whole GPCs greedily.
std::vector<int> home_tables(const std::vector<int> &gpc_of_smid, const std::vector<int> &count, int nt) {
    const int n = (int)gpc_of_smid.size();
    std::vector<int> home(n, 0);
    std::map<int, std::vector<int>> groups;  // gpc -> smids (unknown ids: own group)
    for (int s = 0; s < n; ++s) groups[gpc_of_smid[s] >= 0 ? gpc_of_smid[s] : 100000 + s].push_back(s);
    long total = 0;
    for (int t = 0; t < nt; ++t) total += count[t];
    const int mode = env_int("O1D_HOME_MODE", 0);
    if (mode == 1 && (int)groups.size() >= nt) {
        std::vector<std::pair<int, int>> order;  // (size, gpc)
        for (auto &g : groups) order.push_back({-(int)g.second.size(), g.first});
        std::sort(order.begin(), order.end());
        std::vector<double> assigned(nt, 0.0);
        for (auto &o : order) {
            int best = 0;
            double bd = -1;
            for (int t = 0; t < nt; ++t) {
                const double deficit = count[t] / (assigned[t] + 1e-9);
                if (deficit > bd) bd = deficit, best = t;
            }
            assigned[best] += -o.first;
            for (int sm : groups[o.second]) home[sm] = best;
        }
        return home;
    }
    std::vector<int> ordered;
    for (auto &g : groups) ordered.insert(ordered.end(), g.second.begin(), g.second.end());
    if (env_int("O1D_HOME_REV", 0)) std::reverse(ordered.begin(), ordered.end());  // experiment: SM order reversed
    long acc = 0;
    int t = 0;
    const int m = (int)ordered.size();
    for (int i = 0; i < m; i += 2) {  // TPC pairs stay together
        const double pos = (i + 1.0) * (double)total / m;
        while (t < nt - 1 && pos >= acc + count[t]) acc += count[t], ++t;
        home[ordered[i]] = t;
        if (i + 1 < m) home[ordered[i + 1]] = t;
    }
    return home;
}

// Issue-count proxy of each table's case in a generated v2 kernel: packed and scalar
// FMAs plus shared-memory loads between "case t: {" and its "break;" (the measured
// per-item tap-loop times of the eight S1 tables track this within ~5%).
std::vector<long> case_costs(const std::string &src, int nt) {
    std::vector<long> c(nt, 1);
    for (int t = 0; t < nt; ++t) {
        const std::string key = "    case " + std::to_string(t) + ": {";
        const size_t a = src.rfind(key);
        if (a == std::string::npos) continue;
        const size_t b = src.find("break;", a);
        const std::string body = src.substr(a, b == std::string::npos ? std::string::npos : b - a);
        long n = 0;
        for (const char *tok : {"ffma2(", "fmaf(", "LD(", "LDT("}) {
            for (size_t pos = body.find(tok); pos != std::string::npos; pos = body.find(tok, pos + 1)) ++n;
        }
        c[t] = std::max(1L, n);
    }
    return c;
}

// Host-only part: eligibility, geometry and generated sources (no CUDA calls).
// Returns false (and no sources) when the plan is not eligible.
bool spec_prepare(const o1d_plan *pl, SpecSet *sp, std::string src[3], int nsm, const std::vector<int> *gpc) {
    const o1d_desc &d = pl->d;
    const int es = (int)dtype_size(d.dtype);
    if (d.stride != 1) return false;
    if ((d.W * es) % 16 != 0 || d.K > 64) return false;
    if (pl->n_distinct > 16 || (long)d.N * d.C >= (1L << 22)) return false;
    sp->BR = (pl->P + R - 1) / R;
    sp->BC = (pl->Q + S - 1) / S;
    const int bcg = (sp->BC + 7) / 8, brg = (sp->BR + 3) / 4;
    sp->wpg = bcg * brg;
    sp->G = env_int("O1D_G", (sp->wpg <= 2 && d.K >= 8) ? 2 : 1);  // tap groups per plane
    if (sp->G < 1 || sp->G > 4) return false;
    sp->nthreads = 32 * sp->wpg * sp->G;
    sp->nt = pl->n_distinct;
    sp->nsm = nsm;
    std::vector<int> rep(sp->nt, -1);  // one representative channel per distinct table
    sp->count.assign(sp->nt, 0);
    for (int c = 0; c < d.C; ++c) {
        if (rep[pl->table_of[c]] < 0) rep[pl->table_of[c]] = c;
        sp->count[pl->table_of[c]] += d.N;
    }
    for (int t = 0; t < sp->nt; ++t) {
        const int c = rep[t];
        sp->fwd.push_back(make_geo(&pl->oh[(size_t)c * d.K], &pl->ow[(size_t)c * d.K], d.K, false, sp->BR, sp->BC, es, d.W));
        sp->bwd.push_back(make_geo(&pl->oh[(size_t)c * d.K], &pl->ow[(size_t)c * d.K], d.K, true, sp->BR, sp->BC, es, pl->Q));
        for (const Geo *g : {&sp->fwd.back(), &sp->bwd.back()})
            if (g->pitch > 256 || g->rows > 256 || g->bytes > 100 * 1024) return false;
    }
    if (d.W > 256 || d.H > 256 || sp->nthreads > 1024) return false;
    if (sp->BC > 8) return false;  // one 8-block column group per band (W <= 56)
    Ctx x{d.N, d.C, d.K, pl->P, pl->Q, sp->BR, sp->BC, sp->wpg, sp->G, sp->nt, nsm};
    x.ffma2 = env_int("O1D_FFMA2", 1) != 0;
    g_parity_groups = env_int("O1D_PARITY", 0) != 0;
    x.ffma2_w = env_int("O1D_FFMA2_W", g_parity_groups ? 1 : 0) != 0;
    x.act = d.dtype;
    x.convert = x.act != O1D_F32 && env_int("O1D_CONVERT", 0) != 0;
    if (gpc && !gpc->empty()) {
        // SMs per table in proportion to the table's work: planes x estimated issue cost per 7x7
        // block (FMA instructions + footprint loads; measured: cheap 45/135-degree tables otherwise
        // finish early and their SMs idle through the tail)
        std::vector<int> work(sp->nt);
        for (int t = 0; t < sp->nt; ++t)
            work[t] = sp->count[t] * (env_int("O1D_COSTW", 1) ? range_cost(sp->fwd[t], 0, (int)sp->fwd[t].taps.size()) + 100 : 1);
        x.home = home_tables(*gpc, work, sp->nt);
        if (env_int("O1D_ADAPT", 0)) {  // GPC-ordered SM list for the device-side placement update
            std::map<int, std::vector<int>> groups;
            for (int sm = 0; sm < (int)gpc->size(); ++sm) groups[(*gpc)[sm] >= 0 ? (*gpc)[sm] : 100000 + sm].push_back(sm);
            for (auto &gq : groups) x.order.insert(x.order.end(), gq.second.begin(), gq.second.end());
            if (x.order.size() > 256 || sp->nt > 16) x.order.clear();
        }
        // every table has home SMs: no stealing needed for completion
        std::vector<int> seen(sp->nt, 0);
        for (int h : x.home) seen[h] = 1;
        bool all = true;
        for (int v : seen) all = all && v;
        // fewer planes than SMs: the grid does not cover every SM, so a table's home SMs may
        // run no CTA -> CTAs must move on to other tables once theirs is exhausted
        const bool partial_grid = (long)d.N * d.C < 4L * nsm;  // (v1 runs up to 3 CTAs per SM)
        x.steal = !all || partial_grid || env_int("O1D_STEAL", 0) != 0;
        if (partial_grid) x.order.clear();  // adaptive placement assumes one CTA on every SM
    }
    x.minb = env_int("O1D_MINB", 3);
    x.gw = env_int("O1D_GW", 2);
    if (x.gw < 1 || x.gw > 8) return false;
    {
        int maxd = 0;
        for (auto &g : sp->fwd)
            for (int gi = 0; gi < x.gw; ++gi) maxd = std::max(maxd, (int)group_taps(g, gi, x.gw).size());
        if (maxd > 32) return false;
    }
    std::vector<int> table_of(pl->table_of.begin(), pl->table_of.end());
    // v2 pipeline per pass (O1D_V2 bit mask: 1 forward + backward_input, 2 backward_weight)
    const int mask = x.convert ? 0 : env_int("O1D_V2", 3);
    int maxd_all = 0;
    for (auto &g : sp->fwd) maxd_all = std::max(maxd_all, (int)g.taps.size());
    const int hin[3] = {d.H, pl->P, d.H};
    for (int i = 0; i < 3; ++i) {
        const Lay2 L = lay2(x, i == 1 ? sp->bwd : sp->fwd, es, hin[i], i == 2);
        const bool want = (mask >> (i == 2 ? 1 : 0)) & 1;
        sp->v2p[i] = want && sp->BC <= 8 && (i < 2 || maxd_all <= 32) && L.NB >= 2 && L.total + 16 <= 227 * 1024;
        if (sp->v2p[i]) {
            Ctx xi = x;
            xi.G = 1;
            sp->pitch2[i] = L.pitch;
            sp->rows2[i] = hin[i];
            sp->ns2 = L.NS;
            auto gen = [&]() {
                return i < 2 ? gen_stencil2(xi, i == 0 ? sp->fwd : sp->bwd, table_of, sp->count, hin[i], L)
                             : gen_wgrad2(xi, sp->fwd, table_of, sp->count, hin[i], L);
            };
            src[i] = gen();
            if (gpc && !gpc->empty() && env_int("O1D_COSTW", 1) == 1) {
                // home tables of THIS pass from its own generated code: SMs per table in proportion
                // to planes x issue count of the table's case (packed/scalar FMAs + loads); measured:
                // the wgrad's per-table costs differ from the stencil's (pairing varies by angle)
                const std::vector<long> cost = case_costs(src[i], sp->nt);
                std::vector<int> work(sp->nt);
                long mx = 1;
                for (long c : cost) mx = std::max(mx, c);
                // per-item cost outside the case (issue units).  Measured flat from 100 to 500 (the
                // two-SM placement granularity dominates), 0 costs 7% in backward_weight
                const long ovh = env_int("O1D_COST_OVH", 100);
                for (int t = 0; t < sp->nt; ++t)
                    work[t] = (int)std::min<long>(1L << 30, (long)sp->count[t] * (cost[t] + ovh) * 1000 / (mx + ovh));
                xi.home = home_tables(*gpc, work, sp->nt);
                src[i] = gen();
            }
            sp->home2[i] = xi.home;
        }
    }
    sp->v2 = sp->v2p[0] || sp->v2p[1] || sp->v2p[2];
    Ctx xw = x;
    xw.G = x.gw;
    for (int i = 0; i < 2; ++i)
        if (!sp->v2p[i] && stencil_smem(x, i == 0 ? sp->fwd : sp->bwd) > 220 * 1024) return false;
    if (!sp->v2p[2] && wgrad_smem(xw, sp->fwd) > 220 * 1024) return false;
    if (!sp->v2p[0]) src[0] = gen_stencil(x, sp->fwd, table_of, sp->count);
    if (!sp->v2p[1]) src[1] = gen_stencil(x, sp->bwd, table_of, sp->count);
    if (!sp->v2p[2]) src[2] = gen_wgrad(xw, sp->fwd, table_of, sp->count);
    if (sp->v2p[0]) sp->G = 1, sp->nthreads = 32 * lay2(x, sp->fwd, es, d.H, false).ncw();
    sp->gw = x.gw;
    return true;
}

o1d_status spec_create(o1d_plan *pl) {
    pl->spec = nullptr;
    const o1d_desc &d = pl->d;
    Driver &dr = drv();
    if (!dr.err.empty()) return O1D_OK;  // no driver entry points: generic path
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pl->device) != cudaSuccess || nsm < 1)
        return fail(O1D_CUDA_ERROR, "cannot query the SM count");
    SpecSet *sp = new SpecSet();
    std::string src[3];
    std::vector<int> gpc;
    if (!gpc_map(pl->device, &gpc)) gpc.clear();
    if (!spec_prepare(pl, sp, src, nsm, &gpc)) {
        delete sp;
        return O1D_OK;
    }
    const char *names[3] = {"o1d_fwd.cu", "o1d_bwd_in.cu", "o1d_wgrad.cu"};
    if (const char *dir = getenv("O1D_DUMP_SOURCE")) {
        for (int i = 0; i < 3; ++i) {
            FILE *f = fopen((std::string(dir) + "/" + names[i]).c_str(), "w");
            if (f) {
                fputs(src[i].c_str(), f);
                fclose(f);
            }
        }
    }
    std::vector<char> cubin[3];
    std::string logs[3];
    bool ok[3];
    {
        std::vector<std::thread> th;
        for (int i = 0; i < 3; ++i)
            th.emplace_back([&, i] { ok[i] = compile_cubin(src[i], names[i], &cubin[i], &logs[i]); });
        for (auto &t : th) t.join();
    }
    for (int i = 0; i < 3; ++i)
        if (!ok[i]) {
            delete sp;
            return fail(O1D_JIT_ERROR, std::string("NVRTC failed for ") + names[i] + ":\n" + logs[i].substr(0, 4000));
        }
    Ctx x{d.N, d.C, d.K, pl->P, pl->Q, sp->BR, sp->BC, sp->wpg, sp->G, sp->nt, nsm};
    x.act = d.dtype;
    x.convert = x.act != O1D_F32 && env_int("O1D_CONVERT", 0) != 0;
    {
        const int es = (int)dtype_size(d.dtype);
        const Lay2 L[3] = {lay2(x, sp->fwd, es, d.H, false), lay2(x, sp->bwd, es, pl->P, false),
                           lay2(x, sp->fwd, es, d.H, true)};
        Ctx x1 = x;
        x1.G = env_int("O1D_G", (sp->wpg <= 2 && d.K >= 8) ? 2 : 1);
        Ctx xw = x;
        xw.G = sp->gw;
        for (int i = 0; i < 3; ++i) {
            if (sp->v2p[i]) {
                sp->smem[i] = L[i].total + 16, sp->threads[i] = 32 * (L[i].ncw() + L[i].NPROD);
            } else if (i < 2) {
                sp->smem[i] = stencil_smem(x1, i == 0 ? sp->fwd : sp->bwd);
                sp->threads[i] = 32 * (sp->wpg * x1.G + 1);
            } else {
                sp->threads[2] = 32 * (sp->wpg * sp->gw + 1);
                sp->smem[2] = wgrad_smem(xw, sp->fwd);
            }
        }
    }
    const char *fnames[3] = {"o1d_stencil", "o1d_stencil", "o1d_wgrad"};
    PFN_cuOccupancyMaxActiveBlocksPerMultiprocessor_v6050 occ = nullptr;
    std::string e;
    entry("cuOccupancyMaxActiveBlocksPerMultiprocessor", &occ, &e);
    const long planes = (long)d.N * d.C;
    for (int i = 0; i < 3; ++i) {
        CUresult r = dr.moduleLoadData(&sp->mod[i], cubin[i].data());
        if (r == CUDA_SUCCESS) r = dr.moduleGetFunction(&sp->fn[i], sp->mod[i], fnames[i]);
        if (r == CUDA_SUCCESS && i == 2) r = dr.moduleGetFunction(&sp->fin, sp->mod[i], "o1d_wgrad_finalize");
        if (r == CUDA_SUCCESS)
            r = dr.funcSetAttribute(sp->fn[i], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)sp->smem[i]);
        int blocks = 0;
        if (r == CUDA_SUCCESS && occ) r = occ(&blocks, sp->fn[i], sp->threads[i], sp->smem[i]);
        if (r != CUDA_SUCCESS || blocks < 1) {
            for (int j = 0; j <= i; ++j)
                if (sp->mod[j]) dr.moduleUnload(sp->mod[j]);
            delete sp;
            return fail(O1D_CUDA_ERROR, std::string("loading specialised kernel: ") +
                                            (r != CUDA_SUCCESS ? cu_err(r) : "zero occupancy"));
        }
        sp->grid[i] = (int)std::min<long>(planes, (long)blocks * nsm);
        const std::string &lg = logs[i];
        size_t fpos = lg.find(std::string("for ") + fnames[i] + "\n");
        if (fpos == std::string::npos) fpos = lg.find(std::string("Compiling entry function '") + fnames[i] + "'");
        size_t pos = lg.find("Used ", fpos == std::string::npos ? 0 : fpos);
        sp->regs[i] = pos == std::string::npos ? "?" : lg.substr(pos, lg.find('\n', pos) - pos);
    }
    const size_t nsched = (size_t)3 * kSlots * (sp->nt + 1) * kCS + d.C;
    if (cudaMalloc(&sp->d_sched, sizeof(unsigned) * nsched) != cudaSuccess ||
        cudaMemset(sp->d_sched, 0, sizeof(unsigned) * nsched) != cudaSuccess) {
        for (int j = 0; j < 3; ++j) dr.moduleUnload(sp->mod[j]);
        delete sp;
        return fail(O1D_CUDA_ERROR, "scheduler counter allocation failed");
    }
    if (env_flag("O1D_TRACE") && cudaMalloc(&sp->d_trace, kTraceBytes) == cudaSuccess)
        cudaMemset(sp->d_trace, 0, kTraceBytes);
    if (sp->v2 && !gpc.empty() && env_int("O1D_ADAPT", 0) && cudaMalloc(&sp->d_bal, 3 * kBalBytes) == cudaSuccess) {
        std::vector<unsigned char> init(3 * kBalBytes, 0);
        for (int i = 0; i < 3; ++i) {
            unsigned *home = reinterpret_cast<unsigned *>(init.data() + i * kBalBytes + 16 * 8 + 16 * 4 + 16 * 4 + 8);
            for (size_t k = 0; k < sp->home2[i].size() && k < 256; ++k) home[k] = (unsigned)sp->home2[i][k];
        }
        if (cudaMemcpy(sp->d_bal, init.data(), init.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaFree(sp->d_bal);
            sp->d_bal = nullptr;
        }
    }
    pl->spec = sp;
    char buf[768];
    snprintf(buf, sizeof buf,
             "spec%s(persistent warp-specialised, 7x7 blocks, %d consumer threads/CTA (%d tap groups), %d tap tables, TMA 4-D %d-slot ring; "
             "fwd grid %d smem %zu [%s]; bwd_in grid %d [%s]; wgrad grid %d smem %zu [%s])",
             sp->v2 ? "-v2" : "", sp->nthreads, sp->G, sp->nt, sp->v2 ? sp->ns2 : 2, sp->grid[0], sp->smem[0], sp->regs[0].c_str(), sp->grid[1], sp->regs[1].c_str(),
             sp->grid[2], sp->smem[2], sp->regs[2].c_str());
    pl->describe = buf;
    if (env_flag("O1D_VERBOSE")) fprintf(stderr, "[o1d] %s\n", buf);
    return O1D_OK;
}

void spec_destroy(o1d_plan *pl) {
    SpecSet *sp = pl->spec;
    if (!sp) return;
    for (int i = 0; i < 3; ++i)
        if (sp->mod[i]) drv().moduleUnload(sp->mod[i]);
    if (sp->d_sched) cudaFree(sp->d_sched);
    if (sp->d_trace) cudaFree(sp->d_trace);
    if (sp->d_bal) cudaFree(sp->d_bal);
    delete sp;
    pl->spec = nullptr;
}

bool spec_has(const o1d_plan *pl, int pass) { return pl->spec && pass >= 0 && pass < 3; }
// batch windows (o1d_step_host pipelining): every pass on the v2 kernels with the default
// channel-major item order, single-plane wgrad items and the default scheduler
bool spec_window_ok(const o1d_plan *pl) {
    const SpecSet *sp = pl->spec;
    return sp && sp->v2p[0] && sp->v2p[1] && sp->v2p[2] && env_int("O1D_CMAJOR", 1) && env_int("O1D_WB", 1) == 1 &&
           !env_int("O1D_SCHED2", 0) && !env_int("O1D_SEQ", 0);
}
o1d_status spec_finalize(const o1d_plan *pl, float *dW, const float *ws, void *stream) {
    const SpecSet *sp = pl->spec;
    const void *wsp = ws;
    void *fargs[] = {&wsp, &dW};
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
    fc.numAttrs = env_int("O1D_PDL", 1) != 0 ? 1 : 0;
    const CUresult r = drv().launchKernelEx(&fc, sp->fin, fargs, nullptr);
    if (r != CUDA_SUCCESS) return fail(O1D_CUDA_ERROR, "launch of wgrad finalize: " + cu_err(r));
    return O1D_OK;
}
int spec_launches(const o1d_plan *, int pass) { return pass == 2 ? 2 : 1; }
size_t spec_workspace_bytes(const o1d_plan *pl) {
    if (!pl->spec) return 0;
    return sizeof(float) * (size_t)pl->d.N * pl->d.C * pl->spec->wpg * pl->d.K;
}

o1d_status spec_run(const o1d_plan *pl, int pass, const void *a, const float *w, const void *b, float *dW, float *ws,
                    void *stream, int n0, int nlen, bool finalize, bool nowait) {
    if (nlen > 0 && !spec_window_ok(pl)) return fail(O1D_UNSUPPORTED, "batch windows need the v2 kernels");
    const SpecSet *sp = pl->spec;
    const o1d_desc &d = pl->d;
    const int nt = sp->nt;
    alignas(64) unsigned char blob[sizeof(CUtensorMap) * 17 + 12 * sizeof(void *)];
    CUtensorMap *maps = reinterpret_cast<CUtensorMap *>(blob);
    const std::vector<Geo> &geo = pass == 1 ? sp->bwd : sp->fwd;
    // input maps (x for forward / wgrad, dy for backward_input), one box per table
    const int inW = pass == 1 ? pl->Q : d.W, inH = pass == 1 ? pl->P : d.H;
    for (int t = 0; t < nt; ++t) {
        // v2: one box for every table (uniform pitch, image rows only); v1: the table's own footprint
        const int bw = sp->v2p[pass] ? sp->pitch2[pass] : geo[t].pitch, bh = sp->v2p[pass] ? sp->rows2[pass] : geo[t].rows;
        if (o1d_status st = encode(&maps[t], a, d.dtype, inW, inH, d.C, d.N, bw, bh)) return st;
    }
    if (pass != 2) {  // dense output band box for the TMA store
        const int oW = pass == 1 ? d.W : pl->Q, oH = pass == 1 ? d.H : pl->P;
        if (o1d_status st = encode(&maps[nt], b, d.dtype, oW, oH, d.C, d.N, oW, std::min(oH, 4 * R))) return st;
    } else {  // dy plane, rows padded to whole 7-row blocks (zero-filled)
        const int vec = 16 / (int)dtype_size(d.dtype);
        if (o1d_status st = encode(&maps[nt], b, d.dtype, pl->Q, pl->P, d.C, d.N, (S * sp->BC + vec - 1) & ~(vec - 1), R * sp->BR))
            return st;
    }
    void **ptrs = reinterpret_cast<void **>(blob + sizeof(CUtensorMap) * (nt + 1));
    ptrs[0] = const_cast<float *>(w);
    ptrs[1] = const_cast<void *>(b);
    ptrs[2] = ws;
    const unsigned slot = const_cast<SpecSet *>(sp)->launch_seq.fetch_add(1) % kSlots;
    ptrs[3] = sp->d_sched + ((size_t)pass * kSlots + slot) * (nt + 1) * kCS;
    ptrs[4] = sp->d_sched + (size_t)3 * kSlots * (nt + 1) * kCS;
    ptrs[5] = dW;
    int *only = reinterpret_cast<int *>(ptrs + 6);
    *only = -1;
    {
        static std::atomic<unsigned> adapt_seq{0};
        const int k = std::max(1, env_int("O1D_ADAPT_EVERY", 8));
        only[1] = (adapt_seq.fetch_add(1) % (unsigned)k) == 0 ? 1 : 0;
    }
    ptrs[7] = sp->d_trace;
    ptrs[8] = (sp->d_bal && sp->v2p[pass] && sp->home2[pass].size() > 0) ? sp->d_bal + (size_t)pass * kBalBytes : nullptr;
    int *win = reinterpret_cast<int *>(ptrs + 9);
    win[0] = nlen > 0 ? n0 : 0;
    win[1] = nlen > 0 ? nlen : 0;
    *reinterpret_cast<int *>(ptrs + 10) = (nowait && sp->v2p[pass]) ? 1 : 0;
    void *args[] = {blob};
    CUlaunchAttribute attr[1];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[0].value.programmaticStreamSerializationAllowed = 1;
    const bool pdl = env_int("O1D_PDL", 1) != 0;
    CUlaunchConfig cfg{};
    cfg.gridDimX = (unsigned)sp->grid[pass];
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = (unsigned)sp->threads[pass];
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.sharedMemBytes = (unsigned)sp->smem[pass];
    cfg.hStream = static_cast<CUstream>(stream);
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (ptrs[8] && env_int("O1D_ADAPT_DEBUG", 0)) {  // diagnostics: the placement state this launch starts from
        std::vector<unsigned char> hb(kBalBytes);
        cudaDeviceSynchronize();
        cudaMemcpy(hb.data(), ptrs[8], kBalBytes, cudaMemcpyDeviceToHost);
        const float *ema = reinterpret_cast<const float *>(hb.data() + 192);
        const unsigned *home = reinterpret_cast<const unsigned *>(hb.data() + 264);
        std::vector<int> cnt(nt, 0);
        for (int q = 0; q < sp->nsm && q < 256; ++q) cnt[home[q] < (unsigned)nt ? home[q] : 0]++;
        fprintf(stderr, "[o1d adapt] pass %d SMs/table:", pass);
        for (int t = 0; t < nt; ++t) fprintf(stderr, " %d", cnt[t]);
        fprintf(stderr, "  ema:");
        for (int t = 0; t < nt; ++t) fprintf(stderr, " %.0f", ema[t]);
        fprintf(stderr, "\n");
    }
    CUresult r = CUDA_SUCCESS;
    if (env_int("O1D_SEQ", 0) != 0 && nt > 1) {
        // table-sequential: one launch per distinct table, the whole GPU on one code path at a time
        for (int t = 0; t < nt && r == CUDA_SUCCESS; ++t) {
            *only = t;
            const unsigned sl = const_cast<SpecSet *>(sp)->launch_seq.fetch_add(1) % kSlots;
            ptrs[3] = sp->d_sched + ((size_t)pass * kSlots + sl) * (nt + 1) * kCS;
            r = drv().launchKernelEx(&cfg, sp->fn[pass], args, nullptr);
        }
    } else {
        r = drv().launchKernelEx(&cfg, sp->fn[pass], args, nullptr);
    }
    if (r != CUDA_SUCCESS) return fail(O1D_CUDA_ERROR, "launch of specialised kernel: " + cu_err(r));
    if (pass == 2 && finalize) {
        const void *wsp = ws;
        void *fargs[] = {&wsp, &dW};
        CUlaunchConfig fc = cfg;
        fc.gridDimX = (unsigned)d.C;
        fc.blockDimX = 256;
        fc.sharedMemBytes = 0;
        r = drv().launchKernelEx(&fc, sp->fin, fargs, nullptr);
        if (r != CUDA_SUCCESS) return fail(O1D_CUDA_ERROR, "launch of wgrad finalize: " + cu_err(r));
    }
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
    std::string src[3];
    if (pass < 0 || pass > 2) return fail(O1D_INVALID_ARG, "pass must be 0, 1 or 2");
    if (!spec_prepare(pl, &sp, src, 148, nullptr)) return fail(O1D_UNSUPPORTED, "plan is not eligible for specialised kernels");
    *out = src[pass];
    return O1D_OK;
}

}  // namespace o1d
