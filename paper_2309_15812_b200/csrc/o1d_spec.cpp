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
#include <mutex>
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
                  entry("cuTensorMapEncodeTiled", &d.encodeTiled, &e) && entry("cuGetErrorString", &d.getErrorString, &e);
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
    int rows, pitch;       // TMA box (rows x pitch floats) = shared-memory tile
    int x0;                // first tile column (image coords), 16-byte aligned: TMA needs an
                           // aligned innermost start coordinate
    uint32_t bytes;
};

int pitch_for(int cols) {
    int p = cols;
    while (p % 16 != 8) ++p;  // 7*pitch = 8 or 24 mod 32 -> conflict-free LDS.32
    return p;
}

Geo make_geo(const int16_t *oh, const int16_t *ow, int K, bool negate, int BR, int BC, int es) {
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
    const int vec = 16 / es;
    g.x0 = g.minDW >= 0 ? (g.minDW / vec) * vec : -((-g.minDW + vec - 1) / vec) * vec;
    g.rows = R * BR + (g.maxDH - g.minDH);
    g.pitch = pitch_for(S * BC + (g.maxDW - g.x0));
    g.bytes = (uint32_t)(g.rows * g.pitch * es);
    return g;
}

}  // namespace

struct SpecSet {
    int BR = 0, BC = 0, nthreads = 0, nwarps = 0, nt = 0;
    int sdy_pitch = 0;
    std::vector<Geo> fwd, bwd;  // per distinct table
    CUmodule mod[3] = {nullptr, nullptr, nullptr};
    CUfunction fn[3] = {nullptr, nullptr, nullptr};
    size_t smem[3] = {0, 0, 0};
    unsigned *d_counters = nullptr;
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
  TmaDesc aux_map;
  const float* w;
  float* ws;
  unsigned* cnt;
  float* dW;
};
__device__ __forceinline__ u32 sa(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* b, u32 n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(n));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(u64* b, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* b, u32 ph) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
               :: "r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const TmaDesc* m, int x, int y, int z, int w, u64* b) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
               :: "r"(sa(dst)), "l"(m), "r"(x), "r"(y), "r"(z), "r"(w), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void tma_store(const TmaDesc* m, const void* src, int x, int y, int z, int w) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
               :: "l"(m), "r"(sa(src)), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
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
)";

struct Ctx {
    int N, C, K, Ho, Wo, BR, BC, nthreads, nwarps, nt;
    int sdy_pitch;
};

void emit_header(std::ostringstream &os, const Ctx &x, const std::vector<int> &table_of) {
    os << "#define NT " << x.nt << "\n" << kPrelude;
    os << "__constant__ unsigned char TABLE_OF[" << x.C << "] = {";
    for (int c = 0; c < x.C; ++c) os << (c ? "," : "") << table_of[c];
    os << "};\n";
}

// thread -> 7x7 block map: lanes cover 8 block-columns x 4 block-rows
void emit_thread_map(std::ostringstream &os, const Ctx &x) {
    const int bcg = (x.BC + 7) / 8;
    os << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n"
       << "  int bc = (lane & 7) + 8 * (warp % " << bcg << "), br = (lane >> 3) + 4 * (warp / " << bcg << ");\n"
       << "  const bool active = bc < " << x.BC << " && br < " << x.BR << ";\n"
       << "  if (!active) { bc = 0; br = 0; }\n";
}

// For each footprint row i (relative to the block's top row), the (r, tap) pairs
// reading it; emit one LDS per needed input pixel and the FMAs that consume it.
template <typename F>
void for_each_pixel(const Geo &g, F &&f) {
    for (int i = g.minDH; i <= g.maxDH + R - 1; ++i) {
        std::vector<std::pair<int, int>> pairs;  // (r, distinct tap)
        for (int r = 0; r < R; ++r)
            for (int d = 0; d < (int)g.taps.size(); ++d)
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

void emit_weights(std::ostringstream &os, const Geo &g, int K) {
    for (int k = 0; k < K; ++k) os << "    const float w" << k << " = __ldg(wp + " << k << ");\n";
    for (int d = 0; d < (int)g.taps.size(); ++d) {
        os << "    const float m" << d << " = ";
        for (size_t i = 0; i < g.taps[d].ks.size(); ++i) os << (i ? " + " : "") << "w" << g.taps[d].ks[i];
        os << ";\n";
    }
}

std::string gen_stencil(const Ctx &x, const std::vector<Geo> &geo, const std::vector<int> &table_of) {
    std::ostringstream os;
    emit_header(os, x, table_of);
    size_t tile_bytes = (size_t)x.Ho * x.Wo * 4;
    for (auto &g : geo) tile_bytes = std::max(tile_bytes, (size_t)g.bytes);
    tile_bytes = (tile_bytes + 127) & ~(size_t)127;
    os << "extern \"C\" __global__ void __launch_bounds__(" << x.nthreads << ") o1d_stencil(const __grid_constant__ Params p) {\n"
       << "  extern __shared__ __align__(1024) unsigned char smem[];\n"
       << "  float* tile = reinterpret_cast<float*>(smem);\n"
       << "  u64* bar = reinterpret_cast<u64*>(smem + " << tile_bytes << ");\n"
       << "  const int c = blockIdx.x / " << x.N << ", n = blockIdx.x - c * " << x.N << ";\n"
       << "  const int t = TABLE_OF[c];\n";
    emit_thread_map(os, x);
    os << "  if (tid == 0) {\n    mbar_init(bar, 1);\n    switch (t) {\n";
    for (int t = 0; t < x.nt; ++t)
        os << "      case " << t << ": mbar_expect(bar, " << geo[t].bytes << "u); tma_load(tile, &p.in_map[" << t
           << "], " << geo[t].x0 << ", " << geo[t].minDH << ", c, n, bar); break;\n";
    os << "    }\n  }\n  const float* wp = p.w + c * " << x.K << ";\n";
    os << "  switch (t) {\n";
    const bool ragged = (R * x.BR != x.Ho) || (S * x.BC != x.Wo);
    for (int t = 0; t < x.nt; ++t) {
        const Geo &g = geo[t];
        os << "  case " << t << ": {\n";
        emit_weights(os, g, x.K);
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s) os << "    float a" << r << "_" << s << " = 0.f;\n";
        os << "    const float* tb = tile + (" << R << " * br) * " << g.pitch << " + " << S << " * bc;\n";
        os << "    __syncthreads();\n    mbar_wait(bar, 0);\n";
        for_each_pixel(g, [&](int i, int j, const std::vector<std::pair<int, std::pair<int, int>>> &uses) {
            os << "    { const float v = tb[" << (i - g.minDH) * g.pitch + (j - g.x0) << "];";
            for (auto &u : uses) {
                const int r = u.second.first, s = u.second.second;
                os << " a" << r << "_" << s << " = fmaf(v, m" << u.first << ", a" << r << "_" << s << ");";
            }
            os << " }\n";
        });
        os << "    __syncthreads();\n    if (active) {\n      float* o = tile + (" << R << " * br) * " << x.Wo << " + "
           << S << " * bc;\n";
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s) {
                os << "      ";
                if (ragged) os << "if (" << R << " * br + " << r << " < " << x.Ho << " && " << S << " * bc + " << s
                               << " < " << x.Wo << ") ";
                os << "o[" << r * x.Wo + s << "] = a" << r << "_" << s << ";\n";
            }
        os << "    }\n    break;\n  }\n";
    }
    os << "  }\n  fence_async_smem();\n  __syncthreads();\n"
       << "  if (tid == 0) tma_store(&p.aux_map, tile, 0, 0, c, n);\n}\n";
    return os.str();
}

std::string gen_wgrad(const Ctx &x, const std::vector<Geo> &geo, const std::vector<int> &table_of) {
    std::ostringstream os;
    emit_header(os, x, table_of);
    size_t tile_bytes = 0;
    for (auto &g : geo) tile_bytes = std::max(tile_bytes, (size_t)g.bytes);
    tile_bytes = (tile_bytes + 1023) & ~(size_t)1023;
    const size_t dy_bytes = ((size_t)R * x.BR * x.sdy_pitch * 4 + 127) & ~(size_t)127;
    const int rounds = (x.K + 31) / 32;
    os << "__constant__ unsigned char K2D[" << x.nt << "][" << x.K << "] = {";
    for (int t = 0; t < x.nt; ++t) {
        os << (t ? "," : "") << "{";
        for (int k = 0; k < x.K; ++k) os << (k ? "," : "") << geo[t].k2d[k];
        os << "}";
    }
    os << "};\n";
    os << "extern \"C\" __global__ void __launch_bounds__(" << x.nthreads << ") o1d_wgrad(const __grid_constant__ Params p) {\n"
       << "  extern __shared__ __align__(1024) unsigned char smem[];\n"
       << "  float* tile = reinterpret_cast<float*>(smem);\n"
       << "  float* sdy = reinterpret_cast<float*>(smem + " << tile_bytes << ");\n"
       << "  float* red = reinterpret_cast<float*>(smem + " << tile_bytes + dy_bytes << ");\n"
       << "  u64* bar = reinterpret_cast<u64*>(smem + " << tile_bytes + dy_bytes + 4 * 32 * rounds * x.nwarps << ");\n"
       << "  __shared__ int s_last;\n"
       << "  const int c = blockIdx.x / " << x.N << ", n = blockIdx.x - c * " << x.N << ";\n"
       << "  const int t = TABLE_OF[c];\n";
    emit_thread_map(os, x);
    os << "  if (tid == 0) {\n    mbar_init(bar, 1);\n    switch (t) {\n";
    const uint32_t dyb = (uint32_t)(R * x.BR * x.sdy_pitch * 4);
    for (int t = 0; t < x.nt; ++t)
        os << "      case " << t << ": mbar_expect(bar, " << geo[t].bytes + dyb << "u); tma_load(tile, &p.in_map[" << t
           << "], " << geo[t].x0 << ", " << geo[t].minDH << ", c, n, bar); break;\n";
    os << "    }\n    tma_load(sdy, &p.aux_map, 0, 0, c, n, bar);\n  }\n";
    os << "  float v0[32]";
    for (int rd = 1; rd < rounds; ++rd) os << ", v" << rd << "[32]";
    os << ";\n  __syncthreads();\n  mbar_wait(bar, 0);\n";
    os << "  const float* gb = sdy + (" << R << " * br) * " << x.sdy_pitch << " + " << S << " * bc;\n";
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s)
            os << "  const float g" << r << "_" << s << " = active ? gb[" << r * x.sdy_pitch + s << "] : 0.f;\n";
    os << "  switch (t) {\n";
    for (int t = 0; t < x.nt; ++t) {
        const Geo &g = geo[t];
        const int nd = (int)g.taps.size();
        os << "  case " << t << ": {\n";
        for (int d = 0; d < nd; ++d) os << "    float q" << d << " = 0.f;\n";
        os << "    const float* tb = tile + (" << R << " * br) * " << g.pitch << " + " << S << " * bc;\n";
        for_each_pixel(g, [&](int i, int j, const std::vector<std::pair<int, std::pair<int, int>>> &uses) {
            os << "    { const float v = tb[" << (i - g.minDH) * g.pitch + (j - g.x0) << "];";
            for (auto &u : uses)
                os << " q" << u.first << " = fmaf(g" << u.second.first << "_" << u.second.second << ", v, q" << u.first
                   << ");";
            os << " }\n";
        });
        for (int d = 0; d < 32 * rounds; ++d)
            os << "    v" << d / 32 << "[" << d % 32 << "] = " << (d < nd ? "q" + std::to_string(d) : "0.f") << ";\n";
        os << "    break;\n  }\n";
    }
    os << "  }\n";
    for (int rd = 0; rd < rounds; ++rd)
        os << "  red[warp * " << 32 * rounds << " + " << 32 * rd << " + lane] = reduce_scatter32(v" << rd << ", lane);\n";
    os << "  __syncthreads();\n"
       << "  float* wsp = p.ws + (u64)blockIdx.x * " << x.K << ";\n"
       << "  if (tid < " << x.K << ") {\n    const int d = K2D[t][tid];\n    float s = 0.f;\n"
       << "    for (int w = 0; w < " << x.nwarps << "; ++w) s += red[w * " << 32 * rounds << " + d];\n"
       << "    wsp[tid] = s;\n  }\n"
       << "  __threadfence();\n  __syncthreads();\n"
       << "  if (tid == 0) {\n    const unsigned old = atomicAdd(p.cnt + c, 1u);\n"
       << "    s_last = ((old + 1u) % " << x.N << "u) == 0u;\n  }\n  __syncthreads();\n"
       << "  if (s_last) {\n    __threadfence();\n"
       << "    for (int k = tid; k < " << x.K << "; k += " << x.nthreads << ") {\n      double s = 0.0;\n"
       << "      const float* col = p.ws + (u64)c * " << x.N << " * " << x.K << " + k;\n"
       << "      for (int i = 0; i < " << x.N << "; ++i) s += (double)__ldcg(col + (u64)i * " << x.K << ");\n"
       << "      p.dW[c * " << x.K << " + k] = (float)s;\n    }\n  }\n}\n";
    return os.str();
}

// host mirror of the generated Params (layout must match the emitted struct)
struct alignas(64) HostParamsHead {
    CUtensorMap maps[1];
};

size_t params_size(int nt) { return sizeof(CUtensorMap) * (nt + 1) + 4 * sizeof(void *); }

bool env_flag(const char *n) {
    const char *v = getenv(n);
    return v && *v && strcmp(v, "0") != 0;
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

// Host-only part: eligibility, geometry and generated sources (no CUDA calls).
// Returns false (and no sources) when the plan is not eligible.
bool spec_prepare(const o1d_plan *pl, SpecSet *sp, std::string src[3]) {
    const o1d_desc &d = pl->d;
    if (d.stride != 1 || d.dtype != O1D_F32) return false;
    if ((d.W * 4) % 16 != 0 || d.K > 64) return false;
    if (pl->n_distinct > 16) return false;
    sp->BR = (pl->P + R - 1) / R;
    sp->BC = (pl->Q + S - 1) / S;
    const int bcg = (sp->BC + 7) / 8, brg = (sp->BR + 3) / 4;
    sp->nwarps = bcg * brg;
    sp->nthreads = 32 * sp->nwarps;
    sp->nt = pl->n_distinct;
    sp->sdy_pitch = (S * sp->BC + 3) & ~3;
    std::vector<int> rep(sp->nt, -1);  // one representative channel per distinct table
    for (int c = 0; c < d.C; ++c)
        if (rep[pl->table_of[c]] < 0) rep[pl->table_of[c]] = c;
    for (int t = 0; t < sp->nt; ++t) {
        const int c = rep[t];
        sp->fwd.push_back(make_geo(&pl->oh[(size_t)c * d.K], &pl->ow[(size_t)c * d.K], d.K, false, sp->BR, sp->BC, 4));
        sp->bwd.push_back(make_geo(&pl->oh[(size_t)c * d.K], &pl->ow[(size_t)c * d.K], d.K, true, sp->BR, sp->BC, 4));
        for (const Geo *g : {&sp->fwd.back(), &sp->bwd.back()})
            if (g->pitch > 256 || g->rows > 256 || g->bytes > 160 * 1024) return false;
    }
    if (d.W > 256 || d.H > 256 || sp->nthreads > 1024) return false;
    Ctx x{d.N, d.C, d.K, pl->P, pl->Q, sp->BR, sp->BC, sp->nthreads, sp->nwarps, sp->nt, sp->sdy_pitch};
    std::vector<int> table_of(pl->table_of.begin(), pl->table_of.end());
    src[0] = gen_stencil(x, sp->fwd, table_of);
    src[1] = gen_stencil(x, sp->bwd, table_of);
    src[2] = gen_wgrad(x, sp->fwd, table_of);
    return true;
}

o1d_status spec_create(o1d_plan *pl) {
    pl->spec = nullptr;
    const o1d_desc &d = pl->d;
    Driver &dr = drv();
    if (!dr.err.empty()) return O1D_OK;  // no driver entry points: generic path
    SpecSet *sp = new SpecSet();
    std::string src[3];
    if (!spec_prepare(pl, sp, src)) {
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
    // size the shared memory of each kernel (must match the emitted offsets)
    size_t tile_f = (size_t)pl->P * pl->Q * 4, tile_b = tile_f, tile_w = 0;
    for (auto &g : sp->fwd) tile_f = std::max(tile_f, (size_t)g.bytes), tile_w = std::max(tile_w, (size_t)g.bytes);
    for (auto &g : sp->bwd) tile_b = std::max(tile_b, (size_t)g.bytes);
    tile_f = (tile_f + 127) & ~(size_t)127;
    tile_b = (tile_b + 127) & ~(size_t)127;
    tile_w = (tile_w + 1023) & ~(size_t)1023;
    const size_t dy_bytes = ((size_t)R * sp->BR * sp->sdy_pitch * 4 + 127) & ~(size_t)127;
    sp->smem[0] = tile_f + 16;
    sp->smem[1] = tile_b + 16;
    sp->smem[2] = tile_w + dy_bytes + 4 * 32 * ((d.K + 31) / 32) * sp->nwarps + 16;
    const char *fnames[3] = {"o1d_stencil", "o1d_stencil", "o1d_wgrad"};
    for (int i = 0; i < 3; ++i) {
        CUresult r = dr.moduleLoadData(&sp->mod[i], cubin[i].data());
        if (r == CUDA_SUCCESS) r = dr.moduleGetFunction(&sp->fn[i], sp->mod[i], fnames[i]);
        if (r == CUDA_SUCCESS)
            r = dr.funcSetAttribute(sp->fn[i], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)sp->smem[i]);
        if (r != CUDA_SUCCESS) {
            for (int j = 0; j <= i; ++j)
                if (sp->mod[j]) dr.moduleUnload(sp->mod[j]);
            delete sp;
            return fail(O1D_CUDA_ERROR, std::string("loading specialised kernel: ") + cu_err(r));
        }
        // keep the ptxas register / spill line for describe()
        const std::string &lg = logs[i];
        size_t pos = lg.find("Used ");
        sp->regs[i] = pos == std::string::npos ? "?" : lg.substr(pos, lg.find('\n', pos) - pos);
    }
    if (cudaMalloc(&sp->d_counters, sizeof(unsigned) * d.C) != cudaSuccess ||
        cudaMemset(sp->d_counters, 0, sizeof(unsigned) * d.C) != cudaSuccess) {
        for (int j = 0; j < 3; ++j) dr.moduleUnload(sp->mod[j]);
        delete sp;
        return fail(O1D_CUDA_ERROR, "counter allocation failed");
    }
    pl->spec = sp;
    char buf[512];
    snprintf(buf, sizeof buf,
             "spec(7x7 blocks, %d threads/plane, %d tap tables, TMA 4-D; fwd %zu B smem [%s]; bwd_in [%s]; "
             "wgrad %zu B smem [%s])",
             sp->nthreads, sp->nt, sp->smem[0], sp->regs[0].c_str(), sp->regs[1].c_str(), sp->smem[2],
             sp->regs[2].c_str());
    pl->describe = buf;
    if (env_flag("O1D_VERBOSE")) fprintf(stderr, "[o1d] %s\n", buf);
    return O1D_OK;
}

void spec_destroy(o1d_plan *pl) {
    SpecSet *sp = pl->spec;
    if (!sp) return;
    for (int i = 0; i < 3; ++i)
        if (sp->mod[i]) drv().moduleUnload(sp->mod[i]);
    if (sp->d_counters) cudaFree(sp->d_counters);
    delete sp;
    pl->spec = nullptr;
}

bool spec_has(const o1d_plan *pl, int pass) { return pl->spec && pass >= 0 && pass < 3; }
int spec_launches(const o1d_plan *, int) { return 1; }
size_t spec_workspace_bytes(const o1d_plan *pl) {
    if (!pl->spec) return 0;
    return sizeof(float) * (size_t)pl->d.N * pl->d.C * pl->d.K;
}

o1d_status spec_run(const o1d_plan *pl, int pass, const void *a, const float *w, const void *b, float *dW, float *ws,
                    void *stream) {
    const SpecSet *sp = pl->spec;
    const o1d_desc &d = pl->d;
    const int nt = sp->nt;
    std::vector<unsigned char> blob(params_size(nt) + 64);
    unsigned char *base = blob.data();
    base += (64 - (reinterpret_cast<uintptr_t>(base) & 63)) & 63;
    CUtensorMap *maps = reinterpret_cast<CUtensorMap *>(base);
    const std::vector<Geo> &geo = pass == 1 ? sp->bwd : sp->fwd;
    // input maps: x for forward / wgrad, dy for backward_input; per table box
    const int inW = pass == 1 ? pl->Q : d.W, inH = pass == 1 ? pl->P : d.H;
    for (int t = 0; t < nt; ++t)
        if (o1d_status st = encode(&maps[t], a, d.dtype, inW, inH, d.C, d.N, geo[t].pitch, geo[t].rows)) return st;
    if (pass == 2) {
        // dy (b) staged as a zero-padded 7*BR x sdy_pitch box
        if (o1d_status st = encode(&maps[nt], b, d.dtype, pl->Q, pl->P, d.C, d.N, sp->sdy_pitch, R * sp->BR)) return st;
    } else {
        const int oW = pass == 1 ? d.W : pl->Q, oH = pass == 1 ? d.H : pl->P;
        if (o1d_status st = encode(&maps[nt], b, d.dtype, oW, oH, d.C, d.N, oW, oH)) return st;
    }
    void **ptrs = reinterpret_cast<void **>(base + sizeof(CUtensorMap) * (nt + 1));
    ptrs[0] = const_cast<float *>(w);
    ptrs[1] = ws;
    ptrs[2] = sp->d_counters;
    ptrs[3] = dW;
    void *args[] = {base};
    const unsigned grid = (unsigned)(d.N * d.C);
    CUresult r = drv().launchKernel(sp->fn[pass], grid, 1, 1, sp->nthreads, 1, 1, (unsigned)sp->smem[pass],
                                    static_cast<CUstream>(stream), args, nullptr);
    if (r != CUDA_SUCCESS) return fail(O1D_CUDA_ERROR, "launch of specialised kernel: " + cu_err(r));
    return O1D_OK;
}

o1d_status spec_source(const o1d_plan *pl, int pass, std::string *out) {
    SpecSet sp;
    std::string src[3];
    if (pass < 0 || pass > 2) return fail(O1D_INVALID_ARG, "pass must be 0, 1 or 2");
    if (!spec_prepare(pl, &sp, src)) return fail(O1D_UNSUPPORTED, "plan is not eligible for specialised kernels");
    *out = src[pass];
    return O1D_OK;
}

}  // namespace o1d
