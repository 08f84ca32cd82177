// nbk_capi.cu -- the extern "C" boundary of libnbk.so (include/nbk.h) and the
// host orchestration of the hot path: kernel dispatch over N, the CG loop
// captured once into a CUDA graph per (precision, niter), device-resident
// scalars, one D2H copy of the history per solve; multi-rank z-slabs (NCCL
// face exchange + all-gather of per-rank partials, or in-process virtual
// slabs on one device).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "nbk_internal.h"
#include "nbk_kernels.cuh"

using namespace nbk;

static thread_local std::string g_err;

#define NBK_CUDA(ctx, ...)                                                                \
    do {                                                                                  \
        cudaError_t e__ = (__VA_ARGS__);                                                  \
        if (e__ != cudaSuccess) {                                                         \
            std::string m__ = std::string(#__VA_ARGS__) + ": " + cudaGetErrorString(e__); \
            if (ctx) (ctx)->err = m__; else g_err = m__;                                  \
            return NBK_ECUDA;                                                             \
        }                                                                                 \
    } while (0)

static nbk_status fail(nbk_ctx* ctx, nbk_status st, const std::string& msg)
{
    if (ctx) ctx->err = msg; else g_err = msg;
    return st;
}

static int vec_grid(int64_t n)
{
    int64_t g = (n + 255) / 256;
    if (g < 1) g = 1;
    return (int)(g > NBK_VEC_GRID_MAX ? NBK_VEC_GRID_MAX : g);
}


// ------------------------------------------------------------ dispatchers
// Launch with the programmatic-stream-serialization attribute (PDL) when pdl:
// the kernel may start while its predecessor drains; it calls griddepcontrol.wait
// before touching the predecessor's results.
static bool g_pdl_enabled = [] {
    const char* e = getenv("NBK_PDL");  // opt-in: measured no gain on C2
    return e && e[0] == '1';
}();

template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                            cudaStream_t s, bool pdl, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    const bool on = pdl && g_pdl_enabled;
    cfg.attrs = on ? attr : nullptr;
    cfg.numAttrs = on ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}
// attr_only: set the dynamic shared-memory limit (done once at set-up, never
// under stream capture).
template <typename T, int N, int FUSED, bool VP = false>
static cudaError_t launch_ax_n(const AxArgs<T>& a, cudaStream_t s, bool attr_only = false,
                               bool pdl = false)
{
    constexpr int EPB = ax_epb<T>(N);
    const size_t smem = (size_t)ax_smem_bytes<T>(N);
    if (attr_only)
        return cudaFuncSetAttribute(k_ax<T, N, FUSED, VP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem);
    const unsigned grid = (unsigned)((a.mesh.E + EPB - 1) / EPB);
    return launch_k(k_ax<T, N, FUSED, VP>, grid, ax_threads<T>(N), smem, s, pdl, a);
}

#define NBK_SWITCH_N(N, CALL)                 \
    switch (N) {                              \
    case 2: return CALL(2);                   \
    case 3: return CALL(3);                   \
    case 4: return CALL(4);                   \
    case 5: return CALL(5);                   \
    case 6: return CALL(6);                   \
    case 7: return CALL(7);                   \
    case 8: return CALL(8);                   \
    case 9: return CALL(9);                   \
    case 10: return CALL(10);                 \
    case 11: return CALL(11);                 \
    case 12: return CALL(12);                 \
    case 13: return CALL(13);                 \
    case 14: return CALL(14);                 \
    case 15: return CALL(15);                 \
    case 16: return CALL(16);                 \
    default: return cudaErrorInvalidValue;    \
    }

template <typename T, int FUSED, bool VP = false>
static cudaError_t launch_ax(const AxArgs<T>& a, cudaStream_t s, bool attr_only = false,
                             bool pdl = false)
{
#define AXN(n) launch_ax_n<T, n, FUSED, VP>(a, s, attr_only, pdl)
    if constexpr (VP) {  // VPREC emulation kernels: N <= NBK_VPREC_MAXN (compile time)
        switch (a.mesh.N) {
        case 2: return AXN(2);
        case 3: return AXN(3);
        case 4: return AXN(4);
        case 5: return AXN(5);
        case 6: return AXN(6);
        case 7: return AXN(7);
        case 8: return AXN(8);
        case 9: return AXN(9);
        case 10: return AXN(10);
        case 11: return AXN(11);
        case 12: return AXN(12);
        default: return cudaErrorNotSupported;
        }
    } else {
        NBK_SWITCH_N(a.mesh.N, AXN)
    }
#undef AXN
}

// Resident CTAs of a kernel on the whole device (SM count x occupancy), cached
// per kernel: grids of the streaming kernels are sized to exactly one wave.
static int resident_grid(const void* kern, int block, size_t smem)
{
    static std::map<const void*, int> cache;
    auto it = cache.find(kern);
    if (it != cache.end()) return it->second;
    int dev = 0, sms = 148, nb = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, block, smem) != cudaSuccess || nb < 1) nb = 1;
    int g = nb * sms;
    if (g > NBK_VEC_GRID_MAX) g = NBK_VEC_GRID_MAX;
    cache[kern] = g;
    return g;
}

template <typename T, int V, int MODE, bool VP>
static cudaError_t launch_vec_v(const VecArgs<T>& a, cudaStream_t s, bool pdl)
{
    const int cap = resident_grid((const void*)k_vec<T, V, MODE, VP>, 256, 0);
    int64_t g = (a.n / 4 + 511) / 512;  // >= 2 chunks of 4 points per thread
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return launch_k(k_vec<T, V, MODE, VP>, (unsigned)g, 256, 0, s, pdl, a);
}

// one vector kernel for every N: chunks of 4 points (even N) or 1 (odd N)
template <typename T, int MODE, bool VP = false>
static cudaError_t launch_vec(const VecArgs<T>& a, cudaStream_t s, bool pdl = false)
{
    if (a.mesh.N < 2 || a.mesh.N > 16) return cudaErrorInvalidValue;
    return a.mesh.N % 2 == 0 ? launch_vec_v<T, 4, MODE, VP>(a, s, pdl) : launch_vec_v<T, 1, MODE, VP>(a, s, pdl);
}

template <typename T, bool FUSED, bool VP = false>
static int dssum_grid_t(int ntiles)
{
    const int cap = resident_grid((const void*)k_dssum<T, FUSED, VP>, 256, 0);
    return ntiles < 1 ? 1 : (ntiles > cap ? cap : ntiles);
}

template <typename T, bool FUSED, bool VP = false>
static cudaError_t launch_dssum(const DssumArgs<T>& a, cudaStream_t s, bool pdl = false)
{
    return launch_k(k_dssum<T, FUSED, VP>, dssum_grid_t<T, FUSED, VP>(a.ntiles), 256, 0, s, pdl, a);
}

// ------------------------------------------------------------ NCCL (dlopen)
// NCCL is loaded at run time only when a context has nranks > 1 and a unique
// id, so that the process uses the one libnccl.so.2 torch has already loaded
// (dlopen by soname returns the loaded copy) and 1-rank use needs no NCCL.
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
};

static const NcclApi* nccl_api(std::string& why)
{
    static NcclApi api;
    static int state = 0;  // 0 untried, 1 ok, -1 failed
    static std::string err;
    if (state == 0) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
#ifdef NBK_NCCL_LIB
        if (!h) h = dlopen(NBK_NCCL_LIB, RTLD_NOW | RTLD_GLOBAL);
#endif
        if (!h) {
            err = std::string("cannot load libnccl.so.2: ") + dlerror();
            state = -1;
        } else {
#define NBK_SYM(f, n) api.f = (decltype(api.f))dlsym(h, n)
            NBK_SYM(getUniqueId, "ncclGetUniqueId");
            NBK_SYM(commInitRank, "ncclCommInitRank");
            NBK_SYM(commDestroy, "ncclCommDestroy");
            NBK_SYM(groupStart, "ncclGroupStart");
            NBK_SYM(groupEnd, "ncclGroupEnd");
            NBK_SYM(send, "ncclSend");
            NBK_SYM(recv, "ncclRecv");
            NBK_SYM(allGather, "ncclAllGather");
            NBK_SYM(errorString, "ncclGetErrorString");
#undef NBK_SYM
            const bool ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.groupStart &&
                            api.groupEnd && api.send && api.recv && api.allGather && api.errorString;
            state = ok ? 1 : -1;
            if (!ok) err = "libnccl.so.2 lacks a required symbol";
        }
    }
    if (state < 0) { why = err; return nullptr; }
    return &api;
}

// ------------------------------------------------------------ teams
// The contexts whose work one call enqueues: {self} for a 1-rank or an NCCL
// rank context, or all P contexts of an in-process virtual-slab group (every
// slab on this device; faces and partials are shared by pointer aliasing and
// the phases of all slabs are enqueued in order on the first member's stream).
struct Team {
    std::vector<nbk_ctx*> m;
    bool multi = false;   // nranks > 1: face exchange + rank-ordered reductions
    cudaStream_t s = nullptr;
};

static Team team_self(nbk_ctx* c)
{
    Team t;
    t.m.push_back(c);
    t.multi = c->nranks > 1;
    t.s = c->stream;
    return t;
}

template <typename T>
static T* fld(nbk_ctx* c, int which, bool fp32)
{
    // which: 0 x, 1 r, 2 p, 3 w, 4 dinv
    void* v64[5] = {c->x64, c->r64, c->p64, c->w64, c->dinv64};
    void* v32[5] = {c->x32, c->r32, c->p32, c->w32, c->dinv32};
    return (T*)(fp32 ? v32[which] : v64[which]);
}

// Exchange the packed face layers with the neighbour ranks (NCCL mode).  In a
// virtual group the receive buffers alias the neighbours' send buffers.
template <typename T>
static cudaError_t xchg_faces(const Team& t, cudaStream_t s, std::string& err)
{
    for (nbk_ctx* c : t.m) {
        if (!c->comm) continue;
        std::string why;
        const NcclApi* A = nccl_api(why);
        if (!A) { err = why; return cudaErrorUnknown; }
        ncclComm_t comm = (ncclComm_t)c->comm;
        const ncclDataType_t ty = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
        const size_t cnt = (size_t)c->nlayer;
        ncclResult_t r = A->groupStart();
        if (c->has_lo && r == ncclSuccess) r = A->send(c->send_lo, cnt, ty, c->rank - 1, comm, s);
        if (c->has_lo && r == ncclSuccess) r = A->recv(c->recv_lo, cnt, ty, c->rank - 1, comm, s);
        if (c->has_hi && r == ncclSuccess) r = A->send(c->send_hi, cnt, ty, c->rank + 1, comm, s);
        if (c->has_hi && r == ncclSuccess) r = A->recv(c->recv_hi, cnt, ty, c->rank + 1, comm, s);
        ncclResult_t r2 = A->groupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess) {
            err = std::string("NCCL face exchange: ") + A->errorString(r != ncclSuccess ? r : r2);
            return cudaErrorUnknown;
        }
    }
    return cudaSuccess;
}

// All-gather of the per-rank dd partials, in place (slot = gather + rank).
static cudaError_t xchg_gather(const Team& t, cudaStream_t s, std::string& err)
{
    for (nbk_ctx* c : t.m) {
        if (!c->comm) continue;
        std::string why;
        const NcclApi* A = nccl_api(why);
        if (!A) { err = why; return cudaErrorUnknown; }
        ncclResult_t r = A->allGather(c->gather + 2 * c->rank, c->gather, 4, ncclFloat64,
                                      (ncclComm_t)c->comm, s);
        if (r != ncclSuccess) {
            err = std::string("NCCL allgather: ") + A->errorString(r);
            return cudaErrorUnknown;
        }
    }
    return cudaSuccess;
}

// ------------------------------------------------------------ helpers
template <typename T>
static AxArgs<T> ax_args(nbk_ctx* c, const T* D, const T* G)
{
    AxArgs<T> a{};
    a.D = D;
    a.G = G;
    a.mesh = c->view;
    a.st = c->st;
    a.parts = c->parts;
    return a;
}

template <typename T>
static int ax_blocks_n(int64_t E, int N)
{
#define EPBN(n) (int)((E + ax_epb<T>(n) - 1) / ax_epb<T>(n))
    NBK_SWITCH_N(N, EPBN)
#undef EPBN
}

template <typename T>
static DssumArgs<T> dssum_args(nbk_ctx* c, T* w)
{
    DssumArgs<T> d{};
    d.w = w;
    d.g2 = c->g2; d.g4 = c->g4; d.g8 = c->g8;
    d.toff = c->toff; d.ntiles = (int)c->ntiles;
    d.st = c->st; d.trace = c->trace; d.mesh = c->view; d.mask = 0; d.fin = 1;
    return d;
}

template <typename T>
static FaceArgs<T> face_args(nbk_ctx* c, T* w)
{
    FaceArgs<T> f{};
    f.w = w;
    f.send_lo = (T*)c->send_lo; f.send_hi = (T*)c->send_hi;
    f.recv_lo = (const T*)c->recv_lo; f.recv_hi = (const T*)c->recv_hi;
    f.has_lo = c->has_lo; f.has_hi = c->has_hi;
    f.parts = c->parts; f.st = c->st; f.slot = c->gather + 2 * c->rank; f.mesh = c->view;
    return f;
}

// vector kernels: two banks of NBK_VEC_GRID_MAX partials (rtr, rtz) at the end
static dd* vec_parts(nbk_ctx* c) { return c->parts + c->nparts - 2 * NBK_VEC_GRID_MAX; }

// dssum (+ mask) of w over a team.  fused: shared-node pap terms, alpha.
// One rank: K_B (its last block forms alpha).  Several: K_B (publish only) and
// the face pack, exchange, face merge (reduces this rank's pap), all-gather,
// k_fin (rank-ordered combination, alpha).
template <typename T, bool FUSED, bool VP = false>
static cudaError_t dssum_team(const Team& t, const std::vector<T*>& w, const std::vector<const T*>& p,
                              int mask, bool pdl, std::string& err, int rev = 0, int single = 0,
                              int vp_t = 0)
{
    cudaError_t e;
    const cudaStream_t s = t.s;
    for (size_t q = 0; q < t.m.size(); ++q) {
        nbk_ctx* c = t.m[q];
        DssumArgs<T> d = dssum_args<T>(c, w[q]);
        d.mask = mask;
        d.rev = rev;
        d.single = single;
        d.vp_t = vp_t;
        if (FUSED) {
            d.p = p[q];
            d.parts = c->parts;
            d.nA = ax_blocks_n<T>(c->E, c->N);
            d.fin = t.multi ? 0 : 1;
        }
        if ((e = launch_dssum<T, FUSED, VP>(d, s, pdl && !t.multi)) != cudaSuccess) return e;
        if (t.multi) {
            FaceArgs<T> f = face_args<T>(c, w[q]);
            k_face_pack<T><<<vec_grid(2 * c->nlayer), 256, 0, s>>>(f);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
    }
    if (!t.multi) return cudaSuccess;
    if ((e = xchg_faces<T>(t, s, err)) != cudaSuccess) return e;
    for (size_t q = 0; q < t.m.size(); ++q) {
        nbk_ctx* c = t.m[q];
        FaceArgs<T> f = face_args<T>(c, w[q]);
        f.mask = mask;
        f.single = single;
        if (FUSED) {
            f.p = p[q];
            f.nprev = ax_blocks_n<T>(c->E, c->N) + dssum_grid_t<T, FUSED, VP>((int)c->ntiles);
        }
        const int64_t nodes = (int64_t)(c->has_lo + c->has_hi) * c->nplane;
        k_face_merge<T, FUSED><<<vec_grid(nodes), 256, 0, s>>>(f);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (FUSED) {
        if ((e = xchg_gather(t, s, err)) != cudaSuccess) return e;
        for (nbk_ctx* c : t.m) {
            k_fin<0><<<1, 32, 0, s>>>(c->gather, c->nranks, c->st, c->hist, c->trace, single, vp_t);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

// Vector kernel (K_C and the other modes) over a team: one rank finalises in
// its last block; several publish per-rank partials, all-gather, k_fin.
template <typename T, int MODE, bool VP = false>
static cudaError_t vec_team(const Team& t, const std::vector<VecArgs<T>>& args, bool pdl,
                            std::string& err)
{
    cudaError_t e;
    for (size_t q = 0; q < t.m.size(); ++q) {
        VecArgs<T> a = args[q];
        a.slot = t.multi ? t.m[q]->gather + 2 * t.m[q]->rank : nullptr;
        if ((e = launch_vec<T, MODE, VP>(a, t.s, pdl && !t.multi)) != cudaSuccess) return e;
    }
    if (!t.multi) return cudaSuccess;
    if ((e = xchg_gather(t, t.s, err)) != cudaSuccess) return e;
    for (size_t q = 0; q < t.m.size(); ++q) {
        nbk_ctx* c = t.m[q];
        k_fin<1 + MODE><<<1, 32, 0, t.s>>>(c->gather, c->nranks, c->st, c->hist, c->trace,
                                          args[q].single, args[q].vp_t);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <typename T>
static VecArgs<T> vec_args(nbk_ctx* c)
{
    VecArgs<T> v{};
    v.n = c->n; v.parts = vec_parts(c); v.st = c->st; v.hist = c->hist; v.trace = c->trace;
    v.mesh = c->view;
    return v;
}

// ax (+ dssum + mask) of per-member fields over a team (standalone / final check).
template <typename T>
static cudaError_t ax_team(const Team& t, const std::vector<const T*>& u, const std::vector<T*>& w,
                           int flags, bool fp32, std::string& err)
{
    cudaError_t e;
    for (size_t q = 0; q < t.m.size(); ++q) {
        nbk_ctx* c = t.m[q];
        AxArgs<T> a = fp32 ? ax_args<T>(c, (const T*)c->D32, (const T*)c->G32)
                           : ax_args<T>(c, (const T*)c->D64, (const T*)c->G64);
        a.u = u[q]; a.w = w[q]; a.mask = (flags & NBK_AX_MASK) ? 1 : 0;
        if ((e = launch_ax<T, 0>(a, t.s)) != cudaSuccess) return e;
    }
    if (flags & NBK_AX_DSSUM) return dssum_team<T, false>(t, w, {}, 0, false, err);
    return cudaSuccess;
}

// Enqueue one CG solve (T1 loop, fixed niter) for the team; used under capture.
template <typename T, bool VP = false>
static cudaError_t enqueue_solve(const Team& t, int niter, nbk_graph* g, bool fp32, bool profiling,
                                 std::string& err, int single = 0)
{
    const cudaStream_t s = t.s;
    const size_t P = t.m.size();
    cudaError_t e;
    int64_t launches = 0;
    std::vector<T*> x(P), r(P), p(P), w(P);
    std::vector<const T*> pc(P);
    for (size_t q = 0; q < P; ++q) {
        x[q] = fld<T>(t.m[q], 0, fp32); r[q] = fld<T>(t.m[q], 1, fp32);
        p[q] = fld<T>(t.m[q], 2, fp32); w[q] = fld<T>(t.m[q], 3, fp32);
        pc[q] = p[q];
    }
    const int64_t per_fin = t.multi ? 1 : 0;  // k_fin launches per reduction and member
    const int64_t nface = t.multi ? 2 : 0;    // pack + merge per dssum and member

    // Jacobi PCG (NEXT-1): z = r * dinv formed in K_A and K_C, rtz reduced beside rtr
    const bool jac = !VP && t.m[0]->precond == NBK_PRECOND_JACOBI;
    const int vp_t = VP ? t.m[0]->vp_t : 0;  // VPREC emulation (NEXT-4)
    std::vector<VecArgs<T>> vi(P), vr(P);
    for (size_t q = 0; q < P; ++q) {
        vi[q] = vec_args<T>(t.m[q]);
        vi[q].r = r[q]; vi[q].x = x[q]; vi[q].p = p[q]; vi[q].f = t.m[q]->f64;
        vi[q].dinv = fld<T>(t.m[q], 4, fp32);
        vi[q].single = single;
        vi[q].vp_t = vp_t;
        vr[q] = vi[q];
        vr[q].w = w[q];
    }
    e = jac ? vec_team<T, VEC_INIT_J>(t, vi, false, err) : vec_team<T, VEC_INIT, VP>(t, vi, false, err);
    if (e != cudaSuccess) return e;
    launches += (int64_t)P * (1 + per_fin);

    // sweep directions alternate kernel by kernel: K_A f, K_B b, K_C f, K_A b, ...
    int rev = 0;
    for (int k = 1; k <= niter; ++k) {
        const bool prof = g && profiling && P == 1;
        if (prof) cudaEventRecordWithFlags(g->prof_events[4 * (k - 1)], s, cudaEventRecordExternal);
        const bool pdl = !prof;  // events between kernels break PDL edges
        for (size_t q = 0; q < P; ++q) {
            nbk_ctx* c = t.m[q];
            AxArgs<T> aa = fp32 ? ax_args<T>(c, (const T*)c->D32, (const T*)c->G32)
                                : ax_args<T>(c, (const T*)c->D64, (const T*)c->G64);
            aa.u = nullptr; aa.w = w[q]; aa.p = p[q]; aa.r = r[q]; aa.x = x[q]; aa.mask = 1;
            aa.rev = rev;
            aa.dinv = fld<T>(c, 4, fp32);
            aa.single = single;
            aa.vp_t = vp_t;
            e = jac ? launch_ax<T, 2>(aa, s, false, pdl) : launch_ax<T, 1, VP>(aa, s, false, pdl);
            if (e != cudaSuccess) return e;
        }
        if (prof) cudaEventRecordWithFlags(g->prof_events[4 * (k - 1) + 1], s, cudaEventRecordExternal);
        if ((e = dssum_team<T, true, VP>(t, w, pc, 0, pdl, err, !rev, single, vp_t)) != cudaSuccess)
            return e;
        if (prof) cudaEventRecordWithFlags(g->prof_events[4 * (k - 1) + 2], s, cudaEventRecordExternal);
        for (size_t q = 0; q < P; ++q) vr[q].rev = rev;
        e = jac ? vec_team<T, VEC_RUPD_J>(t, vr, pdl, err) : vec_team<T, VEC_RUPD, VP>(t, vr, pdl, err);
        if (e != cudaSuccess) return e;
        if (prof) cudaEventRecordWithFlags(g->prof_events[4 * (k - 1) + 3], s, cudaEventRecordExternal);
        rev = !rev;
        launches += (int64_t)P * (3 + nface + 2 * per_fin);
    }
    for (size_t q = 0; q < P; ++q) {
        nbk_ctx* c = t.m[q];
        k_tail_x<T, VP><<<vec_grid(c->n), 256, 0, s>>>(x[q], p[q], c->st, c->n, vp_t);
        ++launches;
        // final FP64 residual check (C12): x64 = (double)x ; r_true = f - A x64
        if (fp32) {
            k_upcast<<<vec_grid(c->n), 256, 0, s>>>(c->x64, (const float*)x[q], c->n);
            ++launches;
        }
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    std::vector<const double*> x64(P);
    std::vector<double*> w64(P);
    std::vector<VecArgs<double>> vt(P);
    for (size_t q = 0; q < P; ++q) {
        nbk_ctx* c = t.m[q];
        x64[q] = c->x64; w64[q] = c->w64;
        vt[q] = vec_args<double>(c);
        vt[q].r = c->r64; vt[q].w = c->w64; vt[q].f = c->f64;
    }
    if ((e = ax_team<double>(t, x64, w64, NBK_AX_DSSUM | NBK_AX_MASK, false, err)) != cudaSuccess) return e;
    if ((e = vec_team<double, VEC_TRUE>(t, vt, false, err)) != cudaSuccess) return e;
    launches += (int64_t)P * (3 + nface + per_fin);
    if (g) g->launches = launches;
    return cudaSuccess;
}

static nbk_status get_graph(const Team& t, int niter, nbk_precision prec, nbk_graph** out)
{
    nbk_ctx* c = t.m[0];
    auto key = std::make_tuple((int)prec + 4 * (prec == NBK_VPREC ? c->vp_t : 0), niter,
                               c->profiling * 2 + c->precond);
    auto it = c->graphs.find(key);
    if (it != c->graphs.end()) { *out = &it->second; return NBK_OK; }
    nbk_graph g;
    if (c->profiling && t.m.size() == 1) {
        g.prof_events.resize(4 * niter);
        for (auto& ev : g.prof_events) NBK_CUDA(c, cudaEventCreate(&ev));
    }
    NBK_CUDA(c, cudaStreamBeginCapture(t.s, cudaStreamCaptureModeThreadLocal));
    std::string err;
    cudaError_t e = prec == NBK_FP64    ? enqueue_solve<double>(t, niter, &g, false, c->profiling, err)
                    : prec == NBK_VPREC ? enqueue_solve<double, true>(t, niter, &g, false, c->profiling, err)
                                        : enqueue_solve<float>(t, niter, &g, true, c->profiling, err,
                                                               prec == NBK_FP32S ? 1 : 0);
    cudaGraph_t graph = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(t.s, &graph);
    if (e != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        return fail(c, err.empty() ? NBK_ECUDA : NBK_ENCCL,
                    std::string("capture: ") + (err.empty() ? cudaGetErrorString(e) : err));
    }
    if (e2 != cudaSuccess) return fail(c, NBK_ECUDA, std::string("end capture: ") + cudaGetErrorString(e2));
    g.graph = graph;
    NBK_CUDA(c, cudaGraphInstantiate(&g.exec, graph, 0));
    auto res = c->graphs.emplace(key, std::move(g));
    *out = &res.first->second;
    return NBK_OK;
}

static void destroy_graphs(nbk_ctx* c)
{
    for (auto& kv : c->graphs) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
        for (auto ev : kv.second.prof_events) cudaEventDestroy(ev);
    }
    c->graphs.clear();
}

static cudaError_t set_ax_attrs(nbk_ctx* c)
{
    AxArgs<double> a64{};
    a64.mesh = c->view;
    AxArgs<float> a32{};
    a32.mesh = c->view;
    cudaError_t e;

    if ((e = launch_ax<double, 0>(a64, c->stream, true)) != cudaSuccess) return e;
    if (c->N <= NBK_VPREC_MAXN && (e = launch_ax<double, 1, true>(a64, c->stream, true)) != cudaSuccess)
        return e;
    if ((e = launch_ax<double, 1>(a64, c->stream, true)) != cudaSuccess) return e;
    if ((e = launch_ax<double, 2>(a64, c->stream, true)) != cudaSuccess) return e;
    if ((e = launch_ax<float, 0>(a32, c->stream, true)) != cudaSuccess) return e;
    if ((e = launch_ax<float, 1>(a32, c->stream, true)) != cudaSuccess) return e;
    return launch_ax<float, 2>(a32, c->stream, true);
}

// glsc3 over a team (synchronous); result identical on every member.
template <typename T>
static nbk_status glsc3_team(const Team& t, const std::vector<const T*>& a, const std::vector<const T*>& b,
                             double* out, int single = 0)
{
    nbk_ctx* c0 = t.m[0];
    std::vector<VecArgs<T>> v(t.m.size());
    for (size_t q = 0; q < t.m.size(); ++q) {
        v[q] = vec_args<T>(t.m[q]);
        v[q].a = a[q]; v[q].b = b[q];
        v[q].single = single;
    }
    std::string err;
    cudaError_t e = vec_team<T, VEC_DOT>(t, v, false, err);
    if (e != cudaSuccess) return fail(c0, err.empty() ? NBK_ECUDA : NBK_ENCCL, err.empty() ? cudaGetErrorString(e) : err);
    NBK_CUDA(c0, cudaMemcpyAsync(out, &c0->st->dot, 8, cudaMemcpyDeviceToHost, t.s));
    NBK_CUDA(c0, cudaStreamSynchronize(t.s));
    return NBK_OK;
}

static nbk_status refresh_fp32(nbk_ctx* c)
{
    cudaStream_t s = c->stream;
    c->dinv_dirty = 1;  // the operator may have changed: own diagonal re-assembled on demand
    if (c->G32) {
        k_downcast<<<vec_grid(6 * c->n), 256, 0, s>>>(c->G32, c->G64, 6 * c->n);
        k_downcast<<<1, 256, 0, s>>>(c->D32, c->D64, (int64_t)c->N * c->N);
        NBK_CUDA(c, cudaGetLastError());
    }
    c->h0_dirty = 1;
    return NBK_OK;
}

// h0 (FP64) = sqrt(glsc3(f, c, f)) for the relative true residual (C12).
static nbk_status refresh_h0(const Team& t)
{
    bool dirty = false;
    for (nbk_ctx* c : t.m) dirty = dirty || c->h0_dirty;
    if (!dirty) return NBK_OK;
    std::vector<const double*> f(t.m.size());
    for (size_t q = 0; q < t.m.size(); ++q) f[q] = t.m[q]->f64;
    double dot = 0.0;
    nbk_status st = glsc3_team<double>(t, f, f, &dot);
    if (st != NBK_OK) return st;
    for (nbk_ctx* c : t.m) {
        c->h0_64 = std::sqrt(dot);
        c->h0_dirty = 0;
    }
    return NBK_OK;
}

// Jacobi data (NEXT-1): the library's own assembled diagonal -- per-element
// diag(A_e) (FP64), the team's dssum (slab faces exchanged like any dssum),
// masked entries 1, inverse, RN32 copy -- unless loaded (nbk_load_precond).
static nbk_status refresh_dinv(const Team& t)
{
    bool dirty = false;
    for (nbk_ctx* c : t.m) dirty = dirty || c->dinv_dirty;
    if (!dirty) return NBK_OK;
    nbk_ctx* c0 = t.m[0];
    std::vector<double*> d(t.m.size());
    for (size_t q = 0; q < t.m.size(); ++q) {
        d[q] = t.m[q]->dinv64;
        NBK_CUDA(c0, local_diag(t.m[q], d[q]));
    }
    std::string err;
    cudaError_t e = dssum_team<double, false>(t, d, {}, 0, false, err);
    if (e != cudaSuccess)
        return fail(c0, err.empty() ? NBK_ECUDA : NBK_ENCCL, err.empty() ? cudaGetErrorString(e) : err);
    for (size_t q = 0; q < t.m.size(); ++q) NBK_CUDA(c0, finish_dinv(t.m[q], d[q]));
    NBK_CUDA(c0, cudaStreamSynchronize(t.s));
    for (nbk_ctx* c : t.m) c->dinv_dirty = 0;
    return NBK_OK;
}

// Team of a call made on one context: errors for virtual-group members.
static nbk_status self_team(nbk_ctx* c, Team& t)
{
    if (c->nranks > 1 && !c->comm)
        return fail(c, NBK_ESTATE, "virtual-slab context: use the nbk_group_* calls");
    t = team_self(c);
    return NBK_OK;
}

static nbk_status solve_team(const Team& t, int32_t niter, nbk_precision prec, double* hist_host,
                             double* trace_host, nbk_result* result)
{
    nbk_ctx* c = t.m[0];
    if (niter < 1 || niter > NBK_MAX_NITER) return fail(c, NBK_EINVAL, "niter out of range");
    if (prec != NBK_FP64 && prec != NBK_FP32 && prec != NBK_FP32S && prec != NBK_VPREC)
        return fail(c, NBK_EINVAL, "bad precision");
    for (nbk_ctx* m : t.m) {
        if ((prec == NBK_FP32 || prec == NBK_FP32S) && !m->G32)
            return fail(c, NBK_ESTATE, "context was set up without FP32 arrays");
        if (prec == NBK_VPREC && m->vp_t != c->vp_t) return fail(c, NBK_EINVAL, "members differ in VPREC t");
        if (prec == NBK_VPREC && m->N > NBK_VPREC_MAXN) return fail(c, NBK_EINVAL, "VPREC emulation supports N <= 12");
    }
    nbk_status st = refresh_h0(t);
    if (st != NBK_OK) return st;
    if (c->precond == NBK_PRECOND_JACOBI) {
        for (nbk_ctx* m : t.m)
            if (m->precond != c->precond) return fail(c, NBK_EINVAL, "members differ in preconditioner");
        st = refresh_dinv(t);
        if (st != NBK_OK) return st;
    }
    nbk_graph* g = nullptr;
    st = get_graph(t, niter, prec, &g);
    if (st != NBK_OK) return st;
    cudaStream_t s = t.s;
    NBK_CUDA(c, cudaEventRecord(c->ev0, s));
    NBK_CUDA(c, cudaGraphLaunch(g->exec, s));
    NBK_CUDA(c, cudaEventRecord(c->ev1, s));
    CgState hs;
    NBK_CUDA(c, cudaMemcpyAsync(&hs, c->st, sizeof(CgState), cudaMemcpyDeviceToHost, s));
    if (hist_host) NBK_CUDA(c, cudaMemcpyAsync(hist_host, c->hist, 8 * (size_t)(niter + 1), cudaMemcpyDeviceToHost, s));
    if (trace_host) NBK_CUDA(c, cudaMemcpyAsync(trace_host, c->trace, 8 * 5 * (size_t)niter, cudaMemcpyDeviceToHost, s));
    NBK_CUDA(c, cudaStreamSynchronize(s));
    for (nbk_ctx* m : t.m) m->last_solved_precision = (int)prec;
    if (result) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->ev0, c->ev1);
        result->solve_ms = ms;
        result->true_res = std::sqrt(hs.true_rtr);
        result->true_res_rel = c->h0_64 > 0 ? result->true_res / c->h0_64 : 0.0;
        result->defect_iter = hs.defect;
        result->niter = niter;
        float ka = 0.f;
        float kb = 0.f, kc = 0.f;
        if (c->profiling && !g->prof_events.empty()) {
            for (int k = 0; k < niter; ++k) {
                float t0 = 0.f, t1 = 0.f, t2 = 0.f;
                cudaEventElapsedTime(&t0, g->prof_events[4 * k], g->prof_events[4 * k + 1]);
                cudaEventElapsedTime(&t1, g->prof_events[4 * k + 1], g->prof_events[4 * k + 2]);
                cudaEventElapsedTime(&t2, g->prof_events[4 * k + 2], g->prof_events[4 * k + 3]);
                ka += t0;
                kb += t1;
                kc += t2;
            }
        }
        result->kA_ms = ka;
        result->kB_ms = kb;
        result->kC_ms = kc;
    }
    return hs.defect ? fail(c, NBK_EDEFECT, "CG defect: pap <= 0 or non-finite scalar") : NBK_OK;
}

// ================================================================== ABI
extern "C" {

const char* nbk_version(void) { return "nbk 0.2 (sm_100a; z-slab multi-rank)"; }

const char* nbk_last_error(const nbk_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

nbk_status nbk_workspace_bytes(const nbk_mesh* mesh, nbk_precision precision, const nbk_dist* dist,
                               size_t* bytes_out)
{
    std::string why;
    if (!bytes_out) return fail(nullptr, NBK_EINVAL, "bytes_out is NULL");
    if (!validate_mesh(mesh, dist, why)) return fail(nullptr, NBK_EINVAL, why);
    if (precision != NBK_FP64 && precision != NBK_FP32) return fail(nullptr, NBK_EINVAL, "bad precision");
    Layout L = compute_layout(mesh, precision, dist);
    *bytes_out = L.total;
    return NBK_OK;
}

nbk_status nbk_partition(const nbk_mesh* mesh, const nbk_dist* dist, nbk_info* info)
{
    std::string why;
    if (!info) return fail(nullptr, NBK_EINVAL, "info is NULL");
    if (!validate_mesh(mesh, dist, why)) return fail(nullptr, NBK_EINVAL, why);
    Layout L = compute_layout(mesh, NBK_FP64, dist);
    info->n_local = L.n;
    info->n_global = L.n_global;
    info->e_local = L.E;
    info->e_offset = L.e_offset;
    info->n_shared = L.nseg;
    info->n_copies = L.ncopies;
    info->N = mesh->N;
    info->has_fp32 = 0;
    info->face_layer = (L.has_lo + L.has_hi) ? L.nlayer : 0;
    info->face_nodes = (L.has_lo + L.has_hi) * L.nplane;
    return NBK_OK;
}

nbk_status nbk_nccl_unique_id(void* out128)
{
    if (!out128) return fail(nullptr, NBK_EINVAL, "out is NULL");
    std::string why;
    const NcclApi* A = nccl_api(why);
    if (!A) return fail(nullptr, NBK_ENCCL, why);
    ncclUniqueId id;
    ncclResult_t r = A->getUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, NBK_ENCCL, A->errorString(r));
    std::memcpy(out128, &id, sizeof(id));
    return NBK_OK;
}

nbk_status nbk_cg_setup(const nbk_mesh* mesh, nbk_precision precision, const nbk_dist* dist,
                        void* dev_workspace, size_t ws_bytes, nbk_ctx** out)
{
    std::string why;
    if (!out) return fail(nullptr, NBK_EINVAL, "out is NULL");
    *out = nullptr;
    if (!validate_mesh(mesh, dist, why)) return fail(nullptr, NBK_EINVAL, why);
    if (precision != NBK_FP64 && precision != NBK_FP32) return fail(nullptr, NBK_EINVAL, "bad precision");
    if (!dev_workspace) return fail(nullptr, NBK_EINVAL, "workspace is NULL");
    if (((uintptr_t)dev_workspace & 255) != 0) return fail(nullptr, NBK_EINVAL, "workspace not 256-byte aligned");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(nullptr, NBK_ECUDA, "no CUDA device (libnbk has no CPU fallback)");
    nbk_dist d1{0, 1, 0, nullptr, nullptr};
    const nbk_dist* d = dist ? dist : &d1;
    if (cudaSetDevice(d->device) != cudaSuccess) return fail(nullptr, NBK_ECUDA, "cudaSetDevice failed");
    Layout L = compute_layout(mesh, precision, d);
    if (ws_bytes < L.total) return fail(nullptr, NBK_ENOMEM, "workspace too small");

    nbk_ctx* c = new (std::nothrow) nbk_ctx();
    if (!c) return fail(nullptr, NBK_ENOMEM, "host allocation failed");
    c->mesh = *mesh;
    c->dist = *d;
    c->setup_precision = precision;
    c->stream = (cudaStream_t)d->stream;
    c->N = mesh->N;
    c->E = L.E;
    c->n = L.n;
    c->n_global = L.n_global;
    c->e_offset = L.e_offset;
    c->nseg = L.nseg;
    c->ncopies = L.ncopies;
    c->nparts = L.nparts;
    c->view = make_view(mesh, d);
    c->rank = d->rank;
    c->nranks = d->nranks;
    c->has_lo = L.has_lo;
    c->has_hi = L.has_hi;
    c->nlayer = L.nlayer;
    c->nplane = L.nplane;
    unsigned char* b = (unsigned char*)dev_workspace;
    c->st = (CgState*)(b + L.off_state);
    c->D64 = (double*)(b + L.off_D64);
    c->D32 = (float*)(b + L.off_D32);
    c->hist = (double*)(b + L.off_hist);
    c->trace = (double*)(b + L.off_trace);
    c->parts = (dd*)(b + L.off_parts);
    c->seg_off = (int32_t*)(b + L.off_segoff);
    c->seg_idx = (int32_t*)(b + L.off_segidx);
    c->grp = (int32_t*)(b + L.off_grp);
    c->toff = (int32_t*)(b + L.off_toff);
    if (c->has_lo || c->has_hi) {
        const size_t fb = 8 * (size_t)L.nlayer;
        c->send_lo = b + L.off_face;
        c->send_hi = b + L.off_face + fb;
        c->recv_lo = b + L.off_face + 2 * fb;
        c->recv_hi = b + L.off_face + 3 * fb;
    }
    c->gather_own = (dd*)(b + L.off_gather);
    c->gather = c->gather_own;
    c->G64 = (double*)(b + L.off_G64);
    c->f64 = (double*)(b + L.off_f64);
    c->dinv64 = (double*)(b + L.off_dinv64);
    const size_t v64 = ((size_t)8 * c->n + 255) & ~(size_t)255;
    c->x64 = (double*)(b + L.off_vec64);
    c->r64 = (double*)(b + L.off_vec64 + v64);
    c->p64 = (double*)(b + L.off_vec64 + 2 * v64);
    c->w64 = (double*)(b + L.off_vec64 + 3 * v64);
    c->scratch = b + L.off_vec64;
    c->scratch_bytes = (precision == NBK_FP32 ? L.off_G32 : L.total) - L.off_vec64;
    if (precision == NBK_FP32) {
        const size_t v32 = ((size_t)4 * c->n + 255) & ~(size_t)255;
        c->G32 = (float*)(b + L.off_G32);
        c->x32 = (float*)(b + L.off_vec32);
        c->r32 = (float*)(b + L.off_vec32 + v32);
        c->p32 = (float*)(b + L.off_vec32 + 2 * v32);
        c->w32 = (float*)(b + L.off_vec32 + 3 * v32);
        c->dinv32 = (float*)(b + L.off_dinv32);
    }
    // NCCL communicator (collective over the ranks) when an id is given
    if (c->nranks > 1 && d->nccl_id) {
        const NcclApi* A = nccl_api(why);
        if (!A) { delete c; return fail(nullptr, NBK_ENCCL, why); }
        ncclUniqueId id;
        std::memcpy(&id, d->nccl_id, sizeof(id));
        ncclComm_t comm = nullptr;
        ncclResult_t r = A->commInitRank(&comm, c->nranks, id, c->rank);
        if (r != ncclSuccess) { delete c; return fail(nullptr, NBK_ENCCL, std::string("ncclCommInitRank: ") + A->errorString(r)); }
        c->comm = comm;
    }
    nbk_status st = NBK_OK;
    cudaError_t e = set_ax_attrs(c);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->st, 0, sizeof(CgState), c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->gather_own, 0, 2 * sizeof(dd) * NBK_MAX_RANKS, c->stream);
    if (e == cudaSuccess) e = setup_device(c, L);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        std::string m = std::string("set-up: ") + cudaGetErrorString(e);
        nbk_destroy(c);
        return fail(nullptr, NBK_ECUDA, m);
    }
    // vectors start at zero (the plan used their space as scratch)
    e = cudaMemsetAsync(c->x64, 0, 4 * v64, c->stream);
    if (e != cudaSuccess) { nbk_destroy(c); return fail(nullptr, NBK_ECUDA, cudaGetErrorString(e)); }
    st = refresh_fp32(c);
    if (st == NBK_OK && !(c->nranks > 1 && !c->comm)) st = refresh_h0(team_self(c));
    if (st != NBK_OK) { std::string m = c->err; nbk_destroy(c); return fail(nullptr, st, m); }
    cudaEventCreate(&c->ev0);
    cudaEventCreate(&c->ev1);
    *out = c;
    return NBK_OK;
}

nbk_status nbk_load_arrays(nbk_ctx* c, const double* D_host, const double* G_host, const double* f_host)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    cudaStream_t s = c->stream;
    if (D_host) NBK_CUDA(c, cudaMemcpyAsync(c->D64, D_host, 8 * c->N * c->N, cudaMemcpyHostToDevice, s));
    if (G_host) NBK_CUDA(c, cudaMemcpyAsync(c->G64, G_host, 8 * 6 * c->n, cudaMemcpyHostToDevice, s));
    if (f_host) NBK_CUDA(c, cudaMemcpyAsync(c->f64, f_host, 8 * c->n, cudaMemcpyHostToDevice, s));
    nbk_status st = refresh_fp32(c);
    if (st != NBK_OK) return st;
    NBK_CUDA(c, cudaStreamSynchronize(s));
    return NBK_OK;
}

nbk_status nbk_get_arrays(nbk_ctx* c, double* D_host, double* G_host, double* f_host)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    cudaStream_t s = c->stream;
    if (D_host) NBK_CUDA(c, cudaMemcpyAsync(D_host, c->D64, 8 * c->N * c->N, cudaMemcpyDeviceToHost, s));
    if (G_host) NBK_CUDA(c, cudaMemcpyAsync(G_host, c->G64, 8 * 6 * c->n, cudaMemcpyDeviceToHost, s));
    if (f_host) NBK_CUDA(c, cudaMemcpyAsync(f_host, c->f64, 8 * c->n, cudaMemcpyDeviceToHost, s));
    NBK_CUDA(c, cudaStreamSynchronize(s));
    return NBK_OK;
}

static nbk_status ax_apply_team(const Team& t, const void* const* u_dev, void* const* w_dev, int32_t flags,
                                nbk_precision prec)
{
    nbk_ctx* c = t.m[0];
    if (flags & ~(NBK_AX_DSSUM | NBK_AX_MASK)) return fail(c, NBK_EINVAL, "bad flags");
    if (prec != NBK_FP64 && prec != NBK_FP32) return fail(c, NBK_EINVAL, "bad precision");
    const size_t P = t.m.size();
    for (size_t q = 0; q < P; ++q) {
        if (!u_dev[q] || !w_dev[q] || u_dev[q] == w_dev[q]) return fail(c, NBK_EINVAL, "u/w must be distinct non-NULL");
        if (prec == NBK_FP32 && !t.m[q]->G32) return fail(c, NBK_ESTATE, "context has no FP32 arrays");
    }
    std::string err;
    cudaError_t e;
    if (prec == NBK_FP64) {
        std::vector<const double*> u(P);
        std::vector<double*> w(P);
        for (size_t q = 0; q < P; ++q) { u[q] = (const double*)u_dev[q]; w[q] = (double*)w_dev[q]; }
        e = ax_team<double>(t, u, w, flags, false, err);
    } else {
        std::vector<const float*> u(P);
        std::vector<float*> w(P);
        for (size_t q = 0; q < P; ++q) { u[q] = (const float*)u_dev[q]; w[q] = (float*)w_dev[q]; }
        e = ax_team<float>(t, u, w, flags, true, err);
    }
    if (e != cudaSuccess)
        return fail(c, err.empty() ? NBK_ECUDA : NBK_ENCCL, err.empty() ? cudaGetErrorString(e) : err);
    return NBK_OK;
}

nbk_status nbk_ax_apply(nbk_ctx* c, const void* u_dev, void* w_dev, int32_t flags, nbk_precision prec)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    Team t;
    nbk_status st = self_team(c, t);
    if (st != NBK_OK) return st;
    return ax_apply_team(t, &u_dev, &w_dev, flags, prec);
}

static nbk_status dssum_team_abi(const Team& t, void* const* f_dev, int32_t apply_mask, nbk_precision prec)
{
    nbk_ctx* c = t.m[0];
    const size_t P = t.m.size();
    for (size_t q = 0; q < P; ++q)
        if (!f_dev[q]) return fail(c, NBK_EINVAL, "f is NULL");
    std::string err;
    cudaError_t e;
    if (prec == NBK_FP64) {
        std::vector<double*> w(P);
        for (size_t q = 0; q < P; ++q) w[q] = (double*)f_dev[q];
        e = dssum_team<double, false>(t, w, {}, apply_mask ? 1 : 0, false, err);
        for (size_t q = 0; e == cudaSuccess && apply_mask && q < P; ++q) {
            k_mask<double><<<vec_grid(t.m[q]->n), 256, 0, t.s>>>(w[q], t.m[q]->view);
            e = cudaGetLastError();
        }
    } else if (prec == NBK_FP32) {
        std::vector<float*> w(P);
        for (size_t q = 0; q < P; ++q) w[q] = (float*)f_dev[q];
        e = dssum_team<float, false>(t, w, {}, apply_mask ? 1 : 0, false, err);
        for (size_t q = 0; e == cudaSuccess && apply_mask && q < P; ++q) {
            k_mask<float><<<vec_grid(t.m[q]->n), 256, 0, t.s>>>(w[q], t.m[q]->view);
            e = cudaGetLastError();
        }
    } else {
        return fail(c, NBK_EINVAL, "bad precision");
    }
    if (e != cudaSuccess)
        return fail(c, err.empty() ? NBK_ECUDA : NBK_ENCCL, err.empty() ? cudaGetErrorString(e) : err);
    return NBK_OK;
}

nbk_status nbk_dssum(nbk_ctx* c, void* f_dev, int32_t apply_mask, nbk_precision prec)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    Team t;
    nbk_status st = self_team(c, t);
    if (st != NBK_OK) return st;
    return dssum_team_abi(t, &f_dev, apply_mask, prec);
}

static nbk_status glsc3_team_abi(const Team& t, const void* const* a_dev, const void* const* b_dev,
                                 nbk_precision prec, double* out)
{
    nbk_ctx* c = t.m[0];
    const size_t P = t.m.size();
    if (!out) return fail(c, NBK_EINVAL, "NULL argument");
    for (size_t q = 0; q < P; ++q)
        if (!a_dev[q] || !b_dev[q]) return fail(c, NBK_EINVAL, "NULL argument");
    if (prec == NBK_FP64) {
        std::vector<const double*> a(P), b(P);
        for (size_t q = 0; q < P; ++q) { a[q] = (const double*)a_dev[q]; b[q] = (const double*)b_dev[q]; }
        return glsc3_team<double>(t, a, b, out);
    } else if (prec == NBK_FP32 || prec == NBK_FP32S) {
        std::vector<const float*> a(P), b(P);
        for (size_t q = 0; q < P; ++q) { a[q] = (const float*)a_dev[q]; b[q] = (const float*)b_dev[q]; }
        return glsc3_team<float>(t, a, b, out, prec == NBK_FP32S ? 1 : 0);
    }
    return fail(c, NBK_EINVAL, "bad precision");
}

nbk_status nbk_glsc3(nbk_ctx* c, const void* a_dev, const void* b_dev, nbk_precision prec, double* out)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    Team t;
    nbk_status st = self_team(c, t);
    if (st != NBK_OK) return st;
    return glsc3_team_abi(t, &a_dev, &b_dev, prec, out);
}

nbk_status nbk_set_vprec(nbk_ctx* c, int32_t t)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    if (t < 1 || t > 52) return fail(c, NBK_EINVAL, "VPREC mantissa bits must lie in [1, 52]");
    c->vp_t = t;
    return NBK_OK;
}

nbk_status nbk_set_precond(nbk_ctx* c, int32_t precond)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    if (precond != NBK_PRECOND_NONE && precond != NBK_PRECOND_JACOBI)
        return fail(c, NBK_EINVAL, "bad preconditioner");
    c->precond = precond;
    return NBK_OK;
}

nbk_status nbk_load_precond(nbk_ctx* c, const double* dinv_host)
{
    if (!c || !dinv_host) return fail(c, NBK_EINVAL, "NULL argument");
    NBK_CUDA(c, cudaMemcpyAsync(c->dinv64, dinv_host, 8 * (size_t)c->n, cudaMemcpyHostToDevice, c->stream));
    if (c->dinv32) {
        k_downcast<<<vec_grid(c->n), 256, 0, c->stream>>>(c->dinv32, c->dinv64, c->n);
        NBK_CUDA(c, cudaGetLastError());
    }
    NBK_CUDA(c, cudaStreamSynchronize(c->stream));
    c->dinv_dirty = 0;
    return NBK_OK;
}

nbk_status nbk_get_precond(nbk_ctx* c, double* dinv_host)
{
    if (!c || !dinv_host) return fail(c, NBK_EINVAL, "NULL argument");
    Team t;
    if (c->group.empty()) {
        nbk_status st = self_team(c, t);
        if (st != NBK_OK) return st;
    } else {
        t.m = c->group;
        t.multi = true;
        t.s = c->group[0]->stream;
    }
    nbk_status st = refresh_dinv(t);
    if (st != NBK_OK) return st;
    NBK_CUDA(c, cudaMemcpyAsync(dinv_host, c->dinv64, 8 * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
    NBK_CUDA(c, cudaStreamSynchronize(c->stream));
    return NBK_OK;
}

nbk_status nbk_set_profiling(nbk_ctx* c, int32_t enable)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    c->profiling = enable ? 1 : 0;
    return NBK_OK;
}

nbk_status nbk_cg_solve(nbk_ctx* c, int32_t niter, nbk_precision prec, double* hist_host,
                        double* trace_host, nbk_result* result)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    Team t;
    nbk_status st = self_team(c, t);
    if (st != NBK_OK) return st;
    return solve_team(t, niter, prec, hist_host, trace_host, result);
}

nbk_status nbk_cg_solve_host(nbk_ctx* c, const double* f_host, int32_t niter, nbk_precision prec,
                             double* x_host, double* hist_host, nbk_result* result)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    if (f_host) {
        NBK_CUDA(c, cudaMemcpyAsync(c->f64, f_host, 8 * (size_t)c->n, cudaMemcpyHostToDevice, c->stream));
        nbk_status st0 = refresh_fp32(c);  // new RHS: new h0 for the relative residual
        if (st0 != NBK_OK) return st0;
        c->h0_dirty = 1;
    }
    nbk_status st = nbk_cg_solve(c, niter, prec, hist_host, nullptr, result);
    if (st != NBK_OK && st != NBK_EDEFECT) return st;
    if (x_host) {
        NBK_CUDA(c, cudaMemcpyAsync(x_host, c->x64, 8 * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
        NBK_CUDA(c, cudaStreamSynchronize(c->stream));
    }
    return st;
}

nbk_status nbk_get_solution(nbk_ctx* c, double* x_host)
{
    if (!c || !x_host) return fail(c, NBK_EINVAL, "NULL argument");
    if (c->last_solved_precision < 0) return fail(c, NBK_ESTATE, "no solve yet");
    NBK_CUDA(c, cudaMemcpyAsync(x_host, c->x64, 8 * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
    NBK_CUDA(c, cudaStreamSynchronize(c->stream));
    return NBK_OK;
}

nbk_status nbk_solution_ptr(nbk_ctx* c, nbk_precision prec, void** x_dev)
{
    if (!c || !x_dev) return fail(c, NBK_EINVAL, "NULL argument");
    if (prec == NBK_FP32 && !c->x32) return fail(c, NBK_ESTATE, "no FP32 arrays");
    *x_dev = prec == NBK_FP32 ? (void*)c->x32 : (void*)c->x64;
    return NBK_OK;
}

nbk_status nbk_query(const nbk_ctx* c, nbk_info* info)
{
    if (!c || !info) return fail(nullptr, NBK_EINVAL, "NULL argument");
    info->n_local = c->n;
    info->n_global = c->n_global;
    info->e_local = c->E;
    info->e_offset = c->e_offset;
    info->n_shared = c->nseg;
    info->n_copies = c->ncopies;
    info->N = c->N;
    info->has_fp32 = c->G32 ? 1 : 0;
    info->face_layer = (c->has_lo + c->has_hi) ? c->nlayer : 0;
    info->face_nodes = (int64_t)(c->has_lo + c->has_hi) * c->nplane;
    return NBK_OK;
}

nbk_status nbk_solve_launches(const nbk_ctx* c, int32_t niter, nbk_precision prec, int64_t* launches)
{
    if (!c || !launches) return fail(nullptr, NBK_EINVAL, "NULL argument");
    const int64_t multi = c->nranks > 1 ? 1 : 0;
    // init (+fin), per iteration K_A, K_B, K_C (+ pack, merge, 2 fin), tail_x, [upcast],
    // final check K_A, K_B, K_C (+ pack, merge, fin)
    *launches = (1 + multi) + (3 + 4 * multi) * (int64_t)niter + 1 +
                ((prec == NBK_FP32 || prec == NBK_FP32S) ? 1 : 0) +
                (3 + 3 * multi);
    return NBK_OK;
}

// ------------------------------------------------------------ virtual slabs
static nbk_status group_team(nbk_ctx* const* ctxs, int32_t P, Team& t)
{
    if (!ctxs || P < 1 || P > NBK_MAX_RANKS) return fail(nullptr, NBK_EINVAL, "bad context array");
    for (int r = 0; r < P; ++r)
        if (!ctxs[r]) return fail(nullptr, NBK_EINVAL, "NULL context");
    nbk_ctx* c0 = ctxs[0];
    if ((int)c0->group.size() != P) return fail(c0, NBK_ESTATE, "contexts are not linked (nbk_group_link)");
    for (int r = 0; r < P; ++r)
        if (c0->group[r] != ctxs[r]) return fail(c0, NBK_EINVAL, "context order differs from the linked group");
    t.m.assign(ctxs, ctxs + P);
    t.multi = P > 1;
    t.s = c0->stream;
    return NBK_OK;
}

nbk_status nbk_group_link(nbk_ctx* const* ctxs, int32_t P)
{
    if (!ctxs || P < 1 || P > NBK_MAX_RANKS) return fail(nullptr, NBK_EINVAL, "bad context array");
    for (int r = 0; r < P; ++r) {
        nbk_ctx* c = ctxs[r];
        if (!c) return fail(nullptr, NBK_EINVAL, "NULL context");
        if (c->rank != r || c->nranks != P) return fail(c, NBK_EINVAL, "context r must be rank r of P");
        if (c->comm) return fail(c, NBK_ESTATE, "NCCL context cannot join a virtual group");
        if (std::memcmp(&c->mesh, &ctxs[0]->mesh, sizeof(nbk_mesh)) != 0)
            return fail(c, NBK_EINVAL, "contexts of a group must share the mesh");
        if (c->stream != ctxs[0]->stream) return fail(c, NBK_EINVAL, "contexts of a group must share the stream");
        if (c->dist.device != ctxs[0]->dist.device) return fail(c, NBK_EINVAL, "contexts of a group must share the device");
        if ((c->G32 != nullptr) != (ctxs[0]->G32 != nullptr)) return fail(c, NBK_EINVAL, "mixed set-up precisions");
    }
    for (int r = 0; r < P; ++r) {
        nbk_ctx* c = ctxs[r];
        c->group.assign(ctxs, ctxs + P);
        c->gather = ctxs[0]->gather_own;      // one shared partial array
        if (c->has_lo) c->recv_lo = ctxs[r - 1]->send_hi;
        if (c->has_hi) c->recv_hi = ctxs[r + 1]->send_lo;
        c->h0_dirty = 1;
        c->dinv_dirty = 1;
        destroy_graphs(c);
    }
    return NBK_OK;
}

nbk_status nbk_group_ax_apply(nbk_ctx* const* ctxs, int32_t P, const void* const* u_devs,
                              void* const* w_devs, int32_t flags, nbk_precision prec)
{
    Team t;
    nbk_status st = group_team(ctxs, P, t);
    if (st != NBK_OK) return st;
    if (!u_devs || !w_devs) return fail(ctxs[0], NBK_EINVAL, "NULL pointer array");
    return ax_apply_team(t, u_devs, w_devs, flags, prec);
}

nbk_status nbk_group_dssum(nbk_ctx* const* ctxs, int32_t P, void* const* f_devs, int32_t apply_mask,
                           nbk_precision prec)
{
    Team t;
    nbk_status st = group_team(ctxs, P, t);
    if (st != NBK_OK) return st;
    if (!f_devs) return fail(ctxs[0], NBK_EINVAL, "NULL pointer array");
    return dssum_team_abi(t, f_devs, apply_mask, prec);
}

nbk_status nbk_group_glsc3(nbk_ctx* const* ctxs, int32_t P, const void* const* a_devs,
                           const void* const* b_devs, nbk_precision prec, double* out_host)
{
    Team t;
    nbk_status st = group_team(ctxs, P, t);
    if (st != NBK_OK) return st;
    if (!a_devs || !b_devs) return fail(ctxs[0], NBK_EINVAL, "NULL pointer array");
    return glsc3_team_abi(t, a_devs, b_devs, prec, out_host);
}

nbk_status nbk_group_cg_solve(nbk_ctx* const* ctxs, int32_t P, int32_t niter, nbk_precision prec,
                              double* hist_host, double* trace_host, nbk_result* result)
{
    Team t;
    nbk_status st = group_team(ctxs, P, t);
    if (st != NBK_OK) return st;
    return solve_team(t, niter, prec, hist_host, trace_host, result);
}

void nbk_destroy(nbk_ctx* c)
{
    if (!c) return;
    destroy_graphs(c);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->comm) {
        std::string why;
        const NcclApi* A = nccl_api(why);
        if (A) A->commDestroy((ncclComm_t)c->comm);
    }
    // unlink from a virtual group: the others must not alias this workspace
    for (nbk_ctx* o : std::vector<nbk_ctx*>(c->group)) {
        if (o == c) continue;
        o->group.clear();
        destroy_graphs(o);
    }
    delete c;
}

}  // extern "C"
