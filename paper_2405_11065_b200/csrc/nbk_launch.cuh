// nbk_launch.cuh -- kernel launchers and the solve enqueue of libnbk, shared by
// the translation units that instantiate them: nbk_capi.cu (the ABI and the
// FP64 / FP32 solvers) and nbk_emu_*.cu (one precision-emulation mode each, so
// the heavy emulation kernels compile in parallel).  Host code only.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "nbk_internal.h"
#include "nbk_kernels.cuh"
#include "nbk_axl.cuh"
#include "nbk_kbw.cuh"

namespace nbk {

inline int vec_grid(int64_t n)
{
    int64_t g = (n + 255) / 256;
    if (g < 1) g = 1;
    return (int)(g > NBK_VEC_GRID_MAX ? NBK_VEC_GRID_MAX : g);
}


// ------------------------------------------------------------ dispatchers
// Launch with the programmatic-stream-serialization attribute (PDL) when pdl:
// the kernel may start while its predecessor drains; it calls griddepcontrol.wait
// before touching the predecessor's results.
// Edges of the CG loop that get PDL: bit 0 K_C -> K_A, bit 1 K_A -> K_B, bit 2 K_B -> K_C.
// Measured: K_C -> K_A alone +3 % on C2, neutral on C4 (K_A issues its
// G bulk copy while K_C's last CTA reduces); K_A -> K_B costs up to 12 %.  NBK_PDL overrides.
inline int g_pdl_mask = [] {
    const char* e = getenv("NBK_PDL");
    return e ? atoi(e) : 1;
}();
inline bool g_pdl_enabled = true;
// K_A issues p / x loads before the PDL wait from iteration 2 on (NBK_P_EARLY=0: after).
inline int g_p_early = [] {
    const char* e = getenv("NBK_P_EARLY");
    return e ? atoi(e) : 1;
}();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
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
template <typename T, int N, int FUSED, int PM = PM_NONE>
inline cudaError_t launch_ax_n(const AxArgs<T>& a, cudaStream_t s, bool attr_only = false,
                               bool pdl = false)
{
    if constexpr (axl_on<T>(N, FUSED, PM)) {  // line-owner K_A (nbk_axl.cuh)
        constexpr int EPB = axl_epb<T>(N);
        const size_t smem = (size_t)axl_smem_bytes<T>(N);
        if (attr_only)
            return cudaFuncSetAttribute(k_axl<T, N, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem);
        const unsigned grid = (unsigned)((a.en0 + EPB - 1) / EPB + (a.en1 + EPB - 1) / EPB);
        if (grid == 0) return cudaSuccess;
        DMat<T, N> dc{};
        for (int q = 0; q < N * N; ++q) {
            dc.d[q] = a.Dh[q];
            dc.dt[(q % N) * N + q / N] = a.Dh[q];
        }
        return launch_k(k_axl<T, N, FUSED>, grid, axl_threads<T>(N), smem, s, pdl, a, dc);
    }
    constexpr int EPB = ax_epb<T>(N);
    const size_t smem = (size_t)ax_smem_bytes<T>(N, FUSED);
    if (attr_only)
        return cudaFuncSetAttribute(k_ax<T, N, FUSED, PM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem);
    const unsigned grid = (unsigned)((a.en0 + EPB - 1) / EPB + (a.en1 + EPB - 1) / EPB);
    if (grid == 0) return cudaSuccess;
    DConst<T> dc{};
    for (int q = 0; q < N * N; ++q) dc.v[q] = a.Dh[q];
    return launch_k(k_ax<T, N, FUSED, PM>, grid, ax_threads<T>(N), smem, s, pdl, a, dc);
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

template <typename T, int FUSED, int PM = PM_NONE>
inline cudaError_t launch_ax(const AxArgs<T>& a, cudaStream_t s, bool attr_only = false,
                             bool pdl = false)
{
#define AXN(n) launch_ax_n<T, n, FUSED, PM>(a, s, attr_only, pdl)
    if constexpr (PM == PM_VPREC) {  // emulation kernels: N <= NBK_VPREC_MAXN (compile time)
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
    } else if constexpr (PM != PM_NONE) {  // Monte Carlo modes: N <= NBK_MC_MAXN
        switch (a.mesh.N) {
        case 2: return AXN(2);
        case 3: return AXN(3);
        case 4: return AXN(4);
        case 5: return AXN(5);
        case 6: return AXN(6);
        case 7: return AXN(7);
        case 8: return AXN(8);
        default: return cudaErrorNotSupported;
        }
    } else {
        NBK_SWITCH_N(a.mesh.N, AXN)
    }
#undef AXN
}

// Resident CTAs of a kernel on the whole device (SM count x occupancy), cached
// per kernel: grids of the streaming kernels are sized to exactly one wave.
inline int resident_grid(const void* kern, int block, size_t smem)
{
    static std::map<std::pair<const void*, size_t>, int> cache;
    auto it = cache.find({kern, smem});
    if (it != cache.end()) return it->second;
    int dev = 0, sms = 148, nb = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, block, smem) != cudaSuccess || nb < 1) nb = 1;
    int g = nb * sms;
    if (g > NBK_VEC_GRID_MAX) g = NBK_VEC_GRID_MAX;
    cache[{kern, smem}] = g;
    return g;
}

template <typename T, int V, int MODE, int PM>
inline cudaError_t launch_vec_v(const VecArgs<T>& a, cudaStream_t s, bool pdl)
{
    const int cap = resident_grid((const void*)k_vec<T, V, MODE, PM>, 256, 0);
    int64_t g = (a.n / 4 + 511) / 512;  // >= 2 chunks of 4 points per thread
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return launch_k(k_vec<T, V, MODE, PM>, (unsigned)g, 256, 0, s, pdl, a);
}

// one vector kernel for every N: chunks of 4 points (even N) or 1 (odd N)
template <typename T, int MODE, int PM = PM_NONE>
inline cudaError_t launch_vec(const VecArgs<T>& a, cudaStream_t s, bool pdl = false)
{
    if (a.mesh.N < 2 || a.mesh.N > 16) return cudaErrorInvalidValue;
    return a.mesh.N % 2 == 0 ? launch_vec_v<T, 4, MODE, PM>(a, s, pdl) : launch_vec_v<T, 1, MODE, PM>(a, s, pdl);
}

// K_B index staging: a block's next tile is prefetched while it processes the
// current one, which only pays when blocks own several tiles (large meshes;
// measured: C4 +2-4 %, C2 -2 % where every block owns one tile).
// NBK_DSSUM_STAGE (read at every launch / graph capture): 0 off, 1 auto
// (default: on when the tiles are >= 4 per block), 2 always (tests).
inline int dssum_stage_mode()
{
    const char* e = getenv("NBK_DSSUM_STAGE");
    return e ? atoi(e) : 1;
}

// dynamic shared memory of a staged K_B: two index buffers (+ the gather
// variant's copy and p values of one tile)
template <typename T>
inline size_t dssum_stage_smem(int64_t tile_smem)
{
#if defined(NBK_DSSUM_GATHER)
    return 2 * (size_t)tile_smem + (size_t)tile_smem / 4 * sizeof(T) + (size_t)tile_smem / 8 * sizeof(T) + 16;
#else
    return 2 * (size_t)tile_smem;
#endif
}

template <typename T, bool FUSED, int PM = PM_NONE>
inline int dssum_grid_t(int ntiles, int64_t tile_smem, int* stage_out = nullptr)
{
    if constexpr (kbw_on<T, FUSED, PM>()) {  // warp-stream K_B: one resident wave, no staging
        if (stage_out) *stage_out = 0;
        const int cap = resident_grid((const void*)k_dssum_w<T, FUSED, PM>, 256, 0);
        const int want = (ntiles + 7) / 8;   // a warp per tile at least
        return want < 1 ? 1 : (want > cap ? cap : want);
    }
    const int mode = dssum_stage_mode();
    int stage = 0;
    int cap = resident_grid((const void*)k_dssum<T, FUSED, PM>, NBK_DSSUM_THREADS, 0);
    if (mode != 0) {
        const int cap_s = resident_grid((const void*)k_dssum<T, FUSED, PM>, NBK_DSSUM_THREADS, dssum_stage_smem<T>(tile_smem));
#ifdef NBK_DSSUM_GATHER
        const bool auto_stage = true;   // the gather phase works on staged tiles
#else
        const bool auto_stage = ntiles >= 4 * cap_s;
#endif
        if (mode == 2 || auto_stage) { stage = 1; cap = cap_s; }
    }
    if (stage_out) *stage_out = stage;
    return ntiles < 1 ? 1 : (ntiles > cap ? cap : ntiles);
}

// allow more than 48 KB of dynamic shared memory for a staged K_B (set-up, not captured)
template <typename T, bool FUSED, int PM = PM_NONE>
inline cudaError_t dssum_attrs()
{
    return cudaFuncSetAttribute(k_dssum<T, FUSED, PM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)dssum_stage_smem<T>(NBK_DSSUM_TILE_SMEM));
}

template <typename T, bool FUSED, int PM = PM_NONE>
inline cudaError_t launch_dssum(const DssumArgs<T>& a, cudaStream_t s, bool pdl = false)
{
    DssumArgs<T> d = a;
    const int grid = dssum_grid_t<T, FUSED, PM>(a.ntiles, a.tile_smem, &d.stage);
    if constexpr (kbw_on<T, FUSED, PM>()) return launch_k(k_dssum_w<T, FUSED, PM>, grid, 256, 0, s, pdl, d);
    return launch_k(k_dssum<T, FUSED, PM>, grid, NBK_DSSUM_THREADS, d.stage ? dssum_stage_smem<T>(a.tile_smem) : 0, s, pdl, d);
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

inline const NcclApi* nccl_api(std::string& why)
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

inline Team team_self(nbk_ctx* c)
{
    Team t;
    t.m.push_back(c);
    t.multi = c->nranks > 1;
    t.s = c->stream;
    return t;
}

template <typename T>
inline T* fld(nbk_ctx* c, int which, bool fp32)
{
    // which: 0 x, 1 r, 2 p, 3 w, 4 dinv
    void* v64[5] = {c->x64, c->r64, c->p64, c->w64, c->dinv64};
    void* v32[5] = {c->x32, c->r32, c->p32, c->w32, c->dinv32};
    return (T*)(fp32 ? v32[which] : v64[which]);
}

// Exchange the packed face layers with the neighbour ranks (NCCL mode).  In a
// virtual group the receive buffers alias the neighbours' send buffers.
template <typename T>
inline cudaError_t xchg_faces(const Team& t, cudaStream_t s, std::string& err)
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
inline cudaError_t xchg_gather(const Team& t, cudaStream_t s, std::string& err)
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
inline AxArgs<T> ax_args(nbk_ctx* c, const T* D, const T* G)
{
    AxArgs<T> a{};
    a.eb0 = 0; a.en0 = c->E; a.eb1 = 0; a.en1 = 0; a.part_off = 0;   // all elements, one range
    a.D = D;
    if constexpr (sizeof(T) == 8) a.Dh = (const T*)c->Dh64; else a.Dh = (const T*)c->Dh32;
    a.G = G;
    a.mesh = c->view;
    a.st = c->st;
    a.parts = c->parts;
    return a;
}


template <typename T>
inline DssumArgs<T> dssum_args(nbk_ctx* c, T* w)
{
    DssumArgs<T> d{};
    d.w = w;
    d.g2 = c->g2; d.g4 = c->g4; d.g8 = c->g8;
    d.toff = c->toff; d.ntiles = (int)c->ntiles; d.tile_smem = (int)c->tile_smem;
    d.st = c->st; d.trace = c->trace; d.mesh = c->view; d.mask = 0; d.fin = 1;
    return d;
}

template <typename T>
inline FaceArgs<T> face_args(nbk_ctx* c, T* w)
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
inline dd* vec_parts(nbk_ctx* c) { return c->parts + c->nparts - 2 * NBK_VEC_GRID_MAX; }

// Pack the slab-boundary face layers of every member and start the exchange
// (NCCL send / recv on each member's comm stream, event fork / join).
template <typename T>
inline cudaError_t faces_begin(const Team& t, const std::vector<T*>& w, std::string& err)
{
    cudaError_t e;
    for (size_t q = 0; q < t.m.size(); ++q) {
        FaceArgs<T> f = face_args<T>(t.m[q], w[q]);
        k_face_pack<T><<<vec_grid(2 * t.m[q]->nlayer), 256, 0, t.s>>>(f);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    for (nbk_ctx* c : t.m) {
        if (!c->comm) continue;
        if ((e = cudaEventRecord(c->ev_pack, t.s)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(c->comm_stream, c->ev_pack, 0)) != cudaSuccess) return e;
        if ((e = xchg_faces<T>(team_self(c), c->comm_stream, err)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(c->ev_xchg, c->comm_stream)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// Element ranges of the fused K_A of one member.  One rank: everything.  Several
// ranks: launch 0 = the element layers at the slab faces that are exchanged
// (bottom if has_lo, top if has_hi), launch 1 = the interior layers.
struct KaSplit {
    int64_t eb[2][2], en[2][2];   // [launch][range]
};
inline KaSplit ka_split(const nbk_ctx* c, bool multi)
{
    KaSplit k{};
    if (!multi) {
        k.en[0][0] = c->E;
        return k;
    }
    const int64_t exy = (int64_t)c->view.ex * c->view.ey, L = c->view.ez_local;
    const bool lo = c->has_lo, hi = c->has_hi && (L > 1 || !lo);
    if (lo) { k.eb[0][0] = 0; k.en[0][0] = exy; }
    if (hi) { k.eb[0][1] = (L - 1) * exy; k.en[0][1] = exy; }
    const int64_t ib = lo ? exy : 0, ie = (hi ? (L - 1) * exy : L * exy);
    if (ie > ib) { k.eb[1][0] = ib; k.en[1][0] = ie - ib; }
    return k;
}
// K_A blocks over n elements (EPB elements per block)
template <typename T, int PM = PM_NONE>
inline int ka_blocks(const nbk_ctx* c, int64_t n)
{
    int epb = 1;
#define EPBC(nn) case nn: epb = axl_on<T>(nn, 1, PM) ? axl_epb<T>(nn) : ax_epb<T>(nn); break;
    switch (c->N) {
    EPBC(2) EPBC(3) EPBC(4) EPBC(5) EPBC(6) EPBC(7) EPBC(8) EPBC(9) EPBC(10) EPBC(11) EPBC(12)
    EPBC(13) EPBC(14) EPBC(15) EPBC(16)
    default: break;
    }
#undef EPBC
    return (int)((n + epb - 1) / epb);
}
// K_A launches of a member in one CG step (an empty launch is skipped)
inline int ka_launches(const nbk_ctx* c, bool multi)
{
    const KaSplit k = ka_split(c, multi);
    return (k.en[0][0] + k.en[0][1] > 0 ? 1 : 0) + (k.en[1][0] + k.en[1][1] > 0 ? 1 : 0);
}
// K_A pap partials of a member in the CG step (all launches)
template <typename T, int PM = PM_NONE>
inline int ka_parts(const nbk_ctx* c, bool multi)
{
    const KaSplit k = ka_split(c, multi);
    int n = 0;
    for (int l = 0; l < 2; ++l)
        for (int r = 0; r < 2; ++r) n += ka_blocks<T, PM>(c, k.en[l][r]);
    return n;
}

// dssum (+ mask) of w over a team.  fused: shared-node pap terms, alpha.
// One rank: K_B (its last block forms alpha).  Several: K_B (publish only) and
// the face pack, exchange, face merge (reduces this rank's pap), all-gather,
// k_fin (rank-ordered combination, alpha).
template <typename T, bool FUSED, int PM = PM_NONE>
inline cudaError_t dssum_team(const Team& t, const std::vector<T*>& w, const std::vector<const T*>& p,
                              int mask, bool pdl, std::string& err, int rev = 0, int single = 0,
                              PmArgs pm = PmArgs{52, 0}, int it = 0, bool faces_started = false)
{
    cudaError_t e;
    const cudaStream_t s = t.s;
    // Several ranks: pack the slab-boundary face layers and start their NCCL
    // exchange on the comm stream (faces_begin) -- in the CG step right after
    // K_A's slab-boundary layers, so that it overlaps the interior elements'
    // ax and the local dssum (K_B never touches plane nodes); the merge waits
    // for both.  (Virtual slabs: the exchange is pointer aliasing.)
    if (t.multi && !faces_started)
        if ((e = faces_begin<T>(t, w, err)) != cudaSuccess) return e;
    for (size_t q = 0; q < t.m.size(); ++q) {
        nbk_ctx* c = t.m[q];
        DssumArgs<T> d = dssum_args<T>(c, w[q]);
        d.mask = mask;
        d.rev = rev;
        d.single = single;
        d.pm = pm;
        d.it = it;
        if (FUSED) {
            d.p = p[q];
            d.parts = c->parts;
            d.nA = ka_parts<T, PM>(c, t.multi);
            d.fin = t.multi ? 0 : 1;
        }
        if ((e = launch_dssum<T, FUSED, PM>(d, s, pdl && !t.multi)) != cudaSuccess) return e;
    }
    if (!t.multi) return cudaSuccess;
    for (nbk_ctx* c : t.m)
        if (c->comm && (e = cudaStreamWaitEvent(s, c->ev_xchg, 0)) != cudaSuccess) return e;
    for (size_t q = 0; q < t.m.size(); ++q) {
        nbk_ctx* c = t.m[q];
        FaceArgs<T> f = face_args<T>(c, w[q]);
        f.mask = mask;
        f.single = single;
        if (FUSED) {
            f.p = p[q];
            f.nprev = ka_parts<T, PM>(c, t.multi) + dssum_grid_t<T, FUSED, PM>((int)c->ntiles, c->tile_smem);
            f.nskip = ka_parts<T, PM>(c, t.multi);
        }
        const int64_t nodes = (int64_t)(c->has_lo + c->has_hi) * c->nplane;
        k_face_merge<T, FUSED><<<vec_grid(nodes), 256, 0, s>>>(f);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (FUSED) {
        if ((e = xchg_gather(t, s, err)) != cudaSuccess) return e;
        for (nbk_ctx* c : t.m) {
            k_fin<0><<<1, 32, 0, s>>>(c->gather, c->nranks, c->st, c->hist, c->trace, single, PM, pm);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

// Vector kernel (K_C and the other modes) over a team: one rank finalises in
// its last block; several publish per-rank partials, all-gather, k_fin.
template <typename T, int MODE, int PM = PM_NONE>
inline cudaError_t vec_team(const Team& t, const std::vector<VecArgs<T>>& args, bool pdl,
                            std::string& err)
{
    cudaError_t e;
    for (size_t q = 0; q < t.m.size(); ++q) {
        VecArgs<T> a = args[q];
        a.slot = t.multi ? t.m[q]->gather + 2 * t.m[q]->rank : nullptr;
        if ((e = launch_vec<T, MODE, PM>(a, t.s, pdl && !t.multi)) != cudaSuccess) return e;
    }
    if (!t.multi) return cudaSuccess;
    if ((e = xchg_gather(t, t.s, err)) != cudaSuccess) return e;
    for (size_t q = 0; q < t.m.size(); ++q) {
        nbk_ctx* c = t.m[q];
        k_fin<1 + MODE><<<1, 32, 0, t.s>>>(c->gather, c->nranks, c->st, c->hist, c->trace,
                                          args[q].single, PM, args[q].pm);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// Binary32-accumulating vector kernel over a team (NEXT-2 paper single solver).
template <int MODE>
inline cudaError_t vec_a_team(const Team& t, const std::vector<VecArgs<float>>& args, std::string& err)
{
    cudaError_t e;
    for (size_t q = 0; q < t.m.size(); ++q) {
        VecArgs<float> a = args[q];
        a.slot = t.multi ? t.m[q]->gather + 2 * t.m[q]->rank : nullptr;
        const bool v4 = a.mesh.N % 2 == 0;
        const void* kern = v4 ? (const void*)k_vec_a<4, MODE> : (const void*)k_vec_a<1, MODE>;
        const int cap = resident_grid(kern, 256, 0);
        int64_t g = (a.n / 4 + 511) / 512;
        if (g < 1) g = 1;
        if (g > cap) g = cap;
        if (v4) k_vec_a<4, MODE><<<(unsigned)g, 256, 0, t.s>>>(a);
        else k_vec_a<1, MODE><<<(unsigned)g, 256, 0, t.s>>>(a);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (!t.multi) return cudaSuccess;
    if ((e = xchg_gather(t, t.s, err)) != cudaSuccess) return e;
    for (nbk_ctx* c : t.m) {
        constexpr int KIND = MODE == VA_PAP ? 0 : (MODE == VA_INIT ? 1 + VEC_INIT : 1 + VEC_RUPD);
        k_fin<KIND><<<1, 32, 0, t.s>>>(c->gather, c->nranks, c->st, c->hist, c->trace, 2, PM_NONE,
                                      PmArgs{52, 0});
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <typename T>
inline VecArgs<T> vec_args(nbk_ctx* c)
{
    VecArgs<T> v{};
    v.n = c->n; v.parts = vec_parts(c); v.st = c->st; v.hist = c->hist; v.trace = c->trace;
    v.mesh = c->view;
    return v;
}

// Field permutation natural <-> split layout (one pass).
template <typename T>
inline cudaError_t perm_sl(nbk_ctx* c, T* dst, const T* src, bool to_sl, cudaStream_t s)
{
    if (to_sl) k_perm_sl<T, true><<<vec_grid(c->n), 256, 0, s>>>(dst, src, c->view);
    else k_perm_sl<T, false><<<vec_grid(c->n), 256, 0, s>>>(dst, src, c->view);
    return cudaGetLastError();
}

// The solver's w buffer of precision T: scratch of the public natural-order calls
// (dead between solves).
template <typename T>
inline T* sl_scratch(nbk_ctx* c) { return (T*)(sizeof(T) == 8 ? (void*)c->w64 : (void*)c->w32); }

// ax (+ dssum + mask) of per-member fields over a team.  sl: u, w are CG vectors
// in the split layout (final check); otherwise natural-order public arrays --
// with DSSUM, K_A writes SL into the member's scratch, the SL plan sums it and
// the result is permuted into w.
template <typename T>
inline cudaError_t ax_team(const Team& t, const std::vector<const T*>& u, const std::vector<T*>& w,
                           int flags, bool fp32, std::string& err, bool sl = false)
{
    cudaError_t e;
    const bool ds = (flags & NBK_AX_DSSUM) != 0;
    std::vector<T*> wsl(t.m.size());
    for (size_t q = 0; q < t.m.size(); ++q) {
        nbk_ctx* c = t.m[q];
        AxArgs<T> a = fp32 ? ax_args<T>(c, (const T*)c->D32, (const T*)c->G32)
                           : ax_args<T>(c, (const T*)c->D64, (const T*)c->G64);
        wsl[q] = (sl || !ds) ? w[q] : sl_scratch<T>(c);
        a.u = u[q]; a.w = wsl[q]; a.mask = (flags & NBK_AX_MASK) ? 1 : 0;
        a.in_sl = sl ? 1 : 0;
        a.out_sl = (sl || ds) ? 1 : 0;
        if ((e = launch_ax<T, 0>(a, t.s)) != cudaSuccess) return e;
    }
    if (!ds) return cudaSuccess;
    if ((e = dssum_team<T, false>(t, wsl, {}, 0, false, err)) != cudaSuccess) return e;
    if (sl) return cudaSuccess;
    for (size_t q = 0; q < t.m.size(); ++q)
        if ((e = perm_sl<T>(t.m[q], w[q], wsl[q], false, t.s)) != cudaSuccess) return e;
    return cudaSuccess;
}

// Enqueue one CG solve (T1 loop, fixed niter) for the team; used under capture.
// Final FP64 residual check (C12) after the loop: w = A x64 (K_A, dssum, mask),
// r_true = f - w, glsc3 -- plain binary64 kernels, defined once (nbk_capi.cu).
cudaError_t enqueue_final_check(const Team& t, std::string& err);

template <typename T, int PM = PM_NONE>
inline cudaError_t enqueue_solve(const Team& t, int niter, nbk_graph* g, bool fp32, bool profiling,
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
    const bool jac = PM == PM_NONE && t.m[0]->precond == NBK_PRECOND_JACOBI;
    const PmArgs pm{t.m[0]->vp_t, t.m[0]->pm_seed};  // precision emulation (NEXT-4)
    std::vector<VecArgs<T>> vi(P), vr(P);
    for (size_t q = 0; q < P; ++q) {
        vi[q] = vec_args<T>(t.m[q]);
        vi[q].r = r[q]; vi[q].x = x[q]; vi[q].p = p[q]; vi[q].f = t.m[q]->f64;
        vi[q].dinv = fld<T>(t.m[q], 4, fp32);
        vi[q].single = single;
        vi[q].pm = pm;
        vi[q].it = 0;
        vr[q] = vi[q];
        vr[q].w = w[q];
    }
    // the paper's single-precision solver (NEXT-2, R11c): binary32 accumulation of
    // pap and rtr in separate kernels (K_B runs as a plain dssum)
    const bool acc32 = single == 2;
    if constexpr (sizeof(T) == 4) {
        if (acc32) {
            std::vector<VecArgs<float>> v32(P);
            for (size_t q = 0; q < P; ++q) v32[q] = *(const VecArgs<float>*)&vi[q];
            e = vec_a_team<VA_INIT>(t, v32, err);
        }
    }
    if (!acc32)
        e = jac ? vec_team<T, VEC_INIT_J>(t, vi, false, err) : vec_team<T, VEC_INIT, PM>(t, vi, false, err);
    if (e != cudaSuccess) return e;
    launches += (int64_t)P * (1 + per_fin);

    // sweep directions alternate kernel by kernel: K_A f, K_B b, K_C f, K_A b, ...
    int rev = 0;
    for (int k = 1; k <= niter; ++k) {
        const bool prof = g && profiling && P == 1;
        if (prof) cudaEventRecordWithFlags(g->prof_events[4 * (k - 1)], s, cudaEventRecordExternal);
        const bool pdl = !prof;  // events between kernels break PDL edges
        // K_A; several ranks: slab-face layers, start of the face exchange, interior layers
        for (int l = 0; l < (t.multi ? 2 : 1); ++l) {
            if (l == 1 && (e = faces_begin<T>(t, w, err)) != cudaSuccess) return e;
            for (size_t q = 0; q < P; ++q) {
                nbk_ctx* c = t.m[q];
                AxArgs<T> aa = fp32 ? ax_args<T>(c, (const T*)c->D32, (const T*)c->G32)
                                    : ax_args<T>(c, (const T*)c->D64, (const T*)c->G64);
                aa.u = nullptr; aa.w = w[q]; aa.p = p[q]; aa.r = r[q]; aa.x = x[q]; aa.mask = 1;
                aa.rev = rev;
                aa.dinv = fld<T>(c, 4, fp32);
                aa.single = single;
                aa.pm = pm;
                aa.it = k;
                aa.p_ready = k >= 2 && g_p_early;
                const KaSplit ks = ka_split(c, t.multi);
                aa.eb0 = ks.eb[l][0]; aa.en0 = ks.en[l][0];
                aa.eb1 = ks.eb[l][1]; aa.en1 = ks.en[l][1];
                aa.part_off = l == 0 ? 0 : ka_blocks<T, PM>(c, ks.en[0][0]) + ka_blocks<T, PM>(c, ks.en[0][1]);
                const bool pa = pdl && (g_pdl_mask & 1) && l == 0;
                e = jac ? launch_ax<T, 2>(aa, s, false, pa) : launch_ax<T, 1, PM>(aa, s, false, pa);
                if (e != cudaSuccess) return e;
            }
        }
        if (prof) cudaEventRecordWithFlags(g->prof_events[4 * (k - 1) + 1], s, cudaEventRecordExternal);
        if (acc32) {
            if ((e = dssum_team<T, false>(t, w, {}, 0, false, err, !rev, 0, PmArgs{52, 0}, 0, t.multi)) !=
                cudaSuccess)
                return e;
            if constexpr (sizeof(T) == 4) {
                std::vector<VecArgs<float>> vp(P);
                for (size_t q = 0; q < P; ++q) {
                    vp[q] = *(const VecArgs<float>*)&vr[q];
                    vp[q].p = (float*)p[q];
                    vp[q].rev = rev;
                }
                if ((e = vec_a_team<VA_PAP>(t, vp, err)) != cudaSuccess) return e;
            }
            launches += (int64_t)P * (1 + per_fin);
        } else if ((e = dssum_team<T, true, PM>(t, w, pc, 0, pdl && (g_pdl_mask & 2), err, !rev, single, pm, k,
                                                t.multi)) != cudaSuccess) {
            return e;
        }
        if (prof) cudaEventRecordWithFlags(g->prof_events[4 * (k - 1) + 2], s, cudaEventRecordExternal);
        for (size_t q = 0; q < P; ++q) {
            vr[q].rev = rev;
            vr[q].it = k;
        }
        const bool pc_ = pdl && (g_pdl_mask & 4);
        if constexpr (sizeof(T) == 4) {
            if (acc32) {
                std::vector<VecArgs<float>> v32(P);
                for (size_t q = 0; q < P; ++q) v32[q] = *(const VecArgs<float>*)&vr[q];
                e = vec_a_team<VA_RUPD>(t, v32, err);
            }
        }
        if (!acc32)
            e = jac ? vec_team<T, VEC_RUPD_J>(t, vr, pc_, err) : vec_team<T, VEC_RUPD, PM>(t, vr, pc_, err);
        if (e != cudaSuccess) return e;
        if (prof) cudaEventRecordWithFlags(g->prof_events[4 * (k - 1) + 3], s, cudaEventRecordExternal);
        rev = !rev;
        launches += (int64_t)P * (2 + nface + 2 * per_fin);
        for (size_t q = 0; q < P; ++q) launches += ka_launches(t.m[q], t.multi);
    }
    for (size_t q = 0; q < P; ++q) {
        nbk_ctx* c = t.m[q];
        k_tail_x<T, PM><<<vec_grid(c->n), 256, 0, s>>>(x[q], p[q], c->st, c->n, pm, niter + 1, c->view);
        ++launches;
        // final FP64 residual check (C12): x64 = (double)x ; r_true = f - A x64
        if (fp32) {
            k_upcast<<<vec_grid(c->n), 256, 0, s>>>(c->x64, (const float*)x[q], c->n);
            ++launches;
        }
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = enqueue_final_check(t, err)) != cudaSuccess) return e;
    launches += (int64_t)P * (3 + nface + per_fin);
    if (g) g->launches = launches;
    return cudaSuccess;
}


// Emulated solves (NBK_VPREC precision; nbk_emu_*.cu): enqueue_solve<double, PM>.
cudaError_t enqueue_emulated(const Team& t, int niter, nbk_graph* g, bool profiling, std::string& err,
                             int mode);
cudaError_t emulated_attrs(nbk_ctx* c);

}  // namespace nbk
