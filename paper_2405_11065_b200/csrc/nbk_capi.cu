// nbk_capi.cu -- the extern "C" boundary of libnbk.so (include/nbk.h) and the
// host orchestration of the hot path: kernel dispatch over N, the CG loop
// captured once into a CUDA graph per (precision, niter), device-resident
// scalars, one D2H copy of the history per solve.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

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
template <typename T, int N, bool FUSED>
static cudaError_t launch_ax_n(const AxArgs<T>& a, cudaStream_t s, bool attr_only = false,
                               bool pdl = false)
{
    constexpr int EPB = ax_epb<T>(N);
    const size_t smem = (size_t)ax_smem_bytes<T>(N);
    if (attr_only)
        return cudaFuncSetAttribute(k_ax<T, N, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem);
    const unsigned grid = (unsigned)((a.mesh.E + EPB - 1) / EPB);
    return launch_k(k_ax<T, N, FUSED>, grid, ax_threads<T>(N), smem, s, pdl, a);
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

template <typename T, bool FUSED>
static cudaError_t launch_ax(const AxArgs<T>& a, cudaStream_t s, bool attr_only = false,
                             bool pdl = false)
{
#define AXN(n) launch_ax_n<T, n, FUSED>(a, s, attr_only, pdl)
    NBK_SWITCH_N(a.mesh.N, AXN)
#undef AXN
}

template <typename T, int MODE>
static cudaError_t launch_vec(const VecArgs<T>& a, cudaStream_t s, bool pdl = false)
{
    const int g = vec_grid(a.n);
#define VECN(n) launch_k(k_vec<T, n, MODE>, g, 256, 0, s, pdl, a)
    NBK_SWITCH_N(a.mesh.N, VECN)
#undef VECN
}

template <typename T, bool FUSED>
static cudaError_t launch_dssum(const DssumArgs<T>& a, cudaStream_t s, bool pdl = false)
{
    const int g = vec_grid((a.n2 + a.n4 + a.n8 + a.nother + 1) / 2);
    return launch_k(k_dssum<T, FUSED>, g, 256, 0, s, pdl, a);
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
    d.n2 = c->n2; d.n4 = c->n4; d.n8 = c->n8;
    d.seg_off = c->seg_off; d.seg_idx = c->seg_idx; d.nother = c->nother;
    d.st = c->st; d.trace = c->trace; d.mesh = c->view; d.mask = 0;
    return d;
}

// Enqueue one CG solve (T1 loop, fixed niter) on the stream; used under capture.
template <typename T>
static cudaError_t enqueue_solve(nbk_ctx* c, int niter, nbk_graph* g, bool fp32)
{
    cudaStream_t s = c->stream;
    const T* D = fp32 ? (const T*)c->D32 : (const T*)c->D64;
    const T* G = fp32 ? (const T*)c->G32 : (const T*)c->G64;
    T* x = fp32 ? (T*)c->x32 : (T*)c->x64;
    T* r = fp32 ? (T*)c->r32 : (T*)c->r64;
    T* p = fp32 ? (T*)c->p32 : (T*)c->p64;
    T* w = fp32 ? (T*)c->w32 : (T*)c->w64;
    cudaError_t e;
    int64_t launches = 0;

    VecArgs<T> vi{};
    vi.r = r; vi.x = x; vi.p = p; vi.f = c->f64; vi.n = c->n; vi.parts = c->parts + c->nparts - NBK_VEC_GRID_MAX;
    vi.st = c->st; vi.hist = c->hist; vi.trace = c->trace; vi.mesh = c->view;
    if ((e = launch_vec<T, VEC_INIT>(vi, s)) != cudaSuccess) return e;
    ++launches;

    AxArgs<T> aa = ax_args<T>(c, D, G);
    aa.u = nullptr; aa.w = w; aa.p = p; aa.r = r; aa.x = x; aa.mask = 1;
    DssumArgs<T> da = dssum_args<T>(c, w);
    da.p = p; da.parts = c->parts; da.nA = ax_blocks_n<T>(c->E, c->N);
    VecArgs<T> vr = vi;
    vr.w = w;
    for (int k = 1; k <= niter; ++k) {
        if (g && c->profiling) cudaEventRecordWithFlags(g->prof_events[2 * (k - 1)], s, cudaEventRecordExternal);
        const bool pdl = !(g && c->profiling);  // events between kernels break PDL edges
        if ((e = launch_ax<T, true>(aa, s, false, pdl)) != cudaSuccess) return e;
        if (g && c->profiling) cudaEventRecordWithFlags(g->prof_events[2 * (k - 1) + 1], s, cudaEventRecordExternal);
        if ((e = launch_dssum<T, true>(da, s, pdl)) != cudaSuccess) return e;
        if ((e = launch_vec<T, VEC_RUPD>(vr, s, pdl)) != cudaSuccess) return e;
        launches += 3;
    }
    k_tail_x<T><<<vec_grid(c->n), 256, 0, s>>>(x, p, c->st, c->n);
    ++launches;

    // final FP64 residual check (C12): x64 = (double)x ; r_true = f - A x64
    if (fp32) {
        k_upcast<<<vec_grid(c->n), 256, 0, s>>>(c->x64, (const float*)x, c->n);
        ++launches;
    }
    AxArgs<double> a64 = ax_args<double>(c, c->D64, c->G64);
    a64.u = c->x64; a64.w = c->w64; a64.mask = 1;
    if ((e = launch_ax<double, false>(a64, s)) != cudaSuccess) return e;
    DssumArgs<double> d64 = dssum_args<double>(c, c->w64);
    if ((e = launch_dssum<double, false>(d64, s)) != cudaSuccess) return e;
    VecArgs<double> vt{};
    vt.r = c->r64; vt.w = c->w64; vt.f = c->f64; vt.n = c->n; vt.parts = vi.parts; vt.st = c->st;
    vt.hist = c->hist; vt.trace = c->trace; vt.mesh = c->view;
    if ((e = launch_vec<double, VEC_TRUE>(vt, s)) != cudaSuccess) return e;
    launches += 3;
    if (g) g->launches = launches;
    return cudaSuccess;
}

static nbk_status get_graph(nbk_ctx* c, int niter, nbk_precision prec, nbk_graph** out)
{
    auto key = std::make_tuple((int)prec, niter, c->profiling);
    auto it = c->graphs.find(key);
    if (it != c->graphs.end()) { *out = &it->second; return NBK_OK; }
    nbk_graph g;
    if (c->profiling) {
        g.prof_events.resize(2 * niter);
        for (auto& ev : g.prof_events) NBK_CUDA(c, cudaEventCreate(&ev));
    }
    NBK_CUDA(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = prec == NBK_FP32 ? enqueue_solve<float>(c, niter, &g, true)
                                     : enqueue_solve<double>(c, niter, &g, false);
    cudaGraph_t graph = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(c->stream, &graph);
    if (e != cudaSuccess) return fail(c, NBK_ECUDA, std::string("capture: ") + cudaGetErrorString(e));
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
    if ((e = launch_ax<double, false>(a64, c->stream, true)) != cudaSuccess) return e;
    if ((e = launch_ax<double, true>(a64, c->stream, true)) != cudaSuccess) return e;
    if ((e = launch_ax<float, false>(a32, c->stream, true)) != cudaSuccess) return e;
    return launch_ax<float, true>(a32, c->stream, true);
}

static nbk_status refresh_fp32_and_h0(nbk_ctx* c)
{
    cudaStream_t s = c->stream;
    if (c->G32) {
        k_downcast<<<vec_grid(6 * c->n), 256, 0, s>>>(c->G32, c->G64, 6 * c->n);
        k_downcast<<<1, 256, 0, s>>>(c->D32, c->D64, (int64_t)c->N * c->N);
        NBK_CUDA(c, cudaGetLastError());
    }
    // h0 (FP64) = sqrt(glsc3(f, c, f)) for the relative true residual
    VecArgs<double> v{};
    v.a = c->f64; v.b = c->f64; v.n = c->n; v.parts = c->parts + c->nparts - NBK_VEC_GRID_MAX;
    v.st = c->st; v.mesh = c->view;
    NBK_CUDA(c, launch_vec<double, VEC_DOT>(v, s));
    double dot = 0.0;
    NBK_CUDA(c, cudaMemcpyAsync(&dot, &c->st->dot, 8, cudaMemcpyDeviceToHost, s));
    NBK_CUDA(c, cudaStreamSynchronize(s));
    c->h0_64 = std::sqrt(dot);
    return NBK_OK;
}

// ================================================================== ABI
extern "C" {

const char* nbk_version(void) { return "nbk 0.1 (sm_100a)"; }

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
    nbk_dist d1{0, 1, 0, nullptr};
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
    c->G64 = (double*)(b + L.off_G64);
    c->f64 = (double*)(b + L.off_f64);
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
    }
    nbk_status st = NBK_OK;
    cudaError_t e = set_ax_attrs(c);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->st, 0, sizeof(CgState), c->stream);
    if (e == cudaSuccess) e = setup_device(c, L);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        std::string m = std::string("set-up: ") + cudaGetErrorString(e);
        delete c;
        return fail(nullptr, NBK_ECUDA, m);
    }
    // vectors start at zero (the plan used their space as scratch)
    e = cudaMemsetAsync(c->x64, 0, 4 * v64, c->stream);
    if (e != cudaSuccess) { delete c; return fail(nullptr, NBK_ECUDA, cudaGetErrorString(e)); }
    st = refresh_fp32_and_h0(c);
    if (st != NBK_OK) { std::string m = c->err; delete c; return fail(nullptr, st, m); }
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
    return refresh_fp32_and_h0(c);
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

nbk_status nbk_ax_apply(nbk_ctx* c, const void* u_dev, void* w_dev, int32_t flags, nbk_precision prec)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    if (!u_dev || !w_dev || u_dev == w_dev) return fail(c, NBK_EINVAL, "u/w must be distinct non-NULL");
    if (flags & ~(NBK_AX_DSSUM | NBK_AX_MASK)) return fail(c, NBK_EINVAL, "bad flags");
    if (prec == NBK_FP32 && !c->G32) return fail(c, NBK_ESTATE, "context has no FP32 arrays");
    cudaStream_t s = c->stream;
    if (prec == NBK_FP64) {
        AxArgs<double> a = ax_args<double>(c, c->D64, c->G64);
        a.u = (const double*)u_dev; a.w = (double*)w_dev; a.mask = (flags & NBK_AX_MASK) ? 1 : 0;
        NBK_CUDA(c, launch_ax<double, false>(a, s));
        if (flags & NBK_AX_DSSUM) {
            DssumArgs<double> d = dssum_args<double>(c, (double*)w_dev);
            NBK_CUDA(c, launch_dssum<double, false>(d, s));
        }
    } else if (prec == NBK_FP32) {
        AxArgs<float> a = ax_args<float>(c, c->D32, c->G32);
        a.u = (const float*)u_dev; a.w = (float*)w_dev; a.mask = (flags & NBK_AX_MASK) ? 1 : 0;
        NBK_CUDA(c, launch_ax<float, false>(a, s));
        if (flags & NBK_AX_DSSUM) {
            DssumArgs<float> d = dssum_args<float>(c, (float*)w_dev);
            NBK_CUDA(c, launch_dssum<float, false>(d, s));
        }
    } else {
        return fail(c, NBK_EINVAL, "bad precision");
    }
    return NBK_OK;
}

nbk_status nbk_dssum(nbk_ctx* c, void* f_dev, int32_t apply_mask, nbk_precision prec)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    if (!f_dev) return fail(c, NBK_EINVAL, "f is NULL");
    cudaStream_t s = c->stream;
    if (prec == NBK_FP64) {
        DssumArgs<double> d = dssum_args<double>(c, (double*)f_dev);
        NBK_CUDA(c, launch_dssum<double, false>(d, s));
        if (apply_mask) { k_mask<double><<<vec_grid(c->n), 256, 0, s>>>((double*)f_dev, c->view); NBK_CUDA(c, cudaGetLastError()); }
    } else if (prec == NBK_FP32) {
        DssumArgs<float> d = dssum_args<float>(c, (float*)f_dev);
        NBK_CUDA(c, launch_dssum<float, false>(d, s));
        if (apply_mask) { k_mask<float><<<vec_grid(c->n), 256, 0, s>>>((float*)f_dev, c->view); NBK_CUDA(c, cudaGetLastError()); }
    } else {
        return fail(c, NBK_EINVAL, "bad precision");
    }
    return NBK_OK;
}

nbk_status nbk_glsc3(nbk_ctx* c, const void* a_dev, const void* b_dev, nbk_precision prec, double* out)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    if (!a_dev || !b_dev || !out) return fail(c, NBK_EINVAL, "NULL argument");
    cudaStream_t s = c->stream;
    dd* parts = c->parts + c->nparts - NBK_VEC_GRID_MAX;
    if (prec == NBK_FP64) {
        VecArgs<double> v{};
        v.a = (const double*)a_dev; v.b = (const double*)b_dev; v.n = c->n; v.parts = parts;
        v.st = c->st; v.mesh = c->view;
        NBK_CUDA(c, launch_vec<double, VEC_DOT>(v, s));
    } else if (prec == NBK_FP32) {
        VecArgs<float> v{};
        v.a = (const float*)a_dev; v.b = (const float*)b_dev; v.n = c->n; v.parts = parts;
        v.st = c->st; v.mesh = c->view;
        NBK_CUDA(c, launch_vec<float, VEC_DOT>(v, s));
    } else {
        return fail(c, NBK_EINVAL, "bad precision");
    }
    NBK_CUDA(c, cudaMemcpyAsync(out, &c->st->dot, 8, cudaMemcpyDeviceToHost, s));
    NBK_CUDA(c, cudaStreamSynchronize(s));
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
    if (niter < 1 || niter > NBK_MAX_NITER) return fail(c, NBK_EINVAL, "niter out of range");
    if (prec != NBK_FP64 && prec != NBK_FP32) return fail(c, NBK_EINVAL, "bad precision");
    if (prec == NBK_FP32 && !c->G32) return fail(c, NBK_ESTATE, "context was set up without FP32 arrays");
    nbk_graph* g = nullptr;
    nbk_status st = get_graph(c, niter, prec, &g);
    if (st != NBK_OK) return st;
    cudaStream_t s = c->stream;
    NBK_CUDA(c, cudaEventRecord(c->ev0, s));
    NBK_CUDA(c, cudaGraphLaunch(g->exec, s));
    NBK_CUDA(c, cudaEventRecord(c->ev1, s));
    CgState hs;
    NBK_CUDA(c, cudaMemcpyAsync(&hs, c->st, sizeof(CgState), cudaMemcpyDeviceToHost, s));
    if (hist_host) NBK_CUDA(c, cudaMemcpyAsync(hist_host, c->hist, 8 * (size_t)(niter + 1), cudaMemcpyDeviceToHost, s));
    if (trace_host) NBK_CUDA(c, cudaMemcpyAsync(trace_host, c->trace, 8 * 5 * (size_t)niter, cudaMemcpyDeviceToHost, s));
    NBK_CUDA(c, cudaStreamSynchronize(s));
    c->last_solved_precision = (int)prec;
    if (result) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->ev0, c->ev1);
        result->solve_ms = ms;
        result->true_res = std::sqrt(hs.true_rtr);
        result->true_res_rel = c->h0_64 > 0 ? result->true_res / c->h0_64 : 0.0;
        result->defect_iter = hs.defect;
        result->niter = niter;
        float ka = 0.f;
        if (c->profiling) {
            for (int k = 0; k < niter; ++k) {
                float t = 0.f;
                cudaEventElapsedTime(&t, g->prof_events[2 * k], g->prof_events[2 * k + 1]);
                ka += t;
            }
        }
        result->kA_ms = ka;
    }
    return hs.defect ? fail(c, NBK_EDEFECT, "CG defect: pap <= 0 or non-finite scalar") : NBK_OK;
}

nbk_status nbk_cg_solve_host(nbk_ctx* c, const double* f_host, int32_t niter, nbk_precision prec,
                             double* x_host, double* hist_host, nbk_result* result)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    if (f_host) {
        NBK_CUDA(c, cudaMemcpyAsync(c->f64, f_host, 8 * (size_t)c->n, cudaMemcpyHostToDevice, c->stream));
        nbk_status st0 = refresh_fp32_and_h0(c);  // new RHS: new h0 for the relative residual
        if (st0 != NBK_OK) return st0;
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
    return NBK_OK;
}

nbk_status nbk_solve_launches(const nbk_ctx* c, int32_t niter, nbk_precision prec, int64_t* launches)
{
    if (!c || !launches) return fail(nullptr, NBK_EINVAL, "NULL argument");
    *launches = 1 + 3 * (int64_t)niter + 1 + (prec == NBK_FP32 ? 1 : 0) + 3;
    return NBK_OK;
}

void nbk_destroy(nbk_ctx* c)
{
    if (!c) return;
    destroy_graphs(c);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    delete c;
}

}  // extern "C"
