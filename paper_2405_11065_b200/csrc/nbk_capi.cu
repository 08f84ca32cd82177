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

#include "nbk_launch.cuh"

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

namespace nbk {
cudaError_t enqueue_emulated_1(const Team&, int, nbk_graph*, bool, std::string&);
cudaError_t enqueue_emulated_2(const Team&, int, nbk_graph*, bool, std::string&);
cudaError_t enqueue_emulated_3(const Team&, int, nbk_graph*, bool, std::string&);
cudaError_t emulated_attrs_1(nbk_ctx*);
cudaError_t emulated_attrs_2(nbk_ctx*);
cudaError_t emulated_attrs_3(nbk_ctx*);

cudaError_t enqueue_emulated(const Team& t, int niter, nbk_graph* g, bool profiling, std::string& err,
                             int mode)
{
    switch (mode) {
    case PM_VPREC: return enqueue_emulated_1(t, niter, g, profiling, err);
    case PM_RR: return enqueue_emulated_2(t, niter, g, profiling, err);
    case PM_MCA: return enqueue_emulated_3(t, niter, g, profiling, err);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t enqueue_final_check(const Team& t, std::string& err)
{
    const size_t P = t.m.size();
    std::vector<const double*> x64(P);
    std::vector<double*> w64(P);
    std::vector<VecArgs<double>> vt(P);
    for (size_t q = 0; q < P; ++q) {
        nbk_ctx* c = t.m[q];
        x64[q] = c->x64; w64[q] = c->w64;
        vt[q] = vec_args<double>(c);
        vt[q].r = c->r64; vt[q].w = c->w64; vt[q].f = c->f64;
    }
    cudaError_t e;
    if ((e = ax_team<double>(t, x64, w64, NBK_AX_DSSUM | NBK_AX_MASK, false, err, true)) != cudaSuccess) return e;
    return vec_team<double, VEC_TRUE>(t, vt, false, err);
}

cudaError_t emulated_attrs(nbk_ctx* c)
{
    cudaError_t e;
    if ((e = emulated_attrs_1(c)) != cudaSuccess) return e;
    if ((e = emulated_attrs_2(c)) != cudaSuccess) return e;
    return emulated_attrs_3(c);
}
}  // namespace nbk

static nbk_status get_graph(const Team& t, int niter, nbk_precision prec, nbk_graph** out)
{
    nbk_ctx* c = t.m[0];
    // emulated solves: one graph per (mode, t, seed) -- the seed is a kernel argument
    auto key = std::make_tuple((int)prec + (prec == NBK_VPREC ? 4 * (c->vp_t + 64 * c->pm_mode) : 0), niter,
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
                    : prec == NBK_VPREC ? enqueue_emulated(t, niter, &g, c->profiling, err, c->pm_mode)
                                        : enqueue_solve<float>(t, niter, &g, true, c->profiling, err,
                                                               prec == NBK_FP32S ? 1 : (prec == NBK_FP32A ? 2 : 0));
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

    if ((e = dssum_attrs<double, true>()) != cudaSuccess) return e;
    if ((e = dssum_attrs<double, false>()) != cudaSuccess) return e;
    if ((e = dssum_attrs<float, true>()) != cudaSuccess) return e;
    if ((e = dssum_attrs<float, false>()) != cudaSuccess) return e;
    if ((e = launch_ax<double, 0>(a64, c->stream, true)) != cudaSuccess) return e;
    if (c->N <= NBK_VPREC_MAXN && (e = emulated_attrs(c)) != cudaSuccess) return e;
    if ((e = launch_ax<double, 1>(a64, c->stream, true)) != cudaSuccess) return e;
    if ((e = launch_ax<double, 2>(a64, c->stream, true)) != cudaSuccess) return e;
    if ((e = launch_ax<float, 0>(a32, c->stream, true)) != cudaSuccess) return e;
    if ((e = launch_ax<float, 1>(a32, c->stream, true)) != cudaSuccess) return e;
    return launch_ax<float, 2>(a32, c->stream, true);
}

// glsc3 over a team (synchronous); result identical on every member.
// natural: a, b are public natural-order arrays (else SL vectors of the library)
template <typename T>
static nbk_status glsc3_team(const Team& t, const std::vector<const T*>& a, const std::vector<const T*>& b,
                             double* out, int single = 0, bool natural = true)
{
    nbk_ctx* c0 = t.m[0];
    std::vector<VecArgs<T>> v(t.m.size());
    for (size_t q = 0; q < t.m.size(); ++q) {
        v[q] = vec_args<T>(t.m[q]);
        v[q].a = a[q]; v[q].b = b[q];
        v[q].single = single;
        v[q].natural = natural ? 1 : 0;
    }
    std::string err;
    cudaError_t e = vec_team<T, VEC_DOT>(t, v, false, err);
    if (e != cudaSuccess) return fail(c0, err.empty() ? NBK_ECUDA : NBK_ENCCL, err.empty() ? cudaGetErrorString(e) : err);
    NBK_CUDA(c0, cudaMemcpyAsync(out, &c0->st->dot, 8, cudaMemcpyDeviceToHost, t.s));
    NBK_CUDA(c0, cudaStreamSynchronize(t.s));
    return NBK_OK;
}

// The operator (D and / or G) changed: re-derive the FP32 copies (C11) and
// re-assemble the own Jacobi diagonal on demand.  A new RHS alone only needs
// a new h0 (callers set h0_dirty): G is not re-downcast and a diagonal loaded
// with nbk_load_precond stays in use.
static nbk_status refresh_fp32(nbk_ctx* c)
{
    cudaStream_t s = c->stream;
    c->dinv_dirty = 1;  // own diagonal re-assembled on demand
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
    nbk_status st = glsc3_team<double>(t, f, f, &dot, 0, false);   // f64 is an SL vector
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
    if (prec != NBK_FP64 && prec != NBK_FP32 && prec != NBK_FP32S && prec != NBK_VPREC && prec != NBK_FP32A)
        return fail(c, NBK_EINVAL, "bad precision");
    for (nbk_ctx* m : t.m) {
        if (prec == NBK_FP32A && m->precond != NBK_PRECOND_NONE)
            return fail(c, NBK_EINVAL, "the binary32-accumulating solver is unpreconditioned");
        if ((prec == NBK_FP32 || prec == NBK_FP32S || prec == NBK_FP32A) && !m->G32)
            return fail(c, NBK_ESTATE, "context was set up without FP32 arrays");
        if (prec == NBK_VPREC && m->vp_t != c->vp_t) return fail(c, NBK_EINVAL, "members differ in VPREC t");
        if (prec == NBK_VPREC && m->N > NBK_VPREC_MAXN) return fail(c, NBK_EINVAL, "VPREC emulation supports N <= 12");
        if (prec == NBK_VPREC && m->pm_mode != PM_VPREC && m->N > NBK_MC_MAXN)
            return fail(c, NBK_EINVAL, "RR / MCA emulation supports N <= 8");
        if (prec == NBK_VPREC && t.multi) return fail(c, NBK_EINVAL, "precision emulation runs on one rank");
        if (prec == NBK_VPREC && m->precond != NBK_PRECOND_NONE)
            return fail(c, NBK_EINVAL, "precision emulation runs the unpreconditioned CG only");
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

// Public dssum of natural-order fields: permute into the member's SL scratch,
// sum with the SL plan, permute back, mask (C5) in natural order.
template <typename T>
static cudaError_t dssum_natural(const Team& t, void* const* f_dev, int32_t apply_mask, std::string& err)
{
    const size_t P = t.m.size();
    cudaError_t e;
    std::vector<T*> w(P);
    for (size_t q = 0; q < P; ++q) {
        w[q] = sl_scratch<T>(t.m[q]);
        if ((e = perm_sl<T>(t.m[q], w[q], (const T*)f_dev[q], true, t.s)) != cudaSuccess) return e;
    }
    if ((e = dssum_team<T, false>(t, w, {}, 0, false, err)) != cudaSuccess) return e;
    for (size_t q = 0; q < P; ++q) {
        if ((e = perm_sl<T>(t.m[q], (T*)f_dev[q], w[q], false, t.s)) != cudaSuccess) return e;
        if (apply_mask) {
            k_mask<T><<<vec_grid(t.m[q]->n), 256, 0, t.s>>>((T*)f_dev[q], t.m[q]->view);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
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
    if (!c->stream) {
        // NULL: the legacy default stream cannot be captured into the solve
        // graph; a blocking stream of our own is implicitly ordered with it
        if (cudaStreamCreate(&c->own_stream) != cudaSuccess) {
            delete c;
            return fail(nullptr, NBK_ECUDA, "cannot create the context stream");
        }
        c->stream = c->own_stream;
    }
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
        if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_xchg, cudaEventDisableTiming) != cudaSuccess) {
            nbk_destroy(c);
            return fail(nullptr, NBK_ECUDA, "cannot create the face-exchange stream");
        }
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
    if (D_host) {
        NBK_CUDA(c, cudaMemcpyAsync(c->D64, D_host, 8 * c->N * c->N, cudaMemcpyHostToDevice, s));
        for (int q = 0; q < c->N * c->N; ++q) {
            c->Dh64[q] = D_host[q];
            c->Dh32[q] = (float)D_host[q];  // RN32 (C11)
        }
        // D is a kernel parameter of k_ax: captured solve graphs hold the old values
        destroy_graphs(c);
        for (nbk_ctx* o : c->group) destroy_graphs(o);
    }
    if (G_host) NBK_CUDA(c, cudaMemcpyAsync(c->G64, G_host, 8 * 6 * c->n, cudaMemcpyHostToDevice, s));
    if (f_host) {  // natural order on the host, split layout on the device
        NBK_CUDA(c, cudaMemcpyAsync(c->w64, f_host, 8 * c->n, cudaMemcpyHostToDevice, s));
        NBK_CUDA(c, perm_sl<double>(c, c->f64, c->w64, true, s));
    }
    if (D_host || G_host) {  // operator changed
        nbk_status st = refresh_fp32(c);
        if (st != NBK_OK) return st;
    }
    if (f_host) c->h0_dirty = 1;
    NBK_CUDA(c, cudaStreamSynchronize(s));
    return NBK_OK;
}

nbk_status nbk_get_arrays(nbk_ctx* c, double* D_host, double* G_host, double* f_host)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    cudaStream_t s = c->stream;
    if (D_host) NBK_CUDA(c, cudaMemcpyAsync(D_host, c->D64, 8 * c->N * c->N, cudaMemcpyDeviceToHost, s));
    if (G_host) NBK_CUDA(c, cudaMemcpyAsync(G_host, c->G64, 8 * 6 * c->n, cudaMemcpyDeviceToHost, s));
    if (f_host) {
        NBK_CUDA(c, perm_sl<double>(c, c->w64, c->f64, false, s));
        NBK_CUDA(c, cudaMemcpyAsync(f_host, c->w64, 8 * c->n, cudaMemcpyDeviceToHost, s));
    }
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
        e = dssum_natural<double>(t, f_dev, apply_mask, err);
    } else if (prec == NBK_FP32) {
        for (size_t q = 0; q < P; ++q)
            if (!t.m[q]->w32) return fail(c, NBK_ESTATE, "context has no FP32 arrays");
        e = dssum_natural<float>(t, f_dev, apply_mask, err);
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
    return nbk_set_emulation(c, NBK_EMU_VPREC, t, 0);
}

nbk_status nbk_set_emulation(nbk_ctx* c, int32_t mode, int32_t t, uint64_t seed)
{
    if (!c) return fail(nullptr, NBK_EINVAL, "ctx is NULL");
    if (mode != NBK_EMU_VPREC && mode != NBK_EMU_RR && mode != NBK_EMU_MCA)
        return fail(c, NBK_EINVAL, "bad emulation mode");
    if (t < 1 || t > 52) return fail(c, NBK_EINVAL, "virtual precision t must lie in [1, 52]");
    c->pm_mode = mode;
    c->vp_t = t;
    if (c->pm_seed != seed) {  // the seed is baked into the captured kernel arguments
        for (auto it = c->graphs.begin(); it != c->graphs.end();) {
            if (std::get<0>(it->first) % 4 == NBK_VPREC) {
                if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
                if (it->second.graph) cudaGraphDestroy(it->second.graph);
                for (auto ev : it->second.prof_events) cudaEventDestroy(ev);
                it = c->graphs.erase(it);
            } else {
                ++it;
            }
        }
    }
    c->pm_seed = seed;
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
    NBK_CUDA(c, cudaMemcpyAsync(c->w64, dinv_host, 8 * (size_t)c->n, cudaMemcpyHostToDevice, c->stream));
    NBK_CUDA(c, perm_sl<double>(c, c->dinv64, c->w64, true, c->stream));
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
    NBK_CUDA(c, perm_sl<double>(c, c->w64, c->dinv64, false, c->stream));
    NBK_CUDA(c, cudaMemcpyAsync(dinv_host, c->w64, 8 * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
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
        NBK_CUDA(c, cudaMemcpyAsync(c->w64, f_host, 8 * (size_t)c->n, cudaMemcpyHostToDevice, c->stream));
        NBK_CUDA(c, perm_sl<double>(c, c->f64, c->w64, true, c->stream));
        c->h0_dirty = 1;  // new RHS: new h0 for the relative residual (operator unchanged)
    }
    nbk_status st = nbk_cg_solve(c, niter, prec, hist_host, nullptr, result);
    if (st != NBK_OK && st != NBK_EDEFECT) return st;
    if (x_host) {
        NBK_CUDA(c, perm_sl<double>(c, c->w64, c->x64, false, c->stream));
        NBK_CUDA(c, cudaMemcpyAsync(x_host, c->w64, 8 * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
        NBK_CUDA(c, cudaStreamSynchronize(c->stream));
    }
    return st;
}

nbk_status nbk_cg_solve_host_batch(nbk_ctx* c, int32_t nrhs, const double* const* f_hosts, int32_t niter,
                                   nbk_precision prec, double* const* x_hosts, double* hist_hosts,
                                   nbk_result* results)
{
    if (!c || nrhs < 1 || !f_hosts) return fail(c, NBK_EINVAL, "NULL ctx / f_hosts or nrhs < 1");
    for (int32_t k = 0; k < nrhs; ++k)
        if (!f_hosts[k]) return fail(c, NBK_EINVAL, "f_hosts[k] is NULL");
    const size_t bytes = 8 * (size_t)c->n;
    if (!c->stage_f) {
        NBK_CUDA(c, cudaMalloc(&c->stage_f, bytes));
        NBK_CUDA(c, cudaMalloc(&c->stage_x, bytes));
        NBK_CUDA(c, cudaStreamCreateWithFlags(&c->xs_in, cudaStreamNonBlocking));
        NBK_CUDA(c, cudaStreamCreateWithFlags(&c->xs_out, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&c->ev_in, &c->ev_fused, &c->ev_xready, &c->ev_out})
            NBK_CUDA(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    // RHS 0 in, after the work already queued on the context stream; the context
    // stream is ordered after the copy streams' previous work
    NBK_CUDA(c, cudaEventRecord(c->ev_out, c->xs_out));
    NBK_CUDA(c, cudaEventRecord(c->ev_fused, c->stream));
    NBK_CUDA(c, cudaStreamWaitEvent(c->xs_in, c->ev_fused, 0));
    NBK_CUDA(c, cudaMemcpyAsync(c->stage_f, f_hosts[0], bytes, cudaMemcpyHostToDevice, c->xs_in));
    NBK_CUDA(c, cudaEventRecord(c->ev_in, c->xs_in));
    nbk_status st_all = NBK_OK;
    for (int32_t k = 0; k < nrhs; ++k) {
        // RHS k into the solver's SL vector; then RHS k+1 streams in during solve k
        NBK_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_in, 0));
        NBK_CUDA(c, perm_sl<double>(c, c->f64, c->stage_f, true, c->stream));
        NBK_CUDA(c, cudaEventRecord(c->ev_fused, c->stream));
        c->h0_dirty = 1;
        if (k + 1 < nrhs) {
            NBK_CUDA(c, cudaStreamWaitEvent(c->xs_in, c->ev_fused, 0));
            NBK_CUDA(c, cudaMemcpyAsync(c->stage_f, f_hosts[k + 1], bytes, cudaMemcpyHostToDevice, c->xs_in));
            NBK_CUDA(c, cudaEventRecord(c->ev_in, c->xs_in));
        }
        nbk_status st = nbk_cg_solve(c, niter, prec, hist_hosts ? hist_hosts + (size_t)k * (niter + 1) : nullptr,
                                     nullptr, results ? results + k : nullptr);
        if (st != NBK_OK && st != NBK_EDEFECT) return st;
        if (st == NBK_EDEFECT) st_all = NBK_EDEFECT;
        // solution k out (natural order) while solve k+1 runs; stage_x is free once x_{k-1} left
        if (x_hosts && x_hosts[k]) {
            NBK_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_out, 0));
            NBK_CUDA(c, perm_sl<double>(c, c->stage_x, c->x64, false, c->stream));
            NBK_CUDA(c, cudaEventRecord(c->ev_xready, c->stream));
            NBK_CUDA(c, cudaStreamWaitEvent(c->xs_out, c->ev_xready, 0));
            NBK_CUDA(c, cudaMemcpyAsync(x_hosts[k], c->stage_x, bytes, cudaMemcpyDeviceToHost, c->xs_out));
            NBK_CUDA(c, cudaEventRecord(c->ev_out, c->xs_out));
        }
    }
    NBK_CUDA(c, cudaStreamSynchronize(c->xs_out));
    NBK_CUDA(c, cudaStreamSynchronize(c->xs_in));
    return st_all;
}

nbk_status nbk_get_solution(nbk_ctx* c, double* x_host)
{
    if (!c || !x_host) return fail(c, NBK_EINVAL, "NULL argument");
    if (c->last_solved_precision < 0) return fail(c, NBK_ESTATE, "no solve yet");
    NBK_CUDA(c, perm_sl<double>(c, c->w64, c->x64, false, c->stream));
    NBK_CUDA(c, cudaMemcpyAsync(x_host, c->w64, 8 * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
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
    *launches = (1 + multi) + (2 + 4 * multi + ka_launches(c, multi != 0)) * (int64_t)niter + 1 +
                ((prec == NBK_FP32 || prec == NBK_FP32S || prec == NBK_FP32A) ? 1 : 0) +
                (prec == NBK_FP32A ? (1 + multi) * (int64_t)niter : 0) +   // the binary32 pap kernel (+ fin)
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
    if (c->ev_pack) cudaEventDestroy(c->ev_pack);
    if (c->ev_xchg) cudaEventDestroy(c->ev_xchg);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->xs_in) {
        cudaStreamSynchronize(c->xs_in);
        cudaStreamSynchronize(c->xs_out);
        cudaStreamDestroy(c->xs_in);
        cudaStreamDestroy(c->xs_out);
        for (cudaEvent_t e : {c->ev_in, c->ev_fused, c->ev_xready, c->ev_out})
            if (e) cudaEventDestroy(e);
    }
    if (c->stage_f) cudaFree(c->stage_f);
    if (c->stage_x) cudaFree(c->stage_x);
    if (c->own_stream) {
        cudaStreamSynchronize(c->own_stream);
        cudaStreamDestroy(c->own_stream);
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
