/*
 * nbk.h -- C ABI of libnbk.so, the B200-native (sm_100a) implementation of the
 * data-parallel hot path of Nekbone studied in arXiv 2405.11065: the
 * unpreconditioned conjugate-gradient solve of the 3-D spectral-element
 * Poisson problem, in FP64 and in the paper's mixed form (FP64 set-up, CG loop
 * "exclusively in single precision", FP64 final residual check).
 *
 * Citations: P:n = PAPER.md line n (T1 = tab:cg-profiling);
 * S:n = SPEC.md line n; R#/C# = readings / canonical-order rules in DESIGN.md.
 *
 * Conventions (all entry points):
 *   - extern "C", plain pointers and sizes; no C++ exceptions cross the ABI.
 *   - Every call returns nbk_status; on failure nbk_last_error(ctx) (or
 *     nbk_last_error(NULL) for calls without a context) holds a message.
 *   - Device pointers ("_dev") are CUDA device addresses in the context's
 *     device; host pointers ("_host") are ordinary host memory.
 *   - Local ("E-vector") storage: element-major, i fastest:
 *       u[e][k][j][i], index L = ((e*N + k)*N + j)*N + i, e = ix + ex*(iy + ey*iz)
 *     e is rank-local (the rank's slab starts at global element e_offset).
 *   - Geometric factors: G[e][c][k][j][i], c = g1..g6 = rr, rs, rt, ss, st, tt (R3).
 *   - Work is enqueued on the context's stream; calls that return host data
 *     synchronise that stream.  A context is not re-entrant; use one per
 *     (process, GPU).
 *   - The CUDA path has no CPU fallback: if the device or kernels are not
 *     available, nbk_cg_setup fails with NBK_ECUDA.
 */
#ifndef NBK_H
#define NBK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NBK_OK = 0,
    NBK_EINVAL = 2,  /* bad argument (S:567 exit code 2: config error)          */
    NBK_EDEFECT = 3, /* pap <= 0 or non-finite scalar during CG (exit 3) */
    NBK_ECUDA = 4,   /* CUDA runtime error (message in nbk_last_error)          */
    NBK_ENCCL = 5,   /* NCCL error                                              */
    NBK_ENOMEM = 6,  /* workspace too small                                     */
    NBK_ESTATE = 7   /* call in the wrong state / order                         */
} nbk_status;

typedef enum {
    NBK_FP64 = 0, /* FP64 CG solver (Nekbone's reference precision)                        */
    NBK_FP32 = 1, /* mixed: FP64 set-up, FP32 CG loop with FP64 inner-product accumulation
                     (north_star; reading R11), FP64 final residual check (C12)          */
    NBK_FP32S = 2, /* exactly rounded binary32 (SURVEY 8(f) NEXT-2 variant, reading R11b):
                     as NBK_FP32 but inner products RN32(sum RN32(a b) c), the best value a
                     binary32 accumulator could return, and the scalars alpha, beta, sqrt
                     in binary32 (cg_solve and glsc3 only; bitwise against the oracle)   */
    NBK_VPREC = 3, /* VPREC emulation (NEXT-4): binary64 CG loop with
                     every operation's result rounded to t mantissa bits (nbk_set_vprec;
                     glsc3 terms vp(a b) c, the sum vp(RN64(sum)); alpha, beta, sqrt);
                     set-up data and the final FP64 check are not rounded (cg_solve only) */
    NBK_FP32A = 4  /* the paper's single-precision solver (NEXT-2, "exclusively in
                     single", P:507 math.f in single, P:510 single-precision MPI; reading
                     R11c): inner products ACCUMULATED in binary32 (terms RN32(RN32(a b) c),
                     a fixed binary32 summation tree per rank, the rank sums added in
                     binary32 in rank order), binary32 scalars; unpreconditioned
                     cg_solve only; agrees with the oracle's sequential binary32 loop to
                     rounding, not bitwise                                               */
} nbk_precision;

/* Box mesh (reading R5): cubic elements of edge h = 1/ex on
 * [0,1] x [0,ey/ex] x [0,ez/ex]; homogeneous Dirichlet on all 6 faces (R6).
 * jitter > 0 moves every interior vertex by jitter*h*(2U-1) per coordinate,
 * U from SplitMix64(seed_geom, 3v+d); the element map is trilinear.
 * RHS (R7): b_g = 2U-1 from SplitMix64(seed_rhs, g) on unmasked global nodes. */
typedef struct {
    int32_t ex, ey, ez; /* GLOBAL element counts, >= 1; ez % nranks == 0          */
    int32_t N;          /* GLL points per direction, N = p + 1, 2 <= N <= 16     */
    double jitter;      /* 0 = undeformed; must lie in [0, 0.25]                 */
    uint64_t seed_geom;
    uint64_t seed_rhs;
} nbk_mesh;

/* Process / device placement.  rank owns element layers
 * iz in [rank*ez/nranks, (rank+1)*ez/nranks) (contiguous z-slabs, R21; SURVEY
 * 8(e)); 1 <= nranks <= 64.  Two ways to run nranks > 1:
 *   - NCCL mode (one process per GPU, "nearest-neighbor communications
 *     ... and Allreduce"): nccl_id points at the 128-byte id rank 0 obtained
 *     from nbk_nccl_unique_id and broadcast to every rank; nbk_cg_setup is then
 *     collective (ncclCommInitRank) and so are nbk_ax_apply (with DSSUM),
 *     nbk_dssum, nbk_glsc3, nbk_cg_solve(_host): each exchanges the slab-face
 *     layers with ncclSend/ncclRecv and all-gathers the per-rank inner-product
 *     partials (combined in rank order, identical on every rank).
 *   - virtual slabs (nccl_id == NULL): P contexts in one process on one device
 *     and stream, linked with nbk_group_link and driven by the nbk_group_*
 *     calls; the same kernels run with faces and partials shared by pointer.
 * Either way results are bitwise independent of nranks. */
typedef struct {
    int32_t rank, nranks; /* this context's slab and the number of slabs            */
    int32_t device;       /* CUDA device ordinal                                    */
    void* stream;         /* cudaStream_t the library enqueues on; NULL = a stream the
                             context creates (blocking, so ordered with the legacy
                             default stream) and destroys in nbk_destroy           */
    const void* nccl_id;  /* NCCL mode: 128-byte ncclUniqueId; NULL otherwise       */
} nbk_dist;

typedef struct {
    int64_t n_local;  /* local points on this rank, e_local * N^3 (Nekbone's n)     */
    int64_t n_global; /* unique global GLL nodes of the whole box (R19 DOF unit)    */
    int64_t e_local;  /* elements on this rank                                      */
    int64_t e_offset; /* global id of this rank's first element                     */
    int64_t n_shared; /* unique shared nodes (multiplicity > 1) in the dssum plan   */
    int64_t n_copies; /* local points belonging to shared nodes                     */
    int32_t N;
    int32_t has_fp32; /* FP32 arrays allocated                                      */
    int64_t face_layer; /* values per exchanged face layer (ex*ey*N^2), 0 if 1 rank   */
    int64_t face_nodes; /* global nodes on this rank's slab-boundary planes           */
} nbk_info;

/* Outcome of a solve. */
typedef struct {
    double true_res;      /* sqrt(glsc3(f - A x, c, f - A x)) evaluated in FP64 (C12) */
    double true_res_rel;  /* true_res / h_0                                           */
    int32_t defect_iter;  /* first iteration with pap <= 0 or a non-finite scalar, 0   */
    int32_t niter;
    float solve_ms;       /* device time of the CG loop (CUDA events)                  */
    float kA_ms;          /* summed device time of the fused ax kernel K_A (if profiling) */
    float kB_ms;          /* ... of the dssum phase K_B (+ face exchange when multi-rank) */
    float kC_ms;          /* ... of the r update K_C (+ all-gather when multi-rank)       */
} nbk_result;

typedef struct nbk_ctx nbk_ctx;

/* Preconditioner of nbk_cg_solve (T1 line 2 "solveM"). */
#define NBK_PRECOND_NONE 0   /* z = r (MGRID off): the north_star path                      */
#define NBK_PRECOND_JACOBI 1 /* z = r * dinv, dinv = 1 / diag(A) assembled, masked entries 1
                                (S:376-384); rtz1 = glsc3(r, c, z) replaces rtr_{k-1}        */

/* Flags of nbk_ax_apply. */
#define NBK_AX_LOCAL 0 /* w = ax_e(u) per element only (T1 line 5, F2 ax_e)             */
#define NBK_AX_DSSUM 1 /* ... followed by direct-stiffness summation (dssum)      */
#define NBK_AX_MASK 2  /* ... and the Dirichlet mask (masked points assigned +0, C5)     */

/* Bytes of device workspace nbk_cg_setup needs for this mesh / precision
 * (precision NBK_FP32 also allocates the FP64 arrays used by set-up and the
 * final FP64 check).  Returns NBK_EINVAL for an invalid mesh. */
nbk_status nbk_workspace_bytes(const nbk_mesh* mesh, nbk_precision precision, const nbk_dist* dist,
                               size_t* bytes_out);

/* Slab partition of the mesh for dist (host only, no device needed): local
 * sizes, element offset, local dssum plan size and face sizes.  has_fp32 = 0. */
nbk_status nbk_partition(const nbk_mesh* mesh, const nbk_dist* dist, nbk_info* info);

/* NCCL mode bootstrap: writes a fresh 128-byte ncclUniqueId to out128 (call on
 * rank 0, broadcast it, pass it in nbk_dist.nccl_id).  NBK_ENCCL if
 * libnccl.so.2 cannot be loaded. */
nbk_status nbk_nccl_unique_id(void* out128);

/* cg_setup(mesh, N, precision) (north_star): FP64 set-up on the device:
 * GLL nodes/weights/D, geometric factors g1..g6, RHS, dssum plan (sorted
 * segments over unique global node ids), FP32 copies if precision == NBK_FP32
 * (C11: RN32 of the FP64 values).  dev_workspace (>= nbk_workspace_bytes,
 * 256-byte aligned) is caller-owned and must outlive the context; the library
 * carves every device buffer from it and never frees it.  On success *out is
 * a new context (free it with nbk_destroy). */
nbk_status nbk_cg_setup(const nbk_mesh* mesh, nbk_precision precision, const nbk_dist* dist,
                        void* dev_workspace, size_t ws_bytes, nbk_ctx** out);

/* Parity path (C10): replace the set-up data with host FP64 arrays (e.g. the
 * oracle's): D (N*N, row a = evaluation node), G (e_local*6*N^3), f
 * (e_local*N^3, local storage).  Any pointer may be NULL (keep current).
 * A new D or G re-derives the FP32 copies and invalidates the library's own
 * Jacobi diagonal (a diagonal loaded with nbk_load_precond is kept only when
 * just f changes).  Synchronous. */
nbk_status nbk_load_arrays(nbk_ctx* ctx, const double* D_host, const double* G_host,
                           const double* f_host);

/* Export the context's FP64 set-up data (for independent-set-up comparison).
 * Any pointer may be NULL.  Synchronous. */
nbk_status nbk_get_arrays(nbk_ctx* ctx, double* D_host, double* G_host, double* f_host);

/* ax_apply (north_star; T1 line 5): w = [mask o][dssum o] ax_e(u) for all local
 * elements, ax_e = D^T G D u_e in the canonical order C1-C3.  u_dev / w_dev:
 * e_local*N^3 values of the stated precision (double or float); u and w must
 * not overlap.  Asynchronous on the context stream. */
nbk_status nbk_ax_apply(nbk_ctx* ctx, const void* u_dev, void* w_dev, int32_t flags,
                        nbk_precision precision);

/* dssum (north_star; P:125 gather-scatter): every copy of every global node
 * gets the sum of all its copies, summed in ascending local index (C4); then,
 * if apply_mask, Dirichlet points are assigned +0 (C5).  In place on f_dev.
 * Asynchronous. */
nbk_status nbk_dssum(nbk_ctx* ctx, void* f_dev, int32_t apply_mask, nbk_precision precision);

/* glsc3 (T1 lines 3, 6, 9): sum_L a_L b_L c_L with c = 1/multiplicity, FP64
 * accumulation (double-double, deterministic tree) and one final rounding (C6).
 * FP64 vectors: terms RN64(a b) c; FP32 vectors: (double)a (double)b c.
 * Writes the result to *out_host; synchronous. */
nbk_status nbk_glsc3(nbk_ctx* ctx, const void* a_dev, const void* b_dev, nbk_precision precision,
                     double* out_host);

/* cg_solve(niter) (north_star): fixed-iteration unpreconditioned CG (T1,
 * solveM = identity so rtz1 = previous rtr), x0 = 0, r0 = f, all scalars on
 * the device, the whole loop replayed as one CUDA graph.  precision selects the
 * FP64 or the mixed FP32 solver (the context must have been set up with
 * NBK_FP32 for the latter).  Outputs (host, caller-allocated, may be NULL):
 *   hist_host  : niter+1 doubles, h_k = sqrt(rtr_k) (R13)
 *   trace_host : niter*5 doubles, per iteration rtz1, beta, alpha, pap, rtr
 *   result     : final FP64 true residual (C12), defect iteration, timings.
 * The solution stays on the device (nbk_get_solution).  Returns NBK_EDEFECT
 * if a defect was flagged (results are still written).  Synchronous.
 * 1 <= niter <= 10000. */
nbk_status nbk_cg_solve(nbk_ctx* ctx, int32_t niter, nbk_precision precision, double* hist_host,
                        double* trace_host, nbk_result* result);

/* End-to-end form of cg_solve for host data: copies f_host (e_local*N^3 FP64,
 * NULL = keep the set-up RHS) to the device, solves, and copies the solution
 * (as FP64, exact for the FP32 solver) to x_host (may be NULL).  A new RHS
 * leaves the operator, its FP32 copy and any Jacobi data untouched.
 * Synchronous. */
nbk_status nbk_cg_solve_host(nbk_ctx* ctx, const double* f_host, int32_t niter,
                             nbk_precision precision, double* x_host, double* hist_host,
                             nbk_result* result);

/* Batched end-to-end form (several right-hand sides of one operator, the
 * paper's repeated solves P:559): solves RHS k = 0..nrhs-1 from f_hosts[k]
 * (e_local*N^3 FP64 each, natural order; pinned host memory lets the copies
 * overlap) and writes solution k to x_hosts[k] (x_hosts or an entry may be
 * NULL).  The host->device copy of RHS k+1 and the device->host copy of
 * solution k-1 run on two library-owned copy streams while solve k runs (PCIe
 * is full duplex), so only the first copy in and the last copy out are
 * exposed.  Every RHS gets its own h0 (as nbk_cg_solve_host); hist_hosts
 * (NULL or nrhs*(niter+1) doubles) and results (NULL or nrhs entries) are per
 * RHS.  Allocates two n-double staging buffers on first use (freed by
 * nbk_destroy).  Same results as nrhs calls of nbk_cg_solve_host.  Returns
 * NBK_EDEFECT if any solve flagged a defect.  Synchronous (returns when
 * solution nrhs-1 is in host memory).  Errors: NBK_EINVAL (NULL ctx / f_hosts /
 * f_hosts[k], nrhs < 1), else as nbk_cg_solve. */
nbk_status nbk_cg_solve_host_batch(nbk_ctx* ctx, int32_t nrhs, const double* const* f_hosts,
                                   int32_t niter, nbk_precision precision,
                                   double* const* x_hosts, double* hist_hosts,
                                   nbk_result* results);

/* Copy the last solution (FP64 view: exact upcast of the FP32 solver's x) to
 * host memory, e_local*N^3 doubles.  Synchronous. */
nbk_status nbk_get_solution(nbk_ctx* ctx, double* x_host);

/* Device pointer of the last solution in its native precision (do not free).
 * The library stores its CG vectors (x, r, p, w, f, dinv) per element in the
 * split layout, not in natural order: slots [0, (N-2)^3) hold the element's
 * interior points (i, j, k in 1..N-2, natural order), slots [(N-2)^3, N^3) its
 * boundary points in natural order (so dssum touches only the compact tail of
 * each element).  Every host transfer (nbk_get_solution, nbk_load_arrays,
 * nbk_cg_solve_host, the precond calls) and every public device call
 * (nbk_ax_apply, nbk_dssum, nbk_glsc3) uses natural order; only this pointer
 * exposes the internal layout. */
nbk_status nbk_solution_ptr(nbk_ctx* ctx, nbk_precision precision, void** x_dev);

/* Precision emulation of the following NBK_VPREC solves (SURVEY 8(f) NEXT-4,
 * P:58-68; unpreconditioned CG on one rank, CG-loop scope; N <= 12
 * for VPREC, N <= 8 for RR / MCA):
 *   NBK_EMU_VPREC: every operation's result rounded to t mantissa bits (t = 52
 *     reproduces the NBK_FP64 solver bit for bit);
 *   NBK_EMU_RR: Monte Carlo random rounding of every result, inexact(x) =
 *     x + 2^(e_x - t) xi, xi ~ U[-1/2, 1/2) (Verificarlo "rr" mode);
 *   NBK_EMU_MCA: inexact() on the operands and on the result ("mca" mode).
 * xi = SplitMix64(seed, 4 key + slot) with key = (iteration, phase, global
 * local index, operation number): one seed = one sample, reproducible and
 * identical to the oracle's.  Each correctly rounded glsc3 counts as one
 * operation.  nbk_set_vprec(ctx, t) = nbk_set_emulation(ctx, VPREC, t, 0).
 * An NBK_VPREC solve with NBK_PRECOND_JACOBI selected returns NBK_EINVAL. */
#define NBK_EMU_VPREC 1
#define NBK_EMU_RR 2
#define NBK_EMU_MCA 3
nbk_status nbk_set_emulation(nbk_ctx* ctx, int32_t mode, int32_t t, uint64_t seed);
nbk_status nbk_set_vprec(nbk_ctx* ctx, int32_t t);

/* Select the preconditioner of the following solves (default NBK_PRECOND_NONE).
 * Jacobi: K_A forms z = RN_T(r * dinv_T) for p = beta p + z, K_C reduces
 * rtz = glsc3(r, c, z) beside rtr (the history stays h_k = sqrt(rtr_k)); the
 * FP32 solver uses dinv32 = RN32(dinv) (C11).  In a virtual group every member
 * must be set alike. */
nbk_status nbk_set_precond(nbk_ctx* ctx, int32_t precond);

/* Jacobi data.  By default the library assembles its own FP64 diagonal (per
 * element closed form, dssum, masked entries 1, inverse) at the first Jacobi
 * solve after set-up / nbk_load_arrays.  nbk_load_precond replaces it with a
 * host array dinv_host (e_local*N^3 doubles, local storage; the parity path,
 * C10); nbk_get_precond copies the current dinv (FP64) to the host.
 * Synchronous. */
nbk_status nbk_load_precond(nbk_ctx* ctx, const double* dinv_host);
nbk_status nbk_get_precond(nbk_ctx* ctx, double* dinv_host);

/* Per-kernel timing inside the solve graph (CUDA events around the fused ax
 * kernel each iteration).  Takes effect at the next graph build. */
nbk_status nbk_set_profiling(nbk_ctx* ctx, int32_t enable);

nbk_status nbk_query(const nbk_ctx* ctx, nbk_info* info);

/* Number of kernel launches one nbk_cg_solve(niter, precision) performs. */
nbk_status nbk_solve_launches(const nbk_ctx* ctx, int32_t niter, nbk_precision precision,
                              int64_t* launches);

/* Virtual slabs (nranks > 1 without NCCL; SURVEY 8(e) "virtual-slab mode on
 * one GPU"): link the P contexts ctxs[r] = rank r of P (same mesh, device,
 * stream and set-up precision) so that their face buffers and reduction
 * partials are shared.  The contexts then accept only the nbk_group_* calls
 * below, which take the P contexts in rank order and per-rank arrays of device
 * pointers (u_devs[r] etc., rank r's local storage).  Semantics equal the
 * single-context calls on the whole mesh.  Destroying one member unlinks the
 * group. */
nbk_status nbk_group_link(nbk_ctx* const* ctxs, int32_t P);
nbk_status nbk_group_ax_apply(nbk_ctx* const* ctxs, int32_t P, const void* const* u_devs,
                              void* const* w_devs, int32_t flags, nbk_precision precision);
nbk_status nbk_group_dssum(nbk_ctx* const* ctxs, int32_t P, void* const* f_devs, int32_t apply_mask,
                           nbk_precision precision);
nbk_status nbk_group_glsc3(nbk_ctx* const* ctxs, int32_t P, const void* const* a_devs,
                           const void* const* b_devs, nbk_precision precision, double* out_host);
/* hist/trace/result as nbk_cg_solve (identical on every rank); each member
 * keeps its slab of the solution (nbk_get_solution per context). */
nbk_status nbk_group_cg_solve(nbk_ctx* const* ctxs, int32_t P, int32_t niter, nbk_precision precision,
                              double* hist_host, double* trace_host, nbk_result* result);

const char* nbk_last_error(const nbk_ctx* ctx);
const char* nbk_version(void);
void nbk_destroy(nbk_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* NBK_H */
