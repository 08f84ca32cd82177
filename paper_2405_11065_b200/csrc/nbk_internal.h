// nbk_internal.h -- host-side context of libnbk (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/nbk.h"
#include "nbk_common.cuh"

#define NBK_MAX_NITER 10000
#define NBK_VEC_GRID_MAX (148 * 8)
#define NBK_MAX_RANKS 64
#define NBK_VPREC_MAXN 12  // VPREC emulation kernels are built for N <= 12
#define NBK_MC_MAXN 8      // RR / MCA emulation kernels (per-operation RNG: large code) for N <= 8

struct nbk_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<cudaEvent_t> prof_events;  // 2 per iteration when profiling
    int64_t launches = 0;
};

struct nbk_ctx {
    nbk_mesh mesh{};
    nbk_dist dist{};
    nbk_precision setup_precision = NBK_FP64;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;  // created when dist->stream is NULL (a blocking stream,
                                        // implicitly ordered with the legacy default stream)
    int N = 0;
    int64_t E = 0, n = 0, n_global = 0, e_offset = 0;
    int64_t nseg = 0, ncopies = 0;
    nbk::MeshView view{};
    std::string err;

    // device buffers (carved from the caller's workspace)
    nbk::CgState* st = nullptr;
    double *D64 = nullptr, *G64 = nullptr, *f64 = nullptr;
    double *x64 = nullptr, *r64 = nullptr, *p64 = nullptr, *w64 = nullptr;
    float *D32 = nullptr, *G32 = nullptr;
    double Dh64[256] = {};                // host copies of D (kernel parameter of k_ax2)
    float Dh32[256] = {};
    float *x32 = nullptr, *r32 = nullptr, *p32 = nullptr, *w32 = nullptr;
    double* dinv64 = nullptr;             // Jacobi: 1 / assembled diag(A) (masked: 1)
    float* dinv32 = nullptr;              // RN32(dinv64) (C11)
    int precond = NBK_PRECOND_NONE;
    int vp_t = 23;                        // emulation: virtual precision t (NBK_VPREC solves)
    int pm_mode = 1;                      // NBK_EMU_VPREC / NBK_EMU_RR / NBK_EMU_MCA
    unsigned long long pm_seed = 0;       // RR / MCA sample
    int dinv_dirty = 1;                   // own diagonal to be (re)assembled
    double *hist = nullptr, *trace = nullptr;
    nbk::dd* parts = nullptr;
    int64_t nparts = 0;
    int32_t *seg_off = nullptr, *seg_idx = nullptr;
    int32_t *grp = nullptr;                               // group index storage
    int32_t *g2 = nullptr, *g4 = nullptr, *g8 = nullptr;  // segments grouped by multiplicity
    int64_t n2 = 0, n4 = 0, n8 = 0, nother = 0;
    int32_t* toff = nullptr;              // dssum tiles: (ntiles + 1) x 3 offsets
    int64_t ntiles = 0, tile_elems = 1;
    int64_t tile_smem = 0;                // max index bytes of a tile (K_B smem per buffer)
    unsigned char* scratch = nullptr;  // set-up scratch (aliases the vector region)
    size_t scratch_bytes = 0;

    // multi-rank z-slabs; nranks == 1: none of this is used
    int rank = 0, nranks = 1;
    int has_lo = 0, has_hi = 0;        // neighbour slab below / above
    int64_t nlayer = 0, nplane = 0;    // face layer values ex*ey*N^2, plane nodes Gx*Gy
    void *send_lo = nullptr, *send_hi = nullptr, *recv_lo = nullptr, *recv_hi = nullptr;
    nbk::dd* gather = nullptr;         // P per-rank partials (group-shared in virtual mode)
    nbk::dd* gather_own = nullptr;
    void* comm = nullptr;              // ncclComm_t (NCCL mode)
    cudaStream_t comm_stream = nullptr;  // face exchange, overlapped with the local dssum
    cudaEvent_t ev_pack = nullptr, ev_xchg = nullptr;  // fork / join of comm_stream
    std::vector<nbk_ctx*> group;       // virtual slabs: all P contexts of the process
    int h0_dirty = 0;

    double h0_64 = 0.0;  // sqrt(glsc3(f64, c, f64)) (C12 denominator)
    int profiling = 0;
    std::map<std::tuple<int, int, int>, nbk_graph> graphs;  // (precision, niter, profiling)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int last_solved_precision = -1;
    // nbk_cg_solve_host_batch: library-owned staging buffers (natural order, n doubles each,
    // allocated on first use) and the two copy streams (H2D, D2H run concurrently)
    double *stage_f = nullptr, *stage_x = nullptr;
    cudaStream_t xs_in = nullptr, xs_out = nullptr;
    cudaEvent_t ev_in = nullptr, ev_fused = nullptr, ev_xready = nullptr, ev_out = nullptr;
};

namespace nbk {

struct Layout {
    size_t off_state, off_D64, off_D32, off_hist, off_trace, off_parts, off_segoff, off_segidx, off_grp,
        off_face, off_gather, off_toff, off_dinv64, off_dinv32, off_G64, off_f64, off_vec64, off_G32, off_vec32, total;
    int64_t nlayer, nplane;
    int has_lo, has_hi;
    int64_t E, n, n_global, nseg, ncopies, nparts, e_offset;
    size_t scratch_need;
};

// Host helpers implemented in nbk_setup.cu
bool validate_mesh(const nbk_mesh* m, const nbk_dist* d, std::string& why);
Layout compute_layout(const nbk_mesh* m, nbk_precision prec, const nbk_dist* d);
MeshView make_view(const nbk_mesh* m, const nbk_dist* d);
void gll_host(int N, double* xi, double* rho, double* D);
cudaError_t setup_device(nbk_ctx* ctx, const Layout& L);
cudaError_t build_plan(nbk_ctx* ctx);
cudaError_t local_diag(nbk_ctx* ctx, double* d);        // per-element diag(A_e), FP64
cudaError_t finish_dinv(nbk_ctx* ctx, double* d);       // mask -> 1, invert, RN32 copy

}  // namespace nbk
