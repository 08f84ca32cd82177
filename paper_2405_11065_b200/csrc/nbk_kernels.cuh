// nbk_kernels.cuh -- the hot-path CUDA kernels of libnbk (sm_100a).
//
//   K_A  k_ax      : fused  p = beta p + r  (add2s1, T1 line 4, z = r)
//                           x = x + alpha_prev p_prev  (add2s2, T1 line 7, deferred
//                               one iteration so p is read once)
//                           w = ax_e(p) = D^T G D p_e  (T1 line 5; F2 ax_e,
//                               local_grad3, local_grad3_t) + Dirichlet mask
//                           pap partial over element-interior points
//                               (glsc3(w,c,p), T1 line 6)
//   K_B  k_dssum   : direct-stiffness summation over sorted segments of unique
//                    shared global nodes (gslib gs_op) + the shared-node
//                    part of pap; the last block forms alpha = rtz1/pap.
//   K_C  k_vec     : r = r - alpha w (add2s2, T1 line 8) + rtr = glsc3(r,c,r)
//                    (T1 line 9); the last block forms h_k, beta_{k+1}.
//                    Same kernel (other modes) for the CG initialisation, the
//                    final FP64 residual check and the standalone glsc3.
//
// Canonical evaluation order (DESIGN.md CEO-1, rules C1-C8) is followed
// operation by operation so that results are bitwise equal to the oracle's.
#pragma once
#include "nbk_common.cuh"

namespace nbk {

// Elements per CTA of k_ax: about 256 threads (N^2 per element).
__host__ __device__ constexpr int ax_epb(int N) { return (256 / (N * N)) > 0 ? 256 / (N * N) : 1; }
// CTA size: N^2 * EPB rounded up to whole warps (the extra lanes idle).
__host__ __device__ constexpr int ax_threads(int N) { return (N * N * ax_epb(N) + 31) / 32 * 32; }

template <typename T>
struct AxArgs {
    const T* D;        // N*N, D[a*N+b] = l_b'(xi_a)
    const T* G;        // E*6*N^3
    const T* u;        // input field (plain mode) or p_{k-1} (fused mode)
    T* w;              // output
    T* p;              // fused: p (in/out)
    const T* r;        // fused: r
    T* x;              // fused: x (in/out)
    const CgState* st; // fused: beta, alpha_prev
    dd* parts;         // fused: pap partial per block
    MeshView mesh;
    int mask;          // assign +0 to Dirichlet points of w
};

// ---------------------------------------------------------------- K_A
// Thread layout: (i, j) of one of EPB elements; the k-loop runs in registers.
// smem: D, D^T and per element u_e, wr, ws (3 N^3 values).
template <typename T, int N, bool FUSED>
__global__ void __launch_bounds__(ax_threads(N))
    k_ax(AxArgs<T> a)
{
    constexpr int N2 = N * N, N3 = N * N * N, EPB = ax_epb(N);
    __shared__ T sD[N2], sDt[N2];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* su = reinterpret_cast<T*>(smem_raw);

    const int tid = threadIdx.x;
    const int el = tid / N2, ij = tid - el * N2;
    const int i = ij % N, j = ij / N;
    const int64_t e = (int64_t)blockIdx.x * EPB + el;
    const bool valid = el < EPB && e < a.mesh.E;
    T* ue = su + el * 3 * N3;
    T* wre = ue + N3;
    T* wse = wre + N3;

    for (int q = tid; q < N2; q += blockDim.x) {
        T d = a.D[q];
        sD[q] = d;
        sDt[(q % N) * N + q / N] = d;
    }

    T betaT = 0, alphaT = 0;
    if constexpr (FUSED) {
        if constexpr (sizeof(T) == 8) {
            betaT = (T)a.st->beta;
            alphaT = (T)a.st->alpha;
        } else {
            betaT = (T)a.st->beta32;
            alphaT = (T)a.st->alpha32;
        }
    }

    // ---- load p (fused: p = fma(beta, p, r), x = fma(alpha_prev, p_prev, x))
    T ureg[N];
    const int64_t base = e * N3 + ij;
    if (valid) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const int64_t L = base + k * N2;
            T v;
            if constexpr (FUSED) {
                T po = a.p[L];
                T rr = a.r[L];
                T xx = a.x[L];
                v = fma_t<T>(betaT, po, rr);         // C8: p = fma(betaT, p, r)
                a.x[L] = fma_t<T>(alphaT, po, xx);   // C8: x = fma(alphaT, p, x)
                a.p[L] = v;
            } else {
                v = a.u[L];
            }
            ureg[k] = v;
            ue[k * N2 + ij] = v;
        }
    }
    __syncthreads();

    // ---- gradient (C1), metric (C2), t-part of the transpose (C3: b chain)
    T b[N];
#pragma unroll
    for (int k = 0; k < N; ++k) b[k] = 0;
    if (valid) {
        const T* Ge = a.G + e * 6 * N3 + ij;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            T ur = 0, us = 0, ut = 0;
#pragma unroll
            for (int l = 0; l < N; ++l) ur = fma_t<T>(sDt[l * N + i], ue[k * N2 + j * N + l], ur);
#pragma unroll
            for (int l = 0; l < N; ++l) us = fma_t<T>(sDt[l * N + j], ue[k * N2 + l * N + i], us);
#pragma unroll
            for (int l = 0; l < N; ++l) ut = fma_t<T>(sD[k * N + l], ureg[l], ut);
            const T g1 = Ge[0 * N3 + k * N2], g2 = Ge[1 * N3 + k * N2], g3 = Ge[2 * N3 + k * N2];
            const T g4 = Ge[3 * N3 + k * N2], g5 = Ge[4 * N3 + k * N2], g6 = Ge[5 * N3 + k * N2];
            T wr = mul_t<T>(g1, ur);
            wr = fma_t<T>(g2, us, wr);
            wr = fma_t<T>(g3, ut, wr);
            T ws = mul_t<T>(g2, ur);
            ws = fma_t<T>(g4, us, ws);
            ws = fma_t<T>(g5, ut, ws);
            T wt = mul_t<T>(g3, ur);
            wt = fma_t<T>(g5, us, wt);
            wt = fma_t<T>(g6, ut, wt);
            wre[k * N2 + ij] = wr;
            wse[k * N2 + ij] = ws;
#pragma unroll
            for (int kk = 0; kk < N; ++kk) b[kk] = fma_t<T>(sD[k * N + kk], wt, b[kk]);
        }
    }
    __syncthreads();

    // ---- r/s part of the transpose (C3: a chain), w = a + b, mask, pap
    acc_t acc;
    if (valid) {
        ElemCoord ec = elem_coord(a.mesh, (uint32_t)e);
#pragma unroll
        for (int k = 0; k < N; ++k) {
            T s = 0;
#pragma unroll
            for (int l = 0; l < N; ++l) s = fma_t<T>(sD[l * N + i], wre[k * N2 + j * N + l], s);
#pragma unroll
            for (int l = 0; l < N; ++l) s = fma_t<T>(sD[l * N + j], wse[k * N2 + l * N + i], s);
            T wv = add_t<T>(s, b[k]);
            if (a.mask && is_masked(a.mesh, ec, i, j, k)) wv = 0;   // C5: assign +0
            a.w[base + k * N2] = wv;
            if constexpr (FUSED) {
                // element-interior points (m == 1) contribute w p c here; shared
                // nodes contribute once per node in K_B (bitwise-equal exact sum).
                if (multiplicity(a.mesh, ec, i, j, k) == 1) acc.add(dot_term(wv, ureg[k], 1.0));
            }
        }
    }
    if constexpr (FUSED) {
        dd v = block_reduce_dd(acc.get());
        if (threadIdx.x == 0) a.parts[blockIdx.x] = v;
    }
}

// ---------------------------------------------------------------- K_B
template <typename T>
struct DssumArgs {
    T* w;
    const T* p;               // fused: p (shared-node pap term)
    const int32_t* seg_off;   // nseg+1 offsets into seg_idx
    const int32_t* seg_idx;   // local indices, ascending within a segment
    int64_t nseg;
    dd* parts;                // fused: partials [0, nA) from K_A, [nA, nA+gridDim) here
    int nA;
    CgState* st;
    double* trace;            // fused: per-iteration trace (niter*5)
    int mask;                 // standalone: assign +0 to masked shared nodes
    MeshView mesh;
};

template <typename T, bool FUSED>
__global__ void __launch_bounds__(256) k_dssum(DssumArgs<T> a)
{
    acc_t acc;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.nseg;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t o0 = a.seg_off[s], o1 = a.seg_off[s + 1];
        const int32_t L0 = a.seg_idx[o0];
        T sum = a.w[L0];                              // C4: s = w[L1]
        for (int32_t q = o0 + 1; q < o1; ++q) sum = add_t<T>(sum, a.w[a.seg_idx[q]]);
        if (!FUSED && a.mask) {
            const int N = a.mesh.N;
            const uint32_t e = (uint32_t)(L0 / (N * N * N));
            const int rem = L0 - (int)e * N * N * N;
            ElemCoord ec = elem_coord(a.mesh, e);
            if (is_masked(a.mesh, ec, rem % N, (rem / N) % N, rem / (N * N))) sum = 0;
        }
        for (int32_t q = o0; q < o1; ++q) a.w[a.seg_idx[q]] = sum;
        if constexpr (FUSED) acc.add(dot_term(sum, a.p[L0], 1.0));  // one term per node
    }
    if constexpr (FUSED) {
        dd v = block_reduce_dd(acc.get());
        const unsigned int total = gridDim.x;
        if (publish_and_check_last(a.parts, a.nA + blockIdx.x, v, &a.st->cnt[0], total)) {
            dd pap_dd = reduce_partials(a.parts, a.nA + (int)gridDim.x);
            if (threadIdx.x == 0) {
                CgState* st = a.st;
                const int k = st->it;
                const double pap = pap_dd.hi;
                const double rtz1 = st->rtr;
                double alpha = 0.0;
                if (!st->zero) alpha = rtz1 / pap;                     // C7
                if (!st->zero && st->defect == 0 && (!(pap > 0.0) || !isfinite(pap)))
                    st->defect = k;                                   // C9
                st->alpha = alpha;
                st->alpham = -alpha;
                st->alpha32 = (float)alpha;
                st->alpham32 = -(float)alpha;
                double* tr = a.trace + 5 * (int64_t)(k - 1);
                tr[0] = rtz1;
                tr[1] = st->beta;
                tr[2] = alpha;
                tr[3] = pap;
                st->cnt[0] = 0;
            }
        }
    }
}

// ---------------------------------------------------------------- K_C
enum VecMode { VEC_INIT = 0, VEC_RUPD = 1, VEC_TRUE = 2, VEC_DOT = 3 };

template <typename T>
struct VecArgs {
    T* r;               // INIT: r out; RUPD: r in/out; TRUE: r_true out (double)
    const T* w;         // RUPD/TRUE
    const double* f;    // INIT: f (double); TRUE: f
    T* x;               // INIT: zeroed
    T* p;               // INIT: zeroed
    const T* a;         // DOT
    const T* b;         // DOT
    int64_t n;
    dd* parts;
    CgState* st;
    double* hist;
    double* trace;
    MeshView mesh;
};

template <typename T, int N, int MODE>
__global__ void __launch_bounds__(256) k_vec(VecArgs<T> a)
{
    constexpr int N2 = N * N, N3 = N * N * N;
    acc_t acc;
    T am = 0;
    if constexpr (MODE == VEC_RUPD) {
        if constexpr (sizeof(T) == 8) am = (T)a.st->alpham; else am = (T)a.st->alpham32;
    }
    uint32_t e_cached = 0xffffffffu;
    ElemCoord ec{0, 0, 0};
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < a.n;
         L += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t e = (uint32_t)(L / N3);
        const int rem = (int)(L - (int64_t)e * N3);
        if (e != e_cached) {
            ec = elem_coord(a.mesh, e);
            e_cached = e;
        }
        const double c = inv_mult(multiplicity(a.mesh, ec, rem % N, (rem / N) % N, rem / N2));
        T v;
        if constexpr (MODE == VEC_INIT) {
            v = (T)a.f[L];                 // C11: f32 = RN32(f64)
            a.r[L] = v;
            a.x[L] = 0;
            a.p[L] = 0;
            acc.add(dot_term(v, v, c));
        } else if constexpr (MODE == VEC_RUPD) {
            v = fma_t<T>(am, a.w[L], a.r[L]);  // C8: r = fma(-alphaT, w, r)
            a.r[L] = v;
            acc.add(dot_term(v, v, c));
        } else if constexpr (MODE == VEC_TRUE) {
            v = fma_t<T>((T)-1, a.w[L], (T)a.f[L]);  // C12: r_true = f - w (one rounding)
            a.r[L] = v;
            acc.add(dot_term(v, v, c));
        } else {
            acc.add(dot_term(a.a[L], a.b[L], c));
        }
    }
    dd v = block_reduce_dd(acc.get());
    if (publish_and_check_last(a.parts, blockIdx.x, v, &a.st->cnt[1], gridDim.x)) {
        dd tot = reduce_partials(a.parts, (int)gridDim.x);
        if (threadIdx.x == 0) {
            CgState* st = a.st;
            const double rtr = tot.hi;
            if constexpr (MODE == VEC_INIT) {
                st->rtr = rtr;
                st->rtz2 = 0.0;
                st->beta = 0.0;
                st->beta32 = 0.0f;
                st->alpha = 0.0;
                st->alpha32 = 0.0f;
                st->alpham = 0.0;
                st->alpham32 = 0.0f;
                st->zero = (rtr == 0.0);
                st->defect = 0;
                st->it = 1;
                a.hist[0] = sqrt(rtr);
            } else if constexpr (MODE == VEC_RUPD) {
                const int k = st->it;
                a.hist[k] = sqrt(rtr);                  // h_k (R13)
                a.trace[5 * (int64_t)(k - 1) + 4] = rtr;
                if (!st->zero && st->defect == 0 && !isfinite(rtr)) st->defect = k;
                const double rtz1_next = rtr, rtz2_next = st->rtr;
                st->rtz2 = rtz2_next;
                st->rtr = rtz1_next;
                if (rtz1_next == 0.0) st->zero = 1;     // C9
                const double beta = st->zero ? 0.0 : rtz1_next / rtz2_next;  // C7
                st->beta = beta;
                st->beta32 = (float)beta;
                st->it = k + 1;
            } else if constexpr (MODE == VEC_TRUE) {
                st->true_rtr = rtr;
            } else {
                st->dot = rtr;
            }
            st->cnt[1] = 0;
        }
    }
}

// x = fma(alphaT, p, x) after the last iteration (deferred C8 x update).
template <typename T>
__global__ void __launch_bounds__(256) k_tail_x(T* x, const T* p, const CgState* st, int64_t n)
{
    T al;
    if constexpr (sizeof(T) == 8) al = (T)st->alpha; else al = (T)st->alpha32;
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n;
         L += (int64_t)gridDim.x * blockDim.x)
        x[L] = fma_t<T>(al, p[L], x[L]);
}

// x64 = (double)x32 (exact, C12) ; G32/D32 = RN32(G64/D64) (C11).
__global__ void __launch_bounds__(256) k_upcast(double* dst, const float* src, int64_t n)
{
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n;
         L += (int64_t)gridDim.x * blockDim.x)
        dst[L] = (double)src[L];
}
__global__ void __launch_bounds__(256) k_downcast(float* dst, const double* src, int64_t n)
{
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n;
         L += (int64_t)gridDim.x * blockDim.x)
        dst[L] = __double2float_rn(src[L]);
}

// Standalone mask (C5) over all local points.
template <typename T>
__global__ void __launch_bounds__(256) k_mask(T* w, MeshView m)
{
    const int N = m.N, N3 = N * N * N;
    const int64_t n = m.E * N3;
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n;
         L += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t e = (uint32_t)(L / N3);
        const int rem = (int)(L - (int64_t)e * N3);
        ElemCoord ec = elem_coord(m, e);
        if (is_masked(m, ec, rem % N, (rem / N) % N, rem / (N * N))) w[L] = 0;
    }
}

}  // namespace nbk
