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

// Load N consecutive values of shared memory into registers with the widest
// vector loads the row alignment allows (rows are N*sizeof(T) bytes, and every
// row start used below is a multiple of that).
template <typename T, int N>
__device__ __forceinline__ void lds_row(T (&dst)[N], const T* src)
{
    constexpr int RB = N * (int)sizeof(T);
    if constexpr (RB % 16 == 0) {
#pragma unroll
        for (int q = 0; q < RB / 16; ++q) {
            if constexpr (sizeof(T) == 4) {
                const float4 v = reinterpret_cast<const float4*>(src)[q];
                dst[4 * q] = v.x;
                dst[4 * q + 1] = v.y;
                dst[4 * q + 2] = v.z;
                dst[4 * q + 3] = v.w;
            } else {
                const double2 d = reinterpret_cast<const double2*>(src)[q];
                dst[2 * q] = d.x;
                dst[2 * q + 1] = d.y;
            }
        }
    } else if constexpr (RB % 8 == 0 && sizeof(T) == 4) {
#pragma unroll
        for (int q = 0; q < N / 2; ++q) {
            const float2 v = reinterpret_cast<const float2*>(src)[q];
            dst[2 * q] = v.x;
            dst[2 * q + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int q = 0; q < N; ++q) dst[q] = src[q];
    }
}

// b[kk] = fma(d[kk], t, b[kk]) for kk = 0..N-1 (packed FFMA2 for FP32: per-lane
// numerics identical to __fmaf_rn, so the canonical order is unchanged).
// PM != PM_NONE: b[q] is the t-chain of the point at key kbase + q kstride.
template <typename T, int N, int PM = PM_NONE>
__device__ __forceinline__ void fma_row(T (&b)[N], const T (&d)[N], T t, const PmArgs* P = nullptr,
                                        unsigned long long kbase = 0, unsigned long long kstride = 0)
{
    if constexpr (PM != PM_NONE) {
#pragma unroll
        for (int q = 0; q < N; ++q) b[q] = pfma<PM>(d[q], t, b[q], *P, kbase + q * kstride);
    } else if constexpr (sizeof(T) == 4 && N % 2 == 0) {
        const float2 tt = make_float2(t, t);
#pragma unroll
        for (int q = 0; q < N / 2; ++q) {
            float2 r = __ffma2_rn(make_float2(d[2 * q], d[2 * q + 1]), tt,
                                  make_float2(b[2 * q], b[2 * q + 1]));
            b[2 * q] = r.x;
            b[2 * q + 1] = r.y;
        }
    } else {
#pragma unroll
        for (int q = 0; q < N; ++q) b[q] = fma_t<T>(d[q], t, b[q]);
    }
}

// Emulation keys (NEXT-4) name the operation by the local index L of the point
// it produces (every FP operation perturbed on its own), so under RR /
// MCA the copies of a shared node get independent perturbations and p, x, r are
// not continuous: the shared-node pap is then summed over all copies (K_B).
__device__ __forceinline__ long long global_local_index(const MeshView& m, int64_t L)
{
    return (long long)m.z0 * m.ex * m.ey * m.N * m.N * m.N + L;
}

// glsc3 term: VPREC rounds the product, vp(a b) c (NEXT-4); RR / MCA treat the
// whole correctly rounded glsc3 as one operation (its result is perturbed).
template <int PM, typename T>
__device__ __forceinline__ double dot_term_pm(T a, T b, double c, bool single, const PmArgs& P)
{
    if constexpr (PM == PM_VPREC) return __dmul_rn(vprec_round(mul_t<T>(a, b), P.t), c);
    else return dot_term(a, b, c, single);
}

// ------------------------------------------------------------ K_A config
// Per CTA: EPB elements, one thread per (i, j) of each element (k-loop in
// registers).  STAGE_G: the CTA's G block (EPB*6*N^3 values) and its p/u block
// (EPB*N^3) are staged in shared memory by TMA 1-D bulk copies (even N: 16-byte
// granularity) or a cooperative copy (odd N); wr/ws are written into the G
// slots of g1/g2 once consumed, so smem = 7*EPB*N^3 values.  Without STAGE_G
// (only N=16 FP64, > 227 KB) G is read from global memory per k-slice.
template <typename T>
#ifndef NBK_EPB8_F32
#define NBK_EPB8_F32 2
#endif
#ifndef NBK_EPB8_F64
#define NBK_EPB8_F64 1
#endif
#ifndef NBK_EPB10_F32
#define NBK_EPB10_F32 2
#endif
#ifndef NBK_AX_KP32
#define NBK_AX_KP32 1   // planes per step of K_A's transpose pass (interleaved chains), FP32
#endif
#ifndef NBK_AX_KP64
#define NBK_AX_KP64 2   // ... FP64
#endif
#ifndef NBK_DREG_BYTES
#define NBK_DREG_BYTES 48   // D rows / columns of K_A kept in registers up to this row size
#endif
#ifndef NBK_AX_G1P64
#define NBK_AX_G1P64 1  // planes per step of K_A's gradient pass, FP64
#endif
#ifndef NBK_AX_G1P32
#define NBK_AX_G1P32 1  // ... FP32
#endif
__host__ __device__ constexpr int ax_epb(int N)
{
    if (N == 8) return sizeof(T) == 4 ? NBK_EPB8_F32 : NBK_EPB8_F64;
    if (N == 10) return sizeof(T) == 4 ? NBK_EPB10_F32 : 1;
    if (N == 12) return 1;
    int by_thr = 256 / (N * N) > 0 ? 256 / (N * N) : 1;
    int by_smem = (int)(57344 / (7 * N * N * N * (int)sizeof(T)));
    if (by_smem < 1) by_smem = 1;
    return by_thr < by_smem ? by_thr : by_smem;
}
template <typename T>
__host__ __device__ constexpr bool ax_stage_g(int N)
{
    return 7 * N * N * N * (int)sizeof(T) * ax_epb<T>(N) <= 200 * 1024;
}
// CTA size: N^2 * EPB rounded up to whole warps (the extra lanes idle).
template <typename T>
__host__ __device__ constexpr int ax_threads(int N)
{
    return (N * N * ax_epb<T>(N) + 31) / 32 * 32;
}
template <typename T>
__host__ __device__ constexpr int ax_blocks_by_smem(int N, int slabs)
{
    return (232448 - 1024) / (slabs * ax_epb<T>(N) * N * N * N * (int)sizeof(T) + 1024 +
                              2 * N * N * (int)sizeof(T) + 64);
}
// TMA I/O of the fused CG step (TIO): r and x are bulk-loaded like p and G, and
// p, x, w leave through bulk stores from shared memory -- no per-thread global
// access to the split-layout vectors (their scattered column addresses cost
// address arithmetic and L1 sectors).  Two more N^3 blocks per element: used
// where they do not lower the CTAs per SM (N = 10), and for FP32 at N >= 10
// while >= 3 CTAs fit (N = 12: 4 -> 3 CTAs, still faster).  Measured same-box
// (DESIGN.md section 8): C5 FP32 K_A 2.74 vs 3.04 ms, FP64 5.54 vs 5.82; C3 FP32
// 0.64 vs 0.67; N = 8 (7 -> 6 CTAs) and N = 12 FP64 (2 -> 1) slower.
// NBK_TIO_ALL / NBK_TIO_NONE force it on / off.
template <typename T>
__host__ __device__ constexpr bool ax_tio(int N, int fused)
{
    if (fused != 1 || N % 2 != 0 || 7 * N * N * N * (int)sizeof(T) * ax_epb<T>(N) > 200 * 1024) return false;
#if defined(NBK_TIO_ALL)
    return 9 * N * N * N * (int)sizeof(T) * ax_epb<T>(N) <= 200 * 1024;
#elif defined(NBK_TIO_NONE)
    return false;
#else
    return ax_blocks_by_smem<T>(N, 9) == ax_blocks_by_smem<T>(N, 7) ||
           (sizeof(T) == 4 && N >= 10 && ax_blocks_by_smem<T>(N, 9) >= 3);
#endif
}
template <typename T>
__host__ __device__ constexpr int ax_smem_bytes(int N, int fused = 0)
{
    return (ax_stage_g<T>(N) ? (ax_tio<T>(N, fused) ? 9 : 7) : 3) * ax_epb<T>(N) * N * N * N * (int)sizeof(T);
}
template <typename T>
__host__ __device__ constexpr int ax_min_blocks(int N, int fused = 0)
{
    int by_smem = (232448 - 1024) / (ax_smem_bytes<T>(N, fused) + 1024 + 2 * N * N * (int)sizeof(T) + 64);
    int by_thr = 2048 / ax_threads<T>(N);
    int m = by_smem < by_thr ? by_smem : by_thr;
    return m < 1 ? 1 : m;
}

template <typename T>
struct AxArgs {
    const T* D;        // N*N, D[a*N+b] = l_b'(xi_a)
    const T* Dh;       // host copy of D (the launchers pass it to k_ax as a DConst parameter)
    const T* G;        // E*6*N^3
    const T* u;        // input field (plain mode)
    T* w;              // output
    T* p;              // fused: p (in/out)
    const T* r;        // fused: r
    T* x;              // fused: x (in/out)
    const CgState* st; // fused: beta, alpha_prev
    const T* dinv;     // fused Jacobi PCG: z = r * dinv replaces r in the p update
    int single;        // paper-literal single mode: pap terms RN32(w p) (NEXT-2)
    PmArgs pm;         // precision emulation (NEXT-4; kernels instantiated with PM)
    int it;            // CG iteration (emulation keys)
    dd* parts;         // fused: pap partial per block
    MeshView mesh;
    int mask;          // assign +0 to Dirichlet points of w
    int rev;           // sweep the element tiles in reverse order (L2 reuse, see k_vec)
    int p_ready;       // fused: p is final before the PDL wait (CG iterations >= 2)
    int in_sl, out_sl; // plain ax: u / w in the split layout (SL) instead of natural order
                       // (the fused CG step always works on SL vectors)
    // element ranges of this launch: blocks cover [eb0, eb0 + en0) then
    // [eb1, eb1 + en1) (multi-rank: the slab-boundary layers first, so the face
    // exchange overlaps the interior elements); pap partials at part_off + block
    int64_t eb0, en0, eb1, en1;
    int part_off;
};

// D as a kernel parameter: k_ax reads D[k][*] (t-derivative, t-transpose) with
// compile-time indices, i.e. as constant-bank operands of the FMAs, not from
// shared memory.
template <typename T>
struct DConst {
    T v[256];  // D[a*N+b], N <= 16
};

// ---------------------------------------------------------------- K_A
// FUSED: 0 = plain ax (u -> w); 1 = CG step (p = beta p + r); 2 = Jacobi PCG
// step (p = beta p + z, z = RN(r * dinv) formed here: S:376-384, T1 line 2).
template <typename T, int N, int FUSED, int PM = PM_NONE>
__global__ void __launch_bounds__(ax_threads<T>(N), ax_min_blocks<T>(N, FUSED))
    k_ax(AxArgs<T> a, const __grid_constant__ DConst<T> dc)
{
    // PM: every operation goes through the emulation (NEXT-4); op numbers per point:
    // 0 p, 1 x (these two keyed by the global node), 2.. ur, 2+N.. us, 2+2N.. ut,
    // 2+3N.. metric (9), 11+3N.. r/s transpose (2N), 11+5N.. t transpose (N), 11+6N add
    const PmArgs& P = a.pm;
    constexpr int N2 = N * N, N3 = N * N * N, EPB = ax_epb<T>(N);
    constexpr bool STAGE = ax_stage_g<T>(N);
    constexpr bool TMA = STAGE && (N % 2 == 0);
    constexpr bool TIO = ax_tio<T>(N, FUSED);
    __shared__ __align__(16) T sD[N2];
    __shared__ __align__(16) T sDt[N2];
    __shared__ __align__(8) uint64_t bar[3];   // TMA: p / u (+ x) block, G block, (TIO) r block
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* sG = reinterpret_cast<T*>(smem_raw);                  // STAGE: EPB*6*N3
    T* sU = STAGE ? sG + EPB * 6 * N3 : sG;                  // EPB*N3
    T* sW = sU + EPB * N3;                                   // !STAGE: wr, ws (2*EPB*N3)
    T* sR = sU + EPB * N3;                                   // TIO: r (SL), then u in natural order
    T* sX = sR + EPB * N3;                                   // TIO: x (SL)

    const int tid = threadIdx.x;
    const int el = tid / N2, ij = tid - el * N2;
    const int i = ij % N, j = ij / N;
    const int64_t bl = (int64_t)(a.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
    const int64_t nb0 = (a.en0 + EPB - 1) / EPB;
    const int64_t e0 = bl < nb0 ? a.eb0 + bl * EPB : a.eb1 + (bl - nb0) * EPB;
    const int64_t eend = bl < nb0 ? a.eb0 + a.en0 : a.eb1 + a.en1;
    const int64_t e = e0 + el;
    const int nel = (int)((eend - e0) < EPB ? (eend - e0) : EPB);
    const bool valid = el < nel;
    const T* src_u = FUSED ? a.p : a.u;
    NBK_ASSERT(nel >= 1 && e0 + nel <= a.mesh.E);

    T rreg[FUSED ? N : 1], xreg[FUSED ? N : 1], dreg[FUSED == 2 ? N : 1];
    // ---- stage G and u/p of the CTA's elements in shared memory.  G does not
    // depend on the previous kernel: its bulk copy is issued before the PDL
    // wait and overlaps the previous kernel's tail.
    if constexpr (TMA) {
        // p / u and G on their own barriers: the p update runs while G is in
        // flight.  p (CG step) is final before this kernel starts from
        // iteration 2 on (written by the previous K_A, which completed before
        // K_B and K_C ran), so it is issued first and before the PDL wait when
        // a.p_ready.
        if (tid == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            if (TIO) mbar_init(&bar[2], 1);
            const uint32_t ubytes = (uint32_t)(nel * N3 * sizeof(T));
            const uint32_t gbytes = (uint32_t)(nel * 6 * N3 * sizeof(T));
            // p (and, TIO, x: both written by the previous K_A) on bar[0]
            if (FUSED && a.p_ready) {
                mbar_arrive_expect_tx(&bar[0], TIO ? 2 * ubytes : ubytes);
                tma_load_1d(sU, src_u + e0 * N3, ubytes, &bar[0]);
                if (TIO) tma_load_1d(sX, a.x + e0 * N3, ubytes, &bar[0]);
            }
            mbar_arrive_expect_tx(&bar[1], gbytes);
            tma_load_1d(sG, a.G + e0 * 6 * N3, gbytes, &bar[1]);
            pdl_wait();
            if (!(FUSED && a.p_ready)) {
                mbar_arrive_expect_tx(&bar[0], TIO ? 2 * ubytes : ubytes);
                tma_load_1d(sU, src_u + e0 * N3, ubytes, &bar[0]);
                if (TIO) tma_load_1d(sX, a.x + e0 * N3, ubytes, &bar[0]);
            }
            if (TIO) {  // r: written by the previous K_C (after the PDL wait)
                mbar_arrive_expect_tx(&bar[2], ubytes);
                tma_load_1d(sR, a.r + e0 * N3, ubytes, &bar[2]);
            }
        }
        if constexpr (FUSED && !TIO) {  // x and dinv are final too (x: previous K_A)
            if (valid && a.p_ready) {
                const SlCol cs = sl_col(N, i, j);
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    xreg[k] = a.x[e * N3 + cs.at(N, k)];
                    if constexpr (FUSED == 2) dreg[k] = __ldg(a.dinv + e * N3 + cs.at(N, k));
                }
            }
        }
        pdl_wait();
    } else if constexpr (STAGE) {
        pdl_wait();
        for (int q = tid; q < nel * 6 * N3; q += blockDim.x) sG[q] = a.G[e0 * 6 * N3 + q];
        for (int q = tid; q < nel * N3; q += blockDim.x) sU[q] = src_u[e0 * N3 + q];
    } else {
        pdl_wait();
        for (int q = tid; q < nel * N3; q += blockDim.x) sU[q] = src_u[e0 * N3 + q];
    }
    for (int q = tid; q < N2; q += blockDim.x) {
        T d = a.D[q];
        sD[q] = d;
        sDt[(q % N) * N + q / N] = d;
    }

    const int64_t base = e * N3 + ij;   // natural index of (i, j, 0)
    const long long goff = (long long)a.mesh.z0 * a.mesh.ex * a.mesh.ey * N3;  // global local index
    auto key = [&](int kk, int o) { return pm_key(a.it, PH_A, goff + base + (long long)kk * N2, o); };
    (void)key;
    // storage of the thread's column (i, j, *): SL slots (CG vectors) or natural
    const SlCol cs = sl_col(N, i, j);
    const bool isl = FUSED || a.in_sl, osl = FUSED || a.out_sl;
    NBK_ASSERT(!valid || (cs.at(N, 0) >= 0 && cs.at(N, N - 1) < N3 && cs.at(N, N / 2) < N3));
    auto gin = [&](int kk) -> int64_t { return isl ? e * N3 + cs.at(N, kk) : base + (int64_t)kk * N2; };
    auto gout = [&](int kk) -> int64_t { return osl ? e * N3 + cs.at(N, kk) : base + (int64_t)kk * N2; };
    T betaT = 0, alphaT = 0;
    if constexpr (FUSED) {
        if constexpr (sizeof(T) == 8) {
            betaT = (T)a.st->beta;
            alphaT = (T)a.st->alpha;
        } else {
            betaT = (T)a.st->beta32;
            alphaT = (T)a.st->alpha32;
        }
        if (valid && !TIO) {  // issued before the TMA wait: overlaps with the bulk copies
            const bool early = TMA && a.p_ready;
#pragma unroll
            for (int k = 0; k < N; ++k) {
                rreg[k] = a.r[gin(k)];
                if (!early) {
                    xreg[k] = a.x[gin(k)];
                    if constexpr (FUSED == 2) dreg[k] = __ldg(a.dinv + gin(k));
                }
            }
        }
    }
    __syncthreads();  // barrier init, sD, cooperative copies visible
    if constexpr (TMA) mbar_wait(&bar[0], 0);

    T* ue = sU + el * N3;
    T* wre = STAGE ? sG + el * 6 * N3 : sW + el * N3;            // aliases g1 (STAGE)
    T* wse = STAGE ? sG + el * 6 * N3 + N3 : sW + (EPB + el) * N3;  // aliases g2

    // ---- p = fma(beta, p, r), x = fma(alpha_prev, p_prev, x)  (C8, fused)
    // The staged block is in the storage order of the source: SL (CG vectors)
    // is read per column and re-stored in natural order for the derivatives.
    T ureg[N];
    T* un = ue;   // natural-order u of the element for the derivatives
    if constexpr (TIO) {
        // p, x, r blocks (SL) in shared memory: p and x updated in place and
        // bulk-stored; the natural u goes into the (consumed) r block.
        mbar_wait(&bar[2], 0);
        T* re = sR + el * N3;
        T* xe = sX + el * N3;
        if (valid) {
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const int sk = cs.at(N, k);
                const T po = ue[sk];
                const long long gk = goff + base + (long long)k * N2;  // emulation key: natural local index
                const T v = pfma<PM>(betaT, po, re[sk], P, pm_key(a.it, PH_A, gk, 0));
                xe[sk] = pfma<PM>(alphaT, po, xe[sk], P, pm_key(a.it, PH_A, gk, 1));
                ue[sk] = v;
                ureg[k] = v;
            }
        }
        __syncthreads();  // every r value of the block has been read
        if (valid) {
#pragma unroll
            for (int k = 0; k < N; ++k) re[k * N2 + ij] = ureg[k];
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            const uint32_t ubytes = (uint32_t)(nel * N3 * sizeof(T));
            tma_store_1d(a.p + e0 * N3, sU, ubytes);
            tma_store_1d(a.x + e0 * N3, sX, ubytes);
            bulk_commit();
        }
        un = re;
    } else if (valid) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            T v = ue[isl ? cs.at(N, k) : k * N2 + ij];
            if constexpr (FUSED) {
                const T po = v;
                T zk = rreg[k];
                if constexpr (FUSED == 2) zk = mul_t<T>(rreg[k], dreg[k]);  // solveM (Jacobi)
                const long long gk = goff + base + (long long)k * N2;  // emulation key: natural local index
                v = pfma<PM>(betaT, po, zk, P, pm_key(a.it, PH_A, gk, 0));
                a.x[gin(k)] = pfma<PM>(alphaT, po, xreg[k], P, pm_key(a.it, PH_A, gk, 1));
                a.p[gin(k)] = v;
            }
            ureg[k] = v;
        }
    }
    if (isl && !TIO) {
        __syncthreads();  // every SL value of the block has been read
        if (valid) {
#pragma unroll
            for (int k = 0; k < N; ++k) ue[k * N2 + ij] = ureg[k];
        }
        __syncthreads();
    }

    // D rows / columns of this thread: D[i][l], D[j][l] (gradient) and
    // D[l][i], D[l][j] (transpose), in registers when they fit.
    constexpr bool DREG = N * (int)sizeof(T) <= NBK_DREG_BYTES;

    // ---- gradient (C1), metric (C2), t-part of the transpose (C3: b chain)
    T b[N];
#pragma unroll
    for (int k = 0; k < N; ++k) b[k] = 0;
    if (valid) {
        const T* Ge = STAGE ? sG + el * 6 * N3 + ij : a.G + e * 6 * N3 + ij;
        T Dri[N], Drj[N];
        if constexpr (DREG) {
            lds_row<T, N>(Dri, sD + i * N);
            lds_row<T, N>(Drj, sD + j * N);
        }
        // G1P planes per step (their ur / us / ut chains interleaved; the b update
        // of plane k precedes that of plane k + 1, so every chain keeps its order)
        constexpr int GW = sizeof(T) == 8 ? NBK_AX_G1P64 : NBK_AX_G1P32;
        constexpr int G1P = (N % GW == 0 && PM == PM_NONE) ? GW : 1;
#pragma unroll
        for (int k0 = 0; k0 < N; k0 += G1P) {
            if constexpr (TMA) {
                if (k0 == 0) mbar_wait(&bar[1], 0);
            }
            if constexpr (!DREG) {
                lds_row<T, N>(Dri, sD + i * N);
                lds_row<T, N>(Drj, sD + j * N);
            }
            T wtq[G1P];
#pragma unroll
            for (int q = 0; q < G1P; ++q) {
                const int k = k0 + q;
                T urow[N], Dk[N];
                lds_row<T, N>(urow, un + k * N2 + j * N);   // u[k][j][:]
#ifdef NBK_D_SMEM
                lds_row<T, N>(Dk, sD + k * N);   // D[k][:] (broadcast)
#else
#pragma unroll
                for (int l = 0; l < N; ++l) Dk[l] = dc.v[k * N + l];   // D[k][:] (kernel parameter)
#endif
                T ur = 0, us = 0, ut = 0;
#pragma unroll
                for (int l = 0; l < N; ++l) ur = pfma<PM>(Dri[l], urow[l], ur, P, key(k, 2 + l));
#pragma unroll
                for (int l = 0; l < N; ++l) us = pfma<PM>(Drj[l], un[k * N2 + l * N + i], us, P, key(k, 2 + N + l));
#pragma unroll
                for (int l = 0; l < N; ++l) ut = pfma<PM>(Dk[l], ureg[l], ut, P, key(k, 2 + 2 * N + l));
                const T g1 = Ge[0 * N3 + k * N2], g2 = Ge[1 * N3 + k * N2], g3 = Ge[2 * N3 + k * N2];
                const T g4 = Ge[3 * N3 + k * N2], g5 = Ge[4 * N3 + k * N2], g6 = Ge[5 * N3 + k * N2];
                const int om = 2 + 3 * N;
                T wr = pmul<PM>(g1, ur, P, key(k, om));
                wr = pfma<PM>(g2, us, wr, P, key(k, om + 1));
                wr = pfma<PM>(g3, ut, wr, P, key(k, om + 2));
                T ws = pmul<PM>(g2, ur, P, key(k, om + 3));
                ws = pfma<PM>(g4, us, ws, P, key(k, om + 4));
                ws = pfma<PM>(g5, ut, ws, P, key(k, om + 5));
                T wt = pmul<PM>(g3, ur, P, key(k, om + 6));
                wt = pfma<PM>(g5, us, wt, P, key(k, om + 7));
                wt = pfma<PM>(g6, ut, wt, P, key(k, om + 8));
                // own (i,j,k) slot of g1/g2 is dead after the reads above
                wre[k * N2 + ij] = wr;
                wse[k * N2 + ij] = ws;
                wtq[q] = wt;
            }
#pragma unroll
            for (int q = 0; q < G1P; ++q) {
                const int k = k0 + q;
                T Dk[N];
#ifdef NBK_D_SMEM
                lds_row<T, N>(Dk, sD + k * N);
#else
#pragma unroll
                for (int l = 0; l < N; ++l) Dk[l] = dc.v[k * N + l];
#endif
                // b[kk] = fma(D[k][kk], wt, b[kk]): op 11+5N+k of point (i, j, kk)
                fma_row<T, N, PM>(b, Dk, wtq[q], &P, key(0, 11 + 5 * N + k), key(1, 0) - key(0, 0));
            }
        }
    }
    __syncthreads();

    // ---- r/s part of the transpose (C3: a chain), w = a + b, mask, pap
    acc_t acc;
    if (valid) {
        const ElemCoord ec = elem_coord(a.mesh, (uint32_t)e);
        const int n1 = N - 1;
        const bool mxy = (i == 0 && ec.ax == 0) || (i == n1 && ec.ax == a.mesh.ex - 1) ||
                         (j == 0 && ec.ay == 0) || (j == n1 && ec.ay == a.mesh.ey - 1);
        const bool sxy = (i == 0 && ec.ax > 0) || (i == n1 && ec.ax < a.mesh.ex - 1) ||
                         (j == 0 && ec.ay > 0) || (j == n1 && ec.ay < a.mesh.ey - 1);
        const bool mz0 = ec.azg == 0, mz1 = ec.azg == a.mesh.ezg - 1;
        T Dci[N], Dcj[N];
        if constexpr (DREG) {
            lds_row<T, N>(Dci, sDt + i * N);   // D[:][i]
            lds_row<T, N>(Dcj, sDt + j * N);   // D[:][j]
        }
        // KP planes per step: their chains are independent and interleaved
        // (each point's chain keeps its canonical order)
        // (FP64: 2 planes -- C5 FP64 K_A 5.32 vs 5.61 ms same-box; FP32: no gain, 1)
        constexpr int KPW = sizeof(T) == 8 ? NBK_AX_KP64 : NBK_AX_KP32;
        constexpr int KP = (N % KPW == 0 && PM == PM_NONE) ? KPW : 1;
#pragma unroll
        for (int k0 = 0; k0 < N; k0 += KP) {
            if constexpr (!DREG) {
                lds_row<T, N>(Dci, sDt + i * N);
                lds_row<T, N>(Dcj, sDt + j * N);
            }
            T wrow[KP][N], s[KP];
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                lds_row<T, N>(wrow[q], wre + (k0 + q) * N2 + j * N);  // wr[k][j][:]
                s[q] = 0;
            }
#pragma unroll
            for (int l = 0; l < N; ++l)
#pragma unroll
                for (int q = 0; q < KP; ++q) s[q] = pfma<PM>(Dci[l], wrow[q][l], s[q], P, key(k0 + q, 11 + 3 * N + l));
#pragma unroll
            for (int l = 0; l < N; ++l)
#pragma unroll
                for (int q = 0; q < KP; ++q)
                    s[q] = pfma<PM>(Dcj[l], wse[(k0 + q) * N2 + l * N + i], s[q], P, key(k0 + q, 11 + 4 * N + l));
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                const int k = k0 + q;
                T wv = padd<PM>(s[q], b[k], P, key(k, 11 + 6 * N));
                const bool masked = mxy || (k == 0 && mz0) || (k == n1 && mz1);
                if (a.mask && masked) wv = 0;   // C5: assign +0
                if constexpr (TIO) sG[el * 6 * N3 + 2 * N3 + cs.at(N, k)] = wv;   // dead g3 slots, SL order
                else a.w[gout(k)] = wv;
                if constexpr (FUSED) {
                    // element-interior points (m == 1) contribute w p c here; shared
                    // nodes contribute once per node in K_B (bitwise-equal exact sum).
                    const bool sz = (k == 0 && !mz0) || (k == n1 && !mz1);
                    if (!sxy && !sz) acc.add(dot_term_pm<PM>(wv, ureg[k], 1.0, a.single, P));
                }
            }
        }
    }
    if constexpr (TIO) {  // w leaves by bulk stores (one per element: the g3 slots are strided)
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            for (int q = 0; q < nel; ++q)
                tma_store_1d(a.w + (e0 + q) * N3, sG + q * 6 * N3 + 2 * N3, (uint32_t)(N3 * sizeof(T)));
            bulk_commit();
        }
    }
    pdl_launch_dependents();
    if constexpr (FUSED) {
        dd v = block_reduce_dd(acc.get());
        if (threadIdx.x == 0) a.parts[a.part_off + blockIdx.x] = v;
    }
    if constexpr (TIO) {
        if (tid == 0) bulk_wait_all();   // shared memory stays valid until the stores are done
    }
}

// ------------------------------------------------------- scalar finalisers
// CG scalars from the globally reduced inner products (rules C7, C9); run by
// one thread: the last block of the reducing kernel (1 rank) or k_fin after
// the rank-ordered combination of the per-rank partials (several ranks).
// Scalar operations under an emulation mode (NEXT-4): glsc3 results, division,
// sqrt -- each one operation (keys: iteration, PH_S, 0, op).
__device__ __forceinline__ double pm_scalar(int pm, double r, const PmArgs& P, int it, int o)
{
    const unsigned long long key = pm_key(it, PH_S, 0, o);
    if (pm == PM_VPREC) return vprec_round(r, P.t);
    if (pm == PM_RR || pm == PM_MCA) return pm_inexact(r, P, key, 0);
    return r;
}
__device__ __forceinline__ double pm_opnd_rt(int pm, double x, const PmArgs& P, int it, int o, int slot)
{
    return pm == PM_MCA ? pm_inexact(x, P, pm_key(it, PH_S, 0, o), slot) : x;
}
__device__ __forceinline__ double pm_div(int pm, double a, double b, const PmArgs& P, int it, int o)
{
    return pm_scalar(pm, pm_opnd_rt(pm, a, P, it, o, 1) / pm_opnd_rt(pm, b, P, it, o, 2), P, it, o);
}
__device__ __forceinline__ double pm_sqrt(int pm, double a, const PmArgs& P, int it, int o)
{
    return pm_scalar(pm, sqrt(pm_opnd_rt(pm, a, P, it, o, 1)), P, it, o);
}

__device__ __forceinline__ void fin_alpha(CgState* st, dd pap_dd, double* trace, bool single,
                                          int pm = PM_NONE, PmArgs P = PmArgs{52, 0})
{
    const int k = st->it;
    const double rtz1 = st->rtr;
    double alpha = 0.0, pap;
    if (pm != PM_NONE) {  // NEXT-4: the reduction and the division are emulated operations
        pap = pm_scalar(pm, pap_dd.hi, P, k, 0);
        if (!st->zero) alpha = pm_div(pm, rtz1, pap, P, k, 1);
    } else if (single) {  // NEXT-2: binary32 scalars (rtz1 already a binary32 value)
        const float pap32 = dd_to_float_rn(pap_dd.hi, pap_dd.lo);
        pap = pap32;
        if (!st->zero) alpha = __fdiv_rn((float)rtz1, pap32);
    } else {
        pap = pap_dd.hi;
        if (!st->zero) alpha = rtz1 / pap;                               // C7
    }
    if (!st->zero && st->defect == 0 && (!(pap > 0.0) || !isfinite(pap)))
        st->defect = k;                                                  // C9
    st->alpha = alpha;
    st->alpham = -alpha;
    st->alpha32 = (float)alpha;
    st->alpham32 = -(float)alpha;
    double* tr = trace + 5 * (int64_t)(k - 1);
    tr[0] = rtz1;
    tr[1] = st->beta;
    tr[2] = alpha;
    tr[3] = pap;
}

// VEC_INIT_J / VEC_RUPD_J: the Jacobi PCG forms of INIT / RUPD, which also
// form z = r * dinv and reduce rtz = glsc3(r, c, z) beside rtr.
enum VecMode { VEC_INIT = 0, VEC_RUPD = 1, VEC_TRUE = 2, VEC_DOT = 3, VEC_INIT_J = 4, VEC_RUPD_J = 5 };

__host__ __device__ constexpr bool vec_jacobi(int mode) { return mode == VEC_INIT_J || mode == VEC_RUPD_J; }

// rtr: glsc3(r,c,r) (the residual norm h_k); rtz: glsc3(r,c,z), the
// preconditioned product that drives alpha / beta (= rtr when z = r).
// st->rtr holds the current rtz1.
template <int MODE>
__device__ __forceinline__ void fin_rtr(CgState* st, dd rtr_dd, dd rtz_dd, double* hist, double* trace,
                                        bool single, int pm = PM_NONE, PmArgs P = PmArgs{52, 0})
{
    // single mode (NEXT-2): binary32 sums, sqrt and division; emulation (NEXT-4):
    // rtr, sqrt and beta are emulated operations (unpreconditioned: rtz = rtr)
    const int it = (MODE == VEC_INIT || MODE == VEC_INIT_J) ? 0 : st->it;
    double rtr = single ? (double)dd_to_float_rn(rtr_dd.hi, rtr_dd.lo) : rtr_dd.hi;
    double rtz = single ? (double)dd_to_float_rn(rtz_dd.hi, rtz_dd.lo) : rtz_dd.hi;
    if (pm != PM_NONE) {
        rtr = pm_scalar(pm, rtr, P, it, 2);
        rtz = rtr;
    }
    const double h = single ? (double)__fsqrt_rn((float)rtr)
                            : (pm != PM_NONE ? pm_sqrt(pm, rtr, P, it, 3) : sqrt(rtr));
    if constexpr (MODE == VEC_INIT || MODE == VEC_INIT_J) {
        st->rtr = rtz;
        st->rtz2 = 0.0;
        st->beta = 0.0;
        st->beta32 = 0.0f;
        st->alpha = 0.0;
        st->alpha32 = 0.0f;
        st->alpham = 0.0;
        st->alpham32 = 0.0f;
        st->zero = (rtz == 0.0);
        st->defect = 0;
        st->it = 1;
        hist[0] = h;
    } else if constexpr (MODE == VEC_RUPD || MODE == VEC_RUPD_J) {
        const int k = st->it;
        hist[k] = h;                            // h_k (R13)
        trace[5 * (int64_t)(k - 1) + 4] = rtr;
        if (!st->zero && st->defect == 0 && (!isfinite(rtr) || !isfinite(rtz))) st->defect = k;
        const double rtz1_next = rtz, rtz2_next = st->rtr;
        st->rtz2 = rtz2_next;
        st->rtr = rtz1_next;
        if (rtz1_next == 0.0) st->zero = 1;     // C9
        double beta = 0.0;
        if (!st->zero)
            beta = single ? (double)__fdiv_rn((float)rtz1_next, (float)rtz2_next)
                          : (pm != PM_NONE ? pm_div(pm, rtz1_next, rtz2_next, P, k, 4)
                                           : rtz1_next / rtz2_next);  // C7
        st->beta = beta;
        st->beta32 = (float)beta;
        st->it = k + 1;
    } else if constexpr (MODE == VEC_TRUE) {
        st->true_rtr = rtr;
    } else {
        st->dot = rtr;
    }
}

// ---------------------------------------------------------------- K_B
// The dssum plan groups the segments (unique shared nodes) by multiplicity
// m in {2, 4, 8}: group m is a dense int32 array of m ascending local indices
// per node (one vector load), each group ordered by the node's first copy.
// The domain is cut into tiles of `te` consecutive elements; toff[3t + g] is
// the first node of group g whose first copy lies in tile t or later.  A block
// processes whole tiles -- all three groups of a tile back to back -- so the
// sectors of w a tile touches (its own elements and the neighbours at +1,
// +ex, +ex*ey) are re-used from L2 instead of being streamed from HBM once
// per group.
#ifndef NBK_DSSUM_H
#define NBK_DSSUM_H 2   // nodes per thread per step
#endif
// CTAs per SM of K_B (launch bounds; registers).  With the gather phase the
// chains need few registers: 6 (FP32) / 4 (FP64) CTAs with 512-node tiles,
// measured same-box: C5 FP64 K_B 0.74 vs 0.86 ms, C4 0.25 vs 0.29 ms, FP32 equal.
#ifndef NBK_DSSUM_THREADS
#define NBK_DSSUM_THREADS 256   // threads per K_B block
#endif
#ifndef NBK_DSSUM_MINB64
#define NBK_DSSUM_MINB64 4
#endif
#ifndef NBK_DSSUM_MINB32
#define NBK_DSSUM_MINB32 6
#endif
template <typename T>
struct DssumArgs {
    T* w;
    const T* p;               // fused: p (shared-node pap term)
    const int32_t* g2;        // n2 x 2
    const int32_t* g4;        // n4 x 4
    const int32_t* g8;        // n8 x 8
    const int32_t* toff;      // (ntiles + 1) x 3 tile offsets into g2, g4, g8
    int ntiles;
    dd* parts;                // fused: partials [0, nA) from K_A, [nA, nA+gridDim) here
    int nA;
    CgState* st;
    double* trace;            // fused: per-iteration trace (niter*5)
    int mask;                 // standalone: assign +0 to masked shared nodes
    int fin;                  // fused: 1 = last block forms alpha (1 rank); 0 = publish only
    int rev;                  // visit the tiles in reverse order
    int single;               // paper-literal single mode (NEXT-2)
    PmArgs pm;                // precision emulation (NEXT-4)
    int it;                   // CG iteration (emulation keys)
    int stage;                // index rows of each tile staged in smem by bulk copies
    int tile_smem;            // bytes per staging buffer (two buffers)
    MeshView mesh;
};

// pap terms of a shared node with m copies (rule C6: one term RN(RN(w p) c) per
// copy, c = 1/m, all copies equal after dssum).  FP32 vectors: w p is exact in
// binary64 (RN32(w p) in single mode), so the m terms sum exactly to the one
// term with c = 1.  FP64: RN(w p)/m rounds when it is subnormal, so the m equal
// terms are accumulated (each exact in the double-double accumulator).
template <typename T, int PM = PM_NONE>
__device__ __forceinline__ void add_node_pap(acc_t& acc, T w, T p, int m, int single, const PmArgs& P)
{
    if constexpr (sizeof(T) == 8) {
        const double cm = m == 2 ? 0.5 : (m == 4 ? 0.25 : 0.125);  // 1/m, m in {2, 4, 8}
        const double t = dot_term_pm<PM>(w, p, cm, single != 0, P);
        // t normal: RN(w p)/m was exact, the m terms sum exactly to m t -- one add
        const bool one = fabs(t) >= 2.2250738585072014e-308;
        acc.add(one ? t * (double)m : t);
        if (!one) {  // rare (subnormal t): the other m - 1 copies' terms
#pragma unroll 1
            for (int c = 1; c < m; ++c) acc.add(t);
        }
    } else {
        acc.add(dot_term_pm<PM>(w, p, 1.0, single != 0, P));
    }
}

// Natural local index of the SL position Ls (the plan stores SL positions).
__device__ __forceinline__ int64_t sl_natural(const MeshView& m, int64_t Ls)
{
    const int N = m.N, N3 = N * N * N;
    const int64_t e = Ls / N3;
    int i, j, k;
    sl_point(N, (int)(Ls - e * N3), i, j, k);
    return e * N3 + (k * N + j) * N + i;
}

template <typename T>
__device__ __forceinline__ bool masked_local(const MeshView& m, int32_t Ls)
{
    const int N = m.N, N3 = N * N * N;
    const uint32_t e = (uint32_t)(Ls / N3);
    int i, j, k;
    sl_point(N, Ls - (int)e * N3, i, j, k);
    ElemCoord ec = elem_coord(m, e);
    return is_masked(m, ec, i, j, k);
}

// Load the (ascending) local indices of node q of a tile (q counts the tile's
// g2 nodes, then its g4, then its g8 nodes); returns the multiplicity.
__device__ __forceinline__ int tile_seg_load(const int32_t* g2, const int32_t* g4, const int32_t* g8,
                                             int s2, int n2, int s4, int n4, int s8, int q,
                                             int32_t (&ix)[8])
{
    if (q < n2) {
        const int2 v = reinterpret_cast<const int2*>(g2)[s2 + q];
        ix[0] = v.x; ix[1] = v.y;
        return 2;
    }
    q -= n2;
    if (q < n4) {
        const int4 v = reinterpret_cast<const int4*>(g4)[s4 + q];
        ix[0] = v.x; ix[1] = v.y; ix[2] = v.z; ix[3] = v.w;
        return 4;
    }
    q -= n4;
    const int4* g = reinterpret_cast<const int4*>(g8) + 2 * (int64_t)(s8 + q);
    const int4 v0 = g[0], v1 = g[1];
    ix[0] = v0.x; ix[1] = v0.y; ix[2] = v0.z; ix[3] = v0.w;
    ix[4] = v1.x; ix[5] = v1.y; ix[6] = v1.z; ix[7] = v1.w;
    return 8;
}

// The tiles of this block (grid-stride), node by node (all multiplicities of
// a tile in one loop, two nodes per thread per step, every load of both
// issued before use; p by the read-only path).
// Tile t's segment offsets.
__device__ __forceinline__ void tile_range(const int32_t* toff, int t, int& s2, int& n2, int& s4, int& n4,
                                           int& s8, int& n8)
{
    s2 = __ldg(&toff[3 * t]); s4 = __ldg(&toff[3 * t + 1]); s8 = __ldg(&toff[3 * t + 2]);
    n2 = __ldg(&toff[3 * t + 3]) - s2; n4 = __ldg(&toff[3 * t + 4]) - s4; n8 = __ldg(&toff[3 * t + 5]) - s8;
}

// Thread 0: bulk-copy tile t's index rows into buf (layout: dssum_tile_bytes).
__device__ __forceinline__ void tile_stage(const int32_t* g2, const int32_t* g4, const int32_t* g8,
                                           const int32_t* toff, int t, unsigned char* buf, uint64_t* bar)
{
    int s2, n2, s4, n4, s8, n8;
    tile_range(toff, t, s2, n2, s4, n4, s8, n8);
    const uint32_t b2 = (uint32_t)dssum_g2_bytes(s2, n2), b4 = 16u * n4, b8 = 32u * n8;
    mbar_arrive_expect_tx(bar, b2 + b4 + b8);
    if (b2) tma_load_1d(buf, reinterpret_cast<const unsigned char*>(g2) + ((8 * (int64_t)s2) & ~(int64_t)15), b2, bar);
    if (b4) tma_load_1d(buf + b2, g4 + 4 * (int64_t)s4, b4, bar);
    if (b8) tma_load_1d(buf + b2 + b4, g8 + 8 * (int64_t)s8, b8, bar);
}

// The tiles of this block (grid-stride), node by node (all multiplicities of
// a tile in one loop, NBK_DSSUM_H nodes per thread per step, every load of
// them issued before use; p by the read-only path).  stage: the index rows of
// the block's next tile are bulk-copied into the other shared-memory buffer
// while this tile is processed, so the per-step dependent chain is one global
// latency (w) instead of two (indices, then w).
template <typename T, bool FUSED, int PM = PM_NONE>
__device__ __forceinline__ void dssum_tiles(const DssumArgs<T>& a, acc_t& acc, unsigned char* sbuf,
                                            int tile_smem, uint64_t* bars)
{
    if (a.stage) {
        if (threadIdx.x == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0 && (int)blockIdx.x < a.ntiles)
            tile_stage(a.g2, a.g4, a.g8, a.toff, a.rev ? a.ntiles - 1 - blockIdx.x : blockIdx.x, sbuf, &bars[0]);
    }
    int k = 0;
    for (int i = blockIdx.x; i < a.ntiles; i += gridDim.x, ++k) {
        const int t = a.rev ? a.ntiles - 1 - i : i;
        int s2, n2, s4, n4, s8, n8;
        tile_range(a.toff, t, s2, n2, s4, n4, s8, n8);
        const int32_t *G2 = a.g2, *G4 = a.g4, *G8 = a.g8;
        int S2 = s2, S4 = s4, S8 = s8;
        if (a.stage) {
            const int b = k & 1;
            const int inx = i + (int)gridDim.x;
            if (threadIdx.x == 0 && inx < a.ntiles) {  // the other buffer was released by the last barrier
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tile_stage(a.g2, a.g4, a.g8, a.toff, a.rev ? a.ntiles - 1 - inx : inx,
                           sbuf + (b ^ 1) * tile_smem, &bars[b ^ 1]);
            }
            mbar_wait(&bars[b], (k >> 1) & 1);
            unsigned char* buf = sbuf + b * tile_smem;
            const int b2 = (int)dssum_g2_bytes(s2, n2);
            G2 = reinterpret_cast<const int32_t*>(buf + dssum_g2_lead(s2));
            G4 = reinterpret_cast<const int32_t*>(buf + b2);
            G8 = reinterpret_cast<const int32_t*>(buf + b2 + 16 * n4);
            S2 = S4 = S8 = 0;
        }
        const int tot = n2 + n4 + n8;
        for (int q = threadIdx.x; q < tot; q += NBK_DSSUM_H * blockDim.x) {
            int32_t ix[NBK_DSSUM_H][8];
            int m[NBK_DSSUM_H];
#pragma unroll
            for (int h = 0; h < NBK_DSSUM_H; ++h) {
                const int qh = q + h * blockDim.x;
                m[h] = qh < tot ? tile_seg_load(G2, G4, G8, S2, n2, S4, n4, S8, qh, ix[h]) : 0;
            }
            T v[NBK_DSSUM_H][8];
            T p0[NBK_DSSUM_H];
#pragma unroll
            for (int h = 0; h < NBK_DSSUM_H; ++h) {
                p0[h] = 0;
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (c < m[h]) {
                        NBK_ASSERT(ix[h][c] >= 0 && (int64_t)ix[h][c] < a.mesh.E * a.mesh.N * a.mesh.N * a.mesh.N);
                        v[h][c] = a.w[ix[h][c]];
                    }
                if constexpr (FUSED && !pm_discontinuous(PM))
                    if (m[h]) p0[h] = __ldg(a.p + ix[h][0]);
            }
#pragma unroll
            for (int h = 0; h < NBK_DSSUM_H; ++h) {
                if (!m[h]) continue;
                T sum = v[h][0];                          // C4: ascending local index
#pragma unroll
                for (int c = 1; c < 8; ++c)
                    if (c < m[h])  // chain add c of the node (key: its first copy)
                        sum = padd<PM>(sum, v[h][c], a.pm,
                                       pm_key(a.it, PH_B, global_local_index(a.mesh, sl_natural(a.mesh, ix[h][0])), c));
                if (!FUSED && a.mask && masked_local<T>(a.mesh, ix[h][0])) sum = 0;
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (c < m[h]) a.w[ix[h][c]] = sum;
                if constexpr (FUSED && pm_discontinuous(PM)) {
                    // RR / MCA: the copies of p differ -- one term RN(RN(w p_c) / m) per copy
                    // (C6 over every local point, as the oracle's glsc3)
                    const double cm = m[h] == 2 ? 0.5 : (m[h] == 4 ? 0.25 : 0.125);
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        if (c < m[h]) acc.add(dot_term_pm<PM>(sum, __ldg(a.p + ix[h][c]), cm, false, a.pm));
                } else if constexpr (FUSED) {
                    add_node_pap<T, PM>(acc, sum, p0[h], m[h], a.single, a.pm);
                }
            }
        }
        if (a.stage) __syncthreads();
    }
}

// Gather-phase K_B (staged tiles): the copies of a tile's nodes (and p at each
// node's first copy) are fetched into shared memory by cp.async first -- every
// load of the tile in flight at once, no registers held -- then each node's
// chain is summed from shared memory and scattered.  Memory-level parallelism
// of K_B is otherwise bounded by the registers of the per-thread node chains.
// Dynamic shared memory: 2 index buffers, then the copy values and p values of
// one tile (dssum_gather_smem).
__device__ __forceinline__ void cp_async_4(void* dst_smem, const void* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_8(void* dst_smem, const void* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
template <typename T>
__device__ __forceinline__ void cp_async_t(T* dst_smem, const T* src)
{
    if constexpr (sizeof(T) == 4) cp_async_4(dst_smem, src); else cp_async_8(dst_smem, src);
}

template <typename T, bool FUSED, int PM = PM_NONE>
__device__ __forceinline__ void dssum_tiles_gather(const DssumArgs<T>& a, acc_t& acc, unsigned char* sbuf,
                                                   int tile_smem, uint64_t* bars)
{
    constexpr bool PCOPY = FUSED && !pm_discontinuous(PM);
    T* sval = reinterpret_cast<T*>(sbuf + 2 * tile_smem);      // tile_smem / 4 values
    T* spv = sval + tile_smem / 4;                             // tile_smem / 8 values
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0 && (int)blockIdx.x < a.ntiles)
        tile_stage(a.g2, a.g4, a.g8, a.toff, a.rev ? a.ntiles - 1 - blockIdx.x : blockIdx.x, sbuf, &bars[0]);
    int k = 0;
    // segment offsets of the block's current tile, loaded one tile ahead (their
    // global round trip otherwise opened every tile: ncu C5 FP32, 5 % of the samples)
#ifndef NBK_DSSUM_TOFF_PF
#define NBK_DSSUM_TOFF_PF 1
#endif
    int s2, n2, s4, n4, s8, n8;
    if ((int)blockIdx.x < a.ntiles)
        tile_range(a.toff, a.rev ? a.ntiles - 1 - blockIdx.x : blockIdx.x, s2, n2, s4, n4, s8, n8);
    for (int i = blockIdx.x; i < a.ntiles; i += gridDim.x, ++k) {
        const int b = k & 1;
        const int inx = i + (int)gridDim.x;
        int s2n = 0, n2n = 0, s4n = 0, n4n = 0, s8n = 0, n8n = 0;
        if (!NBK_DSSUM_TOFF_PF) tile_range(a.toff, a.rev ? a.ntiles - 1 - i : i, s2, n2, s4, n4, s8, n8);
        else if (inx < a.ntiles) tile_range(a.toff, a.rev ? a.ntiles - 1 - inx : inx, s2n, n2n, s4n, n4n, s8n, n8n);
        if (threadIdx.x == 0 && inx < a.ntiles) {  // the other buffer was released by the last barrier
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tile_stage(a.g2, a.g4, a.g8, a.toff, a.rev ? a.ntiles - 1 - inx : inx,
                       sbuf + (b ^ 1) * tile_smem, &bars[b ^ 1]);
        }
        mbar_wait(&bars[b], (k >> 1) & 1);
        unsigned char* buf = sbuf + b * tile_smem;
        const int b2 = (int)dssum_g2_bytes(s2, n2);
        const int32_t* G2 = reinterpret_cast<const int32_t*>(buf + dssum_g2_lead(s2));
        const int32_t* G4 = reinterpret_cast<const int32_t*>(buf + b2);
        const int32_t* G8 = reinterpret_cast<const int32_t*>(buf + b2 + 16 * n4);
        const int c2 = 2 * n2, c4 = c2 + 4 * n4, nc = c4 + 8 * n8, tot = n2 + n4 + n8;
        // phase 1: every copy value (and p) of the tile in flight
        for (int r = threadIdx.x; r < nc; r += blockDim.x) {
            const int32_t ix = r < c2 ? G2[r] : (r < c4 ? G4[r - c2] : G8[r - c4]);
            NBK_ASSERT(ix >= 0 && (int64_t)ix < a.mesh.E * a.mesh.N * a.mesh.N * a.mesh.N);
            NBK_ASSERT(r < tile_smem / 4);
            cp_async_t<T>(sval + r, a.w + ix);
        }
        if constexpr (PCOPY) {
            for (int q = threadIdx.x; q < tot; q += blockDim.x) {
                const int32_t ix = q < n2 ? G2[2 * q] : (q < n2 + n4 ? G4[4 * (q - n2)] : G8[8 * (q - n2 - n4)]);
                cp_async_t<T>(spv + q, a.p + ix);
            }
        }
        cp_async_wait_all();
        __syncthreads();
        // phase 2: chains from shared memory (C4), scatter, pap
        for (int q = threadIdx.x; q < tot; q += blockDim.x) {
            int m, r0;
            const int32_t* row;
            if (q < n2) { m = 2; r0 = 2 * q; row = G2 + r0; }
            else if (q < n2 + n4) { m = 4; r0 = 4 * (q - n2); row = G4 + r0; r0 += c2; }
            else { m = 8; r0 = 8 * (q - n2 - n4); row = G8 + r0; r0 += c4; }
            T sum = sval[r0];
            for (int c = 1; c < m; ++c) {
                unsigned long long key = 0;
                if constexpr (PM != PM_NONE)
                    key = pm_key(a.it, PH_B, global_local_index(a.mesh, sl_natural(a.mesh, row[0])), c);
                sum = padd<PM>(sum, sval[r0 + c], a.pm, key);
            }
            if (!FUSED && a.mask && masked_local<T>(a.mesh, row[0])) sum = 0;
            for (int c = 0; c < m; ++c) a.w[row[c]] = sum;
            if constexpr (FUSED && pm_discontinuous(PM)) {
                const double cm = m == 2 ? 0.5 : (m == 4 ? 0.25 : 0.125);
                for (int c = 0; c < m; ++c) acc.add(dot_term_pm<PM>(sum, __ldg(a.p + row[c]), cm, false, a.pm));
            } else if constexpr (FUSED) {
                add_node_pap<T, PM>(acc, sum, spv[q], m, a.single, a.pm);
            }
        }
        __syncthreads();
        if (NBK_DSSUM_TOFF_PF) { s2 = s2n; n2 = n2n; s4 = s4n; n4 = n4n; s8 = s8n; n8 = n8n; }
    }
}

// Gather-phase K_B, multiplicity-specialised (PM_NONE; NBK_DSSUM_GATHER_M, default on).
// Same tiles, same chains (C4: ascending local index), same pap terms as
// dssum_tiles_gather -- bitwise identical -- with fewer issue slots per node
// (ncu C5 FP32: the runtime-m form spent ~100 warp instructions per node
// iteration in phase 2 and 22 per copy in phase 1, issue 61 % busy):
//  phase 1 walks the staged index buffer as one flat int array (the value
//          buffer mirrors it slot for slot; alignment-pad slots are skipped by
//          a range test), no 3-way row selection;
//  phase 2 runs one loop per multiplicity with the chain unrolled and the
//          index row / copy values fetched by 8- and 16-byte shared loads.
#ifndef NBK_DSSUM_GATHER_M
#define NBK_DSSUM_GATHER_M 1
#endif
#ifndef NBK_DSSUM_PF_L2
#define NBK_DSSUM_PF_L2 0   // 1: prefetch.global.L2 of the next tile's copies during phase 2 (experiment)
#endif
template <typename T, int M>
__device__ __forceinline__ void lds_row(const int32_t* row, const T* val, int32_t (&ix)[M], T (&v)[M])
{
    if constexpr (M == 2) {
        const int2 r = *reinterpret_cast<const int2*>(row);
        ix[0] = r.x; ix[1] = r.y;
    } else {
#pragma unroll
        for (int h = 0; h < M / 4; ++h) {
            const int4 r = reinterpret_cast<const int4*>(row)[h];
            ix[4 * h] = r.x; ix[4 * h + 1] = r.y; ix[4 * h + 2] = r.z; ix[4 * h + 3] = r.w;
        }
    }
    if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int h = 0; h < M / 2; ++h) {
            const double2 d = reinterpret_cast<const double2*>(val)[h];
            v[2 * h] = d.x; v[2 * h + 1] = d.y;
        }
    } else if constexpr (M == 2) {
        const float2 f = *reinterpret_cast<const float2*>(val);
        v[0] = f.x; v[1] = f.y;
    } else {
#pragma unroll
        for (int h = 0; h < M / 4; ++h) {
            const float4 f = reinterpret_cast<const float4*>(val)[h];
            v[4 * h] = f.x; v[4 * h + 1] = f.y; v[4 * h + 2] = f.z; v[4 * h + 3] = f.w;
        }
    }
}
// The n nodes of multiplicity M of a tile: index rows at rows[M q], their copy
// values at vals[M q], p of the first copy at pv[q].
template <typename T, bool FUSED, int M>
__device__ __forceinline__ void dssum_nodes_m(const DssumArgs<T>& a, acc_t& acc, const int32_t* rows,
                                              const T* vals, const T* pv, int n)
{
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        int32_t ix[M];
        T v[M];
        lds_row<T, M>(rows + M * q, vals + M * q, ix, v);
        T sum = v[0];                                    // C4: ascending local index
#pragma unroll
        for (int c = 1; c < M; ++c) sum = sum + v[c];
        if (!FUSED && a.mask && masked_local<T>(a.mesh, ix[0])) sum = 0;
#pragma unroll
        for (int c = 0; c < M; ++c) a.w[ix[c]] = sum;
        if constexpr (FUSED) add_node_pap<T, PM_NONE>(acc, sum, pv[q], M, a.single, a.pm);
    }
}
// Thread-private fetch of the copies (and p) of the nodes dssum_nodes_m gives this thread.
template <typename T, bool FUSED, int M>
__device__ __forceinline__ void dssum_fetch_m(const DssumArgs<T>& a, const int32_t* rows, T* vals, T* pv, int n)
{
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        int32_t ix[M];
        if constexpr (M == 2) {
            const int2 r = *reinterpret_cast<const int2*>(rows + 2 * q);
            ix[0] = r.x; ix[1] = r.y;
        } else {
#pragma unroll
            for (int h = 0; h < M / 4; ++h) {
                const int4 r = reinterpret_cast<const int4*>(rows + M * q)[h];
                ix[4 * h] = r.x; ix[4 * h + 1] = r.y; ix[4 * h + 2] = r.z; ix[4 * h + 3] = r.w;
            }
        }
#pragma unroll
        for (int c = 0; c < M; ++c) cp_async_t<T>(vals + M * q + c, a.w + ix[c]);
        if constexpr (FUSED) cp_async_t<T>(pv + q, a.p + ix[0]);
    }
}
template <typename T, bool FUSED>
__device__ __forceinline__ void dssum_tiles_gather_m(const DssumArgs<T>& a, acc_t& acc, unsigned char* sbuf,
                                                     int tile_smem, uint64_t* bars)
{
    T* sval = reinterpret_cast<T*>(sbuf + 2 * tile_smem);      // tile_smem / 4 values, slot = index slot
    T* spv = sval + tile_smem / 4;                             // tile_smem / 8 values, one per node
    const uint32_t nloc = (uint32_t)(a.mesh.E * a.mesh.N * a.mesh.N * a.mesh.N);
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0 && (int)blockIdx.x < a.ntiles)
        tile_stage(a.g2, a.g4, a.g8, a.toff, a.rev ? a.ntiles - 1 - blockIdx.x : blockIdx.x, sbuf, &bars[0]);
    int k = 0;
    int s2 = 0, n2 = 0, s4 = 0, n4 = 0, s8 = 0, n8 = 0;
    if ((int)blockIdx.x < a.ntiles)
        tile_range(a.toff, a.rev ? a.ntiles - 1 - blockIdx.x : blockIdx.x, s2, n2, s4, n4, s8, n8);
    for (int i = blockIdx.x; i < a.ntiles; i += gridDim.x, ++k) {
        const int b = k & 1;
        const int inx = i + (int)gridDim.x;
        int s2n = 0, n2n = 0, s4n = 0, n4n = 0, s8n = 0, n8n = 0;
        if (inx < a.ntiles) tile_range(a.toff, a.rev ? a.ntiles - 1 - inx : inx, s2n, n2n, s4n, n4n, s8n, n8n);
        if (threadIdx.x == 0 && inx < a.ntiles) {  // the other buffer was released by the last barrier
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tile_stage(a.g2, a.g4, a.g8, a.toff, a.rev ? a.ntiles - 1 - inx : inx,
                       sbuf + (b ^ 1) * tile_smem, &bars[b ^ 1]);
        }
        mbar_wait(&bars[b], (k >> 1) & 1);
        const int32_t* ibuf = reinterpret_cast<const int32_t*>(sbuf + b * tile_smem);
        const int lead = n2 ? (int)dssum_g2_lead(s2) >> 2 : 0;   // pad slots before the g2 rows (none without g2 rows)
        const int e2 = lead + 2 * n2;                            // end of the g2 rows
        const int b2i = (int)dssum_g2_bytes(s2, n2) >> 2;        // first g4 slot
        const int b4i = b2i + 4 * n4;                            // first g8 slot
        const int nint = b4i + 8 * n8;
        // phase 1: every copy value (and p at the first copies) of the tile in flight
#if NBK_DSSUM_GATHER_M == 2
        // thread-private form: a thread fetches the copies of exactly the nodes it sums in
        // phase 2 (same q loops), so its own cp.async wait orders the data -- no block
        // barrier between the phases, the warps of a block drift apart within a tile
        dssum_fetch_m<T, FUSED, 2>(a, ibuf + lead, sval + lead, spv, n2);
        dssum_fetch_m<T, FUSED, 4>(a, ibuf + b2i, sval + b2i, spv + n2, n4);
        dssum_fetch_m<T, FUSED, 8>(a, ibuf + b4i, sval + b4i, spv + n2 + n4, n8);
        (void)nloc; (void)e2; (void)nint;
        cp_async_wait_all();
#else
        for (int r = threadIdx.x; r < nint; r += blockDim.x) {
            const int32_t ix = ibuf[r];
            if ((r >= lead) & ((r < e2) | (r >= b2i))) {
                NBK_ASSERT((uint32_t)ix < nloc);
                cp_async_t<T>(sval + r, a.w + ix);
            }
        }
        if constexpr (FUSED) {
            const int tot = n2 + n4 + n8;
            for (int q = threadIdx.x; q < tot; q += blockDim.x) {
                const int r = q < n2 ? lead + 2 * q : (q < n2 + n4 ? b2i + 4 * (q - n2) : b4i + 8 * (q - n2 - n4));
                cp_async_t<T>(spv + q, a.p + ibuf[r]);
            }
        }
        (void)nloc;
        cp_async_wait_all();
        __syncthreads();
#endif
#if NBK_DSSUM_PF_L2
        // L2 prefetch of the next tile's copies (its index rows were bulk-copied during this
        // tile's gather): the next gather then meets L2 instead of DRAM latency
        if (inx < a.ntiles) {
            mbar_wait(&bars[b ^ 1], ((k + 1) >> 1) & 1);
            const int32_t* inext = reinterpret_cast<const int32_t*>(sbuf + (b ^ 1) * tile_smem);
            const int leadn = n2n ? (int)dssum_g2_lead(s2n) >> 2 : 0, e2n = leadn + 2 * n2n;
            const int b2n = (int)dssum_g2_bytes(s2n, n2n) >> 2, nintn = b2n + 4 * n4n + 8 * n8n;
            for (int r = threadIdx.x; r < nintn; r += blockDim.x) {
                const int32_t ix = inext[r];
                if ((r >= leadn) & ((r < e2n) | (r >= b2n)))
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a.w + ix));
            }
        }
#endif
        // phase 2: chains from shared memory (C4), scatter, pap -- one loop per multiplicity
        dssum_nodes_m<T, FUSED, 2>(a, acc, ibuf + lead, sval + lead, spv, n2);
        dssum_nodes_m<T, FUSED, 4>(a, acc, ibuf + b2i, sval + b2i, spv + n2, n4);
        dssum_nodes_m<T, FUSED, 8>(a, acc, ibuf + b4i, sval + b4i, spv + n2 + n4, n8);
        __syncthreads();
        s2 = s2n; n2 = n2n; s4 = s4n; n4 = n4n; s8 = s8n; n8 = n8n;
    }
}

template <typename T, int PM>
__device__ __forceinline__ void dssum_fused_epilogue(const DssumArgs<T>& a, acc_t& acc);

template <typename T, bool FUSED, int PM = PM_NONE>
__global__ void __launch_bounds__(NBK_DSSUM_THREADS, sizeof(T) == 4 ? NBK_DSSUM_MINB32 : NBK_DSSUM_MINB64) k_dssum(DssumArgs<T> a)
{
    acc_t acc;
    extern __shared__ __align__(128) unsigned char dsm_tiles[];
    __shared__ uint64_t dsm_bars[2];
    pdl_wait();
#if defined(NBK_DSSUM_GATHER)
    if (a.stage) {
        if constexpr (PM == PM_NONE && NBK_DSSUM_GATHER_M) dssum_tiles_gather_m<T, FUSED>(a, acc, dsm_tiles, a.tile_smem, dsm_bars);
        else dssum_tiles_gather<T, FUSED, PM>(a, acc, dsm_tiles, a.tile_smem, dsm_bars);
    } else
#endif
    dssum_tiles<T, FUSED, PM>(a, acc, dsm_tiles, a.tile_smem, dsm_bars);
    pdl_launch_dependents();
    if constexpr (FUSED) dssum_fused_epilogue<T, PM>(a, acc);
}

// Fused K_B epilogue (all threads of the block): fold K_A's partials, publish
// the block's pap partial; one rank: the last block forms alpha.
template <typename T, int PM>
__device__ __forceinline__ void dssum_fused_epilogue(const DssumArgs<T>& a, acc_t& acc)
{
    {
        // K_A's nA pap partials are folded in here, a fixed slice per block, so
        // that the serial last-block reduction sees gridDim partials, not nA + gridDim
        dd ka{0.0, 0.0};
        {
            const int lo = (int)((long long)a.nA * blockIdx.x / gridDim.x);
            const int hi = (int)((long long)a.nA * (blockIdx.x + 1) / gridDim.x);
            for (int q = lo + (int)threadIdx.x; q < hi; q += blockDim.x)
                ka = dd_add(ka, dd{__ldcg(&a.parts[q].hi), __ldcg(&a.parts[q].lo)});
        }
        dd v = block_reduce_dd(dd_add(acc.get(), ka));
        if (!a.fin) {
            // multi-rank: the face-merge kernel adds the slab-face terms and
            // reduces the K_B and merge partials of this rank
            if (threadIdx.x == 0) a.parts[a.nA + blockIdx.x] = v;
            return;
        }
        const unsigned int total = gridDim.x;
        if (publish_and_check_last(a.parts, a.nA + blockIdx.x, v, &a.st->cnt[0], total)) {
            dd pap_dd = reduce_partials(a.parts + a.nA, (int)gridDim.x);
            if (threadIdx.x == 0) {
                fin_alpha(a.st, pap_dd, a.trace, a.single, PM, a.pm);
                a.st->cnt[0] = 0;
            }
        }
    }
}

// ---------------------------------------------------------------- K_C

template <typename T>
struct VecArgs {
    T* r;               // INIT: r out; RUPD: r in/out; TRUE: r_true out (double)
    const T* w;         // RUPD/TRUE
    const double* f;    // INIT: f (double); TRUE: f
    T* x;               // INIT: zeroed
    T* p;               // INIT: zeroed
    const T* a;         // DOT
    const T* b;         // DOT
    const T* dinv;      // INIT_J / RUPD_J
    int64_t n;
    dd* parts;
    CgState* st;
    double* hist;
    double* trace;
    dd* slot;           // multi-rank: this rank's reduced partial (NULL: finalise here)
    int single;         // paper-literal single mode: RN32(a b) terms, binary32 scalars
    PmArgs pm;          // precision emulation (NEXT-4)
    int it;             // CG iteration (emulation keys)
    int rev;            // visit the chunks in reverse order
    int natural;        // DOT only: a, b in natural order (public glsc3); else SL vectors
    MeshView mesh;
};

// V consecutive values, 16-byte vector memory operations when V*sizeof(T) >= 16.
template <typename T, int V>
struct VecT {
    T v[V];
    __device__ __forceinline__ void load(const T* p)
    {
        if constexpr (sizeof(T) == 4 && V % 4 == 0) {
#pragma unroll
            for (int q = 0; q < V / 4; ++q) {
                const float4* a = reinterpret_cast<const float4*>(p) + q;
                const float4 f = *a;
                v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
            }
        } else if constexpr (sizeof(T) == 8 && V % 2 == 0) {
#pragma unroll
            for (int q = 0; q < V / 2; ++q) {
                const double2* a = reinterpret_cast<const double2*>(p) + q;
                const double2 d = *a;
                v[2 * q] = d.x; v[2 * q + 1] = d.y;
            }
        } else {
#pragma unroll
            for (int q = 0; q < V; ++q) v[q] = p[q];
        }
    }
    __device__ __forceinline__ void store(T* p) const
    {
        if constexpr (sizeof(T) == 4 && V % 4 == 0) {
#pragma unroll
            for (int q = 0; q < V / 4; ++q)
                reinterpret_cast<float4*>(p)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else if constexpr (sizeof(T) == 8 && V % 2 == 0) {
#pragma unroll
            for (int q = 0; q < V / 2; ++q)
                reinterpret_cast<double2*>(p)[q] = make_double2(v[2 * q], v[2 * q + 1]);
        } else {
#pragma unroll
            for (int q = 0; q < V; ++q) p[q] = v[q];
        }
    }
};

// c = 1/m (R8) of the V consecutive points L..L+V-1 (one element, N3 % V == 0),
// stepping (i, j, k) incrementally from one division (fast division by the
// runtime N and N^3; one vector kernel serves every N).
template <int V>
__device__ __forceinline__ void chunk_weights(const MeshView& m, int64_t L, double (&c)[V])
{
    const int N = m.N, n1 = N - 1;
    const uint32_t Lu = (uint32_t)L;  // n_local < 2^31 (validated at set-up)
    const uint32_t e = fast_div(Lu, m.n3_mul, m.n3_shr);
    const uint32_t rem = Lu - e * (uint32_t)(N * N * N);
    const uint32_t q1 = fast_div(rem, m.n_mul, m.n_shr);
    const uint32_t q2 = fast_div(q1, m.n_mul, m.n_shr);
    int i = (int)(rem - q1 * (uint32_t)N), j = (int)(q1 - q2 * (uint32_t)N), k = (int)q2;
    const ElemCoord ec = elem_coord(m, e);
    const bool xl = ec.ax > 0, xh = ec.ax < m.ex - 1, yl = ec.ay > 0, yh = ec.ay < m.ey - 1;
    const bool zl = ec.azg > 0, zh = ec.azg < m.ezg - 1;
    int myz = (((j == 0 && yl) || (j == n1 && yh)) ? 2 : 1) * (((k == 0 && zl) || (k == n1 && zh)) ? 2 : 1);
    if (N % V == 0) {  // the chunk lies in one (j, k) row
#pragma unroll
        for (int t = 0; t < V; ++t) {
            const int ii = i + t;
            const int mx = ((ii == 0 && xl) || (ii == n1 && xh)) ? 2 : 1;
            c[t] = inv_mult(mx * myz);
        }
        return;
    }
#pragma unroll
    for (int t = 0; t < V; ++t) {
        const int mx = ((i == 0 && xl) || (i == n1 && xh)) ? 2 : 1;
        c[t] = inv_mult(mx * myz);
        if (t + 1 < V && ++i == N) {
            i = 0;
            if (++j == N) { j = 0; ++k; }
            myz = (((j == 0 && yl) || (j == n1 && yh)) ? 2 : 1) * (((k == 0 && zl) || (k == n1 && zh)) ? 2 : 1);
        }
    }
}

// Vector kernel over all local points: chunks of V = 4 consecutive points
// (N^3 % 4 == 0) in one element, 16-byte loads/stores; structural c = 1/m.
// SL weights: sh_tab[f] = boundary code of face slot I^3 + f (bit 0 i = 0,
// 1 i = N-1, 2 j = 0, 3 j = N-1, 4 k = 0, 5 k = N-1), built per block; an
// element's neighbour code nb has the same bits for "a neighbour lies on that
// side".  Bits 0/1 (2/3, 4/5) exclude each other, so popc(code & nb) is the
// number of directions in which the point is shared and m = 2^popc (R8).
#define NBK_SL_TAB 1352   // N^3 - (N-2)^3 at N = 16
__device__ __forceinline__ void sl_tab_build(int N, unsigned char* tab)
{
    const int I = N - 2, F = N * N * N - I * I * I;
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
        int i, j, k;
        sl_point(N, I * I * I + f, i, j, k);
        tab[f] = (unsigned char)((i == 0) | ((i == N - 1) << 1) | ((j == 0) << 2) | ((j == N - 1) << 3) |
                                 ((k == 0) << 4) | ((k == N - 1) << 5));
    }
}
__device__ __forceinline__ unsigned elem_nb(const MeshView& m, uint32_t e)
{
    const ElemCoord ec = elem_coord(m, e);
    return (ec.ax > 0) | ((ec.ax < m.ex - 1) << 1) | ((ec.ay > 0) << 2) | ((ec.ay < m.ey - 1) << 3) |
           ((ec.azg > 0) << 4) | ((ec.azg < m.ezg - 1) << 5);
}
// c = 1/m of the V consecutive SL slots L..L+V-1 (one element; interior slots and
// face slots never share a chunk: I^3 % V == 0).
template <int V>
__device__ __forceinline__ void chunk_weights_sl(const MeshView& m, int64_t L, const unsigned char* tab,
                                                 double (&c)[V])
{
    const int N = m.N, I = N - 2;
    const uint32_t Lu = (uint32_t)L;
    const uint32_t e = fast_div(Lu, m.n3_mul, m.n3_shr);
    const int s = (int)(Lu - e * (uint32_t)(N * N * N)) - I * I * I;
    if (s < 0) {
#pragma unroll
        for (int t = 0; t < V; ++t) c[t] = 1.0;
        return;
    }
    const unsigned nb = elem_nb(m, e);
#pragma unroll
    for (int t = 0; t < V; ++t) c[t] = inv_mult(1 << __popc(tab[s + t] & nb));
}

// Per-chunk loads and arithmetic of each mode (split so that the loads of two
// chunks can be issued before either is used).
template <typename T, int V, int MODE, int PM = PM_NONE>
struct VecChunk {
    VecT<T, V> A, B, C;
    VecT<double, V> F;
    __device__ __forceinline__ void load(const VecArgs<T>& a, int64_t L)
    {
        if constexpr (MODE == VEC_INIT) {
            F.load(a.f + L);
        } else if constexpr (MODE == VEC_RUPD) {
            A.load(a.w + L);
            B.load(a.r + L);
        } else if constexpr (MODE == VEC_TRUE) {
            A.load(a.w + L);
            F.load(a.f + L);
        } else if constexpr (MODE == VEC_INIT_J) {
            F.load(a.f + L);
            C.load(a.dinv + L);
        } else if constexpr (MODE == VEC_RUPD_J) {
            A.load(a.w + L);
            B.load(a.r + L);
            C.load(a.dinv + L);
        } else {
            A.load(a.a + L);
            B.load(a.b + L);
        }
    }
    __device__ __forceinline__ void run(const VecArgs<T>& a, int64_t L, const double (&c)[V], T am,
                                        acc_t& acc, acc_t& acc2)
    {
        if constexpr (MODE == VEC_INIT) {
            VecT<T, V> r, z;
#pragma unroll
            for (int t = 0; t < V; ++t) {
                r.v[t] = (T)F.v[t];  // C11: f32 = RN32(f64)
                z.v[t] = 0;
            }
            r.store(a.r + L);
            z.store(a.x + L);
            z.store(a.p + L);
#pragma unroll
            for (int t = 0; t < V; ++t) acc.add(dot_term_pm<PM>(r.v[t], r.v[t], c[t], a.single, a.pm));
        } else if constexpr (MODE == VEC_RUPD) {
            VecT<T, V> r;
#pragma unroll
            for (int t = 0; t < V; ++t) {  // C8 (emulation key: the point's natural local index, phase C)
                unsigned long long key = 0;
                if constexpr (PM != PM_NONE) key = pm_key(a.it, PH_C, global_local_index(a.mesh, sl_natural(a.mesh, L + t)), 0);
                r.v[t] = pfma<PM>(am, A.v[t], B.v[t], a.pm, key);
            }
            r.store(a.r + L);
#pragma unroll
            for (int t = 0; t < V; ++t) acc.add(dot_term_pm<PM>(r.v[t], r.v[t], c[t], a.single, a.pm));
        } else if constexpr (MODE == VEC_TRUE) {
            VecT<T, V> r;
#pragma unroll
            for (int t = 0; t < V; ++t) r.v[t] = fma_t<T>((T)-1, A.v[t], (T)F.v[t]);  // C12
            r.store(a.r + L);
#pragma unroll
            for (int t = 0; t < V; ++t) acc.add(dot_term_pm<PM>(r.v[t], r.v[t], c[t], a.single, a.pm));
        } else if constexpr (MODE == VEC_INIT_J) {
            VecT<T, V> r, z;
#pragma unroll
            for (int t = 0; t < V; ++t) {
                r.v[t] = (T)F.v[t];  // C11: f32 = RN32(f64)
                z.v[t] = 0;
            }
            r.store(a.r + L);
            z.store(a.x + L);
            z.store(a.p + L);
#pragma unroll
            for (int t = 0; t < V; ++t) {
                acc.add(dot_term_pm<PM>(r.v[t], r.v[t], c[t], a.single, a.pm));
                acc2.add(dot_term(r.v[t], mul_t<T>(r.v[t], C.v[t]), c[t], a.single));  // z = r dinv
            }
        } else if constexpr (MODE == VEC_RUPD_J) {
            VecT<T, V> r;
#pragma unroll
            for (int t = 0; t < V; ++t) r.v[t] = fma_t<T>(am, A.v[t], B.v[t]);  // C8
            r.store(a.r + L);
#pragma unroll
            for (int t = 0; t < V; ++t) {
                acc.add(dot_term_pm<PM>(r.v[t], r.v[t], c[t], a.single, a.pm));
                acc2.add(dot_term(r.v[t], mul_t<T>(r.v[t], C.v[t]), c[t], a.single));  // z = r dinv
            }
        } else {
#pragma unroll
            for (int t = 0; t < V; ++t) acc.add(dot_term(A.v[t], B.v[t], c[t], a.single));
        }
    }
};

// All chunks of this block (grid-stride).  VP: VPREC rounding (NEXT-4).  The CG loop alternates the sweep
// direction from kernel to kernel (K_A forward, K_B backward, K_C forward, next
// K_A backward, ...): each kernel starts where its predecessor ended, on the
// data still resident in the 126 MB L2.
// V = 4 consecutive points per chunk for even N (N^3 % 4 == 0), 1 for odd N.
#ifndef NBK_VEC_U
#define NBK_VEC_U 2
#endif
template <int V>
__device__ __forceinline__ void chunk_weights_any(const MeshView& m, int64_t L, const unsigned char* tab,
                                                  bool natural, double (&c)[V])
{
    if (natural) chunk_weights<V>(m, L, c);
    else chunk_weights_sl<V>(m, L, tab, c);
}

template <typename T, int V, int MODE, int PM = PM_NONE>
__device__ __forceinline__ void vec_loop(const VecArgs<T>& a, T am, acc_t& acc, acc_t& acc2,
                                         const unsigned char* tab)
{
    const bool nat = MODE == VEC_DOT && a.natural;
    const int64_t nch = a.n / V;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t q0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // NBK_VEC_U chunks of V points per thread per step; every load of them is
    // issued before any use (more bytes in flight per thread)
    for (; q0 + (NBK_VEC_U - 1) * stride < nch; q0 += NBK_VEC_U * stride) {
        VecChunk<T, V, MODE, PM> C[NBK_VEC_U];
        int64_t L[NBK_VEC_U];
#pragma unroll
        for (int u = 0; u < NBK_VEC_U; ++u) {
            const int64_t qu = q0 + u * stride;
            L[u] = (a.rev ? nch - 1 - qu : qu) * V;
            NBK_ASSERT(L[u] >= 0 && L[u] + V <= a.n);
            C[u].load(a, L[u]);
        }
#pragma unroll
        for (int u = 0; u < NBK_VEC_U; ++u) {
            double c[V];
            chunk_weights_any<V>(a.mesh, L[u], tab, nat, c);
            C[u].run(a, L[u], c, am, acc, acc2);
        }
    }
    for (; q0 < nch; q0 += stride) {  // tail: fewer than NBK_VEC_U chunks left
        VecChunk<T, V, MODE, PM> C0;
        const int64_t L0 = (a.rev ? nch - 1 - q0 : q0) * V;
        C0.load(a, L0);
        double c[V];
        chunk_weights_any<V>(a.mesh, L0, tab, nat, c);
        C0.run(a, L0, c, am, acc, acc2);
    }
}

template <typename T, int V, int MODE, int PM = PM_NONE>
__global__ void __launch_bounds__(256) k_vec(VecArgs<T> a)
{
    constexpr bool J = vec_jacobi(MODE);
    acc_t acc, acc2;
    T am = 0;
    __shared__ unsigned char sl_tab[NBK_SL_TAB];
    sl_tab_build(a.mesh.N, sl_tab);  // before the PDL wait: overlaps the previous kernel's tail
    pdl_wait();
    if constexpr (MODE == VEC_RUPD || MODE == VEC_RUPD_J) {
        if constexpr (sizeof(T) == 8) am = (T)a.st->alpham; else am = (T)a.st->alpham32;
    }
    __syncthreads();
    vec_loop<T, V, MODE, PM>(a, am, acc, acc2, sl_tab);
    pdl_launch_dependents();
    dd v = block_reduce_dd(acc.get());
    dd v2 = J ? block_reduce_dd(acc2.get()) : dd{0.0, 0.0};
    if (J && threadIdx.x == 0) {  // rtz partials in the second bank (ordered by the release below)
        __stcg(&a.parts[gridDim.x + blockIdx.x].hi, v2.hi);
        __stcg(&a.parts[gridDim.x + blockIdx.x].lo, v2.lo);
    }
    if (publish_and_check_last(a.parts, blockIdx.x, v, &a.st->cnt[1], gridDim.x)) {
        dd tot = reduce_partials(a.parts, (int)gridDim.x);
        dd tot2 = J ? reduce_partials(a.parts + gridDim.x, (int)gridDim.x) : tot;
        if (threadIdx.x == 0) {
            if (a.slot) {
                // multi-rank: publish this rank's partials; k_fin finalises
                a.slot[0] = tot;
                a.slot[1] = tot2;
            } else {
                fin_rtr<MODE>(a.st, tot, tot2, a.hist, a.trace, a.single, PM, a.pm);
            }
            a.st->cnt[1] = 0;
        }
    }
}

// ------------------------------------------------ binary32 accumulation (NEXT-2)
// The paper's single-precision solver (reading R11c): the
// inner products accumulated in binary32.  Terms RN32(RN32(a b) c) are added
// into a binary32 running sum per thread (its chunks in grid-stride order),
// the block sums by a fixed binary32 shuffle tree, the per-block sums by the
// last block (fixed slices, then the same tree), the per-rank sums in binary32
// in rank order (k_fin): a fixed binary32 summation tree, not the oracle's
// sequential loop, so the two agree to rounding (parity by tolerance).  The
// scalars are binary32 (fin_* with single = 1).  Separate from k_vec so the
// FP64-accumulating hot path is untouched.
enum VecAMode { VA_INIT = 0, VA_RUPD = 1, VA_PAP = 2 };

__device__ __forceinline__ float block_reduce_f32(float v)
{
    __shared__ float red32[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = __fadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
    __syncthreads();
    if (lane == 0) red32[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = lane < nw ? red32[lane] : 0.0f;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = __fadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
    }
    return v;
}

template <int V, int MODE>
__global__ void __launch_bounds__(256) k_vec_a(VecArgs<float> a)
{
    __shared__ unsigned char sl_tab[NBK_SL_TAB];
    sl_tab_build(a.mesh.N, sl_tab);
    const float am = MODE == VA_RUPD ? a.st->alpham32 : 0.0f;
    __syncthreads();
    float s = 0.0f;
    const int64_t nch = a.n / V, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nch; q += stride) {
        const int64_t L = (a.rev ? nch - 1 - q : q) * V;
        NBK_ASSERT(L >= 0 && L + V <= a.n);
        double c[V];
        chunk_weights_sl<V>(a.mesh, L, sl_tab, c);
        VecT<float, V> X, Y;
        if constexpr (MODE == VA_INIT) {
            VecT<double, V> F;
            F.load(a.f + L);
            VecT<float, V> z;
#pragma unroll
            for (int t = 0; t < V; ++t) {
                X.v[t] = (float)F.v[t];  // C11
                z.v[t] = 0.0f;
            }
            X.store(a.r + L);
            z.store(a.x + L);
            z.store(a.p + L);
            Y = X;
        } else if constexpr (MODE == VA_RUPD) {
            VecT<float, V> W;
            W.load(a.w + L);
            X.load(a.r + L);
#pragma unroll
            for (int t = 0; t < V; ++t) X.v[t] = __fmaf_rn(am, W.v[t], X.v[t]);  // C8
            X.store(a.r + L);
            Y = X;
        } else {
            X.load(a.w + L);
            Y.load(a.p + L);
        }
#pragma unroll
        for (int t = 0; t < V; ++t) s = __fadd_rn(s, __fmul_rn(__fmul_rn(X.v[t], Y.v[t]), (float)c[t]));
    }
    const float bsum = block_reduce_f32(s);
    if (publish_and_check_last(a.parts, blockIdx.x, dd{(double)bsum, 0.0}, &a.st->cnt[1], gridDim.x)) {
        const int P = gridDim.x;
        const int lo = (int)((int64_t)P * threadIdx.x / blockDim.x);
        const int hi = (int)((int64_t)P * (threadIdx.x + 1) / blockDim.x);
        float t = 0.0f;
        for (int q = lo; q < hi; ++q) t = __fadd_rn(t, (float)__ldcg(&a.parts[q].hi));
        const float tot = block_reduce_f32(t);
        if (threadIdx.x == 0) {
            const dd v{(double)tot, 0.0};
            if (a.slot) {
                a.slot[0] = v;   // multi-rank: k_fin adds the rank sums in binary32, rank order
                a.slot[1] = v;
            } else if constexpr (MODE == VA_PAP) {
                fin_alpha(a.st, v, a.trace, true);
            } else if constexpr (MODE == VA_INIT) {
                fin_rtr<VEC_INIT>(a.st, v, v, a.hist, a.trace, true);
            } else {
                fin_rtr<VEC_RUPD>(a.st, v, v, a.hist, a.trace, true);
            }
            a.st->cnt[1] = 0;
        }
    }
}

// x = fma(alphaT, p, x) after the last iteration (deferred C8 x update).
// PM: the x update of "iteration niter + 1" (emulation key: op 1 of phase A, local index)
template <typename T, int PM = PM_NONE>
__global__ void __launch_bounds__(256) k_tail_x(T* x, const T* p, const CgState* st, int64_t n,
                                                PmArgs P, int it, MeshView m)
{
    T al;
    if constexpr (sizeof(T) == 8) al = (T)st->alpha; else al = (T)st->alpha32;
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n;
         L += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long key = 0;
        if constexpr (PM != PM_NONE) key = pm_key(it, PH_A, global_local_index(m, sl_natural(m, L)), 1);
        x[L] = pfma<PM>(al, p[L], x[L], P, key);
    }
}

// x64 = (double)x32 (exact, C12) ; G32/D32 = RN32(G64/D64) (C11).
static __global__ void __launch_bounds__(256) k_upcast(double* dst, const float* src, int64_t n)
{
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n;
         L += (int64_t)gridDim.x * blockDim.x)
        dst[L] = (double)src[L];
}
static __global__ void __launch_bounds__(256) k_downcast(float* dst, const double* src, int64_t n)
{
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n;
         L += (int64_t)gridDim.x * blockDim.x)
        dst[L] = __double2float_rn(src[L]);
}

// Natural order <-> split layout (SL) of a local-storage field (public-API
// arrays, host transfers of f / x / dinv).  One thread per natural point.
template <typename T, bool TO_SL>
__global__ void __launch_bounds__(256) k_perm_sl(T* dst, const T* src, MeshView m)
{
    const int N = m.N, N3 = N * N * N;
    const int64_t n = m.E * N3;
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n;
         L += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t e = fast_div((uint32_t)L, m.n3_mul, m.n3_shr);
        const uint32_t rem = (uint32_t)L - e * (uint32_t)N3;
        const uint32_t q1 = fast_div(rem, m.n_mul, m.n_shr);
        const uint32_t q2 = fast_div(q1, m.n_mul, m.n_shr);
        const int64_t Ls = (int64_t)e * N3 + sl_slot(N, (int)(rem - q1 * N), (int)(q1 - q2 * N), (int)q2);
        NBK_ASSERT(Ls >= (int64_t)e * N3 && Ls < (int64_t)(e + 1) * N3);
        if (TO_SL) dst[Ls] = src[L]; else dst[L] = src[Ls];
    }
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

// ------------------------------------------------------- multi-rank slabs
// Contiguous z-slabs (R21).  A global node on the plane between
// the slabs of ranks r and r+1 has its copies in the top element layer of
// rank r (k = N-1) and the bottom layer of rank r+1 (k = 0).  The canonical
// chain (C4: ascending GLOBAL local index) visits all of rank r's copies, in
// ascending element order, then all of rank r+1's.  Each rank sends the raw
// face layer of its own copies to the neighbour and both ranks evaluate the
// same chain from the same values: bit-identical sums on both sides, equal to
// the one-rank result.  The local dssum plan excludes these plane nodes.
template <typename T>
struct FaceArgs {
    T* w;
    const T* p;            // fused: p (face pap term, counted by the lower rank)
    T* send_lo;            // own bottom layer (k = 0 of local layer 0), ex*ey*N^2
    T* send_hi;            // own top layer (k = N-1 of the last local layer)
    const T* recv_lo;      // lower neighbour's top layer
    const T* recv_hi;      // upper neighbour's bottom layer
    int has_lo, has_hi;
    int mask;              // standalone: assign +0 to Dirichlet plane nodes (C5)
    dd* parts;             // fused: partials [0, nprev) of K_A and K_B, then this kernel's
    int nprev;
    int nskip;             // K_A's partials (already folded into K_B's)
    CgState* st;
    dd* slot;              // fused: this rank's reduced pap partial
    int single;            // paper-literal single mode (NEXT-2)
    MeshView mesh;
};

// Pack the raw face layers: layer index q = el*N^2 + j*N + i, el = ax + ex*ay.
template <typename T>
__global__ void __launch_bounds__(256) k_face_pack(FaceArgs<T> a)
{
    const int N = a.mesh.N, N2 = N * N, N3 = N2 * N;
    const int64_t nl = (int64_t)a.mesh.ex * a.mesh.ey * N2;
    const int64_t exy = (int64_t)a.mesh.ex * a.mesh.ey;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < 2 * nl;
         q += (int64_t)gridDim.x * blockDim.x) {
        const bool hi = q >= nl;
        const int64_t t = hi ? q - nl : q;
        if (hi ? !a.has_hi : !a.has_lo) continue;
        const int64_t el = t / N2;
        const int pos = (int)(t - el * N2);
        if (hi) {
            const int64_t e = (int64_t)(a.mesh.ez_local - 1) * exy + el;
            a.send_hi[t] = a.w[e * N3 + sl_plane(N, N - 1) + pos];
        } else {
            a.send_lo[t] = a.w[el * N3 + sl_plane(N, 0) + pos];
        }
    }
}

// Elements (ascending) containing global plane coordinate g along one axis.
__device__ __forceinline__ int plane_elems(int g, int ne, int N, int (&ae)[2], int (&loc)[2])
{
    const int n1 = N - 1;
    const int a = g / n1;
    int c = 0;
    if (g - a * n1 == 0) {
        if (a > 0) { ae[c] = a - 1; loc[c] = n1; ++c; }
        if (a < ne) { ae[c] = a; loc[c] = 0; ++c; }
    } else {
        ae[c] = a; loc[c] = g - a * n1; ++c;
    }
    return c;
}

template <typename T, bool FUSED>
__global__ void __launch_bounds__(256) k_face_merge(FaceArgs<T> a)
{
    const MeshView& m = a.mesh;
    const int N = m.N, N2 = N * N, N3 = N2 * N;
    const int Gx = m.ex * (N - 1) + 1, Gy = m.ey * (N - 1) + 1;
    const int64_t np = (int64_t)Gx * Gy;
    const int64_t exy = (int64_t)m.ex * m.ey;
    const int nplanes = a.has_lo + a.has_hi;
    acc_t acc;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nplanes * np;
         q += (int64_t)gridDim.x * blockDim.x) {
        const bool upper = a.has_lo ? (q >= np) : true;   // upper = shared with rank + 1
        const int64_t t = q >= np ? q - np : q;
        const int gy = (int)(t / Gx), gx = (int)(t - (int64_t)gy * Gx);
        int axe[2], il[2], aye[2], jl[2];
        const int nx = plane_elems(gx, m.ex, N, axe, il);
        const int ny = plane_elems(gy, m.ey, N, aye, jl);
        // own copies: layer base element and plane k
        const int64_t ebase = upper ? (int64_t)(m.ez_local - 1) * exy : 0;
        const int kpl = sl_plane(N, upper ? N - 1 : 0);   // SL slot of the face plane's (0, 0)
        const T* other = upper ? a.recv_hi : a.recv_lo;
        T sum = 0;
        bool first = true;
        // chain: lower rank's copies first (ascending element), then the upper's
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            const bool own = upper ? (side == 0) : (side == 1);
            for (int by = 0; by < ny; ++by)
                for (int bx = 0; bx < nx; ++bx) {
                    const int64_t el = axe[bx] + (int64_t)m.ex * aye[by];
                    const int pos = jl[by] * N + il[bx];
                    const T v = own ? a.w[(ebase + el) * N3 + kpl + pos]
                                    : other[el * N2 + pos];
                    sum = first ? v : add_t<T>(sum, v);
                    first = false;
                }
        }
        if (!FUSED && a.mask && (gx == 0 || gx == Gx - 1 || gy == 0 || gy == Gy - 1)) sum = 0;
        T p0 = 0;
        for (int by = 0; by < ny; ++by)
            for (int bx = 0; bx < nx; ++bx) {
                const int64_t el = axe[bx] + (int64_t)m.ex * aye[by];
                const int64_t L = (ebase + el) * N3 + kpl + jl[by] * N + il[bx];
                if (FUSED && by == 0 && bx == 0) p0 = a.p[L];
                a.w[L] = sum;
            }
        if constexpr (FUSED)
            if (upper) add_node_pap<T>(acc, sum, p0, 2 * nx * ny, a.single, PmArgs{52, 0});  // lower rank counts the node
    }
    if constexpr (FUSED) {
        dd v = block_reduce_dd(acc.get());
        if (publish_and_check_last(a.parts, a.nprev + blockIdx.x, v, &a.st->cnt[2], gridDim.x)) {
            dd tot = reduce_partials(a.parts + a.nskip, a.nprev - a.nskip + (int)gridDim.x);
            if (threadIdx.x == 0) {
                a.slot->hi = tot.hi;
                a.slot->lo = tot.lo;
                a.st->cnt[2] = 0;
            }
        }
    }
}

// Combine the P per-rank partials in rank order (identical on every rank)
// and run the scalar finaliser.  KIND: 0 = alpha (pap); 1 + VecMode = rtr etc.
// gather holds two dd per rank: [2r] the value, [2r + 1] rtz (Jacobi modes).
template <int KIND>
__global__ void k_fin(const dd* gather, int P, CgState* st, double* hist, double* trace, int single,
                      int pm, PmArgs pa)
{
    if (threadIdx.x != 0) return;
    dd t{__ldcg(&gather[0].hi), __ldcg(&gather[0].lo)};
    dd t2{__ldcg(&gather[1].hi), __ldcg(&gather[1].lo)};
    if (single == 2) {  // binary32 all-reduce (NEXT-2): rank sums added in binary32, rank order
        float f = (float)t.hi;
        for (int r = 1; r < P; ++r) f = __fadd_rn(f, (float)__ldcg(&gather[2 * r].hi));
        t = t2 = dd{(double)f, 0.0};
        single = 1;
    } else {
        for (int r = 1; r < P; ++r) {
            t = dd_add(t, dd{__ldcg(&gather[2 * r].hi), __ldcg(&gather[2 * r].lo)});
            t2 = dd_add(t2, dd{__ldcg(&gather[2 * r + 1].hi), __ldcg(&gather[2 * r + 1].lo)});
        }
    }
    if constexpr (KIND == 0) fin_alpha(st, t, trace, single, pm, pa);
    else fin_rtr<KIND - 1>(st, t, vec_jacobi(KIND - 1) ? t2 : t, hist, trace, single, pm, pa);
}

}  // namespace nbk
