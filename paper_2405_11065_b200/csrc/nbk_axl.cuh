// nbk_axl.cuh -- K_A in line-owner form (k_axl): the fused CG step of K_A
// (p = beta p + z, x += alpha_prev p_prev, w = D^T G D p_e + mask, element-
// interior pap; T1 lines 4-7) with the tensor contractions of ax_e
// (F2 local_grad3 / local_grad3_t, mxm at P:452-454) computed by LINE OWNERS:
// a thread that owns an r-line (j, k) of an element loads the N values of the
// line once and forms all N chains of that line, so each shared-memory word
// feeds N outputs instead of one.  The pencil form k_ax (nbk_kernels.cuh)
// loads a row or a column per output point: ~2.15 shared-memory wavefronts per
// point (ncu, C5 FP32), which co-bounded it with HBM.
//
// Same operations on the same operands as k_ax (rules C1-C3, C5, C8 of
// DESIGN.md CEO-1), so the result is bitwise identical; only which thread
// evaluates which chain, and when, differs.  Phases (one element = N^2
// threads; EPB elements per CTA):
//   P1  slot-linear (16-byte vectors, split layout order): p' = fma(beta, p, z),
//       x' = fma(alpha, p, x); p', x' stored to global (coalesced), p' kept in
//       shared memory (the p block arrives by TMA; r, x, dinv by vector loads).
//   P1b pencil (i, j): its column of p' from the SL block -> registers (ureg),
//       natural copy U[k][j][i] and transposed copy T[k][i][j].
//   P2  line owners: r-line (j, k): ur(., j, k) = D u(., j, k)   (in place in U)
//                    s-line (i, k): us(i, ., k) = D u(i, ., k)   (in place in T)
//   P3  pencil: ut = D u(i, j, .) from registers, metric (C2), wr -> U, ws -> T
//       in place; the t-part of the transpose b (C3) accumulated in registers.
//   P4  r-line owners: a(., j, k) = sum_l D[l][.] wr(l, j, k)  -> A (padded layout
//       in the dead G region, fewer bank conflicts for the column accesses)
//   P5  s-line owners: a(i, ., k) += sum_l D[l][.] ws(i, l, k)  (the same chain,
//       continued), in place in A
//   P6  pencil: w = a + b, mask (C5) -> P block in SL order (one TMA bulk store),
//       element-interior pap terms (C6).
// Shared memory per element: G (6 N^3, TMA) + P, U, T (N^3 each) = 9 N^3 values.
#pragma once
#include "nbk_kernels.cuh"

namespace nbk {

#ifndef NBK_AXL_EPB10_F32
#define NBK_AXL_EPB10_F32 1
#endif
#ifndef NBK_AXL_EPB8_F64
#define NBK_AXL_EPB8_F64 2
#endif
// N for which the fused CG step uses k_axl (bit N), FP32 / FP64.  Measured
// same-box against the pencil k_ax: C5 (N = 10) FP32 K_A
// 2.42 vs 2.76 ms, FP64 4.78 vs 5.28; C3 (N = 12) FP32 0.60 vs 0.645; C4
// (N = 8) FP32 0.567 vs 0.593 but FP64 1.37 vs 1.19 ms (off).
#ifndef NBK_AXL_MASK32
#define NBK_AXL_MASK32 ((1 << 4) | (1 << 6) | (1 << 8) | (1 << 10) | (1 << 12))
#endif
#ifndef NBK_AXL_MASK64
#define NBK_AXL_MASK64 ((1 << 4) | (1 << 6) | (1 << 10) | (1 << 12))
#endif
#ifdef NBK_AXL_MASK   // one mask for both (A/B builds)
#undef NBK_AXL_MASK32
#undef NBK_AXL_MASK64
#define NBK_AXL_MASK32 NBK_AXL_MASK
#define NBK_AXL_MASK64 NBK_AXL_MASK
#endif

template <typename T>
__host__ __device__ constexpr int axl_epb(int N)
{
    if (N == 10) return sizeof(T) == 4 ? NBK_AXL_EPB10_F32 : 1;
    if (N == 8 && sizeof(T) == 8) return NBK_AXL_EPB8_F64;
    if (N >= 10) return 1;
    // at least 2 warps of work per CTA
    int e = 128 / (N * N);
    return e < 1 ? 1 : e;
}
// Padded layout of the transpose chain a(i, j, k) (P4 -> P5 -> P6) in the dead
// G region: a at i + R j + P k.  Chosen by a bank-conflict search over the
// P4 row stores, the P5 column loads / stores and the P6 pencil loads (lane
// maps as used below): N = 10 wavefront estimate 380 -> 260 per warp group.
#ifndef NBK_AXL_PAD
#define NBK_AXL_PAD 1   // 0: natural layout (A/B)
#endif
__host__ __device__ constexpr int axl_pr(int N)
{
    return !NBK_AXL_PAD ? N : (N == 8 ? 9 : (N == 10 || N == 12 ? 17 : N));
}
__host__ __device__ constexpr int axl_pp(int N)
{
    return !NBK_AXL_PAD ? N * N : (N == 8 ? 72 : (N == 10 ? 170 : (N == 12 ? 204 : N * N)));
}
template <typename T>
__host__ __device__ constexpr int axl_threads(int N)
{
    return (N * N * axl_epb<T>(N) + 31) / 32 * 32;
}
// NBK_AXL_SMEM8: 8 N^3 values per element -- p arrives by vector loads and its
// SL block sits in the T buffer until the copies are made, w leaves from the
// dead G region (one bulk store per element); 0: 9 N^3 (p by TMA into its own block).
// Default (-1): where it was measured faster (same-box, bench events): FP64 N = 12 (124 ->
// 111 KB per element, 1 -> 2 CTAs/SM: C3 FP64 K_A 1.16 vs 1.32 ms with the pencil kernel)
// and FP32 N = 10 (7 instead of 6 CTAs/SM at 72 registers: C5 K_A 2.16 vs 2.21 ms).  Not
// elsewhere: FP64 N = 10 spills (4.77 vs 4.42 ms), FP32 N = 8 / 12 lose (0.53 vs 0.52 ms).
#ifndef NBK_AXL_SMEM8
#define NBK_AXL_SMEM8 -1
#endif
template <typename T>
__host__ __device__ constexpr bool axl_s8(int N)
{
    return NBK_AXL_SMEM8 >= 0 ? NBK_AXL_SMEM8 != 0 : (sizeof(T) == 8 ? N == 12 : N == 10);
}
template <typename T>
__host__ __device__ constexpr int axl_smem_bytes(int N)
{
    return (axl_s8<T>(N) ? 8 : 9) * axl_epb<T>(N) * N * N * N * (int)sizeof(T);
}
template <typename T>
__host__ __device__ constexpr int axl_min_blocks(int N)
{
    // 228 KB of shared memory per SM; per CTA 1 KB reserved + the static 128 B (bars, red)
    int by_smem = 233472 / (axl_smem_bytes<T>(N) + 1024 + 256);
    int by_thr = 2048 / axl_threads<T>(N);
    int m = by_smem < by_thr ? by_smem : by_thr;
    return m < 1 ? 1 : m;
}
// k_axl serves the fused CG step (FUSED 1, 2) without emulation, for even N
// (16-byte bulk copies and vectors) whose 9 N^3 block fits beside >= 2 CTAs/SM.
template <typename T>
__host__ __device__ constexpr bool axl_on(int N, int fused, int pm)
{
    return fused >= 1 && pm == PM_NONE && N % 2 == 0 && N >= 4 &&
           (((sizeof(T) == 4 ? NBK_AXL_MASK32 : NBK_AXL_MASK64) >> N) & 1) &&
           axl_min_blocks<T>(N) >= 2 && axl_smem_bytes<T>(N) <= 200 * 1024;
}

template <typename T, int N>
__device__ __forceinline__ void sts_row(T* dst, const T (&src)[N])
{
    constexpr int RB = N * (int)sizeof(T);
    if constexpr (RB % 16 == 0) {
#pragma unroll
        for (int q = 0; q < RB / 16; ++q) {
            if constexpr (sizeof(T) == 4)
                reinterpret_cast<float4*>(dst)[q] =
                    make_float4(src[4 * q], src[4 * q + 1], src[4 * q + 2], src[4 * q + 3]);
            else
                reinterpret_cast<double2*>(dst)[q] = make_double2(src[2 * q], src[2 * q + 1]);
        }
    } else if constexpr (RB % 8 == 0 && sizeof(T) == 4) {
#pragma unroll
        for (int q = 0; q < N / 2; ++q)
            reinterpret_cast<float2*>(dst)[q] = make_float2(src[2 * q], src[2 * q + 1]);
    } else {
#pragma unroll
        for (int q = 0; q < N; ++q) dst[q] = src[q];
    }
}

// 16-byte vector of T
template <typename T> struct Vec16;
template <> struct Vec16<float> {
    using type = float4;
    static constexpr int n = 4;
};
template <> struct Vec16<double> {
    using type = double2;
    static constexpr int n = 2;
};
template <typename V, typename T>
__device__ __forceinline__ T& vat(V& v, int q)
{
    return reinterpret_cast<T*>(&v)[q];
}

// D and its transpose as a kernel parameter (constant bank): FP32 pairs of
// adjacent coefficients feed packed FFMA2 as one uniform-register operand.
template <typename T, int N>
struct DMat {
    alignas(16) T d[N * N];    // d[a N + b] = D[a][b]
    alignas(16) T dt[N * N];   // dt[a N + b] = D[b][a]
};

// out[o] = sum_l D[o][l] v[l] (TR = 0) or sum_l D[l][o] v[l] (TR = 1), every
// chain from +0 in ascending l (rule C1 / C3).  FP32: chains o, o + 1 in one
// FFMA2 (per-lane numerics of __fmaf_rn, so each chain is unchanged).
template <typename T, int N, int TR>
__device__ __forceinline__ void line_chains(T (&out)[N], const T (&v)[N], const DMat<T, N>& dm)
{
    const T* c = TR ? dm.d : dm.dt;   // c[l N + o] = coefficient of v[l] in out[o]
#pragma unroll
    for (int o = 0; o < N; ++o) out[o] = 0;
    if constexpr (sizeof(T) == 4 && N % 2 == 0) {
#pragma unroll
        for (int l = 0; l < N; ++l) {
            const float2 vv = make_float2(v[l], v[l]);
#pragma unroll
            for (int o = 0; o < N; o += 2) {
                const float2 r = __ffma2_rn(make_float2(c[l * N + o], c[l * N + o + 1]), vv,
                                            make_float2(out[o], out[o + 1]));
                out[o] = r.x;
                out[o + 1] = r.y;
            }
        }
    } else {
#pragma unroll
        for (int l = 0; l < N; ++l)
#pragma unroll
            for (int o = 0; o < N; ++o) out[o] = fma_t<T>(c[l * N + o], v[l], out[o]);
    }
}
// s[o] = fma(D[l][o], v[l], s[o]) for l ascending, continuing existing chains
template <typename T, int N>
__device__ __forceinline__ void line_chains_cont(T (&s)[N], const T (&v)[N], const DMat<T, N>& dm)
{
    if constexpr (sizeof(T) == 4 && N % 2 == 0) {
#pragma unroll
        for (int l = 0; l < N; ++l) {
            const float2 vv = make_float2(v[l], v[l]);
#pragma unroll
            for (int o = 0; o < N; o += 2) {
                const float2 r = __ffma2_rn(make_float2(dm.d[l * N + o], dm.d[l * N + o + 1]), vv,
                                            make_float2(s[o], s[o + 1]));
                s[o] = r.x;
                s[o + 1] = r.y;
            }
        }
    } else {
#pragma unroll
        for (int l = 0; l < N; ++l)
#pragma unroll
            for (int o = 0; o < N; ++o) s[o] = fma_t<T>(dm.d[l * N + o], v[l], s[o]);
    }
}

template <typename T, int N, int FUSED>
__global__ void __launch_bounds__(axl_threads<T>(N), axl_min_blocks<T>(N))
    k_axl(AxArgs<T> a, const __grid_constant__ DMat<T, N> dc)
{
    constexpr int N2 = N * N, N3 = N * N * N, EPB = axl_epb<T>(N), NT = axl_threads<T>(N);
    using V = typename Vec16<T>::type;
    constexpr int VN = Vec16<T>::n;
    constexpr int NVT = (EPB * N3 / VN + NT - 1) / NT;   // vectors per thread in P1
    static_assert((N3 * (int)sizeof(T)) % 16 == 0, "k_axl needs 16-byte element blocks");
    constexpr bool S8 = axl_s8<T>(N);
    __shared__ __align__(8) uint64_t bar[2];   // 0: p block, 1: G block
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* sG = reinterpret_cast<T*>(smem_raw);   // EPB * 6 N^3: G -> a (padded) + w (SL, S8)
    T* sP = sG + EPB * 6 * N3;                // !S8: EPB * N^3: p (SL) -> w (SL)
    T* sU = S8 ? sP : sP + EPB * N3;          // EPB * N^3: u -> ur -> wr (natural)
    T* sT = sU + EPB * N3;                    // EPB * N^3: (S8: p SL ->) u^T -> us^T -> ws^T

    const int tid = threadIdx.x;
    const int el = tid / N2, ij = tid - el * N2;
    const int i = ij % N, j = ij / N;   // pencil (i, j, *)
    const int lo = ij % N, ko = ij / N; // line owner: r-line (j = lo, k = ko), s-line (i = lo, k = ko)
    const int64_t bl = (int64_t)(a.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
    const int64_t nb0 = (a.en0 + EPB - 1) / EPB;
    const int64_t e0 = bl < nb0 ? a.eb0 + bl * EPB : a.eb1 + (bl - nb0) * EPB;
    const int64_t eend = bl < nb0 ? a.eb0 + a.en0 : a.eb1 + a.en1;
    const int64_t e = e0 + el;
    const int nel = (int)((eend - e0) < EPB ? (eend - e0) : EPB);
    const bool valid = el < nel;
    NBK_ASSERT(nel >= 1 && e0 + nel <= a.mesh.E);
    const int nv = nel * N3 / VN;   // vectors of the CTA's slot range

    // ---- loads: G and p by TMA (G before the PDL wait; p too once it is
    // final, CG iterations >= 2), x / dinv / r by 16-byte vector loads in slot order
    const uint32_t pbytes = (uint32_t)(nel * N3 * sizeof(T));
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        if (!S8 && a.p_ready) {
            mbar_arrive_expect_tx(&bar[0], pbytes);
            tma_load_1d(sP, a.p + e0 * N3, pbytes, &bar[0]);
        }
        const uint32_t gbytes = (uint32_t)(nel * 6 * N3 * sizeof(T));
        mbar_arrive_expect_tx(&bar[1], gbytes);
        tma_load_1d(sG, a.G + e0 * 6 * N3, gbytes, &bar[1]);
    }
    const V* xg = reinterpret_cast<const V*>(a.x + e0 * N3);
    const V* rg = reinterpret_cast<const V*>(a.r + e0 * N3);
    const V* dg = reinterpret_cast<const V*>(FUSED == 2 ? a.dinv + e0 * N3 : a.r);
    const V* pgi = reinterpret_cast<const V*>(a.p + e0 * N3);
    V xv[NVT], rv[NVT], dv[FUSED == 2 ? NVT : 1], pv[S8 ? NVT : 1];
    auto load_xd = [&]() {
#pragma unroll
        for (int q = 0; q < NVT; ++q) {
            const int v = tid + q * NT;
            if (v < nv) {
                xv[q] = xg[v];
                if constexpr (S8) pv[q] = pgi[v];
                if constexpr (FUSED == 2) dv[q] = __ldg(dg + v);
            }
        }
    };
    if (a.p_ready) load_xd();
    pdl_wait();
    if (!a.p_ready) {
        if (!S8 && tid == 0) {
            mbar_arrive_expect_tx(&bar[0], pbytes);
            tma_load_1d(sP, a.p + e0 * N3, pbytes, &bar[0]);
        }
        load_xd();
    }
#pragma unroll
    for (int q = 0; q < NVT; ++q) {
        const int v = tid + q * NT;
        if (v < nv) rv[q] = rg[v];
    }
    T betaT, alphaT;
    if constexpr (sizeof(T) == 8) {
        betaT = (T)a.st->beta;
        alphaT = (T)a.st->alpha;
    } else {
        betaT = (T)a.st->beta32;
        alphaT = (T)a.st->alpha32;
    }
    __syncthreads();   // barrier init visible
    if constexpr (!S8) mbar_wait(&bar[0], 0);

    // ---- P1: p = fma(beta, p, z), x = fma(alpha_prev, p_prev, x)  (C8), slot order
    {
        V* sPv = reinterpret_cast<V*>(S8 ? sT : sP);   // p' in SL order
        V* pg = reinterpret_cast<V*>(a.p + e0 * N3);
        V* xo = reinterpret_cast<V*>(a.x + e0 * N3);
#pragma unroll
        for (int q = 0; q < NVT; ++q) {
            const int v = tid + q * NT;
            if (v < nv) {
                V po;
                if constexpr (S8) po = pv[q];
                else po = sPv[v];
                V pn, xn;
#pragma unroll
                for (int c = 0; c < VN; ++c) {
                    T z = vat<const V, const T>(rv[q], c);
                    if constexpr (FUSED == 2) z = mul_t<T>(z, vat<const V, const T>(dv[q], c));  // solveM
                    const T p0 = vat<const V, const T>(po, c);
                    vat<V, T>(pn, c) = fma_t<T>(betaT, p0, z);
                    vat<V, T>(xn, c) = fma_t<T>(alphaT, p0, vat<const V, const T>(xv[q], c));
                }
                sPv[v] = pn;
                pg[v] = pn;
                xo[v] = xn;
            }
        }
    }
    __syncthreads();

    T* Ue = sU + el * N3;
    T* Te = sT + el * N3;
    // w in SL order: !S8 the p block, S8 the dead G region behind the padded a
    T* We = S8 ? sG + el * 6 * N3 + 3 * N3 : sP + el * N3;
    const SlCol cs = sl_col(N, i, j);
    NBK_ASSERT(!valid || (cs.at(N, 0) >= 0 && cs.at(N, N - 1) < N3 && cs.at(N, N / 2) < N3));

    // ---- P1b: the pencil's column of p' (registers) + natural and transposed copies
    T ureg[N];
    if constexpr (S8) {
        if (valid) {
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const T v = Te[cs.at(N, k)];
                ureg[k] = v;
                Ue[k * N2 + j * N + i] = v;
            }
        }
        __syncthreads();   // the SL block in T is consumed
        if (valid) {
#pragma unroll
            for (int k = 0; k < N; ++k) Te[k * N2 + i * N + j] = ureg[k];
        }
    } else if (valid) {
        const T* Pe = sP + el * N3;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const T v = Pe[cs.at(N, k)];
            ureg[k] = v;
            Ue[k * N2 + j * N + i] = v;
            Te[k * N2 + i * N + j] = v;
        }
    }
    __syncthreads();

    // ---- P2: gradient along r and s by line owners (C1), in place
    if (valid) {
        T v[N], o[N];
        lds_row<T, N>(v, Ue + ko * N2 + lo * N);   // u(., lo, ko)
        line_chains<T, N, 0>(o, v, dc);            // ur(o, lo, ko) = sum_l D[o][l] u(l, lo, ko)
        sts_row<T, N>(Ue + ko * N2 + lo * N, o);
        lds_row<T, N>(v, Te + ko * N2 + lo * N);   // u(lo, ., ko)
        line_chains<T, N, 0>(o, v, dc);            // us(lo, o, ko) = sum_l D[o][l] u(lo, l, ko)
        sts_row<T, N>(Te + ko * N2 + lo * N, o);
    }
    __syncthreads();

    // ---- P3: ut from registers (C1), metric (C2), t-part b of the transpose (C3)
    T b[N];
#pragma unroll
    for (int k = 0; k < N; ++k) b[k] = 0;
    if (valid) {
        T ut[N];
        line_chains<T, N, 0>(ut, ureg, dc);   // ut(i, j, o) = sum_l D[o][l] u(i, j, l)
        mbar_wait(&bar[1], 0);
        const T* Ge = sG + el * 6 * N3 + ij;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const T ur = Ue[k * N2 + j * N + i];
            const T us = Te[k * N2 + i * N + j];
            const T g1 = Ge[0 * N3 + k * N2], g2 = Ge[1 * N3 + k * N2], g3 = Ge[2 * N3 + k * N2];
            const T g4 = Ge[3 * N3 + k * N2], g5 = Ge[4 * N3 + k * N2], g6 = Ge[5 * N3 + k * N2];
            T wr, ws;
            if constexpr (sizeof(T) == 4) {  // wr, ws chains side by side (FMUL2 / FFMA2)
                float2 q = __fmul2_rn(make_float2(g1, g2), make_float2(ur, ur));
                q = __ffma2_rn(make_float2(g2, g4), make_float2(us, us), q);
                q = __ffma2_rn(make_float2(g3, g5), make_float2(ut[k], ut[k]), q);
                wr = q.x;
                ws = q.y;
            } else {
                wr = mul_t<T>(g1, ur);
                wr = fma_t<T>(g2, us, wr);
                wr = fma_t<T>(g3, ut[k], wr);
                ws = mul_t<T>(g2, ur);
                ws = fma_t<T>(g4, us, ws);
                ws = fma_t<T>(g5, ut[k], ws);
            }
            T wt = mul_t<T>(g3, ur);
            wt = fma_t<T>(g5, us, wt);
            wt = fma_t<T>(g6, ut[k], wt);
            Ue[k * N2 + j * N + i] = wr;
            Te[k * N2 + i * N + j] = ws;
            T Dk[N];
#pragma unroll
            for (int l = 0; l < N; ++l) Dk[l] = dc.d[k * N + l];
            fma_row<T, N>(b, Dk, wt);   // b(i, j, kk) += D[k][kk] wt(i, j, k)
        }
    }
    __syncthreads();

    // ---- P4: r-part of the transpose chain (C3) by r-line owners -> A (padded,
    // in the dead G region)
    constexpr int PR = axl_pr(N), PP = axl_pp(N);
    static_assert(PR * (N - 1) + N <= PP && PP * N <= 3 * N3, "k_axl: padded a does not fit");
    T* Ae = sG + el * 6 * N3;
    if (valid) {
        T v[N], o[N];
        lds_row<T, N>(v, Ue + ko * N2 + lo * N);   // wr(., lo, ko)
        line_chains<T, N, 1>(o, v, dc);            // a(o, lo, ko) = sum_l D[l][o] wr(l, lo, ko)
#pragma unroll
        for (int q = 0; q < N; ++q) Ae[q + PR * lo + PP * ko] = o[q];
    }
    __syncthreads();

    // ---- P5: s-part of the same chain by s-line owners, in place in A
    if (valid) {
        T v[N], s[N];
#pragma unroll
        for (int o = 0; o < N; ++o) s[o] = Ae[lo + PR * o + PP * ko];   // a(lo, o, ko)
        lds_row<T, N>(v, Te + ko * N2 + lo * N);                        // ws(lo, ., ko)
        line_chains_cont<T, N>(s, v, dc);
#pragma unroll
        for (int o = 0; o < N; ++o) Ae[lo + PR * o + PP * ko] = s[o];
    }
    __syncthreads();

    // ---- P6: w = a + b, mask (C5), SL order into P, element-interior pap (C6)
    acc_t acc;
    if (valid) {
        const ElemCoord ec = elem_coord(a.mesh, (uint32_t)e);
        const int n1 = N - 1;
        const bool mxy = (i == 0 && ec.ax == 0) || (i == n1 && ec.ax == a.mesh.ex - 1) ||
                         (j == 0 && ec.ay == 0) || (j == n1 && ec.ay == a.mesh.ey - 1);
        const bool sxy = (i == 0 && ec.ax > 0) || (i == n1 && ec.ax < a.mesh.ex - 1) ||
                         (j == 0 && ec.ay > 0) || (j == n1 && ec.ay < a.mesh.ey - 1);
        const bool mz0 = ec.azg == 0, mz1 = ec.azg == a.mesh.ezg - 1;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            T wv = add_t<T>(Ae[i + PR * j + PP * k], b[k]);
            const bool masked = mxy || (k == 0 && mz0) || (k == n1 && mz1);
            if (a.mask && masked) wv = 0;   // C5: assign +0
            We[cs.at(N, k)] = wv;
            // element-interior points only; the others add +0, a no-op of the
            // accumulator (its sum starts at +0 and is never -0), so no branch
            const bool sz = (k == 0 && !mz0) || (k == n1 && !mz1);
            // term with c = 1 (rule C6): FP32 vectors (double)w (double)p, exact
            // (single mode: RN32(w p)); FP64 RN(w p) -- dot_term(w, p, 1.0) without the * 1
            double t;
            if constexpr (sizeof(T) == 4)
                t = a.single ? (double)__fmul_rn(wv, ureg[k]) : __dmul_rn((double)wv, (double)ureg[k]);
            else
                t = __dmul_rn(wv, ureg[k]);
            acc.add(!sxy && !sz ? t : 0.0);
        }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
        if constexpr (S8) {
            for (int q = 0; q < nel; ++q)
                tma_store_1d(a.w + (e0 + q) * N3, sG + q * 6 * N3 + 3 * N3, (uint32_t)(N3 * sizeof(T)));
        } else {
            tma_store_1d(a.w + e0 * N3, sP, pbytes);
        }
        bulk_commit();
    }
    pdl_launch_dependents();
    // pap partial of the block: every thread's dd into the dead G region, then
    // warp 0 alone combines them in a fixed order (lane l: entries l, l + 32,
    // ..., then a shuffle tree) -- 8 warp-level dd additions per block instead
    // of 5 per warp plus 5 (block_reduce_dd)
    dd* red = reinterpret_cast<dd*>(sG);
    red[tid] = acc.get();
    __syncthreads();
    if (tid < 32) {
        dd v = red[tid];
#pragma unroll
        for (int q = 1; q < NT / 32; ++q) v = dd_add(v, red[tid + 32 * q]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = dd_add(v, shfl_down_dd(v, off));
        if (tid == 0) {
            a.parts[a.part_off + blockIdx.x] = v;
            bulk_wait_all();   // shared memory stays valid until the store is done
        }
    }
}

}  // namespace nbk
