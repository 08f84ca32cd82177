// nbk_common.cuh -- device helpers shared by the libnbk kernels (sm_100a).
//
//  * double-double (dd) arithmetic for the FP64-accumulated inner products
//    glsc3 (T1 lines 3, 6, 9; north_star "FP64 accumulation even in the FP32
//    solver"; rule C6: one final rounding of a ~106-bit accurate sum);
//  * structural per-point data of the box mesh: Dirichlet mask (R6) and the
//    multiplicity m (c = 1/m, R8), computed from indices -- 0 bytes of HBM;
//  * deterministic warp / block reductions of dd values (fixed trees, no
//    atomics on values: bitwise reproducible for a fixed launch shape).
//
// The whole library is compiled with -fmad=false: no add/mul is contracted
// into an FMA except the explicit __fma_rn / __fmaf_rn calls of the canonical
// evaluation order (CEO-1).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nbk {

// Bounds checks of a debug build (-DNBK_CHECK_BOUNDS; compute-sanitizer is not
// available on the GPU pool): a failed check traps the kernel, the CUDA call
// returns an error and the test fails.
#ifdef NBK_CHECK_BOUNDS
#define NBK_ASSERT(cond) \
    do {                 \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define NBK_ASSERT(cond) \
    do {                 \
    } while (0)
#endif

// ------------------------------------------------------------------ dd
struct dd {
    double hi, lo;
};

// Knuth TwoSum: s + e == a + b exactly (no branch).
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e)
{
    s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// Dekker Fast2Sum (|a| >= |b| or a == 0).
__device__ __forceinline__ void fast_two_sum(double a, double b, double& s, double& e)
{
    s = __dadd_rn(a, b);
    e = __dsub_rn(b, __dsub_rn(s, a));
}

// Non-finite operands: the plain IEEE sum (inf + finite = inf, inf - inf =
// NaN), as the exact sum with special values is defined (TwoSum would turn
// the error terms into NaN).
__device__ __forceinline__ dd dd_add(dd a, dd b)
{
    double s, e, t, f;
    two_sum(a.hi, b.hi, s, e);
    const double plain = s;   // selects below, no branch: this sits in serial reductions
    two_sum(a.lo, b.lo, t, f);
    e = __dadd_rn(e, t);
    fast_two_sum(s, e, s, e);
    e = __dadd_rn(e, f);
    fast_two_sum(s, e, s, e);
    const bool fin = isfinite(plain);
    return dd{fin ? s : plain, fin ? e : 0.0};
}

// Per-thread accumulator: running sum S plus the exact TwoSum errors in C.
struct acc_t {
    double s = 0.0, c = 0.0;
    __device__ __forceinline__ void add(double t)
    {
        double s2, e;
        two_sum(s, t, s2, e);
        s = s2;
        c = __dadd_rn(c, e);
    }
    __device__ __forceinline__ dd get() const
    {
        if (!isfinite(s)) return dd{s, 0.0};  // an infinite / NaN term (S is the plain IEEE sum)
        double h, l;
        two_sum(s, c, h, l);
        return dd{h, l};
    }
};

__device__ __forceinline__ dd shfl_down_dd(dd v, int off)
{
    dd o;
    o.hi = __shfl_down_sync(0xffffffffu, v.hi, off);
    o.lo = __shfl_down_sync(0xffffffffu, v.lo, off);
    return o;
}

// Fixed-tree block reduction; result valid in thread 0.  Must be called by
// every thread of the block (blockDim.x a multiple of 32, <= 1024).
__device__ __forceinline__ dd block_reduce_dd(dd v)
{
    __shared__ dd red_smem[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = dd_add(v, shfl_down_dd(v, off));
    __syncthreads();  // red_smem may be reused by a previous call
    if (lane == 0) red_smem[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = lane < nw ? red_smem[lane] : dd{0.0, 0.0};
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = dd_add(v, shfl_down_dd(v, off));
    }
    return v;
}

// Reduce n dd partials in a fixed order with one block (all threads call).
// Thread t owns partials t, t+T, t+2T, ... (combined in that order); the loads
// of a batch are issued together so the tail costs ~one L2 round trip.
__device__ __forceinline__ dd reduce_partials(const dd* parts, int n)
{
    constexpr int B = 8;
    dd v{0.0, 0.0};
    for (int q0 = threadIdx.x; q0 < n; q0 += B * blockDim.x) {
        dd p[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int q = q0 + b * blockDim.x;
            if (q < n) {
                p[b].hi = __ldcg(&parts[q].hi);
                p[b].lo = __ldcg(&parts[q].lo);
            } else {
                p[b] = dd{0.0, 0.0};
            }
        }
#pragma unroll
        for (int b = 0; b < B; ++b) v = dd_add(v, p[b]);
    }
    return block_reduce_dd(v);
}

// "Last block finalises": every block publishes its partial, then the block
// that increments the counter last reduces all partials (order fixed by the
// partial index, so the result does not depend on which block is last).
// Release/acquire through the counter (atom.acq_rel), no SC fence.
// Returns true in the last block (all threads).
__device__ __forceinline__ bool publish_and_check_last(dd* parts, int slot, dd v,
                                                       unsigned int* counter, unsigned int total)
{
    __shared__ unsigned int last_flag;
    if (threadIdx.x == 0) {
        __stcg(&parts[slot].hi, v.hi);
        __stcg(&parts[slot].lo, v.lo);
        unsigned int prev;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;"
                     : "=r"(prev)
                     : "l"(counter)
                     : "memory");
        last_flag = (prev == total - 1) ? 1u : 0u;
    }
    __syncthreads();
    return last_flag != 0;
}

// Programmatic dependent launch (PDL): let the next kernel in the stream be
// scheduled early / wait for the previous kernel's results.
__device__ __forceinline__ void pdl_launch_dependents()
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ------------------------------------------------------------------ mesh
// Rank-local view of the global box mesh (contiguous z-slab, R21).
struct MeshView {
    int ex, ey;          // elements in x, y
    int ez_local, z0;    // element layers on this rank and the first global layer
    int ezg;             // global element layers
    int N;
    int64_t E;           // local elements
    // magic numbers for division by ex, ex*ey, N and N^3 (uint32 fast division)
    uint32_t ex_mul, ex_shr, exy_mul, exy_shr;
    uint32_t n_mul, n_shr, n3_mul, n3_shr;
};

// q = floor(n / d) with (mul, shr) from make_fast_div (round-up method of
// Granlund & Montgomery; exact for every 32-bit n).
__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t mul, uint32_t shr)
{
    return (uint32_t)(((uint64_t)__umulhi(n, mul) + n) >> shr);
}

struct ElemCoord {
    int ax, ay, azg;
};

__device__ __forceinline__ ElemCoord elem_coord(const MeshView& m, uint32_t e)
{
    uint32_t az = fast_div(e, m.exy_mul, m.exy_shr);
    uint32_t rem = e - az * (uint32_t)(m.ex * m.ey);
    uint32_t ay = fast_div(rem, m.ex_mul, m.ex_shr);
    uint32_t ax = rem - ay * (uint32_t)m.ex;
    return ElemCoord{(int)ax, (int)ay, (int)az + m.z0};
}

// Dirichlet node (R6): on any face of the global box.
__device__ __forceinline__ bool is_masked(const MeshView& m, const ElemCoord& c, int i, int j,
                                          int k)
{
    const int n1 = m.N - 1;
    return (i == 0 && c.ax == 0) || (i == n1 && c.ax == m.ex - 1) || (j == 0 && c.ay == 0) ||
           (j == n1 && c.ay == m.ey - 1) || (k == 0 && c.azg == 0) ||
           (k == n1 && c.azg == m.ezg - 1);
}

// Multiplicity of the node (number of elements sharing it, R8).
__device__ __forceinline__ int multiplicity(const MeshView& m, const ElemCoord& c, int i, int j,
                                            int k)
{
    const int n1 = m.N - 1;
    int mx = ((i == 0 && c.ax > 0) || (i == n1 && c.ax < m.ex - 1)) ? 2 : 1;
    int my = ((j == 0 && c.ay > 0) || (j == n1 && c.ay < m.ey - 1)) ? 2 : 1;
    int mz = ((k == 0 && c.azg > 0) || (k == n1 && c.azg < m.ezg - 1)) ? 2 : 1;
    return mx * my * mz;
}

// ------------------------------------------------------------ split layout
// Element-local storage order of the CG vectors x, r, p, w, f and dinv inside
// the library ("split layout", SL; G and the public-API arrays stay natural,
// i fastest).  Slots [0, I^3) of an element (I = N - 2) hold its interior
// points in natural order; slots [I^3, N^3) its boundary points, also in
// natural order: the k = 0 face (N^2 points), then per inner plane k = 1..N-2
// its ring of R = 4 (N - 1) points (row j = 0, the pairs i = 0 / i = N-1 of
// rows 1..N-2, row j = N-1), then the k = N-1 face.  Every copy of a shared
// node is a boundary point, so dssum reads and writes only the compact tail of
// each element (whole 32-byte sectors) instead of every sector the stride-N
// x-face points of the natural order touch.
__host__ __device__ __forceinline__ int sl_slot(int N, int i, int j, int k)
{
    const int I = N - 2, n1 = N - 1;
    if (i > 0 && i < n1 && j > 0 && j < n1 && k > 0 && k < n1) return ((k - 1) * I + (j - 1)) * I + (i - 1);
    const int B = I * I * I, R = 4 * n1;
    if (k == 0) return B + j * N + i;
    if (k == n1) return B + N * N + (N - 2) * R + j * N + i;
    int r;
    if (j == 0) r = i;
    else if (j == n1) r = N + 2 * (N - 2) + i;
    else r = N + 2 * (j - 1) + (i == n1 ? 1 : 0);
    return B + N * N + (k - 1) * R + r;
}
// Inverse: the natural (i, j, k) of slot s.
__host__ __device__ __forceinline__ void sl_point(int N, int s, int& i, int& j, int& k)
{
    const int I = N - 2, n1 = N - 1, B = I * I * I, R = 4 * n1;
    if (s < B) {
        i = 1 + s % I;
        j = 1 + (s / I) % I;
        k = 1 + s / (I * I);
        return;
    }
    int f = s - B;
    if (f < N * N) { i = f % N; j = f / N; k = 0; return; }
    f -= N * N;
    if (f < (N - 2) * R) {
        k = 1 + f / R;
        int r = f - (k - 1) * R;
        if (r < N) { i = r; j = 0; }
        else if (r < N + 2 * (N - 2)) { r -= N; j = 1 + r / 2; i = (r & 1) ? n1 : 0; }
        else { i = r - N - 2 * (N - 2); j = n1; }
        return;
    }
    f -= (N - 2) * R;
    i = f % N; j = f / N; k = n1;
}
// First SL slot of the k = 0 or the k = N-1 face (N^2 slots in natural (j, i) order).
__host__ __device__ __forceinline__ int sl_plane(int N, int k)
{
    const int I = N - 2;
    return I * I * I + (k == 0 ? 0 : N * N + (N - 2) * 4 * (N - 1));
}
// Per-thread slot bases of column (i, j): slot(k) = k == 0 ? b0 : k == N-1 ? b1 : bm + (k-1) st.
struct SlCol {
    int b0, b1, bm, st;
    __host__ __device__ __forceinline__ int at(int N, int k) const
    {
        return k == 0 ? b0 : (k == N - 1 ? b1 : bm + (k - 1) * st);
    }
};
__host__ __device__ __forceinline__ SlCol sl_col(int N, int i, int j)
{
    SlCol c;
    const int I = N - 2, n1 = N - 1, B = I * I * I, R = 4 * n1;
    c.b0 = B + j * N + i;
    c.b1 = B + N * N + (N - 2) * R + j * N + i;
    if (i > 0 && i < n1 && j > 0 && j < n1) {
        c.bm = (j - 1) * I + (i - 1);
        c.st = I * I;
    } else {
        c.bm = N > 2 ? sl_slot(N, i, j, 1) : 0;
        c.st = R;
    }
    return c;
}

// c = 1/m is exact (m in {1,2,4,8}).
__device__ __forceinline__ double inv_mult(int m)
{
    return m == 1 ? 1.0 : (m == 2 ? 0.5 : (m == 4 ? 0.25 : 0.125));
}

// glsc3 term (C6): FP64 vectors -> RN64(a b) c ; FP32 vectors -> exact product.
__device__ __forceinline__ double dot_term(double a, double b, double c)
{
    return __dmul_rn(__dmul_rn(a, b), c);
}
__device__ __forceinline__ double dot_term(float a, float b, double c)
{
    return __dmul_rn(__dmul_rn((double)a, (double)b), c);
}
// Paper-literal single-precision glsc3 (NEXT-2): the product rounded to
// binary32 first, RN32(a b) c (c = 1/m, exact).  FP64 vectors: unchanged.
__device__ __forceinline__ double dot_term(float a, float b, double c, bool single)
{
    return single ? __dmul_rn((double)__fmul_rn(a, b), c) : dot_term(a, b, c);
}
__device__ __forceinline__ double dot_term(double a, double b, double c, bool)
{
    return dot_term(a, b, c);
}

// VPREC emulation (NEXT-4): a binary64 value rounded to t explicit
// mantissa bits, round to nearest, ties to even, on the bit pattern (binary64
// exponent range; subnormals rounded at the same absolute bit position).
__device__ __forceinline__ double vprec_round(double x, int t)
{
    if (t >= 52 || !isfinite(x)) return x;
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const int drop = 52 - t;
    const unsigned long long mask = (1ull << drop) - 1ull, half = 1ull << (drop - 1);
    const unsigned long long low = b & mask;
    b &= ~mask;
    if (low > half || (low == half && ((b >> drop) & 1ull))) b += 1ull << drop;
    return __longlong_as_double((long long)b);
}
// ---------------------------------------------------------- precision tools
// Emulation modes of the CG-loop operations:
//   PM_NONE  plain IEEE binary64 / binary32;
//   PM_VPREC every result rounded to t mantissa bits (VPREC);
//   PM_RR    Monte Carlo random rounding of the result: inexact(x) = x + 2^(e_x - t) xi,
//            e_x = floor(log2|x|) + 1, xi ~ U[-1/2, 1/2), then RN64 (MCA "rr" mode);
//   PM_MCA   inexact() on the operands and on the result (full MCA).
// The random xi of an operation comes from SplitMix64(seed, 4 key + slot), key =
// (iteration, phase, global local index, op number) -- the oracle numbers the
// operations identically, so emulated runs are bitwise comparable.
enum { PM_NONE = 0, PM_VPREC = 1, PM_RR = 2, PM_MCA = 3 };
// Random perturbation modes draw per operation (per local point): the copies of
// a shared node then differ, so no per-node shortcut of a sum over copies holds.
__host__ __device__ constexpr bool pm_discontinuous(int pm) { return pm == PM_RR || pm == PM_MCA; }
struct PmArgs {
    int t;                    // virtual precision (mantissa bits)
    unsigned long long seed;  // RR / MCA sample seed
};
__device__ __forceinline__ unsigned long long pm_key(int it, int phase, long long Lg, int o)
{
    return (((unsigned long long)it * 8ull + (unsigned long long)phase) * (1ull << 40) +
            (unsigned long long)Lg) * 128ull + (unsigned long long)o;
}
__device__ __forceinline__ double pm_inexact(double x, const PmArgs& P, unsigned long long key, int slot)
{
    if (x == 0.0 || !isfinite(x)) return x;
    unsigned long long z = P.seed + (4ull * key + (unsigned long long)slot + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double xi = __dsub_rn(__dmul_rn((double)(z >> 11), 0x1.0p-53), 0.5);
    int ex;
    frexp(x, &ex);  // x = m 2^ex, m in [0.5, 1): e_x = floor(log2|x|) + 1 = ex
    return __dadd_rn(x, scalbn(xi, ex - P.t));
}
template <int PM>
__device__ __forceinline__ double pm_res(double r, const PmArgs& P, unsigned long long key)
{
    if constexpr (PM == PM_VPREC) return vprec_round(r, P.t);
    else if constexpr (PM == PM_RR || PM == PM_MCA) return pm_inexact(r, P, key, 0);
    else return r;
}
template <int PM>
__device__ __forceinline__ double pm_opnd(double x, const PmArgs& P, unsigned long long key, int slot)
{
    if constexpr (PM == PM_MCA) return pm_inexact(x, P, key, slot); else return x;
}
template <int PM>
__device__ __forceinline__ double pfma(double a, double b, double c, const PmArgs& P, unsigned long long key)
{
    if constexpr (PM == PM_NONE) return __fma_rn(a, b, c);
    else return pm_res<PM>(__fma_rn(pm_opnd<PM>(a, P, key, 1), pm_opnd<PM>(b, P, key, 2),
                                    pm_opnd<PM>(c, P, key, 3)), P, key);
}
template <int PM>
__device__ __forceinline__ double pmul(double a, double b, const PmArgs& P, unsigned long long key)
{
    if constexpr (PM == PM_NONE) return __dmul_rn(a, b);
    else return pm_res<PM>(__dmul_rn(pm_opnd<PM>(a, P, key, 1), pm_opnd<PM>(b, P, key, 2)), P, key);
}
template <int PM>
__device__ __forceinline__ double padd(double a, double b, const PmArgs& P, unsigned long long key)
{
    if constexpr (PM == PM_NONE) return __dadd_rn(a, b);
    else return pm_res<PM>(__dadd_rn(pm_opnd<PM>(a, P, key, 1), pm_opnd<PM>(b, P, key, 2)), P, key);
}
// binary32 kernels are never emulated
template <int PM>
__device__ __forceinline__ float pfma(float a, float b, float c, const PmArgs&, unsigned long long)
{
    static_assert(PM == PM_NONE, "precision emulation runs in binary64");
    return __fmaf_rn(a, b, c);
}
template <int PM>
__device__ __forceinline__ float pmul(float a, float b, const PmArgs&, unsigned long long)
{
    static_assert(PM == PM_NONE, "precision emulation runs in binary64");
    return __fmul_rn(a, b);
}
template <int PM>
__device__ __forceinline__ float padd(float a, float b, const PmArgs&, unsigned long long)
{
    static_assert(PM == PM_NONE, "precision emulation runs in binary64");
    return __fadd_rn(a, b);
}
// key phases
enum { PH_A = 0, PH_B = 1, PH_C = 2, PH_S = 3 };

// RN32 of the sum represented by a double-double (hi = RN64(hi + lo)): RN32(hi)
// unless hi lies exactly half-way between two binary32 neighbours, where the
// sign of lo (the rest of the sum) decides.
__device__ __forceinline__ float dd_to_float_rn(double hi, double lo)
{
    const float f = __double2float_rn(hi);
    if (!isfinite(hi) || (double)f == hi) return f;
    const float a = nextafterf(f, hi > (double)f ? INFINITY : -INFINITY);
    const double mid = __dmul_rn(__dadd_rn((double)f, (double)a), 0.5);
    if (hi != mid || lo == 0.0) return f;
    return lo > 0.0 ? fmaxf(f, a) : fminf(f, a);
}

template <typename T>
__device__ __forceinline__ T fma_t(T a, T b, T c);
template <>
__device__ __forceinline__ double fma_t<double>(double a, double b, double c)
{
    return __fma_rn(a, b, c);
}
template <>
__device__ __forceinline__ float fma_t<float>(float a, float b, float c)
{
    return __fmaf_rn(a, b, c);
}
template <typename T>
__device__ __forceinline__ T mul_t(T a, T b);
template <>
__device__ __forceinline__ double mul_t<double>(double a, double b)
{
    return __dmul_rn(a, b);
}
template <>
__device__ __forceinline__ float mul_t<float>(float a, float b)
{
    return __fmul_rn(a, b);
}
template <typename T>
__device__ __forceinline__ T add_t(T a, T b);
template <>
__device__ __forceinline__ double add_t<double>(double a, double b)
{
    return __dadd_rn(a, b);
}
template <>
__device__ __forceinline__ float add_t<float>(float a, float b)
{
    return __fadd_rn(a, b);
}

// ------------------------------------------------------------ K_B tile staging
// Byte layout of one dssum tile's index rows in shared memory: the g2 rows
// (8 B each) from the 16-byte boundary at or below the first, rounded up to 16
// bytes, then the g4 rows (16 B), then the g8 rows (32 B).
// K_B gathers each staged tile's copies into shared memory first (cp.async;
// measured same-box: C5 FP32 K_B 0.53 vs 0.63 ms, C4 0.18 vs 0.23 ms);
// NBK_DSSUM_NOGATHER restores the per-thread chains.
#if !defined(NBK_DSSUM_NOGATHER) && !defined(NBK_DSSUM_GATHER)
#define NBK_DSSUM_GATHER 1
#endif
#ifndef NBK_DSSUM_TILE_SMEM
#define NBK_DSSUM_TILE_SMEM 22528   // per buffer; two buffers per CTA
#endif
__host__ __device__ inline int64_t dssum_g2_lead(int64_t s2) { return (8 * s2) & 15; }
__host__ __device__ inline int64_t dssum_g2_bytes(int64_t s2, int64_t n2)
{
    return n2 ? ((8 * (s2 + n2) + 15) & ~(int64_t)15) - ((8 * s2) & ~(int64_t)15) : 0;
}
__host__ __device__ inline int64_t dssum_tile_bytes(int64_t s2, int64_t n2, int64_t n4, int64_t n8)
{
    return dssum_g2_bytes(s2, n2) + 16 * n4 + 32 * n8;
}

// ------------------------------------------------------------ TMA / mbarrier
// 1-D bulk copies global -> shared through the tensor memory accelerator
// (cp.async.bulk, SASS UBLKCP) completing on an mbarrier (transaction bytes).
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                            uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 1-D bulk copy shared -> global (TMA store, SASS UBLKCP), bulk-group completion.
__device__ __forceinline__ void tma_store_1d(void* dst_gmem, const void* src_smem, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
                 "r"(smem_u32(src_smem)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until every committed bulk store of this thread has completed (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy writes to shared memory -> visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ------------------------------------------------------------ CG state
// Device-resident CG scalars (rule C7); alpha/beta never leave the device.
struct CgState {
    double rtr;        // rtr of the previous iteration = rtz1 of the current (z = r)
    double rtz2;       // rtz1 of the previous iteration
    double beta;       // beta of the current iteration (for the p update)
    double alpha;      // alpha of the latest completed pap (x update, r update)
    double alpham;     // -alpha
    float beta32, alpha32, alpham32, pad0;   // RN32 of the FP64 scalars, or (single mode) the scalars
    double true_rtr;   // glsc3(f - A x, c, f - A x) of the final FP64 check
    double dot;        // result slot of the standalone glsc3
    int it;            // current iteration k (1-based)
    int zero;          // rtz1 == 0 reached (rule C9): alpha = beta = 0 from then on
    int defect;        // first iteration with pap <= 0 or a non-finite scalar
    int pm;            // precision emulation of the running solve (PM_*; 0 = off)
    unsigned int cnt[4];  // last-block counters (reset by the finaliser)
};

}  // namespace nbk
