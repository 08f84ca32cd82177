// nbk_setup.cu -- cg_setup: the library's own FP64 set-up on the device
// ("Maintain the initialisation part in double precision").
//
//  * GLL nodes / weights / derivative matrix on the host (tiny), by the
//    Legendre-Vandermonde Newton iteration x <- x - (x P_p - P_{p-1}) / (N P_p)
//    from Chebyshev-Gauss-Lobatto guesses (independent of the oracle, which
//    runs Newton on P'_p); D closed form with the negative-sum diagonal (R17).
//  * Geometric factors g1..g6 (R3, R5) with the ANALYTIC trilinear Jacobian
//    (the oracle differentiates the GLL coordinates with D instead).
//  * RHS b_g = 2U-1 from SplitMix64(seed_rhs, g) on unmasked nodes (R7).
//  * dssum plan: local points sorted by (global node id, local index) with a
//    stable radix sort; runs of length > 1 become segments (ascending local
//    index inside a segment = the canonical chain order C4).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "nbk_internal.h"

namespace nbk {

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

bool validate_mesh(const nbk_mesh* m, const nbk_dist* d, std::string& why)
{
    if (!m) { why = "mesh is NULL"; return false; }
    if (m->ex < 1 || m->ey < 1 || m->ez < 1) { why = "element counts must be >= 1"; return false; }
    if (m->N < 2 || m->N > 16) { why = "N must lie in [2, 16]"; return false; }
    if (!(m->jitter >= 0.0 && m->jitter <= 0.25)) { why = "jitter must lie in [0, 0.25]"; return false; }
    int nr = d ? d->nranks : 1, rk = d ? d->rank : 0;
    if (nr < 1 || rk < 0 || rk >= nr) { why = "bad rank / nranks"; return false; }
    if (m->ez % nr != 0) { why = "ez must be divisible by nranks"; return false; }
    if (nr > NBK_MAX_RANKS) { why = "nranks exceeds NBK_MAX_RANKS (64)"; return false; }
    int64_t n = (int64_t)m->ex * m->ey * (m->ez / nr) * m->N * m->N * m->N;
    if (n >= (int64_t)1 << 31) { why = "local point count must fit in int32"; return false; }
    int64_t ng = ((int64_t)m->ex * (m->N - 1) + 1) * ((int64_t)m->ey * (m->N - 1) + 1) *
                 ((int64_t)m->ez * (m->N - 1) + 1);
    if (ng >= (int64_t)1 << 32) { why = "global node count must fit in uint32"; return false; }
    return true;
}

// shared-node counts of an ex*ey*ez box (Appendix B)
static void box_counts(int64_t ex, int64_t ey, int64_t ez, int64_t N, int64_t& nglob,
                       int64_t& nshared)
{
    int64_t Gx = ex * (N - 1) + 1, Gy = ey * (N - 1) + 1, Gz = ez * (N - 1) + 1;
    nglob = Gx * Gy * Gz;
    nshared = nglob - (Gx - (ex - 1)) * (Gy - (ey - 1)) * (Gz - (ez - 1));
}

static void make_fast_div(uint32_t d, uint32_t& mul, uint32_t& shr)
{
    uint32_t l = 0;
    while (((uint64_t)1 << l) < d) ++l;
    mul = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << l) - d)) / d + 1);
    shr = l;
}

MeshView make_view(const nbk_mesh* m, const nbk_dist* d)
{
    int nr = d ? d->nranks : 1, rk = d ? d->rank : 0;
    MeshView v{};
    v.ex = m->ex;
    v.ey = m->ey;
    v.ez_local = m->ez / nr;
    v.z0 = rk * v.ez_local;
    v.ezg = m->ez;
    v.N = m->N;
    v.E = (int64_t)v.ex * v.ey * v.ez_local;
    make_fast_div((uint32_t)v.ex, v.ex_mul, v.ex_shr);
    make_fast_div((uint32_t)(v.ex * v.ey), v.exy_mul, v.exy_shr);
    make_fast_div((uint32_t)v.N, v.n_mul, v.n_shr);
    make_fast_div((uint32_t)(v.N * v.N * v.N), v.n3_mul, v.n3_shr);
    return v;
}

static size_t plan_scratch_bytes(int64_t n, int64_t nseg)
{
    size_t sort_tmp = 0, scan_tmp = 0;
    cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr), vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, kb, vb, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
    const size_t a = 6 * align256((size_t)n * 4), b = 10 * align256((size_t)nseg * 4);
    return (a > b ? a : b) + align256(sort_tmp > scan_tmp ? sort_tmp : scan_tmp) + 256;
}

Layout compute_layout(const nbk_mesh* m, nbk_precision prec, const nbk_dist* d)
{
    Layout L{};
    MeshView v = make_view(m, d);
    const int64_t N = m->N, N3 = N * N * N;
    L.E = v.E;
    L.n = L.E * N3;
    L.e_offset = (int64_t)v.z0 * v.ex * v.ey;
    int64_t ngl, nsh_dummy;
    box_counts(m->ex, m->ey, m->ez, N, L.n_global, nsh_dummy);
    box_counts(m->ex, m->ey, v.ez_local, N, ngl, L.nseg);
    L.ncopies = L.n - (ngl - L.nseg);
    // rank-boundary planes are summed by the face exchange, not the local plan
    const int nr = d ? d->nranks : 1, rk = d ? d->rank : 0;
    L.has_lo = rk > 0;
    L.has_hi = rk < nr - 1;
    const int64_t Gx = (int64_t)m->ex * (N - 1) + 1, Gy = (int64_t)m->ey * (N - 1) + 1;
    const int64_t U = (Gx - m->ex + 1) * (Gy - m->ey + 1);  // plane nodes with one in-plane copy
    const int nb = L.has_lo + L.has_hi;
    L.nlayer = (int64_t)m->ex * m->ey * N * N;
    L.nplane = Gx * Gy;
    L.nseg -= nb * (L.nplane - U);
    L.ncopies -= nb * (L.nlayer - U);
    // partial slots: K_A (<= E CTAs), K_B, face merge (<= 1184 each), vector kernels (2 x 1184)
    L.nparts = L.E + 4 * NBK_VEC_GRID_MAX + 64;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += align256(bytes); return r; };
    L.off_state = take(sizeof(CgState));
    L.off_D64 = take(8 * N * N);
    L.off_D32 = take(4 * N * N);
    L.off_hist = take(8 * (NBK_MAX_NITER + 1));
    L.off_trace = take(8 * 5 * (size_t)NBK_MAX_NITER);
    L.off_parts = take(sizeof(dd) * (size_t)L.nparts);
    L.off_segoff = take(4 * (size_t)(L.nseg + 1));
    L.off_segidx = take(4 * (size_t)(L.ncopies > 0 ? L.ncopies : 1));
    L.off_grp = take(4 * (size_t)L.ncopies + 64);
    L.off_face = take(nb ? 4 * 8 * (size_t)L.nlayer : 8);
    L.off_gather = take(2 * sizeof(dd) * NBK_MAX_RANKS);
    L.off_toff = take(4 * 3 * ((size_t)L.E + 2));
    L.off_G64 = take(8 * 6 * (size_t)L.n);
    L.off_f64 = take(8 * (size_t)L.n);
    L.off_dinv64 = take(8 * (size_t)L.n);
    L.scratch_need = plan_scratch_bytes(L.n, L.nseg);
    size_t vec64 = 4 * align256(8 * (size_t)L.n);
    L.off_vec64 = take(vec64 > L.scratch_need ? vec64 : L.scratch_need);
    if (prec == NBK_FP32) {
        L.off_G32 = take(4 * 6 * (size_t)L.n);
        L.off_vec32 = take(4 * align256(4 * (size_t)L.n));
        L.off_dinv32 = take(4 * (size_t)L.n);
    } else {
        L.off_G32 = L.off_vec32 = L.off_dinv32 = 0;
    }
    L.total = o;
    return L;
}

// ------------------------------------------------------------------ GLL
static void legendre_all(int p, double x, double* P)
{
    P[0] = 1.0;
    if (p >= 1) P[1] = x;
    for (int k = 2; k <= p; ++k) P[k] = ((2.0 * k - 1.0) * x * P[k - 1] - (k - 1.0) * P[k - 2]) / k;
}

void gll_host(int N, double* xi, double* rho, double* D)
{
    const int p = N - 1;
    const double pi = 3.141592653589793238462643;
    double x[32], P[33];
    for (int j = 0; j < N; ++j) x[j] = std::cos(pi * j / p);  // descending
    for (int it = 0; it < 200; ++it) {
        double dmax = 0.0;
        for (int j = 0; j < N; ++j) {
            legendre_all(p, x[j], P);
            double xn = x[j] - (x[j] * P[p] - P[p - 1]) / (N * P[p]);
            dmax = std::fmax(dmax, std::fabs(xn - x[j]));
            x[j] = xn;
        }
        if (dmax <= 2.2e-16) break;
    }
    for (int j = 0; j < N; ++j) xi[j] = -x[j];  // ascending
    xi[0] = -1.0;
    xi[p] = 1.0;
    for (int j = 0; j < N / 2; ++j) {
        double a = 0.5 * (xi[p - j] - xi[j]);
        xi[j] = -a;
        xi[p - j] = a;
    }
    if (N % 2) xi[p / 2] = 0.0;
    double Pp[32];
    for (int j = 0; j < N; ++j) {
        legendre_all(p, xi[j], P);
        Pp[j] = P[p];
        rho[j] = 2.0 / (p * (double)N * P[p] * P[p]);
    }
    for (int a = 0; a < N; ++a) {
        double s = 0.0;
        for (int b = 0; b < N; ++b) {
            if (a == b) continue;
            double v = Pp[a] / (Pp[b] * (xi[a] - xi[b]));
            D[a * N + b] = v;
            s += v;
        }
        D[a * N + a] = -s;
    }
}

// ------------------------------------------------------------ device setup
struct GeoParams {
    double xi[16], rho[16];
    int N;
    double jitter;
    unsigned long long seed_geom, seed_rhs;
    MeshView v;
};

__device__ __forceinline__ unsigned long long splitmix64_dev(unsigned long long seed,
                                                             unsigned long long i)
{
    unsigned long long z = seed + (i + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double pm1_dev(unsigned long long seed, unsigned long long i)
{
    const double u = __dmul_rn((double)(splitmix64_dev(seed, i) >> 11), 0x1.0p-53);
    return __dsub_rn(__dmul_rn(2.0, u), 1.0);
}

// One block per element: 8 vertices in smem, then one thread per point.
__global__ void __launch_bounds__(256) k_geom(GeoParams gp, double* G)
{
    __shared__ double V[8][3];
    const MeshView& m = gp.v;
    const int N = gp.N, N3 = N * N * N;
    const int64_t e = blockIdx.x;
    ElemCoord ec = elem_coord(m, (uint32_t)e);
    const double h = 1.0 / m.ex;
    if (threadIdx.x < 8) {
        const int a = threadIdx.x & 1, b = (threadIdx.x >> 1) & 1, c = threadIdx.x >> 2;
        const long long vx = ec.ax + a, vy = ec.ay + b, vz = ec.azg + c;
        double pos[3] = {vx * h, vy * h, vz * h};
        const bool interior = vx > 0 && vx < m.ex && vy > 0 && vy < m.ey && vz > 0 && vz < m.ezg;
        if (gp.jitter > 0.0 && interior) {
            const long long vid = vx + (long long)(m.ex + 1) * (vy + (long long)(m.ey + 1) * vz);
            for (int d = 0; d < 3; ++d)
                pos[d] += gp.jitter * h * pm1_dev(gp.seed_geom, (unsigned long long)(3 * vid + d));
        }
        for (int d = 0; d < 3; ++d) V[threadIdx.x][d] = pos[d];
    }
    __syncthreads();
    for (int pt = threadIdx.x; pt < N3; pt += blockDim.x) {
        const int i = pt % N, j = (pt / N) % N, k = pt / (N * N);
        const double r = gp.xi[i], s = gp.xi[j], t = gp.xi[k];
        const double fr[2] = {0.5 * (1.0 - r), 0.5 * (1.0 + r)};
        const double fs[2] = {0.5 * (1.0 - s), 0.5 * (1.0 + s)};
        const double ft[2] = {0.5 * (1.0 - t), 0.5 * (1.0 + t)};
        const double dl[2] = {-0.5, 0.5};
        double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // J[d][m] = dx_d/dr_m
        for (int v = 0; v < 8; ++v) {
            const int a = v & 1, b = (v >> 1) & 1, c = v >> 2;
            const double wr = dl[a] * fs[b] * ft[c], ws = fr[a] * dl[b] * ft[c],
                         wt = fr[a] * fs[b] * dl[c];
            for (int d = 0; d < 3; ++d) {
                J[d][0] += wr * V[v][d];
                J[d][1] += ws * V[v][d];
                J[d][2] += wt * V[v][d];
            }
        }
        // adjugate A[m][d] = (J^-1)[m][d] * det
        double A[3][3];
        A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
        A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
        A[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
        A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
        A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
        A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
        A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        const double det = J[0][0] * A[0][0] + J[0][1] * A[1][0] + J[0][2] * A[2][0];
        const double W = gp.rho[i] * gp.rho[j] * gp.rho[k];
        const double sc = W / det;  // G = W det J^-1 J^-T = (W/det) A A^T
        double g[6];
        const int mm[6] = {0, 0, 0, 1, 1, 2}, nn[6] = {0, 1, 2, 1, 2, 2};
        for (int q = 0; q < 6; ++q) {
            const int a = mm[q], b = nn[q];
            g[q] = sc * (A[a][0] * A[b][0] + A[a][1] * A[b][1] + A[a][2] * A[b][2]);
        }
        double* Ge = G + e * 6 * N3 + pt;
        for (int q = 0; q < 6; ++q) Ge[q * N3] = g[q];
    }
}

__device__ __forceinline__ uint32_t point_gid_dev(const MeshView& m, int64_t L, bool* masked)
{
    const int N = m.N, N3 = N * N * N;
    const uint32_t e = (uint32_t)(L / N3);
    const int rem = (int)(L - (int64_t)e * N3);
    const int i = rem % N, j = (rem / N) % N, k = rem / (N * N);
    ElemCoord ec = elem_coord(m, e);
    const uint32_t Gx = (uint32_t)m.ex * (N - 1) + 1, Gy = (uint32_t)m.ey * (N - 1) + 1;
    const uint32_t gx = ec.ax * (N - 1) + i, gy = ec.ay * (N - 1) + j, gz = ec.azg * (N - 1) + k;
    if (masked) *masked = is_masked(m, ec, i, j, k);
    return gx + Gx * (gy + Gy * gz);
}

// SL position (nbk_common.cuh) of natural local index L.
__device__ __forceinline__ int64_t sl_of_natural(const MeshView& m, int64_t L)
{
    const int N = m.N, N3 = N * N * N;
    const int64_t e = L / N3;
    const int rem = (int)(L - e * N3);
    return e * N3 + sl_slot(N, rem % N, (rem / N) % N, rem / (N * N));
}

__global__ void __launch_bounds__(256) k_rhs(MeshView m, unsigned long long seed, double* f)
{
    const int64_t n = m.E * m.N * m.N * m.N;
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n;
         L += (int64_t)gridDim.x * blockDim.x) {
        bool msk;
        uint32_t g = point_gid_dev(m, L, &msk);
        f[sl_of_natural(m, L)] = msk ? 0.0 : pm1_dev(seed, g);   // f in the split layout
    }
}

__global__ void __launch_bounds__(256) k_gid_keys(MeshView m, uint32_t* keys, uint32_t* vals)
{
    const int64_t n = m.E * m.N * m.N * m.N;
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n;
         L += (int64_t)gridDim.x * blockDim.x) {
        keys[L] = point_gid_dev(m, L, nullptr);
        vals[L] = (uint32_t)L;
    }
}

// flag_head[q] = 1 if q starts a run of length > 1; in_run[q] = 1 if q's run has length > 1.
// Points on a rank-boundary plane (all copies of such a node lie on it) are
// left to the face exchange: never part of a local segment.
__global__ void __launch_bounds__(256) k_run_flags(const uint32_t* keys, const uint32_t* vals,
                                                   int64_t n, MeshView m, int has_lo, int has_hi,
                                                   uint32_t* head, uint32_t* inrun)
{
    const int N = m.N, N2 = N * N, N3 = N2 * N;
    const int64_t exy = (int64_t)m.ex * m.ey;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[q];
        const bool same_prev = q > 0 && keys[q - 1] == k;
        const bool same_next = q + 1 < n && keys[q + 1] == k;
        const int64_t L = vals[q];
        const int64_t e = L / N3;
        const int kk = (int)((L / N2) % N);
        const int64_t az = e / exy;
        const bool excl = (has_lo && az == 0 && kk == 0) ||
                          (has_hi && az == m.ez_local - 1 && kk == N - 1);
        head[q] = (!excl && !same_prev && same_next) ? 1u : 0u;
        inrun[q] = (!excl && (same_prev || same_next)) ? 1u : 0u;
    }
}

__global__ void __launch_bounds__(256) k_scatter_plan(const uint32_t* vals, const uint32_t* head,
                                                      const uint32_t* inrun,
                                                      const uint32_t* head_pos,
                                                      const uint32_t* run_pos, int64_t n,
                                                      int32_t* seg_off, int32_t* seg_idx,
                                                      int64_t ncopies, int64_t nseg, MeshView m)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        // copies in ascending NATURAL local index (chain order C4), stored as SL positions
        if (inrun[q]) seg_idx[run_pos[q]] = (int32_t)sl_of_natural(m, vals[q]);
        if (head[q]) seg_off[head_pos[q]] = (int32_t)run_pos[q];
        if (q == 0) seg_off[nseg] = (int32_t)ncopies;
    }
}

// Group the segments by length m in {2, 4, 8} (dense m-wide index rows).
// Segments are visited in the order of their first (smallest) local index so
// that consecutive threads of k_dssum touch neighbouring addresses.
__global__ void __launch_bounds__(256) k_seg_first(const int32_t* off, const int32_t* idx,
                                                   int64_t nseg, uint32_t* first, uint32_t* id)
{
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg;
         s += (int64_t)gridDim.x * blockDim.x) {
        first[s] = (uint32_t)idx[off[s]];
        id[s] = (uint32_t)s;
    }
}

__global__ void __launch_bounds__(256) k_seg_flags(const int32_t* off, const uint32_t* order,
                                                   int64_t nseg, uint32_t* f2, uint32_t* f4,
                                                   uint32_t* f8)
{
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nseg;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = order[t];
        const int m = off[s + 1] - off[s];
        f2[t] = m == 2;
        f4[t] = m == 4;
        f8[t] = m == 8;
    }
}
__global__ void __launch_bounds__(256) k_group_scatter(const int32_t* off, const int32_t* idx,
                                                       const uint32_t* order,
                                                       int64_t nseg, const uint32_t* f2,
                                                       const uint32_t* f4, const uint32_t* f8,
                                                       const uint32_t* p2, const uint32_t* p4,
                                                       const uint32_t* p8, int32_t* g2, int32_t* g4,
                                                       int32_t* g8)
{
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nseg;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t o = off[order[t]];
        if (f2[t]) for (int q = 0; q < 2; ++q) g2[2 * (int64_t)p2[t] + q] = idx[o + q];
        if (f4[t]) for (int q = 0; q < 4; ++q) g4[4 * (int64_t)p4[t] + q] = idx[o + q];
        if (f8[t]) for (int q = 0; q < 8; ++q) g8[8 * (int64_t)p8[t] + q] = idx[o + q];
    }
}

// toff[3t + g] = first node of group g (rows of m = 2, 4, 8 indices) whose
// first copy lies at local index >= t * te * N^3 (binary search; groups are
// ordered by first copy).
__global__ void __launch_bounds__(256) k_tile_offsets(const int32_t* g2, const int32_t* g4,
                                                      const int32_t* g8, int64_t n2, int64_t n4,
                                                      int64_t n8, int64_t ntiles, int64_t te,
                                                      int64_t N3, int32_t* toff)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < 3 * (ntiles + 1);
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = q / 3;
        const int g = (int)(q - 3 * t);
        const int32_t* arr = g == 0 ? g2 : (g == 1 ? g4 : g8);
        const int m = g == 0 ? 2 : (g == 1 ? 4 : 8);
        const int64_t cnt = g == 0 ? n2 : (g == 1 ? n4 : n8);
        const int64_t key = t * te * N3;
        int64_t lo = 0, hi = cnt;
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if ((int64_t)arr[mid * m] < key) lo = mid + 1; else hi = mid;
        }
        toff[q] = (int32_t)lo;
    }
}

static int grid_for(int64_t n, int cap = 148 * 16)
{
    int64_t g = (n + 255) / 256;
    if (g < 1) g = 1;
    return (int)(g > cap ? cap : g);
}

cudaError_t build_plan(nbk_ctx* ctx)
{
    const int64_t n = ctx->n;
    cudaStream_t s = ctx->stream;
    unsigned char* base = ctx->scratch;
    size_t o = 0;
    auto take = [&](size_t bytes) { unsigned char* r = base + o; o += align256(bytes); return r; };
    uint32_t* k0 = (uint32_t*)take(4 * n);
    uint32_t* k1 = (uint32_t*)take(4 * n);
    uint32_t* v0 = (uint32_t*)take(4 * n);
    uint32_t* v1 = (uint32_t*)take(4 * n);
    uint32_t* head = (uint32_t*)take(4 * n);
    uint32_t* inrun = (uint32_t*)take(4 * n);
    void* tmp = base + o;
    size_t tmp_bytes = ctx->scratch_bytes - o;
    k_gid_keys<<<grid_for(n), 256, 0, s>>>(ctx->view, k0, v0);
    cub::DoubleBuffer<uint32_t> kb(k0, k1), vb(v0, v1);
    int end_bit = 1;
    while (end_bit < 32 && ((uint64_t)1 << end_bit) < (uint64_t)ctx->n_global) ++end_bit;
    size_t need = 0;
    cudaError_t err = cub::DeviceRadixSort::SortPairs(nullptr, need, kb, vb, (int)n, 0, end_bit, s);
    if (err != cudaSuccess) return err;
    if (need > tmp_bytes) return cudaErrorMemoryAllocation;
    err = cub::DeviceRadixSort::SortPairs(tmp, need, kb, vb, (int)n, 0, end_bit, s);
    if (err != cudaSuccess) return err;
    uint32_t* keys = kb.Current();
    uint32_t* vals = vb.Current();
    uint32_t* kalt = kb.Alternate();  // reuse as head_pos
    uint32_t* valt = vb.Alternate();  // reuse as run_pos
    k_run_flags<<<grid_for(n), 256, 0, s>>>(keys, vals, n, ctx->view, ctx->has_lo, ctx->has_hi,
                                            head, inrun);
    err = cub::DeviceScan::ExclusiveSum(nullptr, need, head, kalt, (int)n, s);
    if (err != cudaSuccess) return err;
    if (need > tmp_bytes) return cudaErrorMemoryAllocation;
    err = cub::DeviceScan::ExclusiveSum(tmp, need, head, kalt, (int)n, s);
    if (err != cudaSuccess) return err;
    err = cub::DeviceScan::ExclusiveSum(tmp, need, inrun, valt, (int)n, s);
    if (err != cudaSuccess) return err;
    k_scatter_plan<<<grid_for(n), 256, 0, s>>>(vals, head, inrun, kalt, valt, n, ctx->seg_off,
                                              ctx->seg_idx, ctx->ncopies, ctx->nseg, ctx->view);
    // check the counts match the analytic plan size
    uint32_t last_head, last_run, h_last, r_last;
    cudaMemcpyAsync(&last_head, kalt + n - 1, 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&last_run, valt + n - 1, 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&h_last, head + n - 1, 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&r_last, inrun + n - 1, 4, cudaMemcpyDeviceToHost, s);
    err = cudaStreamSynchronize(s);
    if (err != cudaSuccess) return err;
    if ((int64_t)(last_head + h_last) != ctx->nseg || (int64_t)(last_run + r_last) != ctx->ncopies)
        return cudaErrorInvalidValue;

    // ---- group the segments by multiplicity (scratch is free again)
    const int64_t ns = ctx->nseg;
    ctx->n2 = ctx->n4 = ctx->n8 = ctx->nother = 0;
    ctx->g2 = ctx->g4 = ctx->g8 = ctx->grp;
    ctx->ntiles = 0;
    if (ns == 0) return cudaGetLastError();
    o = 0;
    uint32_t* f2 = (uint32_t*)take(4 * ns);
    uint32_t* f4 = (uint32_t*)take(4 * ns);
    uint32_t* f8 = (uint32_t*)take(4 * ns);
    uint32_t* q2 = (uint32_t*)take(4 * ns);
    uint32_t* q4 = (uint32_t*)take(4 * ns);
    uint32_t* q8 = (uint32_t*)take(4 * ns);
    uint32_t* fk0 = (uint32_t*)take(4 * ns);
    uint32_t* fk1 = (uint32_t*)take(4 * ns);
    uint32_t* od0 = (uint32_t*)take(4 * ns);
    uint32_t* od1 = (uint32_t*)take(4 * ns);
    tmp = base + o;
    tmp_bytes = ctx->scratch_bytes - o;
    // order segments by their first local index
    k_seg_first<<<grid_for(ns), 256, 0, s>>>(ctx->seg_off, ctx->seg_idx, ns, fk0, od0);
    {
        cub::DoubleBuffer<uint32_t> fb(fk0, fk1), ob(od0, od1);
        int eb = 1;
        while (eb < 32 && ((uint64_t)1 << eb) < (uint64_t)n) ++eb;
        err = cub::DeviceRadixSort::SortPairs(nullptr, need, fb, ob, (int)ns, 0, eb, s);
        if (err != cudaSuccess) return err;
        if (need > tmp_bytes) return cudaErrorMemoryAllocation;
        err = cub::DeviceRadixSort::SortPairs(tmp, need, fb, ob, (int)ns, 0, eb, s);
        if (err != cudaSuccess) return err;
        od0 = ob.Current();
    }
    const uint32_t* order = od0;
    k_seg_flags<<<grid_for(ns), 256, 0, s>>>(ctx->seg_off, order, ns, f2, f4, f8);
    err = cub::DeviceScan::ExclusiveSum(nullptr, need, f2, q2, (int)ns, s);
    if (err != cudaSuccess) return err;
    if (need > tmp_bytes) return cudaErrorMemoryAllocation;
    uint32_t* fl[3] = {f2, f4, f8};
    uint32_t* ql[3] = {q2, q4, q8};
    uint32_t cnt[3], lastf[3];
    for (int g = 0; g < 3; ++g) {
        err = cub::DeviceScan::ExclusiveSum(tmp, need, fl[g], ql[g], (int)ns, s);
        if (err != cudaSuccess) return err;
        cudaMemcpyAsync(&cnt[g], ql[g] + ns - 1, 4, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&lastf[g], fl[g] + ns - 1, 4, cudaMemcpyDeviceToHost, s);
    }
    err = cudaStreamSynchronize(s);
    if (err != cudaSuccess) return err;
    ctx->n2 = cnt[0] + lastf[0];
    ctx->n4 = cnt[1] + lastf[1];
    ctx->n8 = cnt[2] + lastf[2];
    ctx->nother = ns - ctx->n2 - ctx->n4 - ctx->n8;
    if (ctx->nother != 0) return cudaErrorInvalidValue;  // box slabs: local m in {2, 4, 8}
    ctx->g2 = ctx->grp;
    ctx->g4 = ctx->g2 + ((2 * ctx->n2 + 3) & ~(int64_t)3);   // 16-byte aligned rows
    ctx->g8 = ctx->g4 + 4 * ctx->n4;
    k_group_scatter<<<grid_for(ns), 256, 0, s>>>(ctx->seg_off, ctx->seg_idx, order, ns, f2, f4, f8, q2,
                                                 q4, q8, ctx->g2, ctx->g4, ctx->g8);
    // dssum tiles: ~tile_nodes nodes per tile (several per thread of a 256-thread block)
    const int64_t N3 = (int64_t)ctx->N * ctx->N * ctx->N;
    const int64_t per_elem = (ns + ctx->E - 1) / ctx->E;
    int64_t tile_nodes = 512;   // K_B gather phase: 512-node tiles
    if (const char* env = getenv("NBK_DSSUM_TILE_NODES")) tile_nodes = atol(env) > 0 ? atol(env) : tile_nodes;
    int64_t te = (tile_nodes + per_elem - 1) / per_elem;
    if (te < 1) te = 1;
    // K_B stages each tile's index rows in shared memory (double-buffered bulk
    // copies): halve the tile until its rows fit NBK_DSSUM_TILE_SMEM bytes.
    std::vector<int32_t> th;
    for (;;) {
        ctx->tile_elems = te;
        ctx->ntiles = (ctx->E + te - 1) / te;
        k_tile_offsets<<<grid_for(3 * (ctx->ntiles + 1)), 256, 0, s>>>(ctx->g2, ctx->g4, ctx->g8, ctx->n2,
                                                                     ctx->n4, ctx->n8, ctx->ntiles, te, N3,
                                                                     ctx->toff);
        th.resize(3 * (size_t)(ctx->ntiles + 1));
        err = cudaMemcpyAsync(th.data(), ctx->toff, th.size() * 4, cudaMemcpyDeviceToHost, s);
        if (err == cudaSuccess) err = cudaStreamSynchronize(s);
        if (err != cudaSuccess) return err;
        int64_t mx = 0;
        for (int64_t t = 0; t < ctx->ntiles; ++t) {
            const int64_t b = nbk::dssum_tile_bytes(th[3 * t], th[3 * t + 3] - th[3 * t],
                                                    th[3 * t + 4] - th[3 * t + 1], th[3 * t + 5] - th[3 * t + 2]);
            mx = b > mx ? b : mx;
        }
        ctx->tile_smem = mx;
        if (mx <= NBK_DSSUM_TILE_SMEM || te == 1) break;
        te = (te + 1) / 2;
    }
    return cudaGetLastError();
}

// Jacobi preconditioner (NEXT-1): diagonal of the element matrix
// A_e = sum_mn D_m^T diag(g_mn) D_n at (i,j,k):
//   sum_a D[a][i]^2 g1(a,j,k) + sum_a D[a][j]^2 g4(i,a,k) + sum_a D[a][k]^2 g6(i,j,a)
//   + 2 (D[i][i] D[j][j] g2 + D[i][i] D[k][k] g3 + D[j][j] D[k][k] g5).
// One block per element.  FP64 set-up; assembled by the library's
// own dssum afterwards.
__global__ void __launch_bounds__(256) k_local_diag(const double* G, const double* Dg, int N, double* d)
{
    __shared__ double D[256];
    const int N2 = N * N, N3 = N2 * N;
    for (int q = threadIdx.x; q < N2; q += blockDim.x) D[q] = Dg[q];
    __syncthreads();
    const int64_t e = blockIdx.x;
    const double* g = G + e * 6 * N3;
    for (int pt = threadIdx.x; pt < N3; pt += blockDim.x) {
        const int i = pt % N, j = (pt / N) % N, k = pt / N2;
        double s = 0.0;
        for (int a = 0; a < N; ++a) {
            s += D[a * N + i] * D[a * N + i] * g[0 * N3 + k * N2 + j * N + a];
            s += D[a * N + j] * D[a * N + j] * g[3 * N3 + k * N2 + a * N + i];
            s += D[a * N + k] * D[a * N + k] * g[5 * N3 + a * N2 + j * N + i];
        }
        const double di = D[i * N + i], dj = D[j * N + j], dk = D[k * N + k];
        s += 2.0 * (di * dj * g[1 * N3 + pt] + di * dk * g[2 * N3 + pt] + dj * dk * g[4 * N3 + pt]);
        d[e * N3 + sl_slot(N, i, j, k)] = s;   // split layout, as every CG vector
    }
}

// masked -> 1, dinv = 1/d, dinv32 = RN32(dinv) (C11)
__global__ void __launch_bounds__(256) k_finish_dinv(MeshView m, double* d, float* d32)
{
    const int N = m.N, N3 = N * N * N;
    const int64_t n = m.E * N3;
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n;
         L += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t e = (uint32_t)(L / N3);
        int i, j, k;
        sl_point(N, (int)(L - (int64_t)e * N3), i, j, k);   // d is in the split layout
        ElemCoord ec = elem_coord(m, e);
        double v = d[L];
        if (is_masked(m, ec, i, j, k)) v = 1.0;
        const double inv = 1.0 / v;
        d[L] = inv;
        if (d32) d32[L] = __double2float_rn(inv);
    }
}

cudaError_t local_diag(nbk_ctx* ctx, double* d)
{
    k_local_diag<<<(unsigned)ctx->E, 256, 0, ctx->stream>>>(ctx->G64, ctx->D64, ctx->N, d);
    return cudaGetLastError();
}

cudaError_t finish_dinv(nbk_ctx* ctx, double* d)
{
    k_finish_dinv<<<grid_for(ctx->n), 256, 0, ctx->stream>>>(ctx->view, d, ctx->dinv32);
    return cudaGetLastError();
}

cudaError_t setup_device(nbk_ctx* ctx, const Layout& L)
{
    (void)L;
    GeoParams gp{};
    double D[256];
    gll_host(ctx->N, gp.xi, gp.rho, D);
    for (int q = 0; q < ctx->N * ctx->N; ++q) {
        ctx->Dh64[q] = D[q];
        ctx->Dh32[q] = (float)D[q];  // RN32, as k_downcast (C11)
    }
    gp.N = ctx->N;
    gp.jitter = ctx->mesh.jitter;
    gp.seed_geom = ctx->mesh.seed_geom;
    gp.seed_rhs = ctx->mesh.seed_rhs;
    gp.v = ctx->view;
    cudaStream_t s = ctx->stream;
    cudaError_t err = cudaMemcpyAsync(ctx->D64, D, 8 * ctx->N * ctx->N, cudaMemcpyHostToDevice, s);
    if (err != cudaSuccess) return err;
    err = build_plan(ctx);  // uses the vector region as scratch: before f / vectors
    if (err != cudaSuccess) return err;
    k_geom<<<(unsigned)ctx->E, 256, 0, s>>>(gp, ctx->G64);
    k_rhs<<<grid_for(ctx->n), 256, 0, s>>>(ctx->view, gp.seed_rhs, ctx->f64);
    return cudaGetLastError();
}

}  // namespace nbk
