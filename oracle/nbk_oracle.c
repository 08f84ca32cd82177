/*
 * nbk_oracle.c -- plain, slow, obviously-correct CPU oracle for the Nekbone
 * unpreconditioned CG hot path (arXiv 2405.11065).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * library under paper_2405_11065_b200/ and neither side includes the other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
 * "R#" / "C#" = the readings / canonical-order rules listed in DESIGN.md
 * (section "Readings of the paper").
 *
 * What is computed (in the paper's order, T1 = tab:cg-profiling):
 *   setup (FP64)  : GLL nodes/weights/D, box mesh, geometric factors
 *                          g1..g6, multiplicity c = 1/m, Dirichlet mask, RHS.
 *   ax  (T1 line 5)      : w = mask(dssum(ax_e(p) for every element)).
 *   glsc3 (T1 lines 3,6,9): sum_L a_L b_L c_L, correctly rounded (C6).
 *   add2s1/add2s2 (T1 lines 4,7,8): p = beta p + z, x += alpha p, r -= alpha w.
 *   CG loop in FP64, and in FP32 with FP64 accumulation
 *   of the inner products (north_star), plus the final FP64 residual check.
 *   Jacobi PCG (SURVEY 8(f) NEXT-1, T1 line 2 solveM): assembled diagonal,
 *   z = r * dinv, rtz1 = glsc3(r,c,z).
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (no -ffast-math:
 * IEEE round-to-nearest, gradual underflow, no contraction except the
 * explicit fma()/fmaf() calls the canonical order prescribes).
 *
 * Parity status: every function is pinned by tests/test_oracle_pins.py
 * except the CG residual *history* itself (no closed form exists; it is
 * pinned only by CG theory properties: finite termination, dense-solve
 * agreement, monotone A-norm error) -- "parity unpinned" for the history
 * beyond those properties, see DESIGN.md.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* Mesh description (box of ex*ey*ez hexahedra, N GLL points per dir)  */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t ex, ey, ez; /* element counts of the GLOBAL box              */
    int32_t N;          /* GLL points per direction, N = p + 1 (R1)      */
} ora_mesh;

static int64_t n3(const ora_mesh* m) { return (int64_t)m->N * m->N * m->N; }
static int64_t gnx(const ora_mesh* m) { return (int64_t)m->ex * (m->N - 1) + 1; }
static int64_t gny(const ora_mesh* m) { return (int64_t)m->ey * (m->N - 1) + 1; }
static int64_t gnz(const ora_mesh* m) { return (int64_t)m->ez * (m->N - 1) + 1; }

/* ------------------------------------------------------------------ */
/* SplitMix64, random access (SURVEY 8d "RNG"; readings R5, R7)         */
/* z = seed + (i+1)*0x9E3779B97F4A7C15; three xor-shift-multiply steps  */
/* ------------------------------------------------------------------ */
uint64_t ora_splitmix64(uint64_t seed, uint64_t i)
{
    uint64_t z = seed + (i + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* value in [-1,1): 2U-1 with U = (z>>11) * 2^-53 (exact in binary64) */
double ora_uniform_pm1(uint64_t seed, uint64_t i)
{
    double u = (double)(ora_splitmix64(seed, i) >> 11) * 0x1.0p-53;
    return 2.0 * u - 1.0;
}

/* ------------------------------------------------------------------ */
/* Legendre polynomial P_n(x) by the three-term recurrence             */
/* (n+1) P_{n+1} = (2n+1) x P_n - n P_{n-1}                             */
/* ------------------------------------------------------------------ */
static void legendre(int n, double x, double* pn, double* pnm1)
{
    double p0 = 1.0, p1 = x;
    if (n == 0) { *pn = 1.0; *pnm1 = 0.0; return; }
    for (int k = 1; k < n; ++k) {
        double p2 = ((2.0 * k + 1.0) * x * p1 - k * p0) / (k + 1.0);
        p0 = p1;
        p1 = p2;
    }
    *pn = p1;
    *pnm1 = p0;
}

/*
 * GLL nodes xi (ascending), weights rho, derivative matrix D (row-major,
 * D[a*N+b] = l_b'(xi_a), row a = evaluation node, reading R17).
 * Interior nodes are the roots of P'_p, p = N-1, found by Newton's method
 * from Chebyshev-Gauss-Lobatto guesses; P'' from Legendre's ODE
 * (1-x^2) P'' - 2x P' + p(p+1) P = 0.  Nodes are symmetrised (xi_j = -xi_{p-j}).
 * Weights rho_j = 2 / (p(p+1) P_p(xi_j)^2).
 * D (closed form): D_ab = P_p(xi_a) / (P_p(xi_b) (xi_a - xi_b)), a != b;
 * D_aa = -sum_{b != a} D_ab (R17, negative-sum diagonal).
 * Returns 0 on success, -1 if N is out of [2, 32], -2 if Newton failed.
 */
int ora_gll(int N, double* xi, double* rho, double* D)
{
    if (N < 2 || N > 32) return -1;
    const int p = N - 1;
    const double pi = 3.14159265358979323846;
    xi[0] = -1.0;
    xi[p] = 1.0;
    for (int j = 1; j < p; ++j) {
        double x = -cos(pi * j / p);
        int it;
        for (it = 0; it < 100; ++it) {
            double P, Pm1;
            legendre(p, x, &P, &Pm1);
            double dP = p * (x * P - Pm1) / (x * x - 1.0);        /* P'_p  */
            double d2P = (2.0 * x * dP - p * (p + 1.0) * P) / (1.0 - x * x); /* P''_p */
            double dx = dP / d2P;
            x -= dx;
            if (fabs(dx) <= 1e-16) break;
        }
        if (it == 100) return -2;
        xi[j] = x;
    }
    for (int j = 0; j < N / 2; ++j) { /* symmetrise */
        double a = 0.5 * (xi[p - j] - xi[j]);
        xi[j] = -a;
        xi[p - j] = a;
    }
    if (N % 2 == 1) xi[p / 2] = 0.0;
    double Pv[64];
    for (int j = 0; j < N; ++j) {
        double P, Pm1;
        legendre(p, xi[j], &P, &Pm1);
        Pv[j] = P;
        rho[j] = 2.0 / (p * (p + 1.0) * P * P);
    }
    for (int a = 0; a < N; ++a) {
        double s = 0.0;
        for (int b = 0; b < N; ++b) {
            if (a == b) continue;
            double v = Pv[a] / (Pv[b] * (xi[a] - xi[b]));
            D[a * N + b] = v;
            s += v;
        }
        D[a * N + a] = -s;
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Sizes                                         */
/* out[0]=n_local=E*N^3, out[1]=n_global=prod(G_d), out[2]=interior     */
/* unknowns prod(G_d-2), out[3]=unique shared nodes (multiplicity > 1)  */
/* ------------------------------------------------------------------ */
void ora_sizes(int ex, int ey, int ez, int N, int64_t* out)
{
    ora_mesh m = {ex, ey, ez, N};
    int64_t Gx = gnx(&m), Gy = gny(&m), Gz = gnz(&m);
    out[0] = (int64_t)ex * ey * ez * n3(&m);
    out[1] = Gx * Gy * Gz;
    out[2] = (Gx - 2) * (Gy - 2) * (Gz - 2);
    /* a global coordinate is "on an element interface" if it is a multiple
       of (N-1) strictly inside the box; node shared iff any coordinate is */
    int64_t sx = ex - 1, sy = ey - 1, sz = ez - 1; /* interface planes */
    int64_t nsh = Gx * Gy * Gz - (Gx - sx) * (Gy - sy) * (Gz - sz);
    out[3] = nsh;
}

/* ------------------------------------------------------------------ */
/* Per-point structural data: gid, multiplicity, mask (R6, R8)   */
/* ------------------------------------------------------------------ */
static void point_coords(const ora_mesh* m, int64_t L, int64_t* e, int* i, int* j, int* k)
{
    const int N = m->N;
    int64_t q = L;
    *i = (int)(q % N); q /= N;
    *j = (int)(q % N); q /= N;
    *k = (int)(q % N); q /= N;
    *e = q;
}

static int64_t point_gid(const ora_mesh* m, int64_t L)
{
    int64_t e; int i, j, k;
    point_coords(m, L, &e, &i, &j, &k);
    int64_t ax = e % m->ex, ay = (e / m->ex) % m->ey, az = e / ((int64_t)m->ex * m->ey);
    int64_t gx = ax * (m->N - 1) + i, gy = ay * (m->N - 1) + j, gz = az * (m->N - 1) + k;
    return gx + gnx(m) * (gy + gny(m) * gz);
}

static int point_masked(const ora_mesh* m, int64_t g)
{
    int64_t Gx = gnx(m), Gy = gny(m), Gz = gnz(m);
    int64_t gx = g % Gx, gy = (g / Gx) % Gy, gz = g / (Gx * Gy);
    return gx == 0 || gx == Gx - 1 || gy == 0 || gy == Gy - 1 || gz == 0 || gz == Gz - 1;
}

/* multiplicity = number of elements containing the global node */
static int node_mult(const ora_mesh* m, int64_t g)
{
    int64_t Gx = gnx(m), Gy = gny(m), Gz = gnz(m);
    int64_t gc[3] = {g % Gx, (g / Gx) % Gy, g / (Gx * Gy)};
    int64_t Gd[3] = {Gx, Gy, Gz};
    int mult = 1;
    for (int d = 0; d < 3; ++d) {
        int64_t c = gc[d];
        if (c > 0 && c < Gd[d] - 1 && c % (m->N - 1) == 0) mult *= 2;
    }
    return mult;
}

/* ------------------------------------------------------------------ */
/* Geometry (reading R5): cubic elements of edge h = 1/ex; interior    */
/* vertices jittered by jitter*h*(2U-1) per coordinate, U from          */
/* SplitMix64(seed_geom, 3v+d), v = vx + (ex+1)(vy + (ey+1) vz).        */
/* The element map is trilinear in the 8 vertices; the Jacobian is      */
/* obtained by applying D to the GLL coordinates (local_grad3 of x, y,  */
/* z, as Nekbone's geometry set-up does) -- the CUDA library uses the   */
/* analytic trilinear derivative instead, so the two are independent.   */
/* G_mn = rho_i rho_j rho_k detJ sum_d (dr_m/dx_d)(dr_n/dx_d),          */
/* stored G[e][c][k][j][i] with c = rr, rs, rt, ss, st, tt (R3, R18).   */
/* ------------------------------------------------------------------ */
static void vertex_xyz(const ora_mesh* m, double jitter, uint64_t seed, int64_t vx, int64_t vy,
                       int64_t vz, double out[3])
{
    const double h = 1.0 / m->ex;
    out[0] = vx * h;
    out[1] = vy * h;
    out[2] = vz * h;
    int interior = vx > 0 && vx < m->ex && vy > 0 && vy < m->ey && vz > 0 && vz < m->ez;
    if (jitter > 0.0 && interior) {
        int64_t v = vx + (int64_t)(m->ex + 1) * (vy + (int64_t)(m->ey + 1) * vz);
        for (int d = 0; d < 3; ++d)
            out[d] += jitter * h * ora_uniform_pm1(seed, (uint64_t)(3 * v + d));
    }
}

/*
 * Set-up of the rank-local element range [e0, e1) of the global box.
 * Any output pointer may be NULL.  Local index L is relative to e0.
 *   G    : (e1-e0)*6*N^3 geometric factors
 *   f    : (e1-e0)*N^3   RHS, f_L = b_{gid(L)}, b_g = 2U-1 from
 *          SplitMix64(seed_rhs, g) on unmasked nodes, 0 on masked (R7)
 *   mass : (e1-e0)*N^3   rho_i rho_j rho_k detJ (for pins P4, P7)
 *   gid  : global node id, mult: multiplicity m, mask: 1 = Dirichlet node
 *   xyz  : (e1-e0)*3*N^3 physical GLL coordinates [e][d][k][j][i] (pins P7)
 * Returns 0, or a negative error code.
 */
int ora_setup(int ex, int ey, int ez, int N, double jitter, uint64_t seed_geom, uint64_t seed_rhs,
              int64_t e0, int64_t e1, double* G, double* f, double* mass, int64_t* gid,
              int32_t* mult, uint8_t* mask, double* xyz)
{
    ora_mesh m = {ex, ey, ez, N};
    if (ex < 1 || ey < 1 || ez < 1) return -1;
    double xi[32], rho[32], D[32 * 32];
    int rc = ora_gll(N, xi, rho, D);
    if (rc) return rc;
    const int64_t nn = n3(&m);
    const int64_t E = e1 - e0;
#pragma omp parallel for schedule(static)
    for (int64_t el = 0; el < E; ++el) {
        int64_t e = e0 + el;
        int64_t ax = e % ex, ay = (e / ex) % ey, az = e / ((int64_t)ex * ey);
        double V[2][2][2][3];
        for (int c = 0; c < 2; ++c)
            for (int b = 0; b < 2; ++b)
                for (int a = 0; a < 2; ++a)
                    vertex_xyz(&m, jitter, seed_geom, ax + a, ay + b, az + c, V[c][b][a]);
        double* X = (double*)malloc(sizeof(double) * 3 * nn);
        for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j)
                for (int i = 0; i < N; ++i) {
                    double fr[2] = {0.5 * (1.0 - xi[i]), 0.5 * (1.0 + xi[i])};
                    double fs[2] = {0.5 * (1.0 - xi[j]), 0.5 * (1.0 + xi[j])};
                    double ft[2] = {0.5 * (1.0 - xi[k]), 0.5 * (1.0 + xi[k])};
                    for (int d = 0; d < 3; ++d) {
                        double s = 0.0;
                        for (int c = 0; c < 2; ++c)
                            for (int b = 0; b < 2; ++b)
                                for (int a = 0; a < 2; ++a) s += fr[a] * fs[b] * ft[c] * V[c][b][a][d];
                        X[d * nn + (k * N + j) * N + i] = s;
                    }
                }
        if (xyz) memcpy(xyz + el * 3 * nn, X, sizeof(double) * 3 * nn);
        for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j)
                for (int i = 0; i < N; ++i) {
                    int64_t pt = (k * N + j) * N + i;
                    double J[3][3]; /* J[d][m] = dx_d / dr_m */
                    for (int d = 0; d < 3; ++d) {
                        const double* Xd = X + d * nn;
                        double xr = 0, xs = 0, xt = 0;
                        for (int l = 0; l < N; ++l) {
                            xr += D[i * N + l] * Xd[(k * N + j) * N + l];
                            xs += D[j * N + l] * Xd[(k * N + l) * N + i];
                            xt += D[k * N + l] * Xd[(l * N + j) * N + i];
                        }
                        J[d][0] = xr;
                        J[d][1] = xs;
                        J[d][2] = xt;
                    }
                    /* cofactor matrix: Cf[d][m] = cofactor of J[d][m]; adj = Cf^T */
                    double Cf[3][3];
                    Cf[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
                    Cf[0][1] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
                    Cf[0][2] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
                    Cf[1][0] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
                    Cf[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
                    Cf[1][2] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
                    Cf[2][0] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
                    Cf[2][1] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
                    Cf[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
                    double det = J[0][0] * Cf[0][0] + J[0][1] * Cf[0][1] + J[0][2] * Cf[0][2];
                    /* dr_m/dx_d = Jinv[m][d] = Cf[d][m] / det */
                    double W = rho[i] * rho[j] * rho[k];
                    double Gmn[3][3];
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b) {
                            double s = 0.0;
                            for (int d = 0; d < 3; ++d) s += (Cf[d][a] / det) * (Cf[d][b] / det);
                            Gmn[a][b] = W * det * s;
                        }
                    if (G) {
                        double* Ge = G + el * 6 * nn;
                        Ge[0 * nn + pt] = Gmn[0][0];
                        Ge[1 * nn + pt] = Gmn[0][1];
                        Ge[2 * nn + pt] = Gmn[0][2];
                        Ge[3 * nn + pt] = Gmn[1][1];
                        Ge[4 * nn + pt] = Gmn[1][2];
                        Ge[5 * nn + pt] = Gmn[2][2];
                    }
                    if (mass) mass[el * nn + pt] = W * det;
                }
        free(X);
    }
#pragma omp parallel for schedule(static)
    for (int64_t l = 0; l < E * nn; ++l) {
        int64_t g = point_gid(&m, e0 * nn + l);
        int msk = point_masked(&m, g);
        if (gid) gid[l] = g;
        if (mult) mult[l] = node_mult(&m, g);
        if (mask) mask[l] = (uint8_t)msk;
        if (f) f[l] = msk ? 0.0 : ora_uniform_pm1(seed_rhs, (uint64_t)g);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Local operator ax_e = D^T G D u_e, canonical order CEO-1 (C1-C3)     */
/* (T1 line 5 P:147; F2 P:215-243 local_grad3 / local_grad3_t)*/
/* ------------------------------------------------------------------ */
#define DEFINE_AX_LOCAL(NAME, T, FMA, MUL, ADD)                                               \
    void NAME(int64_t E, int N, const T* D, const T* G, const T* u, T* w)                     \
    {                                                                                         \
        const int64_t nn = (int64_t)N * N * N;                                                \
        _Pragma("omp parallel for schedule(static)") for (int64_t e = 0; e < E; ++e)          \
        {                                                                                     \
            const T* ue = u + e * nn;                                                         \
            const T* Ge = G + e * 6 * nn;                                                     \
            T* we = w + e * nn;                                                               \
            T* wr = (T*)malloc(sizeof(T) * 3 * nn);                                           \
            T* ws = wr + nn;                                                                  \
            T* wt = ws + nn;                                                                  \
            for (int k = 0; k < N; ++k)                                                       \
                for (int j = 0; j < N; ++j)                                                   \
                    for (int i = 0; i < N; ++i) {                                             \
                        int64_t pt = ((int64_t)k * N + j) * N + i;                            \
                        T ur = 0, us = 0, ut = 0; /* C1 gradient */                           \
                        for (int l = 0; l < N; ++l)                                           \
                            ur = FMA(D[i * N + l], ue[((int64_t)k * N + j) * N + l], ur);     \
                        for (int l = 0; l < N; ++l)                                           \
                            us = FMA(D[j * N + l], ue[((int64_t)k * N + l) * N + i], us);     \
                        for (int l = 0; l < N; ++l)                                           \
                            ut = FMA(D[k * N + l], ue[((int64_t)l * N + j) * N + i], ut);     \
                        T g1 = Ge[0 * nn + pt], g2 = Ge[1 * nn + pt], g3 = Ge[2 * nn + pt];   \
                        T g4 = Ge[3 * nn + pt], g5 = Ge[4 * nn + pt], g6 = Ge[5 * nn + pt];   \
                        T a; /* C2 metric */                                                  \
                        a = MUL(g1, ur); a = FMA(g2, us, a); a = FMA(g3, ut, a); wr[pt] = a;  \
                        a = MUL(g2, ur); a = FMA(g4, us, a); a = FMA(g5, ut, a); ws[pt] = a;  \
                        a = MUL(g3, ur); a = FMA(g5, us, a); a = FMA(g6, ut, a); wt[pt] = a;  \
                    }                                                                         \
            for (int k = 0; k < N; ++k)                                                       \
                for (int j = 0; j < N; ++j)                                                   \
                    for (int i = 0; i < N; ++i) {                                             \
                        T a = 0, b = 0; /* C3 transpose */                                    \
                        for (int l = 0; l < N; ++l)                                           \
                            a = FMA(D[l * N + i], wr[((int64_t)k * N + j) * N + l], a);       \
                        for (int l = 0; l < N; ++l)                                           \
                            a = FMA(D[l * N + j], ws[((int64_t)k * N + l) * N + i], a);       \
                        for (int l = 0; l < N; ++l)                                           \
                            b = FMA(D[l * N + k], wt[((int64_t)l * N + j) * N + i], b);       \
                        we[((int64_t)k * N + j) * N + i] = ADD(a, b);                         \
                    }                                                                         \
            free(wr);                                                                         \
        }                                                                                     \
    }

#define PLAIN_MUL(a, b) ((a) * (b))
#define PLAIN_ADD(a, b) ((a) + (b))
#define PLAIN_DIV(a, b) ((a) / (b))
DEFINE_AX_LOCAL(ora_ax_local64, double, fma, PLAIN_MUL, PLAIN_ADD)
DEFINE_AX_LOCAL(ora_ax_local32, float, fmaf, PLAIN_MUL, PLAIN_ADD)

/* ------------------------------------------------------------------ */
/* VPREC emulation ("VPREC intercepts each  */
/* FP operation, performs the computation in double precision and      */
/* rounds the result to the emulated precision", t in       */
/* [3, 52], CG-loop scope).  vp(x) rounds a binary64 value to t         */
/* explicit mantissa bits, round to nearest, ties to even, on the bit  */
/* pattern (binary64 exponent range; a carry into the exponent is the  */
/* correct rounding up; subnormals are rounded at the same absolute bit*/
/* position).  t >= 52 is the identity.                                 */
/* ------------------------------------------------------------------ */
static int g_vp_t = 52;

double ora_vprec_round(double x, int t)
{
    if (t >= 52 || !isfinite(x)) return x;
    uint64_t b;
    memcpy(&b, &x, 8);
    const int drop = 52 - t;
    const uint64_t mask = ((uint64_t)1 << drop) - 1, half = (uint64_t)1 << (drop - 1);
    const uint64_t low = b & mask;
    b &= ~mask;
    if (low > half || (low == half && ((b >> drop) & 1))) b += (uint64_t)1 << drop;
    double y;
    memcpy(&y, &b, 8);
    return y;
}
static double vp(double x) { return ora_vprec_round(x, g_vp_t); }
static double vp_fma(double a, double b, double c) { return vp(fma(a, b, c)); }
static double vp_mul(double a, double b) { return vp(a * b); }
static double vp_add(double a, double b) { return vp(a + b); }
static double vp_div(double a, double b) { return vp(a / b); }
static double vp_sqrt(double a) { return vp(sqrt(a)); }
DEFINE_AX_LOCAL(ora_ax_local_vp, double, vp_fma, vp_mul, vp_add)

/* ------------------------------------------------------------------ */
/* dssum (C4): for every global node, sum its copies in ascending local */
/* index order, s = w[L1]; s = s + w[L2]; ...; write s to every copy.   */
/* Plain form: one pass over L ascending into a global array.           */
/* Operates on the full mesh (all elements).                            */
/* mask (C5): masked points are assigned +0.                            */
/* ------------------------------------------------------------------ */
#define DEFINE_DSSUM(NAME, T, ADD)                                                            \
    void NAME(int ex, int ey, int ez, int N, T* w, int apply_mask)                            \
    {                                                                                         \
        ora_mesh m = {ex, ey, ez, N};                                                         \
        int64_t n = (int64_t)ex * ey * ez * n3(&m);                                           \
        int64_t ng = gnx(&m) * gny(&m) * gnz(&m);                                             \
        T* s = (T*)malloc(sizeof(T) * ng);                                                    \
        uint8_t* seen = (uint8_t*)calloc(ng, 1);                                              \
        for (int64_t L = 0; L < n; ++L) {                                                     \
            int64_t g = point_gid(&m, L);                                                     \
            if (!seen[g]) { s[g] = w[L]; seen[g] = 1; }                                       \
            else s[g] = ADD(s[g], w[L]);                                                      \
        }                                                                                     \
        for (int64_t L = 0; L < n; ++L) {                                                     \
            int64_t g = point_gid(&m, L);                                                     \
            w[L] = (apply_mask && point_masked(&m, g)) ? (T)0 : s[g];                         \
        }                                                                                     \
        free(s);                                                                              \
        free(seen);                                                                           \
    }

DEFINE_DSSUM(ora_dssum64, double, PLAIN_ADD)
DEFINE_DSSUM(ora_dssum32, float, PLAIN_ADD)

#define DEFINE_MASK(NAME, T)                                                                  \
    void NAME(int ex, int ey, int ez, int N, T* w)                                            \
    {                                                                                         \
        ora_mesh m = {ex, ey, ez, N};                                                         \
        int64_t n = (int64_t)ex * ey * ez * n3(&m);                                           \
        for (int64_t L = 0; L < n; ++L)                                                       \
            if (point_masked(&m, point_gid(&m, L))) w[L] = (T)0;                              \
    }
DEFINE_MASK(ora_mask64, double)
DEFINE_MASK(ora_mask32, float)

/* full operator ax = mask o dssum o (ax_e per element)  (T1 line 5)   */
void ora_ax64(int ex, int ey, int ez, int N, const double* D, const double* G, const double* u,
              double* w, int apply_mask)
{
    ora_ax_local64((int64_t)ex * ey * ez, N, D, G, u, w);
    ora_dssum64(ex, ey, ez, N, w, apply_mask);
}
void ora_ax32(int ex, int ey, int ez, int N, const float* D, const float* G, const float* u,
              float* w, int apply_mask)
{
    ora_ax_local32((int64_t)ex * ey * ez, N, D, G, u, w);
    ora_dssum32(ex, ey, ez, N, w, apply_mask);
}

/* ------------------------------------------------------------------ */
/* Exact summation (C6): correctly rounded sum of binary64 terms.       */
/* Shewchuk's non-overlapping partials ("msum"), followed by the        */
/* round-half-even correction of the final partial sum.  The result is  */
/* RN64(exact sum), independent of term order.                          */
/* ------------------------------------------------------------------ */
#define MAXPART 256
typedef struct {
    double p[MAXPART];
    int n;
    double special; /* sum of non-finite terms (propagates inf/nan) */
    int has_special;
} xsum;

static void xsum_init(xsum* s) { s->n = 0; s->special = 0.0; s->has_special = 0; }

static void xsum_add(xsum* s, double x)
{
    if (!isfinite(x)) { s->special += x; s->has_special = 1; return; }
    int i = 0;
    for (int q = 0; q < s->n; ++q) {
        double y = s->p[q];
        if (fabs(x) < fabs(y)) { double t = x; x = y; y = t; }
        double hi = x + y;
        double lo = y - (hi - x);
        if (lo != 0.0) s->p[i++] = lo;
        x = hi;
    }
    s->p[i] = x;
    s->n = i + 1;
}

static double xsum_round(const xsum* s)
{
    if (s->has_special) return s->special;
    int n = s->n;
    double hi = 0.0, lo = 0.0;
    if (n > 0) {
        hi = s->p[--n];
        while (n > 0) {
            double x = hi, y = s->p[--n];
            hi = x + y;
            double yr = hi - x;
            lo = y - yr;
            if (lo != 0.0) break;
        }
        /* half-way case: if the remaining partials push in the same
           direction as lo, rounding hi+lo went the wrong way */
        if (n > 0 && ((lo < 0.0 && s->p[n - 1] < 0.0) || (lo > 0.0 && s->p[n - 1] > 0.0))) {
            double y = lo * 2.0;
            double x = hi + y;
            double yr = x - hi;
            if (y == yr) hi = x;
        }
    }
    return hi;
}

double ora_fsum(int64_t n, const double* t)
{
    xsum s;
    xsum_init(&s);
    for (int64_t i = 0; i < n; ++i) xsum_add(&s, t[i]);
    return xsum_round(&s);
}

/* glsc3 (T1 lines 3,6,9) with exact accumulation (C6):
 * FP64 vectors : t_L = RN64(a_L b_L) * c_L
 * FP32 vectors : t_L = (double)a_L * (double)b_L * c_L  (exact)
 * Parallel version: fixed chunks, each an exact expansion, merged
 * exactly -- so the result is the same correctly rounded value. */
#define CHUNK 65536
#define DEFINE_GLSC3(NAME, T)                                                                  \
    double NAME(int64_t n, const T* a, const T* b, const double* c)                           \
    {                                                                                          \
        int64_t nch = (n + CHUNK - 1) / CHUNK;                                                 \
        xsum* part = (xsum*)malloc(sizeof(xsum) * (nch > 0 ? nch : 1));                        \
        _Pragma("omp parallel for schedule(static)") for (int64_t ch = 0; ch < nch; ++ch)     \
        {                                                                                      \
            xsum_init(&part[ch]);                                                              \
            int64_t lo = ch * CHUNK, hi = lo + CHUNK < n ? lo + CHUNK : n;                     \
            for (int64_t L = lo; L < hi; ++L) {                                                \
                double ab = (double)a[L] * (double)b[L];                                       \
                xsum_add(&part[ch], ab * c[L]);                                                \
            }                                                                                  \
        }                                                                                      \
        xsum tot;                                                                              \
        xsum_init(&tot);                                                                       \
        for (int64_t ch = 0; ch < nch; ++ch) {                                                 \
            if (part[ch].has_special) { tot.special += part[ch].special; tot.has_special = 1; } \
            for (int q = 0; q < part[ch].n; ++q) xsum_add(&tot, part[ch].p[q]);                \
        }                                                                                      \
        free(part);                                                                            \
        return xsum_round(&tot);                                                               \
    }
DEFINE_GLSC3(ora_glsc3_64, double)
DEFINE_GLSC3(ora_glsc3_32, float)

/* RN32 of the exact sum held in an expansion: h = RN64(S); RN32(h) equals
 * RN32(S) unless h is exactly half-way between two binary32 neighbours and
 * S != h, in which case the sign of S - h (from the expansion) decides. */
static float xsum_round32(const xsum* s)
{
    double h = xsum_round(s);
    float f = (float)h;
    if (!isfinite(h) || (double)f == h) return f;
    float a = nextafterf(f, h > (double)f ? INFINITY : -INFINITY);
    double mid = ((double)f + (double)a) * 0.5;  /* exact: two binary32 values */
    if (h != mid) return f;
    xsum t = *s;
    xsum_add(&t, -h);
    double r = xsum_round(&t);
    if (r == 0.0) return f;  /* exact tie: (float)h rounded half to even */
    return r > 0.0 ? (f > a ? f : a) : (f < a ? f : a);
}

/* Paper-literal single-precision glsc3 ("solver
 * runs exclusively in single", P:507 math.f in single; reading R11b in
 * DESIGN.md): terms RN32(a_L b_L) c_L (c = 1/m exact), the sum rounded once
 * to binary32 -- the best a binary32 accumulator can return. */
float ora_glsc3_32s(int64_t n, const float* a, const float* b, const double* c)
{
    int64_t nch = (n + CHUNK - 1) / CHUNK;
    xsum* part = (xsum*)malloc(sizeof(xsum) * (nch > 0 ? nch : 1));
#pragma omp parallel for schedule(static)
    for (int64_t ch = 0; ch < nch; ++ch) {
        xsum_init(&part[ch]);
        int64_t lo = ch * CHUNK, hi = lo + CHUNK < n ? lo + CHUNK : n;
        for (int64_t L = lo; L < hi; ++L) {
            float ab = a[L] * b[L];
            xsum_add(&part[ch], (double)ab * c[L]);
        }
    }
    xsum tot;
    xsum_init(&tot);
    for (int64_t ch = 0; ch < nch; ++ch) {
        if (part[ch].has_special) { tot.special += part[ch].special; tot.has_special = 1; }
        for (int q = 0; q < part[ch].n; ++q) xsum_add(&tot, part[ch].p[q]);
    }
    free(part);
    return xsum_round32(&tot);
}

/* Paper-literal binary32 accumulation (NEXT-2 as the paper ran it: "the
 * solver runs exclusively in single precision", P:507 math.f -- where glsc3
 * lives -- converted to single, P:510 single-precision MPI communication).
 * Nekbone's glsc3 loop, tmp = tmp + a(i)*b(i)*mult(i), in binary32 and in
 * ascending local index, no contraction (-O2; reading R11c): per rank
 * t = RN32(RN32(a_L b_L) c_L), s = RN32(s + t); then the all-reduce, in
 * binary32 and in rank order.  Ranks own contiguous element ranges (z-slabs,
 * R21), i.e. contiguous ranges of L: rank r the range [r n/P, (r+1) n/P). */
static int g_glsc3a_ranks = 1;
float ora_glsc3_32a_p(int64_t n, const float* a, const float* b, const double* c, int nranks)
{
    float tot = 0.0f;
    for (int r = 0; r < nranks; ++r) {
        const int64_t lo = n * r / nranks, hi = n * (r + 1) / nranks;
        float s = 0.0f;
        for (int64_t L = lo; L < hi; ++L) {
            const float ab = a[L] * b[L];
            const float t = ab * (float)c[L];
            s = s + t;
        }
        tot = r == 0 ? s : tot + s;
    }
    return tot;
}
static float ora_glsc3_32a(int64_t n, const float* a, const float* b, const double* c)
{
    return ora_glsc3_32a_p(n, a, b, c, g_glsc3a_ranks);
}

/* RN32 of an exact sum of binary64 terms (pins the GPU's dd -> binary32 step) */
float ora_fsum32(int64_t n, const double* t)
{
    xsum s;
    xsum_init(&s);
    for (int64_t i = 0; i < n; ++i) xsum_add(&s, t[i]);
    return xsum_round32(&s);
}

/* c = 1/m per local point of the whole mesh (R8) */
static double* make_c(const ora_mesh* m)
{
    int64_t n = (int64_t)m->ex * m->ey * m->ez * n3(m);
    double* c = (double*)malloc(sizeof(double) * n);
#pragma omp parallel for schedule(static)
    for (int64_t L = 0; L < n; ++L) c[L] = 1.0 / node_mult(m, point_gid(m, L));
    return c;
}

void ora_multiplicity_weight(int ex, int ey, int ez, int N, double* c_out)
{
    ora_mesh m = {ex, ey, ez, N};
    double* c = make_c(&m);
    int64_t n = (int64_t)ex * ey * ez * n3(&m);
    memcpy(c_out, c, sizeof(double) * n);
    free(c);
}

/* ------------------------------------------------------------------ */
/* Jacobi preconditioner (T1 line 2 "solveM"; */
/* S:376-384): d = diag(A), the assembled diagonal of the stiffness      */
/* operator, masked entries set to 1; dinv = 1/d.                        */
/* A_e = sum_{m,n in r,s,t} D_m^T diag(g_mn) D_n with D_r = I x I x D   */
/* (i fastest) etc., so its diagonal at (i,j,k) is                      */
/*   sum_a D[a][i]^2 g1(a,j,k) + sum_b D[b][j]^2 g4(i,b,k)              */
/*   + sum_c D[c][k]^2 g6(i,j,c)                                        */
/*   + 2 (D[i][i] D[j][j] g2 + D[i][i] D[k][k] g3 + D[j][j] D[k][k] g5) */
/* (only the q = L term survives in the mixed products).  A node occurs */
/* at most once per element, so the assembled diagonal is the dssum of  */
/* the local diagonals.  FP64 throughout (set-up).               */
/* ------------------------------------------------------------------ */
void ora_jacobi_dinv(int ex, int ey, int ez, int N, const double* D, const double* G,
                     double* d_out, double* dinv_out)
{
    ora_mesh m = {ex, ey, ez, N};
    int64_t E = (int64_t)ex * ey * ez, nn = n3(&m), n = E * nn;
    double* d = (double*)malloc(sizeof(double) * n);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        const double* g = G + e * 6 * nn;
        for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j)
                for (int i = 0; i < N; ++i) {
                    int64_t q = ((int64_t)k * N + j) * N + i;
                    double s = 0.0;
                    for (int a = 0; a < N; ++a)
                        s += D[a * N + i] * D[a * N + i] * g[0 * nn + ((int64_t)k * N + j) * N + a];
                    for (int b = 0; b < N; ++b)
                        s += D[b * N + j] * D[b * N + j] * g[3 * nn + ((int64_t)k * N + b) * N + i];
                    for (int c = 0; c < N; ++c)
                        s += D[c * N + k] * D[c * N + k] * g[5 * nn + ((int64_t)c * N + j) * N + i];
                    s += 2.0 * (D[i * N + i] * D[j * N + j] * g[1 * nn + q] +
                                D[i * N + i] * D[k * N + k] * g[2 * nn + q] +
                                D[j * N + j] * D[k * N + k] * g[4 * nn + q]);
                    d[e * nn + q] = s;
                }
    }
    ora_dssum64(ex, ey, ez, N, d, 0);
    for (int64_t L = 0; L < n; ++L) {
        if (point_masked(&m, point_gid(&m, L))) d[L] = 1.0;
        if (d_out) d_out[L] = d[L];
        if (dinv_out) dinv_out[L] = 1.0 / d[L];
    }
    free(d);
}

/* ------------------------------------------------------------------ */
/* Fixed-iteration CG (T1 P:142-152; C7-C9; R9, R10), unpreconditioned  */
/* (dinv == NULL: solveM is the identity, z = r, MGRID off) or   */
/* Jacobi-preconditioned (z = RN_T(r * dinv_T)).             */
/*   x0 = 0; r0 = f; p0 = 0; rtr0 = glsc3(r,c,r); h0 = sqrt(rtr0)       */
/*   for k = 1..niter:                                                  */
/*     z = solveM(r); rtz1 = glsc3(r,c,z)  (= rtr_{k-1} when z = r)     */
/*     beta = 0 if k == 1 else rtz1/rtz2                                */
/*     p = beta p + z       (add2s1)                                    */
/*     w = ax(p)            (ax: local, dssum, mask)                    */
/*     pap = glsc3(w,c,p); alpha = rtz1/pap                             */
/*     x = x + alpha p      (add2s2); r = r + (-alpha) w (add2s2)        */
/*     rtr = glsc3(r,c,r); h_k = sqrt(rtr); rtz2 = rtz1                 */
/* hist[0..niter], trace[5*(k-1) + {0..4}] = rtz1, beta, alpha, pap, rtr */
/* Returns the first iteration with pap <= 0 or a non-finite scalar     */
/* (defect) or 0.                                                */
/* ------------------------------------------------------------------ */
#define DEFINE_CG(NAME, T, S, FMA, SQRT, DIV, AXLOCAL, DSSUM, GLSC3)                                          \
    int NAME(int ex, int ey, int ez, int N, const T* D, const T* G, const T* f, const T* dinv,  \
             int niter, T* x, double* hist, double* trace)                                      \
    {                                                                                           \
        ora_mesh m = {ex, ey, ez, N};                                                           \
        int64_t E = (int64_t)ex * ey * ez, n = E * n3(&m);                                      \
        double* c = make_c(&m);                                                                 \
        T* r = (T*)malloc(sizeof(T) * n);                                                       \
        T* p = (T*)malloc(sizeof(T) * n);                                                       \
        T* w = (T*)malloc(sizeof(T) * n);                                                       \
        T* z = dinv ? (T*)malloc(sizeof(T) * n) : r;                                            \
        for (int64_t L = 0; L < n; ++L) { x[L] = 0; r[L] = f[L]; p[L] = 0; }                    \
        S rtr = GLSC3(n, r, r, c);                                                              \
        hist[0] = (double)SQRT(rtr);                                                            \
        S rtz = rtr;                                                                            \
        if (dinv) {                                                                             \
            for (int64_t L = 0; L < n; ++L) z[L] = r[L] * dinv[L];                              \
            rtz = GLSC3(n, r, z, c);                                                            \
        }                                                                                       \
        S rtz2 = 0;                                                                             \
        int defect = 0, zero = 0;                                                               \
        for (int k = 1; k <= niter; ++k) {                                                      \
            S rtz1 = rtz, beta = 0, alpha = 0, pap;                                             \
            if (rtz1 == 0.0) zero = 1;                                                          \
            if (!zero && k > 1) beta = DIV(rtz1, rtz2);                                         \
            T betaT = (T)beta;                                                                  \
            for (int64_t L = 0; L < n; ++L) p[L] = FMA(betaT, p[L], z[L]);                      \
            AXLOCAL(E, N, D, G, p, w);                                                          \
            DSSUM(ex, ey, ez, N, w, 1);                                                         \
            pap = GLSC3(n, w, p, c);                                                            \
            if (!zero) alpha = DIV(rtz1, pap);                                                  \
            T alphaT = (T)alpha, alphmT = -alphaT;                                              \
            for (int64_t L = 0; L < n; ++L) x[L] = FMA(alphaT, p[L], x[L]);                     \
            for (int64_t L = 0; L < n; ++L) r[L] = FMA(alphmT, w[L], r[L]);                     \
            rtr = GLSC3(n, r, r, c);                                                            \
            hist[k] = (double)SQRT(rtr);                                                        \
            rtz = rtr;                                                                          \
            if (dinv) {                                                                         \
                for (int64_t L = 0; L < n; ++L) z[L] = r[L] * dinv[L];                          \
                rtz = GLSC3(n, r, z, c);                                                        \
            }                                                                                   \
            if (!zero && !defect &&                                                             \
                (!(pap > 0.0) || !isfinite(pap) || !isfinite(rtr) || !isfinite(rtz)))           \
                defect = k;                                                                     \
            if (trace) {                                                                        \
                double* tr = trace + 5 * (int64_t)(k - 1);                                      \
                tr[0] = rtz1; tr[1] = beta; tr[2] = alpha; tr[3] = pap; tr[4] = rtr;            \
            }                                                                                   \
            rtz2 = rtz1;                                                                        \
        }                                                                                       \
        free(c); free(r); free(p); free(w);                                                     \
        if (dinv) free(z);                                                                      \
        return defect;                                                                          \
    }

DEFINE_CG(ora_cg64_core, double, double, fma, sqrt, PLAIN_DIV, ora_ax_local64, ora_dssum64, ora_glsc3_64)
DEFINE_CG(ora_cg32_core, float, double, fmaf, sqrt, PLAIN_DIV, ora_ax_local32, ora_dssum32, ora_glsc3_32)
/* paper-literal single precision: binary32 inner products (above) and binary32
 * scalars: beta = rtz1/rtz2, alpha = rtz1/pap, sqrt in binary32 (NEXT-2) */
DEFINE_CG(ora_cg32s_core, float, float, fmaf, sqrtf, PLAIN_DIV, ora_ax_local32, ora_dssum32, ora_glsc3_32s)
/* the paper's single-precision solver (NEXT-2, reading R11c): binary32
 * accumulation of every inner product and binary32 scalars */
DEFINE_CG(ora_cg32a_core, float, float, fmaf, sqrtf, PLAIN_DIV, ora_ax_local32, ora_dssum32, ora_glsc3_32a)

/* VPREC CG loop (NEXT-4): binary64 loop with every operation of the CG
 * kernels rounded to t bits (ax: every fma / mul / add; dssum adds; the
 * p, x, r updates; glsc3 terms vp(a b) c and the glsc3 result vp(RN64(sum));
 * alpha, beta, sqrt).  Set-up data (D, G, f) are not rounded (CG scope). */
static double ora_glsc3_vp(int64_t n, const double* a, const double* b, const double* c)
{
    int64_t nch = (n + CHUNK - 1) / CHUNK;
    xsum* part = (xsum*)malloc(sizeof(xsum) * (nch > 0 ? nch : 1));
#pragma omp parallel for schedule(static)
    for (int64_t ch = 0; ch < nch; ++ch) {
        xsum_init(&part[ch]);
        int64_t lo = ch * CHUNK, hi = lo + CHUNK < n ? lo + CHUNK : n;
        for (int64_t L = lo; L < hi; ++L) xsum_add(&part[ch], vp(a[L] * b[L]) * c[L]);
    }
    xsum tot;
    xsum_init(&tot);
    for (int64_t ch = 0; ch < nch; ++ch) {
        if (part[ch].has_special) { tot.special += part[ch].special; tot.has_special = 1; }
        for (int q = 0; q < part[ch].n; ++q) xsum_add(&tot, part[ch].p[q]);
    }
    free(part);
    return vp(xsum_round(&tot));
}
DEFINE_DSSUM(ora_dssum_vp, double, vp_add)
DEFINE_CG(ora_cgvp_core, double, double, vp_fma, vp_sqrt, vp_div, ora_ax_local_vp, ora_dssum_vp, ora_glsc3_vp)

int ora_cgvp(int ex, int ey, int ez, int N, const double* D, const double* G, const double* f, int t,
             int niter, double* x, double* hist, double* trace)
{
    g_vp_t = t;
    int rc = ora_cgvp_core(ex, ey, ez, N, D, G, f, NULL, niter, x, hist, trace);
    g_vp_t = 52;
    return rc;
}

int ora_cg64(int ex, int ey, int ez, int N, const double* D, const double* G, const double* f,
             int niter, double* x, double* hist, double* trace)
{
    return ora_cg64_core(ex, ey, ez, N, D, G, f, NULL, niter, x, hist, trace);
}

/* Mixed precision: FP64 setup data are converted once to
 * binary32 (C11: D32, G32, f32 = RN32), the loop runs in FP32. */
int ora_cg32(int ex, int ey, int ez, int N, const double* D, const double* G, const double* f,
             int niter, float* x32, double* hist, double* trace)
{
    int64_t E = (int64_t)ex * ey * ez, nn = (int64_t)N * N * N, n = E * nn;
    float* D32 = (float*)malloc(sizeof(float) * N * N);
    float* G32 = (float*)malloc(sizeof(float) * 6 * n);
    float* f32 = (float*)malloc(sizeof(float) * n);
    for (int q = 0; q < N * N; ++q) D32[q] = (float)D[q];
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < 6 * n; ++q) G32[q] = (float)G[q];
    for (int64_t q = 0; q < n; ++q) f32[q] = (float)f[q];
    int rc = ora_cg32_core(ex, ey, ez, N, D32, G32, f32, NULL, niter, x32, hist, trace);
    free(D32); free(G32); free(f32);
    return rc;
}

/* Paper-literal single-precision solver (NEXT-2): as ora_cg32 / ora_pcg32
 * but the inner products and the CG scalars are binary32 too (dinv may be
 * NULL: unpreconditioned). */
int ora_cg32s(int ex, int ey, int ez, int N, const double* D, const double* G, const double* f,
              const double* dinv, int niter, float* x32, double* hist, double* trace)
{
    int64_t E = (int64_t)ex * ey * ez, nn = (int64_t)N * N * N, n = E * nn;
    float* D32 = (float*)malloc(sizeof(float) * N * N);
    float* G32 = (float*)malloc(sizeof(float) * 6 * n);
    float* f32 = (float*)malloc(sizeof(float) * n);
    float* di32 = dinv ? (float*)malloc(sizeof(float) * n) : NULL;
    for (int q = 0; q < N * N; ++q) D32[q] = (float)D[q];
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < 6 * n; ++q) G32[q] = (float)G[q];
    for (int64_t q = 0; q < n; ++q) {
        f32[q] = (float)f[q];
        if (di32) di32[q] = (float)dinv[q];
    }
    int rc = ora_cg32s_core(ex, ey, ez, N, D32, G32, f32, di32, niter, x32, hist, trace);
    free(D32); free(G32); free(f32); free(di32);
    return rc;
}

int ora_cg32a(int ex, int ey, int ez, int N, const double* D, const double* G, const double* f,
              const double* dinv, int nranks, int niter, float* x32, double* hist, double* trace)
{
    int64_t E = (int64_t)ex * ey * ez, nn = (int64_t)N * N * N, n = E * nn;
    float* D32 = (float*)malloc(sizeof(float) * N * N);
    float* G32 = (float*)malloc(sizeof(float) * 6 * n);
    float* f32 = (float*)malloc(sizeof(float) * n);
    float* di32 = dinv ? (float*)malloc(sizeof(float) * n) : NULL;
    for (int q = 0; q < N * N; ++q) D32[q] = (float)D[q];
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < 6 * n; ++q) G32[q] = (float)G[q];
    for (int64_t q = 0; q < n; ++q) {
        f32[q] = (float)f[q];
        if (di32) di32[q] = (float)dinv[q];
    }
    g_glsc3a_ranks = nranks < 1 ? 1 : nranks;
    int rc = ora_cg32a_core(ex, ey, ez, N, D32, G32, f32, di32, niter, x32, hist, trace);
    g_glsc3a_ranks = 1;
    free(D32); free(G32); free(f32); free(di32);
    return rc;
}

/* ------------------------------------------------------------------ */
/* Precision-emulated CG (NEXT-4), the CG loop of   */
/* T1 written out with every operation through an emulation op:         */
/*   VPREC (mode 1): result rounded to t mantissa bits;                 */
/*   RR    (mode 2): result -> x + 2^(e_x - t) xi (random rounding);    */
/*   MCA   (mode 3): operands and result perturbed (full MCA);          */
/* xi = SplitMix64(seed, 4 key + slot) - 1/2 in [-1/2, 1/2), e_x =       */
/* floor(log2|x|) + 1, slot 0 = result, 1.. = operands in order.        */
/* key = ((it*8 + phase) * 2^40 + L) * 128 + op, phases A (ax step: ops  */
/* per output point: 0 p update, 1 x update [key of iteration it+1, the  */
/* iteration whose step applies it], 2.. ur, 2+N.. us, 2+2N.. ut chains, */
/* 2+3N.. metric (9), 11+3N.. r/s transpose chain (2N), 11+5N+l t chain, */
/* 11+6N final add), B (dssum: chain add c of a node, L = first copy),   */
/* C (r update), S (scalars, L = 0: 0 pap, 1 alpha, 2 rtr, 3 sqrt, 4     */
/* beta of the next iteration; iteration 0 = initial rtr, h0).  L is the */
/* local index of the point the operation produces: every dynamic FP     */
/* operation draws its own xi ("the result and/or operands of   */
/* each FP operation is replaced by a perturbed computation"), so the    */
/* pointwise updates of the copies of a shared node are perturbed        */
/* independently and, under RR / MCA, p, x and r are not continuous;     */
/* dssum still writes one chain sum per node to every copy (C4).  Each   */
/* correctly rounded glsc3 is one operation (VPREC also rounds the       */
/* products of its terms).  This function shares no code with the       */
/* macro-generated VPREC loop above (cross-checked in the pins).         */
/* ------------------------------------------------------------------ */
static int g_pm_mode = 0, g_pm_t = 52;
static uint64_t g_pm_seed = 0;
enum { ORA_PH_A = 0, ORA_PH_B = 1, ORA_PH_C = 2, ORA_PH_S = 3 };

static uint64_t pm_key(int it, int ph, int64_t L, int o)
{
    return (((uint64_t)it * 8u + (uint64_t)ph) * ((uint64_t)1 << 40) + (uint64_t)L) * 128u + (uint64_t)o;
}
static double pm_inexact(double x, uint64_t key, int slot)
{
    if (x == 0.0 || !isfinite(x)) return x;
    uint64_t z = ora_splitmix64(g_pm_seed, 4 * key + (uint64_t)slot);
    double xi = (double)(z >> 11) * 0x1.0p-53 - 0.5;
    int ex;
    frexp(x, &ex);
    return x + ldexp(xi, ex - g_pm_t);
}
static double pm_res(double r, uint64_t key)
{
    if (g_pm_mode == 1) return ora_vprec_round(r, g_pm_t);
    if (g_pm_mode >= 2) return pm_inexact(r, key, 0);
    return r;
}
static double pm_in(double x, uint64_t key, int slot) { return g_pm_mode == 3 ? pm_inexact(x, key, slot) : x; }
static double P_FMA(double a, double b, double c, uint64_t k)
{
    return pm_res(fma(pm_in(a, k, 1), pm_in(b, k, 2), pm_in(c, k, 3)), k);
}
static double P_MUL(double a, double b, uint64_t k) { return pm_res(pm_in(a, k, 1) * pm_in(b, k, 2), k); }
static double P_ADD(double a, double b, uint64_t k) { return pm_res(pm_in(a, k, 1) + pm_in(b, k, 2), k); }
static double P_DIV(double a, double b, uint64_t k) { return pm_res(pm_in(a, k, 1) / pm_in(b, k, 2), k); }
static double P_SQRT(double a, uint64_t k) { return pm_res(sqrt(pm_in(a, k, 1)), k); }

static void pm_ax_local(int it, int64_t E, int N, const double* D, const double* G, const double* u,
                        double* w)
{
    const int64_t nn = (int64_t)N * N * N;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        const double* ue = u + e * nn;
        const double* Ge = G + e * 6 * nn;
        double* we = w + e * nn;
        double* wr = (double*)malloc(sizeof(double) * 3 * nn);
        double* ws = wr + nn;
        double* wt = ws + nn;
        for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j)
                for (int i = 0; i < N; ++i) {
                    int64_t pt = ((int64_t)k * N + j) * N + i, L = e * nn + pt;
                    double ur = 0, us = 0, ut = 0;
                    for (int l = 0; l < N; ++l)
                        ur = P_FMA(D[i * N + l], ue[((int64_t)k * N + j) * N + l], ur, pm_key(it, ORA_PH_A, L, 2 + l));
                    for (int l = 0; l < N; ++l)
                        us = P_FMA(D[j * N + l], ue[((int64_t)k * N + l) * N + i], us, pm_key(it, ORA_PH_A, L, 2 + N + l));
                    for (int l = 0; l < N; ++l)
                        ut = P_FMA(D[k * N + l], ue[((int64_t)l * N + j) * N + i], ut, pm_key(it, ORA_PH_A, L, 2 + 2 * N + l));
                    const double g1 = Ge[0 * nn + pt], g2 = Ge[1 * nn + pt], g3 = Ge[2 * nn + pt];
                    const double g4 = Ge[3 * nn + pt], g5 = Ge[4 * nn + pt], g6 = Ge[5 * nn + pt];
                    const int om = 2 + 3 * N;
                    double a;
                    a = P_MUL(g1, ur, pm_key(it, ORA_PH_A, L, om));
                    a = P_FMA(g2, us, a, pm_key(it, ORA_PH_A, L, om + 1));
                    a = P_FMA(g3, ut, a, pm_key(it, ORA_PH_A, L, om + 2));
                    wr[pt] = a;
                    a = P_MUL(g2, ur, pm_key(it, ORA_PH_A, L, om + 3));
                    a = P_FMA(g4, us, a, pm_key(it, ORA_PH_A, L, om + 4));
                    a = P_FMA(g5, ut, a, pm_key(it, ORA_PH_A, L, om + 5));
                    ws[pt] = a;
                    a = P_MUL(g3, ur, pm_key(it, ORA_PH_A, L, om + 6));
                    a = P_FMA(g5, us, a, pm_key(it, ORA_PH_A, L, om + 7));
                    a = P_FMA(g6, ut, a, pm_key(it, ORA_PH_A, L, om + 8));
                    wt[pt] = a;
                }
        for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j)
                for (int i = 0; i < N; ++i) {
                    int64_t L = e * nn + ((int64_t)k * N + j) * N + i;
                    double a = 0, b = 0;
                    for (int l = 0; l < N; ++l)
                        a = P_FMA(D[l * N + i], wr[((int64_t)k * N + j) * N + l], a, pm_key(it, ORA_PH_A, L, 11 + 3 * N + l));
                    for (int l = 0; l < N; ++l)
                        a = P_FMA(D[l * N + j], ws[((int64_t)k * N + l) * N + i], a, pm_key(it, ORA_PH_A, L, 11 + 4 * N + l));
                    for (int l = 0; l < N; ++l)
                        b = P_FMA(D[l * N + k], wt[((int64_t)l * N + j) * N + i], b, pm_key(it, ORA_PH_A, L, 11 + 5 * N + l));
                    we[((int64_t)k * N + j) * N + i] = P_ADD(a, b, pm_key(it, ORA_PH_A, L, 11 + 6 * N));
                }
        free(wr);
    }
}

static void pm_dssum_mask(int it, const ora_mesh* m, double* w)
{
    int64_t n = (int64_t)m->ex * m->ey * m->ez * n3(m);
    int64_t ng = gnx(m) * gny(m) * gnz(m);
    double* s = (double*)malloc(sizeof(double) * ng);
    int64_t* first = (int64_t*)malloc(sizeof(int64_t) * ng);
    int* cnt = (int*)calloc(ng, sizeof(int));
    for (int64_t L = 0; L < n; ++L) {
        int64_t g = point_gid(m, L);
        if (cnt[g] == 0) { s[g] = w[L]; first[g] = L; }
        else s[g] = P_ADD(s[g], w[L], pm_key(it, ORA_PH_B, first[g], cnt[g]));
        cnt[g]++;
    }
    for (int64_t L = 0; L < n; ++L) {
        int64_t g = point_gid(m, L);
        w[L] = point_masked(m, g) ? 0.0 : s[g];
    }
    free(s); free(first); free(cnt);
}

/* glsc3 as one emulated operation: exact sum of the terms (VPREC rounds the
 * products), then the result through the emulation op */
static double pm_glsc3(int64_t n, const double* a, const double* b, const double* c, uint64_t key)
{
    xsum tot;
    xsum_init(&tot);
    for (int64_t L = 0; L < n; ++L) {
        double ab = a[L] * b[L];
        if (g_pm_mode == 1) ab = ora_vprec_round(ab, g_pm_t);
        xsum_add(&tot, ab * c[L]);
    }
    return pm_res(xsum_round(&tot), key);
}

int ora_cgpm(int ex, int ey, int ez, int N, const double* D, const double* G, const double* f, int mode,
             int t, uint64_t seed, int niter, double* x, double* hist, double* trace)
{
    ora_mesh m = {ex, ey, ez, N};
    int64_t E = (int64_t)ex * ey * ez, n = E * n3(&m);
    g_pm_mode = mode;
    g_pm_t = t;
    g_pm_seed = seed;
    double* c = make_c(&m);
    double* r = (double*)malloc(sizeof(double) * n);
    double* p = (double*)malloc(sizeof(double) * n);
    double* w = (double*)malloc(sizeof(double) * n);
    for (int64_t L = 0; L < n; ++L) { x[L] = 0; r[L] = f[L]; p[L] = 0; }
    double rtr = pm_glsc3(n, r, r, c, pm_key(0, ORA_PH_S, 0, 2));
    hist[0] = P_SQRT(rtr, pm_key(0, ORA_PH_S, 0, 3));
    double rtz = rtr, rtz2 = 0.0;
    int defect = 0, zero = 0;
    for (int k = 1; k <= niter; ++k) {
        double rtz1 = rtz, beta = 0.0, alpha = 0.0, pap;
        if (rtz1 == 0.0) zero = 1;
        if (!zero && k > 1) beta = P_DIV(rtz1, rtz2, pm_key(k - 1, ORA_PH_S, 0, 4));
        for (int64_t L = 0; L < n; ++L) p[L] = P_FMA(beta, p[L], r[L], pm_key(k, ORA_PH_A, L, 0));
        pm_ax_local(k, E, N, D, G, p, w);
        pm_dssum_mask(k, &m, w);
        pap = pm_glsc3(n, w, p, c, pm_key(k, ORA_PH_S, 0, 0));
        if (!zero) alpha = P_DIV(rtz1, pap, pm_key(k, ORA_PH_S, 0, 1));
        for (int64_t L = 0; L < n; ++L) x[L] = P_FMA(alpha, p[L], x[L], pm_key(k + 1, ORA_PH_A, L, 1));
        for (int64_t L = 0; L < n; ++L) r[L] = P_FMA(-alpha, w[L], r[L], pm_key(k, ORA_PH_C, L, 0));
        rtr = pm_glsc3(n, r, r, c, pm_key(k, ORA_PH_S, 0, 2));
        hist[k] = P_SQRT(rtr, pm_key(k, ORA_PH_S, 0, 3));
        rtz = rtr;
        if (!zero && !defect && (!(pap > 0.0) || !isfinite(pap) || !isfinite(rtr))) defect = k;
        if (trace) {
            double* tr = trace + 5 * (int64_t)(k - 1);
            tr[0] = rtz1; tr[1] = beta; tr[2] = alpha; tr[3] = pap; tr[4] = rtr;
        }
        rtz2 = rtz1;
    }
    free(c); free(r); free(p); free(w);
    g_pm_mode = 0; g_pm_t = 52; g_pm_seed = 0;
    return defect;
}

/* Jacobi PCG (NEXT-1): dinv is data (FP64, e.g. from ora_jacobi_dinv);
 * the FP32 loop uses dinv32 = RN32(dinv) (C11). */
int ora_pcg64(int ex, int ey, int ez, int N, const double* D, const double* G, const double* f,
              const double* dinv, int niter, double* x, double* hist, double* trace)
{
    return ora_cg64_core(ex, ey, ez, N, D, G, f, dinv, niter, x, hist, trace);
}

int ora_pcg32(int ex, int ey, int ez, int N, const double* D, const double* G, const double* f,
              const double* dinv, int niter, float* x32, double* hist, double* trace)
{
    int64_t E = (int64_t)ex * ey * ez, nn = (int64_t)N * N * N, n = E * nn;
    float* D32 = (float*)malloc(sizeof(float) * N * N);
    float* G32 = (float*)malloc(sizeof(float) * 6 * n);
    float* f32 = (float*)malloc(sizeof(float) * n);
    float* di32 = (float*)malloc(sizeof(float) * n);
    for (int q = 0; q < N * N; ++q) D32[q] = (float)D[q];
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < 6 * n; ++q) G32[q] = (float)G[q];
    for (int64_t q = 0; q < n; ++q) { f32[q] = (float)f[q]; di32[q] = (float)dinv[q]; }
    int rc = ora_cg32_core(ex, ey, ez, N, D32, G32, f32, di32, niter, x32, hist, trace);
    free(D32); free(G32); free(f32); free(di32);
    return rc;
}

/* Final FP64 residual check (C12, reading R12): x64 = (double)x (exact),
 * w = ax64(x64) with dssum and mask, r_true = f - w, returns
 * sqrt(glsc3(r_true, c, r_true)).  out_h0 (optional) = sqrt(glsc3(f,c,f)). */
double ora_true_residual(int ex, int ey, int ez, int N, const double* D, const double* G,
                         const double* f, const double* x64, double* out_h0)
{
    ora_mesh m = {ex, ey, ez, N};
    int64_t n = (int64_t)ex * ey * ez * n3(&m);
    double* c = make_c(&m);
    double* w = (double*)malloc(sizeof(double) * n);
    ora_ax64(ex, ey, ez, N, D, G, x64, w, 1);
    for (int64_t L = 0; L < n; ++L) w[L] = f[L] - w[L];
    double rr = ora_glsc3_64(n, w, w, c);
    if (out_h0) *out_h0 = sqrt(ora_glsc3_64(n, f, f, c));
    free(w);
    free(c);
    return sqrt(rr);
}

int ora_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
