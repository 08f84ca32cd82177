"""Pins of the CPU oracle against facts the paper's setting and the mathematics
fix (not against itself).  Each test names the pin id of DESIGN.md / SURVEY
8(c) c4 and the passage it follows.  CPU only (no GPU)."""
import math

import numpy as np
import pytest

from tests import inputs

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


# ---------------------------------------------------------------- helpers
def dense_stiffness(ora, mesh):
    """Brute force: assemble the global stiffness A = sum_e Q_e^T A_e Q_e with
    A_e = sum_mn D_m^T diag(g_mn) D_n built from Kronecker products (i fastest),
    independent of the oracle's tensor-product loops (pin P9)."""
    s = ora.setup(mesh, want=("G", "gid"))
    _, _, D = ora.gll(mesh.N)
    N = mesh.N
    I = np.eye(N)
    Dr = np.kron(I, np.kron(I, D))
    Ds = np.kron(I, np.kron(D, I))
    Dt = np.kron(D, np.kron(I, I))
    Dm = [Dr, Ds, Dt]
    comp = {(0, 0): 0, (0, 1): 1, (0, 2): 2, (1, 1): 3, (1, 2): 4, (2, 2): 5}
    ng = mesh.sizes()["n_global"]
    A = np.zeros((ng, ng))
    for e in range(mesh.E):
        Ge = s["G"][e].reshape(6, -1)
        Ae = np.zeros((N ** 3, N ** 3))
        for m in range(3):
            for n in range(3):
                g = Ge[comp[(min(m, n), max(m, n))]]
                Ae += Dm[m].T @ (g[:, None] * Dm[n])
        gid = s["gid"][e].reshape(-1)
        A[np.ix_(gid, gid)] += Ae
    return A, s["gid"].reshape(-1)


def global_mask(ora, mesh):
    s = ora.setup(mesh, want=("gid", "mask"))
    ng = mesh.sizes()["n_global"]
    mg = np.zeros(ng, dtype=bool)
    mg[s["gid"].reshape(-1)] = s["mask"].reshape(-1).astype(bool)
    return mg


def continuous(ora, mesh, vglob):
    gid = ora.setup(mesh, want=("gid",))["gid"]
    return vglob[gid]


# ------------------------------------------------------------ RNG (R5/R7)
def test_splitmix64_reference_vector(ora):
    # Published SplitMix64 output stream for state 0 (Steele, Lea & Flood 2014;
    # Vigna's reference splitmix64.c): z_i for i = 0, 1, 2.
    assert ora.splitmix64(0, 0) == 0xE220A8397B1DCDAF
    assert ora.splitmix64(0, 1) == 0x6E789E6AA1B965F4
    assert ora.splitmix64(0, 2) == 0x06C45D188009454F
    # random access: index i of seed s equals index 0 of seed s + i*gamma
    g = 0x9E3779B97F4A7C15
    assert ora.splitmix64(12345, 7) == ora.splitmix64((12345 + 7 * g) % 2**64, 0)
    v = [ora.uniform_pm1(1001, i) for i in range(2000)]
    assert min(v) >= -1.0 and max(v) < 1.0 and abs(np.mean(v)) < 0.05


# ------------------------------------------------------------- P1 GLL
def test_gll_closed_forms(ora):
    xi, rho, D = ora.gll(2)
    assert xi.tolist() == [-1.0, 1.0] and rho.tolist() == [1.0, 1.0]
    assert D.tolist() == [[-0.5, 0.5], [-0.5, 0.5]]
    xi, rho, D = ora.gll(3)  # Simpson: {1/3, 4/3, 1/3}
    assert xi.tolist() == [-1.0, 0.0, 1.0]
    np.testing.assert_allclose(rho, [1 / 3, 4 / 3, 1 / 3], rtol=0, atol=4e-16)


@pytest.mark.parametrize("N", list(range(2, 17)))
def test_gll_nodes_weights_vs_library(ora, N):
    xi, rho, _ = ora.gll(N)
    p = N - 1
    roots = np.sort(np.polynomial.legendre.Legendre.basis(p).deriv().roots().real) if p > 1 else []
    ref = np.concatenate([[-1.0], roots, [1.0]])
    np.testing.assert_allclose(xi, ref, rtol=0, atol=2e-14)
    assert abs(math.fsum(rho) - 2.0) <= 2e-15
    # GLL quadrature is exact for degree <= 2N-3
    for q in range(0, 2 * N - 2):
        exact = 0.0 if q % 2 else 2.0 / (q + 1)
        assert abs(np.dot(rho, xi ** q) - exact) <= 2e-14, (N, q)


# --------------------------------------------------------------- P2 D
@pytest.mark.parametrize("N", [2, 3, 5, 8, 10, 12, 16])
def test_derivative_matrix_exact_on_polynomials(ora, N):
    xi, _, D = ora.gll(N)
    assert np.abs(D @ np.ones(N)).max() <= 1e-13
    for q in range(1, N):
        err = np.abs(D @ xi ** q - q * xi ** (q - 1)).max()
        assert err <= 2e-12 * q, (N, q, err)


# ------------------------------------------------ P3 / P4 geometry
@pytest.mark.parametrize("N", [3, 8])
def test_undeformed_geometric_factors_closed_form(ora, N):
    m = ora.Mesh(3, 2, 2, N)
    G = ora.setup(m, want=("G",))["G"]
    _, rho, _ = ora.gll(N)
    W = rho[None, None, :] * rho[None, :, None] * rho[:, None, None]  # [k][j][i]
    h = 1.0 / m.ex
    for c in (0, 3, 5):
        ref = np.broadcast_to(0.5 * h * W, G[:, c].shape)
        # D-based Jacobian: rounding-level agreement in the max norm
        assert np.abs(G[:, c] - ref).max() <= 2e-14 * np.abs(ref).max()
    for c in (1, 2, 4):
        assert np.abs(G[:, c]).max() <= 2e-14 * np.abs(G[:, 0]).max()


@pytest.mark.parametrize("N", [4, 8, 12])
def test_jittered_mass_sums_to_volume(ora, N):
    m = ora.Mesh(3, 3, 2, N, jitter=0.1, seed_geom=2003)
    s = ora.setup(m, want=("mass", "G", "xyz"))
    vol = 1.0 * (m.ey / m.ex) * (m.ez / m.ex)
    assert abs(s["mass"].sum() - vol) <= 1e-13
    assert s["mass"].min() > 0
    # the metric is symmetric positive definite at every point
    Gc = s["G"]
    M = np.stack([np.stack([Gc[:, 0], Gc[:, 1], Gc[:, 2]], -1),
                  np.stack([Gc[:, 1], Gc[:, 3], Gc[:, 4]], -1),
                  np.stack([Gc[:, 2], Gc[:, 4], Gc[:, 5]], -1)], -2)
    assert np.linalg.eigvalsh(M.reshape(-1, 3, 3)).min() > 0
    # the jitter moves interior vertices only: the box boundary is exact
    x = s["xyz"]
    assert abs(x[:, 0].min()) <= 4e-16 and abs(x[:, 0].max() - 1.0) <= 4e-16


def test_coordinates_continuous_across_elements(ora):
    m = ora.Mesh(3, 2, 2, 6, jitter=0.1, seed_geom=7)
    s = ora.setup(m, want=("xyz", "gid"))
    xyz = np.moveaxis(s["xyz"], 1, -1).reshape(-1, 3)
    gid = s["gid"].reshape(-1)
    ref = np.zeros((gid.max() + 1, 3))
    ref[gid] = xyz
    assert np.abs(ref[gid] - xyz).max() <= 1e-15


# --------------------------------------------------- P5 gid / c / mask
def test_multiplicity_and_mask_structure(ora):
    m = ora.Mesh(2, 1, 1, 5)  # 2x1x1 interface has m = 2
    s = ora.setup(m, want=("mult", "mask", "gid"))
    assert (s["mult"][0, :, :, 4] == 2).all() and (s["mult"][1, :, :, 0] == 2).all()
    assert (s["mult"][0, :, :, :4] == 1).all()
    m = ora.Mesh(2, 2, 2, 2)  # centre corner of 2x2x2 has m = 8
    s = ora.setup(m, want=("mult", "gid"))
    centre = s["gid"][0, 1, 1, 1]
    assert (s["mult"][s["gid"] == centre] == 8).all() and (s["gid"] == centre).sum() == 8
    for mesh in (ora.Mesh(2, 2, 2, 8), ora.Mesh(3, 2, 4, 5)):
        sz = mesh.sizes()
        s = ora.setup(mesh, want=("mult", "mask", "gid"))
        one = np.ones((mesh.E, mesh.N, mesh.N, mesh.N))
        assert (ora.dssum(mesh, one) == s["mult"]).all()  # dssum(1) = m
        c = ora.multiplicity_weight(mesh)
        assert (c * s["mult"] == 1.0).all()  # c m = 1 exactly (R8)
        ng = sz["n_global"]
        assert np.unique(s["gid"]).size == ng
        mg = np.zeros(ng, bool)
        mg[s["gid"].reshape(-1)] = s["mask"].reshape(-1).astype(bool)
        assert ng - mg.sum() == sz["n_interior"]
        assert (np.bincount(s["gid"].reshape(-1)) > 1).sum() == sz["n_shared"]


def test_sizes_match_survey_table(ora):
    # SURVEY 8 per-config size table (Appendix B formulas)
    assert ora.Mesh(2, 2, 2, 8).sizes() == dict(n_local=4096, n_global=3375, n_interior=2197,
                                                n_shared=631)
    c2 = ora.Mesh(16, 16, 16, 8).sizes()
    assert (c2["n_local"], c2["n_global"], c2["n_interior"]) == (2097152, 1442897, 1367631)
    c3 = ora.Mesh(32, 32, 32, 12).sizes()
    assert (c3["n_local"], c3["n_global"]) == (56623104, 43986977)
    c5 = ora.Mesh(64, 64, 64, 10).sizes()
    assert c5["n_global"] == 192100033


# ---------------------------------------------------------- dssum / mask
def test_dssum_chain_order_bruteforce(ora):
    """C4: copies summed in ascending local index, pure-Python loop."""
    m = ora.Mesh(2, 2, 2, 3)
    gid = ora.setup(m, want=("gid",))["gid"].reshape(-1)
    w = inputs.uniform_field(gid.size, 11)
    out = ora.dssum(m, w.reshape(m.E, 3, 3, 3)).reshape(-1)
    acc = {}
    for L in range(gid.size):
        g = int(gid[L])
        acc[g] = float(w[L]) if g not in acc else acc[g] + float(w[L])
    ref = np.array([acc[int(g)] for g in gid])
    assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))
    for dt in (np.float32,):
        w32 = w.astype(dt)
        out32 = ora.dssum(m, w32.reshape(m.E, 3, 3, 3)).reshape(-1)
        acc = {}
        for L in range(gid.size):
            g = int(gid[L])
            acc[g] = w32[L] if g not in acc else np.float32(acc[g] + w32[L])
        assert np.array_equal(out32, np.array([acc[int(g)] for g in gid], dtype=dt))


def test_dssum_idempotent_with_multiplicity(ora):
    m = ora.Mesh(2, 2, 2, 4)  # gs(c * gs(f)) == gs(f)
    f = inputs.uniform_field((m.E, 4, 4, 4), 3)
    c = ora.multiplicity_weight(m)
    g = ora.dssum(m, f)
    np.testing.assert_allclose(ora.dssum(m, c * g), g, rtol=1e-15, atol=1e-15)
    msk = ora.setup(m, want=("mask",))["mask"].astype(bool)
    gm = ora.dssum(m, f, apply_mask=True)
    assert (gm[msk] == 0).all() and not np.signbit(gm[msk]).any()  # C5: +0 assigned
    assert np.array_equal(gm[~msk], g[~msk])


# ---------------------------------------------------- operator pins
@pytest.mark.parametrize("mesh_args", [(1, 1, 1, 3, 0.0), (2, 1, 1, 4, 0.0), (2, 2, 2, 3, 0.1),
                                       (2, 2, 1, 5, 0.1)])
def test_ax_matches_dense_assembled_matrix(ora, mesh_args):
    ex, ey, ez, N, jit = mesh_args
    m = ora.Mesh(ex, ey, ez, N, jitter=jit, seed_geom=5)
    A, gid = dense_stiffness(ora, m)
    assert np.abs(A - A.T).max() <= 1e-15 * np.abs(A).max()
    v = inputs.uniform_global(A.shape[0], 21)
    u = v[gid].reshape(m.E, N, N, N)
    _, _, D = ora.gll(N)
    G = ora.setup(m, want=("G",))["G"]
    w = ora.ax(m, D, G, u, apply_mask=False)
    ref = (A @ v)[gid].reshape(w.shape)
    assert np.abs(w - ref).max() <= 1e-14 * np.abs(ref).max()
    # masked operator = dense with Dirichlet rows zeroed
    mg = global_mask(ora, m)
    wm = ora.ax(m, D, G, u, apply_mask=True)
    refm = np.where(mg, 0.0, A @ v)[gid].reshape(w.shape)
    assert np.abs(wm - refm).max() <= 1e-14 * np.abs(ref).max()


def test_c1_dense_and_spd(ora):
    """P9 + P10 on C1 (2x2x2, N=8): dense agreement and SPD interior block."""
    m = ora.Mesh(2, 2, 2, 8)
    A, gid = dense_stiffness(ora, m)
    mg = global_mask(ora, m)
    Ai = A[np.ix_(~mg, ~mg)]
    ev = np.linalg.eigvalsh(Ai)
    assert ev.min() > 0 and Ai.shape[0] == 2197
    v = inputs.uniform_global(A.shape[0], 99)
    _, _, D = ora.gll(8)
    G = ora.setup(m, want=("G",))["G"]
    w = ora.ax(m, D, G, v[gid].reshape(m.E, 8, 8, 8), apply_mask=False)
    ref = (A @ v)[gid].reshape(w.shape)
    assert np.abs(w - ref).max() <= 2e-15 * np.abs(ref).max() * 8


@pytest.mark.parametrize("jit", [0.0, 0.1])
def test_null_space_of_unmasked_operator(ora, jit):
    m = ora.Mesh(3, 2, 2, 8, jitter=jit, seed_geom=2005)  # north_star: constants in null space
    _, _, D = ora.gll(8)
    G = ora.setup(m, want=("G",))["G"]
    w = ora.ax(m, D, G, np.ones((m.E, 8, 8, 8)), apply_mask=False)
    assert np.abs(w).max() <= 2e-15 * np.abs(G).max() * 64


def _poly_check(ora, m, fun, lap, tol):
    _, _, D = ora.gll(m.N)
    s = ora.setup(m, want=("G", "xyz", "mass", "mask"))
    x, y, z = s["xyz"][:, 0], s["xyz"][:, 1], s["xyz"][:, 2]
    w = ora.ax(m, D, s["G"], fun(x, y, z), apply_mask=False)
    B = ora.dssum(m, s["mass"])
    ref = -B * lap(x, y, z)
    um = ~s["mask"].astype(bool)
    err = np.abs(w - ref)[um].max() / np.abs(ref[um]).max()
    assert err <= tol, err


@pytest.mark.parametrize("N", [4, 8])
def test_polynomial_exactness_undeformed_tensor_degree_p(ora, N):
    """P7 (north_star: 'ax is exact for polynomials of degree <= p on the
    undeformed box'): A u = -B Laplace(u) at unmasked points, u in Q_p."""
    p = N - 1
    m = ora.Mesh(2, 2, 2, N)
    _poly_check(ora, m, lambda x, y, z: x ** p * y ** p * z ** p + x * x,
                lambda x, y, z: p * (p - 1) * (x ** (p - 2) * y ** p * z ** p
                                               + x ** p * y ** (p - 2) * z ** p
                                               + x ** p * y ** p * z ** (p - 2)) + 2.0,
                2e-12)
    _poly_check(ora, m, lambda x, y, z: x * x + y * y + z * z, lambda x, y, z: 6.0 + 0 * x, 2e-13)


@pytest.mark.parametrize("N", [8, 10, 12])
def test_polynomial_exactness_jittered_degree2_and_patch(ora, N):
    m = ora.Mesh(3, 3, 3, N, jitter=0.1, seed_geom=2003)
    _poly_check(ora, m, lambda x, y, z: x * x - 2 * y * z + 3 * z * z + x,
                lambda x, y, z: 2.0 + 6.0 + 0 * x, 5e-11)
    _, _, D = ora.gll(N)
    s = ora.setup(m, want=("G", "xyz", "mask"))
    lin = 1.0 + 2 * s["xyz"][:, 0] - s["xyz"][:, 1] + 0.5 * s["xyz"][:, 2]
    w = ora.ax(m, D, s["G"], lin, apply_mask=False)
    um = ~s["mask"].astype(bool)
    assert np.abs(w[um]).max() <= 1e-13  # patch test


def test_operator_symmetry_random_continuous(ora):
    """P8: glsc3(x, c, A y) = glsc3(y, c, A x) for continuous masked x, y."""
    m = ora.Mesh(3, 2, 2, 8, jitter=0.1, seed_geom=9)
    _, _, D = ora.gll(8)
    s = ora.setup(m, want=("G", "gid", "mask"))
    ng = m.sizes()["n_global"]
    msk = s["mask"].astype(bool)
    x = np.where(msk, 0.0, inputs.uniform_global(ng, 1)[s["gid"]])
    y = np.where(msk, 0.0, inputs.uniform_global(ng, 2)[s["gid"]])
    c = ora.multiplicity_weight(m)
    a = ora.glsc3(x, ora.ax(m, D, s["G"], y), c)
    b = ora.glsc3(y, ora.ax(m, D, s["G"], x), c)
    assert abs(a - b) <= 1e-14 * abs(a)
    assert ora.glsc3(x, ora.ax(m, D, s["G"], x), c) > 0  # positive definite


def test_fp32_ax_accuracy(ora):
    """P15: binary32 ax on binary32-rounded inputs vs binary64 ax of the same
    inputs: max-norm relative error well under the north_star 2e-6."""
    m = ora.Mesh(3, 3, 2, 10, jitter=0.1, seed_geom=4)
    xi, _, D = ora.gll(10)
    G = ora.setup(m, want=("G",))["G"]
    u = inputs.uniform_field((m.E, 10, 10, 10), 8)
    D32, G32, u32 = D.astype(np.float32), G.astype(np.float32), u.astype(np.float32)
    w32 = ora.ax(m, D32, G32, u32)
    w64 = ora.ax(m, D32.astype(np.float64), G32.astype(np.float64), u32.astype(np.float64))
    err = np.abs(w32 - w64).max() / np.abs(w64).max()
    assert err < 2e-6 and err > 0
    assert ora.ax(m, D32, G32, np.zeros_like(u32)).max() == 0  # ax(0) = 0


# -------------------------------------------------------- P14 glsc3
def test_glsc3_examples(ora):
    assert ora.glsc3(np.ones(3), np.ones(3), np.ones(3)) == 3.0
    assert ora.glsc3(np.array([1.0, 2.0]), np.array([3.0, 4.0]), np.array([1.0, 0.5])) == 7.0
    assert ora.glsc3(np.zeros(0), np.zeros(0), np.zeros(0)) == 0.0


@pytest.mark.parametrize("n,cancel", [(1, False), (4096, False), (4096, True), (200_000, True),
                                      (70_001, False)])
def test_fsum_correctly_rounded(ora, n, cancel):
    for seed in range(6):
        t = inputs.lognormal_terms(n, seed * 13 + n, cancel=cancel)
        assert ora.fsum(t) == math.fsum(t)
        c = np.ones(n)
        assert ora.glsc3(t, np.ones(n), c) == math.fsum(t)


def test_fsum_halfway_cases(ora):
    cases = [[1.0, 2.0 ** -53, 2.0 ** -106], [1.0, -2.0 ** -54, -2.0 ** -108],
             [2.0 ** 53, 1.0, 2.0 ** -30], [0.1] * 10,
             [1.0, 1e100, 1.0, -1e100]]
    for t in cases:
        assert ora.fsum(np.array(t)) == math.fsum(t), t


def test_glsc3_fp32_terms_are_exact(ora):
    """FP32 loop (north_star: FP64 accumulation): t = (double)a (double)b c is exact."""
    a = inputs.uniform_field(50_000, 1, np.float32)
    b = inputs.uniform_field(50_000, 2, np.float32)
    c = np.random.default_rng(3).choice([1.0, 0.5, 0.25, 0.125], size=50_000)
    ref = math.fsum(float(x) * float(y) * float(z) for x, y, z in zip(a, b, c))
    assert ora.glsc3(a, b, c) == ref


# ---------------------------------------------------------- CG pins
@pytest.mark.parametrize("mesh_args", [(2, 1, 1, 4), (2, 2, 2, 3), (3, 2, 2, 3), (2, 2, 1, 4)])
def test_cg_finite_termination(ora, mesh_args):
    """P11 (north_star: CG converges in at most n_dof iterations on tiny problems)."""
    m = ora.Mesh(*mesh_args, seed_rhs=17)
    _, _, D = ora.gll(m.N)
    s = ora.setup(m, want=("G", "f"))
    ndof = m.sizes()["n_interior"]
    r = ora.cg(m, D, s["G"], s["f"], ndof + 5)
    rel = r.hist / r.hist[0]
    assert (rel[: ndof + 1] < 1e-12).any(), (ndof, rel.min())
    assert r.defect == 0


def test_cg_matches_dense_solve_and_energy_decreases(ora):
    """S:392 dense-solve agreement; S:417 monotone A-norm error."""
    m = ora.Mesh(2, 2, 1, 4, jitter=0.1, seed_geom=3, seed_rhs=5)
    _, _, D = ora.gll(4)
    s = ora.setup(m, want=("G", "f", "gid"))
    A, gid = dense_stiffness(ora, m)
    mg = global_mask(ora, m)
    fg = np.zeros(A.shape[0])
    fg[gid] = s["f"].reshape(-1)
    xg = np.zeros_like(fg)
    Ai = A[np.ix_(~mg, ~mg)]
    xg[~mg] = np.linalg.solve(Ai, fg[~mg])
    errs = []
    for it in range(1, 40):
        r = ora.cg(m, D, s["G"], s["f"], it)
        e = r.x.reshape(-1)
        eg = np.zeros_like(xg)
        eg[gid] = e
        d = (eg - xg)[~mg]
        errs.append(d @ Ai @ d)
    assert all(errs[i + 1] <= errs[i] * (1 + 1e-9) + 1e-28 for i in range(len(errs) - 1))
    r = ora.cg(m, D, s["G"], s["f"], 60)
    assert np.abs(r.x.reshape(-1) - xg[gid]).max() <= 1e-9
    # scalar trace consistency: h_k = sqrt(rtr_k), rtz1_k = rtr_{k-1}, beta_1 = 0
    np.testing.assert_array_equal(r.hist[1:], np.sqrt(r.trace[:, 4]))
    np.testing.assert_array_equal(r.trace[1:, 0], r.trace[:-1, 4])
    assert r.trace[0, 1] == 0.0


def test_cg_zero_rhs(ora):
    """f = 0 gives x = 0 and residual 0, no defect (C9)."""
    m = ora.Mesh(2, 2, 2, 4)
    _, _, D = ora.gll(4)
    G = ora.setup(m, want=("G",))["G"]
    f = np.zeros((m.E, 4, 4, 4))
    for prec in ("fp64", "fp32"):
        r = ora.cg(m, D, G, f, 10, prec)
        assert (r.hist == 0).all() and (r.x == 0).all() and r.defect == 0


def test_cg_defect_on_indefinite_operator(ora):
    """pap <= 0 is a defect signal (operator not SPD)."""
    m = ora.Mesh(2, 2, 2, 4, seed_rhs=3)
    _, _, D = ora.gll(4)
    s = ora.setup(m, want=("G", "f"))
    r = ora.cg(m, D, -s["G"], s["f"], 5)
    assert r.defect == 1


def test_cg_c1_fp64_and_fp32(ora):
    """P12 / P16 plausibility on C1: FP64 converges ~1e-10 in 100 iterations;
    the FP32 solver tracks FP64 early, its true FP64 residual floors ~1e-6 h0."""
    m = ora.Mesh(2, 2, 2, 8, seed_rhs=1001)
    _, _, D = ora.gll(8)
    s = ora.setup(m, want=("G", "f"))
    r64 = ora.cg(m, D, s["G"], s["f"], 100, "fp64")
    r32 = ora.cg(m, D, s["G"], s["f"], 100, "fp32")
    assert r64.defect == 0 and r32.defect == 0
    assert r64.hist[100] / r64.hist[0] < 1e-8
    rel = np.abs(r32.hist[:20] - r64.hist[:20]) / r64.hist[:20]
    assert rel.max() < 1e-4
    tr64, h0 = ora.true_residual(m, D, s["G"], s["f"], r64.x)
    tr32, _ = ora.true_residual(m, D, s["G"], s["f"], r32.x)
    assert tr64 / h0 < 1e-8
    assert 1e-9 < tr32 / h0 < 1e-4
    xe = np.abs(r32.x - r64.x).max() / np.abs(r64.x).max()
    assert 1e-9 < xe < 1e-4


# ------------------------------------------------ Jacobi PCG pins (NEXT-1)
@pytest.mark.parametrize("mesh_args", [(2, 1, 1, 4, 0.0), (2, 2, 1, 3, 0.15), (1, 2, 2, 5, 0.1)])
def test_jacobi_diagonal_is_dense_diagonal(ora, mesh_args):
    """diag(A) equals the diagonal of the Kronecker-assembled dense
    stiffness (P9 brute force) on unmasked nodes; masked entries are 1."""
    ex, ey, ez, N, jit = mesh_args
    m = ora.Mesh(ex, ey, ez, N, jitter=jit, seed_geom=7)
    _, _, D = ora.gll(N)
    s = ora.setup(m, want=("G", "gid", "mask"))
    d, dinv = ora.jacobi_dinv(m, D, s["G"])
    A, gid = dense_stiffness(ora, m)
    ref = np.diag(A)[gid].reshape(d.shape)
    msk = s["mask"].astype(bool)
    assert np.abs(d[~msk] - ref[~msk]).max() <= 1e-13 * np.abs(ref).max()
    assert (d[msk] == 1.0).all() and (ref[~msk] > 0).all()
    np.testing.assert_array_equal(dinv, 1.0 / d)


def test_jacobi_diagonal_by_indicator_vectors(ora):
    """Second brute force: A_gg = (ax e_g) at a copy of g, with e_g the
    continuous indicator of global node g (all copies 1), unmasked operator."""
    m = ora.Mesh(2, 2, 1, 4, jitter=0.1, seed_geom=11)
    _, _, D = ora.gll(4)
    s = ora.setup(m, want=("G", "gid", "mask"))
    d, _ = ora.jacobi_dinv(m, D, s["G"])
    gid = s["gid"]
    for g in range(0, m.sizes()["n_global"], 3):
        u = (gid == g).astype(np.float64)
        w = ora.ax(m, D, s["G"], u, apply_mask=False)
        L = np.argwhere(gid.reshape(-1) == g)[0, 0]
        if s["mask"].reshape(-1)[L]:
            assert d.reshape(-1)[L] == 1.0
        else:
            assert w.reshape(-1)[L] == pytest.approx(d.reshape(-1)[L], rel=1e-13)


def test_jacobi_apply_inverts_the_diagonal(ora):
    """r = diag(A) * v gives z = r * dinv = v within 1e-13; masked
    points have diagonal 1 so z = r there."""
    m = ora.Mesh(2, 2, 2, 5, jitter=0.1, seed_geom=2)
    _, _, D = ora.gll(5)
    s = ora.setup(m, want=("G", "mask"))
    d, dinv = ora.jacobi_dinv(m, D, s["G"])
    v = inputs.uniform_field(d.shape, 4)
    z = (d * v) * dinv
    assert np.abs(z - v).max() <= 1e-13 * np.abs(v).max()


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_pcg_with_unit_diagonal_is_plain_cg(ora, prec):
    """With dinv = 1, solveM is the identity (z = r bitwise, rtz1 = rtr): the
    preconditioned loop must reproduce the unpreconditioned CG bit for bit."""
    m = ora.Mesh(2, 2, 2, 6, jitter=0.1, seed_geom=5, seed_rhs=8)
    _, _, D = ora.gll(6)
    s = ora.setup(m, want=("G", "f"))
    a = ora.cg(m, D, s["G"], s["f"], 30, prec)
    b = ora.cg(m, D, s["G"], s["f"], 30, prec, dinv=np.ones_like(s["f"]))
    np.testing.assert_array_equal(a.hist, b.hist)
    np.testing.assert_array_equal(a.trace, b.trace)
    np.testing.assert_array_equal(a.x, b.x)


def test_pcg_matches_dense_solve_and_terminates(ora):
    """Jacobi PCG (FP64) reaches the dense solution of the interior system
     and, as CG on the symmetrically scaled system, terminates within
    n_dof iterations (P11); it also needs fewer iterations than CG on a
    jittered mesh."""
    m = ora.Mesh(2, 2, 1, 4, jitter=0.2, seed_geom=3, seed_rhs=5)
    _, _, D = ora.gll(4)
    s = ora.setup(m, want=("G", "f", "gid"))
    _, dinv = ora.jacobi_dinv(m, D, s["G"])
    A, gid = dense_stiffness(ora, m)
    mg = global_mask(ora, m)
    fg = np.zeros(A.shape[0])
    fg[gid] = s["f"].reshape(-1)
    xg = np.zeros_like(fg)
    xg[~mg] = np.linalg.solve(A[np.ix_(~mg, ~mg)], fg[~mg])
    ndof = m.sizes()["n_interior"]
    r = ora.cg(m, D, s["G"], s["f"], ndof + 5, "fp64", dinv=dinv)
    assert r.defect == 0
    assert np.abs(r.x.reshape(-1) - xg[gid]).max() <= 1e-9
    assert (r.hist[: ndof + 1] / r.hist[0] < 1e-12).any()
    # trace: h_k = sqrt(rtr_k); beta_1 = 0; rtz1 > 0
    np.testing.assert_array_equal(r.hist[1:], np.sqrt(r.trace[:, 4]))
    assert r.trace[0, 1] == 0.0 and (r.trace[:ndof, 0] > 0).all()
    plain = ora.cg(m, D, s["G"], s["f"], 12, "fp64")
    prec = ora.cg(m, D, s["G"], s["f"], 12, "fp64", dinv=dinv)
    assert prec.hist[12] < plain.hist[12]


def test_pcg_scaled_problem_equivalence(ora):
    """Jacobi PCG on A is CG on the symmetrically scaled S^-1 A S^-1 (S^2 =
    diag(A)): the A-norm error decreases monotonically -- checked
    against the dense solution."""
    m = ora.Mesh(2, 2, 2, 3, jitter=0.15, seed_geom=9, seed_rhs=2)
    _, _, D = ora.gll(3)
    s = ora.setup(m, want=("G", "f", "gid"))
    _, dinv = ora.jacobi_dinv(m, D, s["G"])
    A, gid = dense_stiffness(ora, m)
    mg = global_mask(ora, m)
    Ai = A[np.ix_(~mg, ~mg)]
    fg = np.zeros(A.shape[0])
    fg[gid] = s["f"].reshape(-1)
    xg = np.zeros_like(fg)
    xg[~mg] = np.linalg.solve(Ai, fg[~mg])
    errs = []
    for it in range(1, 20):
        r = ora.cg(m, D, s["G"], s["f"], it, "fp64", dinv=dinv)
        eg = np.zeros_like(xg)
        eg[gid] = r.x.reshape(-1)
        dd = (eg - xg)[~mg]
        errs.append(dd @ Ai @ dd)
    assert all(errs[i + 1] <= errs[i] * (1 + 1e-9) + 1e-28 for i in range(len(errs) - 1))


# ------------------------------------ paper-literal single precision (NEXT-2)
def _rn32_exact(terms):
    """RN32 (ties to even) of the exact rational sum of binary64 terms."""
    from fractions import Fraction
    S = sum(Fraction(float(t)) for t in terms)
    c = np.float32(float(S))
    cands = [np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))]
    even = lambda v: int(np.frombuffer(np.float32(v).tobytes(), np.uint32)[0]) & 1  # noqa: E731
    return float(min(cands, key=lambda v: (abs(Fraction(float(v)) - S), even(v))))


def test_fsum32_is_correctly_rounded(ora):
    """The binary32 rounding of an exact sum (used by the single-precision glsc3)
    equals the rational-arithmetic RN32, including sums that land exactly on a
    binary32 half-way point and half-way points perturbed by 2^-80."""
    g = inputs.rng(3)
    for trial in range(1500):
        if trial % 3 == 0:
            f = np.float32(g.standard_normal())
            a = np.nextafter(f, np.float32(np.inf))
            mid = (float(f) + float(a)) / 2
            terms = [mid, float(g.choice([-1.0, 0.0, 1.0])) * 2.0 ** -80, 0.0]
        else:
            n = int(g.integers(1, 8))
            terms = g.standard_normal(n) * np.exp2(g.integers(-40, 40, n))
        assert ora.fsum32(terms) == _rn32_exact(terms)


def test_glsc3_single_examples_and_definition(ora):
    """S:336-337 examples in binary32, and the definition RN32(sum RN32(a b) c)."""
    one = np.ones(3, np.float32)
    assert ora.glsc3_single(one, one, np.ones(3)) == 3.0
    assert ora.glsc3_single(np.array([1, 2], np.float32), np.array([3, 4], np.float32),
                            np.array([1.0, 0.5])) == 7.0
    a = inputs.uniform_field(5000, 1, np.float32, -3, 3)
    b = inputs.uniform_field(5000, 2, np.float32)
    c = inputs.rng(5).choice([1.0, 0.5, 0.25, 0.125], 5000)
    terms = (a * b).astype(np.float64) * c   # a*b in binary32 (numpy float32 product)
    assert ora.glsc3_single(a, b, c) == _rn32_exact(terms)


def test_single_solver_plausibility(ora):
    """The paper-literal single solver tracks FP64 early, converges to the
    binary32 floor, and f = 0 gives x = 0."""
    m = ora.Mesh(2, 2, 2, 8, seed_rhs=1001)
    _, _, D = ora.gll(8)
    s = ora.setup(m, want=("G", "f"))
    r64 = ora.cg(m, D, s["G"], s["f"], 60, "fp64")
    r1 = ora.cg(m, D, s["G"], s["f"], 60, "fp32s")
    assert r1.defect == 0
    rel = np.abs(r1.hist[:15] - r64.hist[:15]) / r64.hist[:15]
    assert rel.max() < 1e-3
    # scalars are binary32 values
    assert (r1.trace.astype(np.float32).astype(np.float64) == r1.trace).all()
    assert (r1.hist.astype(np.float32).astype(np.float64) == r1.hist).all()
    tr, h0 = ora.true_residual(m, D, s["G"], s["f"], r1.x)
    assert 1e-9 < tr / h0 < 1e-3
    z = ora.cg(m, D, s["G"], np.zeros_like(s["f"]), 5, "fp32s")
    assert (z.hist == 0).all() and (z.x == 0).all()


# --------------------------------------------------- VPREC emulation (NEXT-4)
def _vprec_exact(x, t):
    """Round a binary64 value to t explicit mantissa bits, ties to even, with
    rational arithmetic (independent of the oracle's bit manipulation)."""
    from fractions import Fraction
    if x == 0.0 or t >= 52:
        return x
    m, e = math.frexp(abs(x))           # |x| = m 2^e, m in [0.5, 1)
    e = max(e, -1021)                   # subnormals: same absolute bit position
    ulp = Fraction(2) ** (e - 1 - t)    # weight of the last kept bit
    q = Fraction(abs(x)) / ulp
    fl = q.numerator // q.denominator
    rem = q - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return math.copysign(float(fl * ulp), x)


def test_vprec_round_matches_rational_rounding(ora):
    g = inputs.rng(8)
    for trial in range(3000):
        t = int(g.integers(1, 53))
        if trial % 4 == 0:   # exact ties: a t+1-bit value with its last bit set
            m = (2 * int(g.integers(1 << t, 1 << (t + 1)))) + 1
            x = math.ldexp(m, int(g.integers(-60, 60)) - (t + 1))
        else:
            x = float(g.standard_normal() * 2.0 ** int(g.integers(-80, 80)))
        assert ora.vprec_round(x, t) == _vprec_exact(x, t), (x, t)
    assert ora.vprec_round(3 * 2.0 ** -1074, 52) == 3 * 2.0 ** -1074  # subnormal, t = 52: exact
    assert ora.vprec_round(1.0 + 2.0 ** -30, 23) == 1.0 and ora.vprec_round(1.75, 1) == 2.0


def test_vprec_cg_t52_is_fp64_and_precision_sweep(ora):
    """t = 52 leaves every operation unchanged: the VPREC loop IS the FP64 solver
    bit for bit.  Lower t: the true residual of the solution degrades as the
    emulated precision drops (P:367-372 'residual becomes smaller as precision
    grows', F4)."""
    m = ora.Mesh(2, 2, 2, 6, jitter=0.1, seed_geom=4, seed_rhs=3)
    _, _, D = ora.gll(6)
    s = ora.setup(m, want=("G", "f"))
    a = ora.cg(m, D, s["G"], s["f"], 80, "fp64")
    b = ora.cg_vprec(m, D, s["G"], s["f"], 80, 52)
    np.testing.assert_array_equal(a.hist, b.hist)
    np.testing.assert_array_equal(a.trace, b.trace)
    np.testing.assert_array_equal(a.x, b.x)
    res = {}
    for t in (6, 10, 16, 23, 36, 52):
        r = ora.cg_vprec(m, D, s["G"], s["f"], 80, t)
        tr, h0 = ora.true_residual(m, D, s["G"], s["f"], r.x)
        res[t] = tr / h0
        # every scalar is a t-bit value
        for v in np.concatenate([r.trace.reshape(-1), r.hist]):
            assert ora.vprec_round(v, t) == v
    assert res[6] > res[16] > res[36] and res[52] < 1e-8
    assert res[23] < 1e-3


def test_emulated_loop_vprec_equals_macro_loop(ora):
    """The explicit-key emulation loop (used for RR / MCA) and the macro-built
    VPREC loop are separate code: in VPREC mode they must agree bit for bit."""
    m = ora.Mesh(3, 2, 2, 5, jitter=0.15, seed_geom=6, seed_rhs=7)
    _, _, D = ora.gll(5)
    s = ora.setup(m, want=("G", "f"))
    for t in (5, 12, 23, 52):
        a = ora.cg_vprec(m, D, s["G"], s["f"], 40, t)
        b = ora.cg_emulated(m, D, s["G"], s["f"], 40, "vprec", t)
        np.testing.assert_array_equal(a.hist, b.hist)
        np.testing.assert_array_equal(a.trace, b.trace)
        np.testing.assert_array_equal(a.x, b.x)


@pytest.mark.parametrize("mode", ["rr", "mca"])
def test_mca_samples_statistics(ora, mode):
    """MCA / RR samples: a sample is reproducible from its seed,
    different seeds differ, the perturbation is at the virtual precision: at
    t = 23 the early iterations keep ~t significant bits (s2 = -log2|sigma/mu|,
    P:380), the sample mean tracks the FP64 history, and t = 40 perturbs far
    less than t = 23."""
    m = ora.Mesh(2, 2, 2, 6, jitter=0.1, seed_geom=4, seed_rhs=3)
    _, _, D = ora.gll(6)
    s = ora.setup(m, want=("G", "f"))
    a = ora.cg_emulated(m, D, s["G"], s["f"], 30, mode, 23, 11)
    b = ora.cg_emulated(m, D, s["G"], s["f"], 30, mode, 23, 11)
    np.testing.assert_array_equal(a.hist, b.hist)
    hs = np.array([ora.cg_emulated(m, D, s["G"], s["f"], 30, mode, 23, sd).hist for sd in range(8)])
    assert len({h.tobytes() for h in hs}) == 8
    r64 = ora.cg(m, D, s["G"], s["f"], 30, "fp64")
    mu, sg = hs.mean(0), hs.std(0)
    s2 = -np.log2(sg[1:6] / np.abs(mu[1:6]))
    assert (s2 > 17).all() and (s2 < 30).all(), s2
    assert np.abs(mu[:10] / r64.hist[:10] - 1).max() < 1e-5
    h40 = np.array([ora.cg_emulated(m, D, s["G"], s["f"], 30, mode, 40, sd).hist for sd in range(4)])
    assert h40.std(0)[1:10].max() < 1e-3 * sg[1:10].max()


# ------------------------------------------------ C7: FP64 scalars in the FP32 solver
def test_fp32_solver_scalars_are_fp64(ora):
    """C7 (north_star "FP64 accumulation even in the FP32 solver", reading R11):
    the mixed FP32 solver forms alpha, beta and h_k in binary64 from the binary64
    inner products and rounds alpha / beta to binary32 only where they enter the
    binary32 vector updates (C8).  Pinned by IEEE identities on the trace
    (Python floats are binary64), by values that are not binary32 numbers, and
    by the first iterate x_1 = RN32(RN32(alpha_1) f32): a solver with binary32
    scalars (alpha = RN32(RN32(rtz1) / RN32(pap))) would fail each of them."""
    m = ora.Mesh(2, 2, 2, 6, jitter=0.1, seed_geom=4, seed_rhs=3)
    _, _, D = ora.gll(6)
    s = ora.setup(m, want=("G", "f"))
    r = ora.cg(m, D, s["G"], s["f"], 30, "fp32")
    rtz1, beta, alpha, pap, rtr = r.trace.T
    for k in range(30):
        assert alpha[k] == rtz1[k] / pap[k]                    # binary64 division
        assert r.hist[k + 1] == math.sqrt(rtr[k])               # binary64 sqrt
        if k:
            assert beta[k] == rtz1[k] / rtz1[k - 1] and rtz1[k] == rtr[k - 1]
    as32 = lambda v: float(np.float32(v)) == v  # noqa: E731
    assert not all(as32(v) for v in alpha) and not all(as32(v) for v in beta[1:])
    assert not all(as32(v) for v in rtr)
    # the binary32 loop uses RN32(alpha_1): x_1 = RN32(RN32(alpha_1) * f32) (p_1 = r_0 = f32)
    r1 = ora.cg(m, D, s["G"], s["f"], 1, "fp32")
    f32 = s["f"].astype(np.float32)
    a1 = r1.trace[0, 2]
    assert np.array_equal(r1.x, (np.float32(a1) * f32).astype(np.float32))
    # the binary32-scalar variant (paper-literal single, R11b) follows another trajectory
    rs = ora.cg(m, D, s["G"], s["f"], 30, "fp32s")
    assert not np.array_equal(rs.hist, r.hist)


# ------------------------------------------------ NEXT-4: one draw per FP operation
@pytest.mark.parametrize("mode", ["rr", "mca"])
def test_mca_draws_per_operation(ora, mode):
    """each FP operation is perturbed by its own draw.  The pointwise
    updates of the m copies of a shared node are separate operations, so under
    RR / MCA the copies of x (and p, r) differ after one iteration, while VPREC
    (deterministic rounding) keeps every copy bitwise equal; dssum still writes
    one sum to every copy (C4).  The first iterate, p_1 = fma(0, 0, r_0) with
    its result perturbed, is x_1 / alpha_1-free: check the copies of x_1."""
    m = ora.Mesh(2, 2, 2, 5, jitter=0.1, seed_geom=4, seed_rhs=3)
    _, _, D = ora.gll(5)
    s = ora.setup(m, want=("G", "f", "gid"))
    gid = s["gid"].reshape(-1)
    order = np.argsort(gid, kind="stable")
    g_sorted = gid[order]
    first = np.r_[True, g_sorted[1:] != g_sorted[:-1]]
    grp = np.cumsum(first) - 1

    def spread(x):  # max over nodes of (max - min) over the node's copies
        v = x.reshape(-1)[order]
        mx = np.maximum.reduceat(v, np.nonzero(first)[0])
        mn = np.minimum.reduceat(v, np.nonzero(first)[0])
        return mx - mn

    e = ora.cg_emulated(m, D, s["G"], s["f"], 3, mode, 23, 5)
    v = ora.cg_emulated(m, D, s["G"], s["f"], 3, "vprec", 23)
    assert (spread(v.x) == 0).all()
    sp = spread(e.x)
    shared = np.bincount(grp) > 1
    assert (sp[shared] > 0).mean() > 0.5       # most shared nodes have differing copies
    assert (sp[~shared] == 0).all()


# ------------------------------------------------ NEXT-2: the paper's binary32 accumulation (R11c)
def test_glsc3_accum32_is_sequential_binary32(ora):
    """P:42 / P:507 / P:510: glsc3 accumulated in binary32 in loop order, per
    rank, then a binary32 all-reduce.  Hand-computed cases: small integers sum
    exactly (S:336-337 examples); 2^24 followed by four ones stays 2^24 in a
    binary32 accumulator (2^24 + 1 rounds to even) while the exactly rounded
    sum (R11b) is 2^24 + 4; the ones first give 2^24 + 4; with two ranks
    [2^24, 1 | 1, 1] gives 2^24 + 2 (rank sums 2^24 and 2); the product is
    rounded to binary32 before the weight (c = 1/2 exact)."""
    one = np.ones(3, np.float32)
    assert ora.glsc3_accum32(one, one, np.ones(3)) == 3.0
    assert ora.glsc3_accum32(np.array([1, 2], np.float32), np.array([3, 4], np.float32),
                             np.array([1.0, 0.5])) == 7.0
    big = np.float32(2.0 ** 24)
    a = np.array([big, 1, 1, 1, 1], np.float32)
    o = np.ones(5, np.float32)
    c = np.ones(5)
    assert ora.glsc3_accum32(a, o, c) == 2.0 ** 24
    assert ora.glsc3_single(a, o, c) == 2.0 ** 24 + 4   # exactly rounded (R11b) differs
    assert ora.glsc3_accum32(a[::-1].copy(), o, c) == 2.0 ** 24 + 4
    a4 = np.array([big, 1, 1, 1], np.float32)
    assert ora.glsc3_accum32(a4, np.ones(4, np.float32), np.ones(4), nranks=2) == 2.0 ** 24 + 2
    # RN32(a b) before the weight: (1 + 2^-12)^2 = 1 + 2^-11 + 2^-24 -> 1 + 2^-11 in binary32
    x = np.float32(1 + 2.0 ** -12)
    assert ora.glsc3_accum32(np.array([x]), np.array([x]), np.array([0.5])) == (1 + 2.0 ** -11) / 2


def test_paper_single_solver_plausibility(ora):
    """The paper's single-precision solver (R11c) on C1: tracks FP64 early,
    scalars are binary32 values, its history differs from the exactly rounded
    binary32 variant (R11b) once accumulation errors matter, and the rank
    split changes the rounding (P:510 all-reduce) but not the early history."""
    m = ora.Mesh(2, 2, 2, 8, seed_rhs=1001)
    _, _, D = ora.gll(8)
    s = ora.setup(m, want=("G", "f"))
    r64 = ora.cg(m, D, s["G"], s["f"], 60, "fp64")
    ra = ora.cg(m, D, s["G"], s["f"], 60, "fp32a")
    rb = ora.cg(m, D, s["G"], s["f"], 60, "fp32s")
    r2 = ora.cg(m, D, s["G"], s["f"], 60, "fp32a", nranks=2)
    assert ra.defect == 0
    rel = np.abs(ra.hist[:15] - r64.hist[:15]) / r64.hist[:15]
    assert rel.max() < 1e-3
    assert (ra.trace.astype(np.float32).astype(np.float64) == ra.trace).all()
    assert not np.array_equal(ra.hist, rb.hist)
    assert not np.array_equal(ra.hist, r2.hist)
    assert np.abs(r2.hist[:10] - ra.hist[:10]).max() / ra.hist[0] < 1e-5
    tr, h0 = ora.true_residual(m, D, s["G"], s["f"], ra.x)
    assert 1e-9 < tr / h0 < 1e-3


def test_uniform_pm1_is_the_dyadic_map_of_splitmix64(ora):
    """R7 / SURVEY 8(d): value = 2 U - 1 with U = (z >> 11) 2^-53, z the SplitMix64
    output.  Pinned by structure and distribution rather than by the formula:
    every value is a multiple of 2^-52 in [-1, 1) whose numerator's top bits are
    those of z (so the map is monotone in z >> 11); the published stream of seed
    0 gives the hand-computed first values; 2e4 samples pass a Kolmogorov-Smirnov
    test against U[-1, 1) and have variance 1/3."""
    for i, z in enumerate((0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F)):
        k = z >> 11
        assert ora.uniform_pm1(0, i) == math.ldexp(k, -52) - 1.0
    v = np.array([ora.uniform_pm1(77, i) for i in range(20000)])
    assert ((v + 1.0) * 2.0 ** 52 == np.floor((v + 1.0) * 2.0 ** 52)).all()
    assert v.min() >= -1.0 and v.max() < 1.0
    assert abs(v.var() - 1.0 / 3.0) < 0.02
    from scipy import stats
    assert stats.kstest(v, "uniform", args=(-1.0, 2.0)).pvalue > 1e-3
    order = np.argsort([ora.splitmix64(77, i) >> 11 for i in range(200)], kind="stable")
    assert (np.diff(v[:200][order]) >= 0).all()
