"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Contract mode (C10): the library ingests the oracle's D, G, f, both
follow the canonical evaluation order CEO-1, and results are compared BITWISE
(stronger than the north_star tolerances: ax 1e-13 / 2e-6 relative, history
1e-10 / 1e-4 relative, which are asserted too).  Independent-set-up mode: the
library's own FP64 set-up is compared with the oracle's within tolerances.
"""
import math

import numpy as np
import pytest

from tests import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def nbk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_11065_b200 as p
    p.load()
    return p


def make(nbk, ora, ex, ey, ez, N, jitter=0.0, seed_geom=0, seed_rhs=0, precision="fp32",
         contract=True):
    spec = nbk.MeshSpec(ex, ey, ez, N, jitter, seed_geom, seed_rhs)
    ctx = nbk.cg_setup(spec, precision)
    om = ora.Mesh(ex, ey, ez, N, jitter, seed_geom, seed_rhs)
    _, _, D = ora.gll(N)
    s = ora.setup(om, want=("G", "f"))
    if contract:
        ctx.load_arrays(D, s["G"], s["f"])
    return ctx, om, D, s


def dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.dtype == b.dtype and a.shape == b.shape
    return np.array_equal(a.view(np.uint8), b.view(np.uint8))


def maxrel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-300))


# ------------------------------------------------------------ set-up
@pytest.mark.parametrize("args", [(2, 2, 2, 8, 0.0), (3, 3, 2, 10, 0.1), (2, 3, 4, 12, 0.1),
                                  (3, 1, 2, 5, 0.25)])
def test_independent_setup_matches_oracle(nbk, ora, args):
    ex, ey, ez, N, jit = args
    ctx, om, D, s = make(nbk, ora, ex, ey, ez, N, jit, 2003, 1003, "fp64", contract=False)
    Dl, Gl, fl = ctx.get_arrays()
    assert np.abs(Dl - D).max() <= 1e-15 * max(1.0, np.abs(D).max()) * 8
    # oracle differentiates coordinates with D (rounding ~1e-14 at N=10-12), the
    # library uses the analytic trilinear Jacobian: rounding-level agreement
    assert maxrel(Gl, s["G"]) <= 5e-14
    assert bits_equal(fl, s["f"])  # SplitMix64 RHS is exact on both sides
    info = ctx.info
    sz = om.sizes()
    assert info["n_local"] == sz["n_local"] and info["n_global"] == sz["n_global"]
    assert info["n_shared"] == sz["n_shared"]


# ------------------------------------------------------------ ax
@pytest.mark.parametrize("N", [2, 3, 4, 7, 8, 9, 10, 12, 16])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_ax_local_bitwise(nbk, ora, N, dtype):
    # ragged element count: not a multiple of the elements-per-CTA of k_ax
    ex, ey, ez = 3, 2, 3 if N <= 12 else 1
    ctx, om, D, s = make(nbk, ora, ex, ey, ez, N, 0.1, 7, 5)
    u = inputs.uniform_field((om.E, N, N, N), 100 + N, dtype)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    ud, wd = dev(u, tdt), torch.empty(u.shape, dtype=tdt, device="cuda")
    ctx.ax_apply(ud, wd, nbk.AX_LOCAL)
    ctx.sync()
    w = wd.cpu().numpy()
    ref = ora.ax_local(D.astype(dtype), s["G"].astype(dtype), u)
    assert bits_equal(w, ref)
    tol = 1e-13 if dtype == np.float64 else 2e-6
    assert maxrel(w, ref) <= tol


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("args", [(2, 2, 2, 8, 0.0), (4, 3, 2, 10, 0.1), (3, 3, 3, 12, 0.1),
                                  (1, 1, 1, 5, 0.0)])
def test_ax_full_operator_bitwise(nbk, ora, dtype, args):
    ex, ey, ez, N, jit = args
    ctx, om, D, s = make(nbk, ora, ex, ey, ez, N, jit, 11, 3)
    u = inputs.uniform_field((om.E, N, N, N), 7, dtype)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    ud, wd = dev(u, tdt), torch.empty(u.shape, dtype=tdt, device="cuda")
    ctx.ax_apply(ud, wd, nbk.AX_DSSUM | nbk.AX_MASK)
    ctx.sync()
    ref = ora.ax(om, D.astype(dtype), s["G"].astype(dtype), u, apply_mask=True)
    assert bits_equal(wd.cpu().numpy(), ref)


def test_fp32_ax_vs_fp64_oracle_on_rounded_inputs(nbk, ora):
    """R15: FP32 ax within 2e-6 of the FP64 oracle on the FP32-rounded inputs."""
    ctx, om, D, s = make(nbk, ora, 4, 4, 2, 12, 0.1, 3, 3)
    u32 = inputs.uniform_field((om.E, 12, 12, 12), 9, np.float32)
    wd = torch.empty(u32.shape, dtype=torch.float32, device="cuda")
    ctx.ax_apply(dev(u32, torch.float32), wd, nbk.AX_DSSUM | nbk.AX_MASK)
    ctx.sync()
    ref = ora.ax(om, D.astype(np.float32).astype(np.float64),
                 s["G"].astype(np.float32).astype(np.float64), u32.astype(np.float64))
    err = maxrel(wd.cpu().numpy(), ref)
    assert err <= 2e-6, err


# ------------------------------------------------------------ dssum
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("mask", [False, True])
def test_dssum_bitwise(nbk, ora, dtype, mask):
    ctx, om, D, s = make(nbk, ora, 3, 4, 2, 6, 0.0, 0, 0)
    f = inputs.uniform_field((om.E, 6, 6, 6), 31, dtype)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    fd = dev(f, tdt)
    ctx.dssum(fd, apply_mask=mask)
    ctx.sync()
    assert bits_equal(fd.cpu().numpy(), ora.dssum(om, f, apply_mask=mask))


def test_dssum_single_element_is_identity(nbk, ora):
    ctx, om, D, s = make(nbk, ora, 1, 1, 1, 4)
    f = inputs.uniform_field((1, 4, 4, 4), 1)
    fd = dev(f, torch.float64)
    ctx.dssum(fd)
    ctx.sync()
    assert bits_equal(fd.cpu().numpy(), f)


# ------------------------------------------------------------ glsc3
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_glsc3_correctly_rounded(nbk, ora, dtype):
    ctx, om, D, s = make(nbk, ora, 4, 3, 5, 8)
    c = ora.multiplicity_weight(om)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    for seed in range(5):
        a = inputs.uniform_field((om.E, 8, 8, 8), seed, dtype, -3.0, 3.0)
        b = inputs.uniform_field((om.E, 8, 8, 8), seed + 50, dtype)
        got = ctx.glsc3(dev(a, tdt), dev(b, tdt))
        terms = (a.astype(np.float64) * b.astype(np.float64)).reshape(-1) * c.reshape(-1)
        assert got == math.fsum(terms) == ora.glsc3(a, b, c)


# ------------------------------------------------------------ CG
def _cg_parity(nbk, ora, args, niter, precision, bitwise=True):
    ex, ey, ez, N, jit, sg, sr = args
    ctx, om, D, s = make(nbk, ora, ex, ey, ez, N, jit, sg, sr, "fp32")
    hist, trace, res = ctx.cg_solve(niter, precision)
    ref = ora.cg(om, D, s["G"], s["f"], niter, precision)
    rel = np.abs(hist - ref.hist) / np.abs(ref.hist)
    tol = 1e-10 if precision == "fp64" else 1e-4
    assert rel.max() <= tol, rel.max()
    if bitwise:
        assert bits_equal(hist, ref.hist)
        assert bits_equal(trace, ref.trace)
    x = ctx.solution()
    xr = ref.x.astype(np.float64)
    if bitwise:
        assert bits_equal(x, xr)
    tr, h0 = ora.true_residual(om, D, s["G"], s["f"], xr)
    assert res["defect_iter"] == ref.defect == 0
    assert res["true_res"] == pytest.approx(tr, rel=1e-12, abs=1e-300)
    return ctx, ref, res


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_cg_c1_history_bitwise(nbk, ora, precision):
    _cg_parity(nbk, ora, (2, 2, 2, 8, 0.0, 0, 1001), 100, precision)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("args", [(3, 3, 3, 12, 0.1, 2003, 1003), (4, 4, 4, 10, 0.1, 2005, 1005),
                                  (5, 3, 2, 4, 0.0, 0, 77)])
def test_cg_small_meshes_history_bitwise(nbk, ora, precision, args):
    _cg_parity(nbk, ora, args, 100, precision)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_cg_c2_history_bitwise(nbk, ora, precision):
    """C2 (16^3, N=8) in the bench's launch configuration; 30 iterations keep
    the oracle to seconds."""
    _cg_parity(nbk, ora, (16, 16, 16, 8, 0.0, 0, 1002), 30, precision)


def test_cg_zero_rhs_and_defect(nbk, ora):
    ctx, om, D, s = make(nbk, ora, 2, 2, 2, 4, contract=False)
    ctx.load_arrays(f=np.zeros((om.E, 4, 4, 4)))
    for prec in ("fp64", "fp32"):
        hist, trace, res = ctx.cg_solve(10, prec)
        assert (hist == 0).all() and res["defect_iter"] == 0
        assert (ctx.solution() == 0).all()
    ctx.load_arrays(G=-s["G"], f=s["f"])  # indefinite operator: pap < 0
    hist, trace, res = ctx.cg_solve(5, "fp64")
    assert res["defect_iter"] == 1
    ref = ora.cg(om, D, -s["G"], s["f"], 5)
    assert ref.defect == 1


def test_e2e_host_solve_matches_device_solve(nbk, ora):
    ctx, om, D, s = make(nbk, ora, 4, 4, 4, 8, 0.0, 0, 5)
    h1, _, r1 = ctx.cg_solve(50, "fp32")
    x1 = ctx.solution()
    xh = np.zeros((om.E, 8, 8, 8))
    h2, r2 = ctx.cg_solve_host(s["f"], 50, "fp32", xh)
    assert bits_equal(h1, h2) and bits_equal(x1, xh)
    assert 0 < r2["true_res_rel"] < 1 and r2["true_res_rel"] == r1["true_res_rel"]


def test_errors(nbk, ora):
    with pytest.raises(nbk.NbkError):
        nbk.cg_setup(nbk.MeshSpec(2, 2, 2, 17), "fp64")
    with pytest.raises(nbk.NbkError):
        nbk.cg_setup(nbk.MeshSpec(2, 2, 2, 8, jitter=0.5), "fp64")
    ctx = nbk.cg_setup(nbk.MeshSpec(2, 2, 2, 4), "fp64")
    with pytest.raises(nbk.NbkError):
        ctx.cg_solve(10, "fp32")  # no FP32 arrays
    with pytest.raises(nbk.NbkError):
        ctx.cg_solve(0, "fp64")


# ------------------------------------------------- full-size samples
@pytest.mark.parametrize("cfg", ["C3", "C5"])
def test_full_size_sampled_ax_and_continuity(nbk, ora, cfg):
    """Full BASELINE sizes in the bench's launch configuration: the library's
    own set-up vs the oracle on sampled elements, ax_e bitwise on sampled
    elements (oracle fed the library's G for those elements), and the
    continuity invariant of dssum (every copy of a node equal) at full size."""
    c = nbk.CONFIGS[cfg]
    spec = nbk.MeshSpec(**c.mesh_args())
    ctx = nbk.cg_setup(spec, "fp32")
    N, E = c.N, spec.E
    rng = np.random.default_rng(5)
    sample = np.unique(np.concatenate([[0, E - 1], rng.integers(0, E, 6)]))
    _, Gl, fl = ctx.get_arrays()
    om = ora.Mesh(**{k: v for k, v in c.mesh_args().items()})
    _, _, D = ora.gll(N)
    # the oracle's D-based Jacobian loses ~u*|D|*|x|/|x_r| ~ 1/h digits to
    # cancellation (coordinates O(1), derivatives O(h)): tolerance grows with ex
    tol = 5e-14 * max(1.0, c.ex / 4)
    for e in sample:
        so = ora.setup(om, int(e), int(e) + 1, want=("G", "f"))
        assert maxrel(Gl[e:e + 1], so["G"]) <= tol
        assert bits_equal(fl[e:e + 1], so["f"])
    del fl
    u = torch.empty(ctx.shape, dtype=torch.float32, device="cuda").uniform_(-1, 1)
    w = torch.empty_like(u)
    ctx.ax_apply(u, w, nbk.AX_LOCAL)
    ctx.sync()
    Dl, _, _ = ctx.get_arrays()
    for e in sample:
        ue = u[e:e + 1].cpu().numpy()
        ref = ora.ax_local(Dl.astype(np.float32), Gl[e:e + 1].astype(np.float32), ue)
        assert bits_equal(w[e:e + 1].cpu().numpy(), ref)
    del Gl
    # continuity: dssum of a field gives equal values on all copies of a node
    ctx.dssum(w)
    ctx.sync()
    gid = torch.from_numpy(ora.setup(om, want=("gid",))["gid"].reshape(-1)).cuda()
    wf = w.reshape(-1)
    mx = torch.full((ctx.n_global,), -float("inf"), device="cuda").scatter_reduce(0, gid, wf, "amax")
    mn = torch.full((ctx.n_global,), float("inf"), device="cuda").scatter_reduce(0, gid, wf, "amin")
    assert torch.equal(mx[gid], wf) and torch.equal(mn[gid], wf)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_glsc3_special_values(nbk, ora, dtype):
    """glsc3 with +-inf / NaN / huge / subnormal entries: the plain IEEE result
    the exact-sum definition gives (inf, NaN for inf - inf), and correctly
    rounded sums of subnormal terms (R25)."""
    ctx, om, D, s = make(nbk, ora, 2, 2, 2, 4)
    c = ora.multiplicity_weight(om)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    big = np.finfo(dtype).max
    tiny = np.finfo(dtype).smallest_subnormal
    base = inputs.uniform_field((om.E, 4, 4, 4), 3, dtype)
    cases = []
    a = base.copy(); a.flat[5] = np.inf; cases.append((a, base))                 # +inf
    a = base.copy(); a.flat[5] = np.inf; a.flat[9] = -np.inf; cases.append((a, np.abs(base) + 1))  # inf - inf
    a = base.copy(); a.flat[7] = np.nan; cases.append((a, base))                 # NaN
    a = np.full_like(base, big); cases.append((a, np.full_like(base, 2.0)))      # overflow of products
    a = np.full_like(base, tiny); cases.append((a, np.full_like(base, 0.75)))    # subnormal terms
    a = base * np.asarray(2.0 ** -500 if dtype == np.float64 else 2.0 ** -60, dtype)
    cases.append((a, a))                                                          # squares underflow
    for a, b in cases:
        got = ctx.glsc3(dev(a, tdt), dev(b, tdt))
        ref = ora.glsc3(a, b, c)
        if np.isnan(ref):
            assert np.isnan(got)
        else:
            assert got == ref, (got, ref)
    ctx.close()
