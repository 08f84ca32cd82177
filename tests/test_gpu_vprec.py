"""VPREC precision emulation of the CG loop (P:60-62,
P:364-372: every floating-point operation of the CG kernels computed in
binary64 and its result rounded to t mantissa bits) through the C ABI, bitwise
against the oracle's emulation, which rounds the same operations in the same
canonical order (CEO-1)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def nbk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_11065_b200 as p
    p.load()
    return p


def bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    assert a.dtype == b.dtype and a.shape == b.shape
    return np.array_equal(a.view(np.uint8), b.view(np.uint8))


def make(nbk, ora, args):
    ex, ey, ez, N, jit, sg, sr = args
    ctx = nbk.cg_setup(nbk.MeshSpec(ex, ey, ez, N, jit, sg, sr), "fp64")
    om = ora.Mesh(ex, ey, ez, N, jit, sg, sr)
    _, _, D = ora.gll(N)
    s = ora.setup(om, want=("G", "f"))
    ctx.load_arrays(D, s["G"], s["f"])
    return ctx, om, D, s


@pytest.mark.parametrize("t", [3, 8, 16, 23, 40])
@pytest.mark.parametrize("args", [(2, 2, 2, 8, 0.0, 0, 1001), (3, 2, 2, 12, 0.1, 2003, 1003),
                                  (3, 3, 2, 5, 0.2, 4, 5)])
def test_vprec_solver_bitwise(nbk, ora, t, args):
    ctx, om, D, s = make(nbk, ora, args)
    ctx.set_vprec(t)
    hist, trace, res = ctx.cg_solve(60, "vprec")
    ref = ora.cg_vprec(om, D, s["G"], s["f"], 60, t)
    assert bits_equal(hist, ref.hist)
    assert bits_equal(trace, ref.trace)
    assert bits_equal(ctx.solution(), ref.x)
    assert res["defect_iter"] == ref.defect
    tr, _ = ora.true_residual(om, D, s["G"], s["f"], ref.x)
    assert res["true_res"] == pytest.approx(tr, rel=1e-12, abs=1e-300)
    ctx.close()


def test_vprec_t52_is_the_fp64_solver(nbk, ora):
    ctx, om, D, s = make(nbk, ora, (4, 4, 4, 10, 0.1, 2005, 1005))
    ctx.set_vprec(52)
    a = ctx.cg_solve(50, "vprec")
    xa = ctx.solution()
    b = ctx.cg_solve(50, "fp64")
    assert bits_equal(a[0], b[0]) and bits_equal(a[1], b[1]) and bits_equal(xa, ctx.solution())
    ctx.close()


def test_vprec_rejects_large_n(nbk, ora):
    ctx = nbk.cg_setup(nbk.MeshSpec(2, 2, 2, 14), "fp64")
    ctx.set_vprec(23)
    with pytest.raises(nbk.NbkError):
        ctx.cg_solve(5, "vprec")
    ctx.close()
    ctx = nbk.cg_setup(nbk.MeshSpec(2, 2, 2, 10), "fp64")
    ctx.set_emulation("mca", 23, 1)       # Monte Carlo kernels are built for N <= 8
    with pytest.raises(nbk.NbkError):
        ctx.cg_solve(5, "vprec")
    ctx.set_vprec(23)                     # VPREC: N <= 12
    ctx.cg_solve(5, "vprec")
    with pytest.raises(nbk.NbkError):
        ctx.set_vprec(60)
    ctx.close()


@pytest.mark.parametrize("mode", ["rr", "mca"])
@pytest.mark.parametrize("args", [(2, 2, 2, 8, 0.0, 0, 1001), (3, 2, 2, 6, 0.15, 4, 5)])
def test_mca_samples_bitwise(nbk, ora, mode, args):
    """Monte Carlo random rounding / full MCA samples: the library
    draws the same xi for the same operation as the oracle (counter-based
    SplitMix64 over (iteration, phase, global index, operation)), so each
    sample is bitwise reproducible and equal to the oracle's."""
    ctx, om, D, s = make(nbk, ora, args)
    for seed in (1, 2):
        ctx.set_emulation(mode, 23, seed)
        hist, trace, res = ctx.cg_solve(40, "vprec")
        ref = ora.cg_emulated(om, D, s["G"], s["f"], 40, mode, 23, seed)
        assert bits_equal(hist, ref.hist)
        assert bits_equal(trace, ref.trace)
        assert bits_equal(ctx.solution(), ref.x)
    ctx.close()


def test_emulation_vprec_mode_matches_set_vprec(nbk, ora):
    ctx, om, D, s = make(nbk, ora, (2, 2, 2, 8, 0.0, 0, 1001))
    ctx.set_vprec(16)
    a = ctx.cg_solve(30, "vprec")[0]
    ctx.set_emulation("vprec", 16, 99)
    b = ctx.cg_solve(30, "vprec")[0]
    assert bits_equal(a, b)
    ctx.close()


def test_emulation_is_single_rank(nbk, ora):
    """The slab-face merge is not emulated: emulated solves need one rank."""
    grp = nbk.Group(nbk.MeshSpec(2, 2, 4, 6), 2, "fp64")
    for c in grp.ctxs:
        c.set_emulation("rr", 23, 5)
    with pytest.raises(nbk.NbkError):
        grp.cg_solve(5, "vprec")
    grp.close()


def _same(a, b):  # bitwise, any NaN matching any NaN
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and bits_equal(np.where(na, 0.0, a), np.where(nb, 0.0, b))


@pytest.mark.parametrize("mode,t", [("vprec", 52), ("vprec", 30), ("vprec", 10), ("mca", 23),
                                    ("rr", 23)])
def test_emulation_long_runs_past_convergence(nbk, ora, mode, t):
    """1200 iterations on C1, far past convergence (products and the per-copy
    glsc3 terms RN(t(a b))/m subnormal): the emulated GPU solve still follows the
    oracle bit for bit."""
    args = (2, 2, 2, 8, 0.0, 0, 1001)
    ctx, om, D, s = make(nbk, ora, args)
    ctx.set_emulation(mode, t, 7)
    niter = 1200
    hist, trace, res = ctx.cg_solve(niter, "vprec")
    if mode == "vprec":
        ref = ora.cg_vprec(om, D, s["G"], s["f"], niter, t)
    else:
        ref = ora.cg_emulated(om, D, s["G"], s["f"], niter, mode, t, 7)
    assert res["defect_iter"] == ref.defect
    assert _same(hist, ref.hist) and _same(trace, ref.trace) and _same(ctx.solution(), ref.x)
    ctx.close()
