"""Jacobi-preconditioned CG (T1 line 2 "solveM", P:144;
S:376-384) through the C ABI, against the oracle.

Contract mode: the library ingests the oracle's D, G, f and dinv (C10) and
both follow CEO-1 with z = RN_T(r * dinv_T) and rtz1 = glsc3(r, c, z): the
history, trace and solution are compared bitwise.  The library's own
assembled diagonal is compared with the oracle's within rounding.
"""
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


def setup(nbk, ora, args, load_dinv=True):
    ex, ey, ez, N, jit, sg, sr = args
    ctx = nbk.cg_setup(nbk.MeshSpec(ex, ey, ez, N, jit, sg, sr), "fp32")
    om = ora.Mesh(ex, ey, ez, N, jit, sg, sr)
    _, _, D = ora.gll(N)
    s = ora.setup(om, want=("G", "f"))
    ctx.load_arrays(D, s["G"], s["f"])
    _, dinv = ora.jacobi_dinv(om, D, s["G"])
    if load_dinv:
        ctx.load_precond(dinv)
    ctx.set_precond("jacobi")
    return ctx, om, D, s, dinv


MESHES = [(2, 2, 2, 8, 0.0, 0, 1001), (3, 3, 3, 12, 0.1, 2003, 1003), (4, 4, 4, 10, 0.1, 2005, 1005),
          (3, 2, 2, 5, 0.2, 4, 5), (1, 1, 1, 3, 0.0, 0, 9)]


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("args", MESHES)
def test_pcg_history_trace_solution_bitwise(nbk, ora, precision, args):
    ctx, om, D, s, dinv = setup(nbk, ora, args)
    hist, trace, res = ctx.cg_solve(100, precision)
    ref = ora.cg(om, D, s["G"], s["f"], 100, precision, dinv=dinv)
    assert bits_equal(hist, ref.hist)
    assert bits_equal(trace, ref.trace)
    assert bits_equal(ctx.solution(), ref.x.astype(np.float64))
    nz = ref.hist > 0
    rel = np.abs(hist[nz] - ref.hist[nz]) / ref.hist[nz]
    assert rel.max() <= (1e-10 if precision == "fp64" else 1e-4)
    assert res["defect_iter"] == ref.defect == 0
    tr, _ = ora.true_residual(om, D, s["G"], s["f"], ref.x.astype(np.float64))
    assert res["true_res"] == pytest.approx(tr, rel=1e-12, abs=1e-300)
    ctx.close()


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_pcg_c2_bitwise(nbk, ora, precision):
    """C2 in the bench's launch configuration (30 iterations keep the oracle short)."""
    ctx, om, D, s, dinv = setup(nbk, ora, (16, 16, 16, 8, 0.0, 0, 1002))
    hist, trace, _ = ctx.cg_solve(30, precision)
    ref = ora.cg(om, D, s["G"], s["f"], 30, precision, dinv=dinv)
    assert bits_equal(hist, ref.hist) and bits_equal(trace, ref.trace)
    ctx.close()


@pytest.mark.parametrize("args", [(2, 2, 2, 8, 0.0, 0, 1), (3, 2, 4, 6, 0.2, 3, 2), (2, 3, 2, 12, 0.1, 7, 3)])
def test_own_diagonal_matches_oracle(nbk, ora, args):
    """The library's assembled diagonal (own kernel + own dssum) from the same G
    equals the oracle's within rounding of a ~3N+3-term sum."""
    ctx, om, D, s, dinv = setup(nbk, ora, args, load_dinv=False)
    got = ctx.get_precond()
    assert np.abs(got - dinv).max() <= 1e-14 * np.abs(dinv).max()
    msk = ora.setup(om, want=("mask",))["mask"].astype(bool)
    assert (got[msk] == 1.0).all()
    ctx.close()


def test_pcg_own_setup_converges_faster_than_cg(nbk, ora):
    """Independent set-up (library's G, f, own diagonal): Jacobi PCG on a
    jittered mesh reduces the residual more than CG in the same iterations,
    and the FP32 and FP64 Jacobi solvers agree early on."""
    spec = nbk.MeshSpec(8, 8, 8, 8, 0.2, 11, 12)
    ctx = nbk.cg_setup(spec, "fp32")
    h_cg, _, _ = ctx.cg_solve(60, "fp64")
    ctx.set_precond("jacobi")
    h64, _, r64 = ctx.cg_solve(60, "fp64")
    h32, _, _ = ctx.cg_solve(60, "fp32")
    assert h64[60] < h_cg[60]
    assert np.abs(h32[:10] - h64[:10]).max() / h64[0] < 1e-4
    assert r64["defect_iter"] == 0
    ctx.close()


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_pcg_virtual_slabs_bitwise(nbk, ora, P, precision):
    """Multi-rank Jacobi PCG (rtr and rtz all-gathered per rank) = oracle."""
    ex, ey, ez, N, jit, sg, sr = (3, 2, 8, 6, 0.15, 21, 22)
    spec = nbk.MeshSpec(ex, ey, ez, N, jit, sg, sr)
    grp = nbk.Group(spec, P, "fp32")
    om = ora.Mesh(ex, ey, ez, N, jit, sg, sr)
    _, _, D = ora.gll(N)
    s = ora.setup(om, want=("G", "f"))
    _, dinv = ora.jacobi_dinv(om, D, s["G"])
    El = om.E // P
    sl = lambda a: [a[r * El:(r + 1) * El] for r in range(P)]  # noqa: E731
    grp.load_arrays(D, sl(s["G"]), sl(s["f"]))
    grp.set_precond("jacobi")
    # own diagonal across slabs (face exchange in the assembly) first ...
    own = np.concatenate([c.get_precond() for c in grp.ctxs])
    assert np.abs(own - dinv).max() <= 1e-14 * np.abs(dinv).max()
    # ... then the oracle's data for the bitwise solve
    grp.load_precond(sl(dinv))
    hist, trace, _ = grp.cg_solve(50, precision)
    ref = ora.cg(om, D, s["G"], s["f"], 50, precision, dinv=dinv)
    assert bits_equal(hist, ref.hist) and bits_equal(trace, ref.trace)
    assert bits_equal(grp.solution(), ref.x.astype(np.float64))
    grp.close()


def test_pcg_zero_rhs(nbk, ora):
    ctx, om, D, s, dinv = setup(nbk, ora, (2, 2, 2, 4, 0.0, 0, 0))
    ctx.load_arrays(f=np.zeros((om.E, 4, 4, 4)))
    ctx.load_precond(dinv)
    for prec in ("fp64", "fp32"):
        hist, _, res = ctx.cg_solve(10, prec)
        assert (hist == 0).all() and res["defect_iter"] == 0 and (ctx.solution() == 0).all()
    ctx.close()
