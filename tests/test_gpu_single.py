"""Paper-literal single-precision solver ("solver
runs exclusively in single") through the C ABI vs the oracle.

Reading R11b: inner products RN32(sum RN32(a_L b_L) c_L) -- the
correctly rounded binary32 value of the binary32 products -- and the scalars
alpha = rtz1/pap, beta = rtz1/rtz2, h = sqrt(rtr) in binary32.  Contract mode,
bitwise comparisons.
"""
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


def bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    assert a.dtype == b.dtype and a.shape == b.shape
    return np.array_equal(a.view(np.uint8), b.view(np.uint8))


def make(nbk, ora, args):
    ex, ey, ez, N, jit, sg, sr = args
    ctx = nbk.cg_setup(nbk.MeshSpec(ex, ey, ez, N, jit, sg, sr), "fp32")
    om = ora.Mesh(ex, ey, ez, N, jit, sg, sr)
    _, _, D = ora.gll(N)
    s = ora.setup(om, want=("G", "f"))
    ctx.load_arrays(D, s["G"], s["f"])
    return ctx, om, D, s


@pytest.mark.parametrize("jacobi", [False, True])
@pytest.mark.parametrize("args", [(2, 2, 2, 8, 0.0, 0, 1001), (3, 3, 3, 12, 0.1, 2003, 1003),
                                  (4, 4, 4, 10, 0.1, 2005, 1005), (3, 2, 2, 5, 0.2, 4, 5)])
def test_single_solver_bitwise(nbk, ora, args, jacobi):
    ctx, om, D, s = make(nbk, ora, args)
    dinv = None
    if jacobi:
        _, dinv = ora.jacobi_dinv(om, D, s["G"])
        ctx.load_precond(dinv)
        ctx.set_precond("jacobi")
    hist, trace, res = ctx.cg_solve(100, "fp32s")
    ref = ora.cg(om, D, s["G"], s["f"], 100, "fp32s", dinv=dinv)
    assert bits_equal(hist, ref.hist)
    assert bits_equal(trace, ref.trace)
    assert bits_equal(ctx.solution(), ref.x.astype(np.float64))
    assert res["defect_iter"] == ref.defect == 0
    ctx.close()


def test_single_solver_c2_bitwise(nbk, ora):
    ctx, om, D, s = make(nbk, ora, (16, 16, 16, 8, 0.0, 0, 1002))
    hist, trace, _ = ctx.cg_solve(30, "fp32s")
    ref = ora.cg(om, D, s["G"], s["f"], 30, "fp32s")
    assert bits_equal(hist, ref.hist) and bits_equal(trace, ref.trace)
    ctx.close()


def test_single_glsc3_bitwise(nbk, ora):
    ctx, om, D, s = make(nbk, ora, (4, 3, 5, 8, 0.0, 0, 0))
    c = ora.multiplicity_weight(om)
    for seed in range(6):
        a = inputs.uniform_field((om.E, 8, 8, 8), seed, np.float32, -3.0, 3.0)
        b = inputs.uniform_field((om.E, 8, 8, 8), seed + 50, np.float32)
        got = ctx.glsc3(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), single=True)
        assert got == ora.glsc3_single(a, b, c)
        assert np.float32(got) == got
    ctx.close()


@pytest.mark.parametrize("P", [2, 4])
def test_single_solver_virtual_slabs(nbk, ora, P):
    ex, ey, ez, N, jit, sg, sr = (3, 2, 8, 6, 0.15, 21, 22)
    grp = nbk.Group(nbk.MeshSpec(ex, ey, ez, N, jit, sg, sr), P, "fp32")
    om = ora.Mesh(ex, ey, ez, N, jit, sg, sr)
    _, _, D = ora.gll(N)
    s = ora.setup(om, want=("G", "f"))
    El = om.E // P
    grp.load_arrays(D, [s["G"][r * El:(r + 1) * El] for r in range(P)],
                    [s["f"][r * El:(r + 1) * El] for r in range(P)])
    hist, trace, _ = grp.cg_solve(50, "fp32s")
    ref = ora.cg(om, D, s["G"], s["f"], 50, "fp32s")
    assert bits_equal(hist, ref.hist) and bits_equal(trace, ref.trace)
    assert bits_equal(grp.solution(), ref.x.astype(np.float64))
    grp.close()


def test_accuracy_report_shapes(nbk, ora):
    """AE/MAE of the two single-precision solvers against the FP64
    solver on C1: both small and finite; reported by bench.py."""
    ctx, om, D, s = make(nbk, ora, (2, 2, 2, 8, 0.0, 0, 1001))
    h64, _, _ = ctx.cg_solve(100, "fp64")
    h32, _, r32 = ctx.cg_solve(100, "fp32")
    h1, _, r1 = ctx.cg_solve(100, "fp32s")
    ae32 = np.abs(h32[1:] - h64[1:])
    ae1 = np.abs(h1[1:] - h64[1:])
    assert np.isfinite(ae32).all() and np.isfinite(ae1).all()
    assert ae32.mean() < 1e-2 * h64[0] and ae1.mean() < 1e-2 * h64[0]
    assert 0 < r32["true_res_rel"] < 1e-3 and 0 < r1["true_res_rel"] < 1e-3
    ctx.close()


@pytest.mark.parametrize("precision", ["fp64", "fp32", "fp32s"])
@pytest.mark.parametrize("args", [(2, 2, 2, 8, 0.0, 0, 1001), (3, 2, 2, 5, 0.2, 4, 5)])
def test_long_runs_past_convergence_bitwise(nbk, ora, precision, args):
    """1500 iterations: far past convergence, where the recursive residual of the
    single-precision solvers runs into binary32 denormals / underflow (the bench's
    convergence study sees the paper-literal solver break down there) -- the
    GPU path must still follow the oracle bit for bit, defect flag included."""
    ctx, om, D, s = make(nbk, ora, args)
    niter = 1500
    hist, trace, res = ctx.cg_solve(niter, precision)
    ref = ora.cg(om, D, s["G"], s["f"], niter, precision)

    def same(a, b):  # bitwise, except that any NaN matches any NaN (payloads differ)
        a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
        na, nb = np.isnan(a), np.isnan(b)
        return np.array_equal(na, nb) and bits_equal(np.where(na, 0.0, a), np.where(nb, 0.0, b))

    assert res["defect_iter"] == ref.defect
    assert same(hist, ref.hist)
    assert same(trace, ref.trace)
    assert same(ctx.solution(), ref.x.astype(np.float64))
    ctx.close()


def _same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and bits_equal(np.where(na, 0.0, a), np.where(nb, 0.0, b))


@pytest.mark.parametrize("precision", ["fp64", "fp32", "fp32s"])
def test_long_jacobi_runs_past_convergence_bitwise(nbk, ora, precision):
    """Jacobi PCG for 1200 iterations (z = RN(r dinv) and the rtz terms reach the
    subnormal range) -- bit for bit with the oracle."""
    ctx, om, D, s = make(nbk, ora, (3, 2, 2, 5, 0.2, 4, 5))
    _, dinv = ora.jacobi_dinv(om, D, s["G"])
    ctx.load_precond(dinv)
    ctx.set_precond("jacobi")
    hist, trace, res = ctx.cg_solve(1200, precision)
    ref = ora.cg(om, D, s["G"], s["f"], 1200, precision, dinv=dinv)
    assert res["defect_iter"] == ref.defect
    assert _same(hist, ref.hist) and _same(trace, ref.trace)
    assert _same(ctx.solution(), ref.x.astype(np.float64))
    ctx.close()


@pytest.mark.parametrize("P", [2, 4])
def test_long_virtual_slab_runs_past_convergence_bitwise(nbk, ora, P):
    """The face merge's pap terms for slab-plane nodes in the subnormal regime."""
    args = (2, 2, 4, 8, 0.0, 0, 1001)
    spec = nbk.MeshSpec(*args)
    grp = nbk.Group(spec, P, "fp32")
    om = ora.Mesh(*args)
    _, _, D = ora.gll(8)
    s = ora.setup(om, want=("G", "f"))
    El = om.E // P
    grp.load_arrays(D, [s["G"][r * El:(r + 1) * El] for r in range(P)],
                    [s["f"][r * El:(r + 1) * El] for r in range(P)])
    for prec in ("fp64", "fp32"):
        hist, trace, res = grp.cg_solve(1200, prec)
        ref = ora.cg(om, D, s["G"], s["f"], 1200, prec)
        assert res["defect_iter"] == ref.defect
        assert _same(hist, ref.hist) and _same(trace, ref.trace)
        assert _same(grp.solution(), ref.x.astype(np.float64))
    grp.close()


@pytest.mark.parametrize("precision", ["fp64", "fp32", "fp32s"])
@pytest.mark.parametrize("scale_exp", [600, -600, 120])
def test_extreme_rhs_scaling_bitwise(nbk, ora, precision, scale_exp):
    """f scaled by 2^600 / 2^-600 / 2^120 (exact): overflow of the inner
    products to inf (defect flag), subnormal / underflowing data from the start,
    and FP32 overflow of the RN32(f) rounding -- the library and the oracle take
    the same path, defect iteration included."""
    ctx, om, D, s = make(nbk, ora, (2, 2, 2, 6, 0.0, 0, 9))
    f = s["f"] * (2.0 ** scale_exp)
    ctx.load_arrays(D, s["G"], f)
    hist, trace, res = ctx.cg_solve(60, precision)
    ref = ora.cg(om, D, s["G"], f, 60, precision)
    assert res["defect_iter"] == ref.defect
    assert _same(hist, ref.hist) and _same(trace, ref.trace)
    assert _same(ctx.solution(), ref.x.astype(np.float64))
    ctx.close()


# ------------------------------------------- the paper's binary32-accumulating solver (R11c)
def _order_insensitive_window(ora, om, D, s, niter, ref):
    """Iterations over which the binary32-accumulating CG does not depend on the
    summation order: the oracle's own runs with 2 and 3 z-slabs (other, equally
    valid binary32 orders) stay within 5e-5 (half the tolerance) of the 1-slab run.  Past it the
    rounding noise of binary32 sums decides the trajectory (on C1 two orders
    differ by 4e-4 at iteration 40 and 6e-2 at 45), so no order is the right one."""
    rel = np.zeros(niter + 1)
    for P in (2, 3):
        o = ora.cg(om, D, s["G"], s["f"], niter, "fp32a", nranks=P)
        rel = np.maximum(rel, np.abs(o.hist - ref.hist) / ref.hist)
    bad = np.nonzero(rel > 5e-5)[0]
    return int(bad[0]) if len(bad) else niter + 1


@pytest.mark.parametrize("args", [(2, 2, 2, 8, 0.0, 0, 1001), (3, 3, 3, 10, 0.1, 2005, 1005)])
def test_accum32_solver_tracks_oracle(nbk, ora, args):
    """NEXT-2 as the paper ran it (R11c): binary32
    accumulation of every glsc3.  The oracle sums sequentially, the library by a
    fixed binary32 tree: the two are different roundings of the same sums, so
    parity is the north_star FP32 tolerance (1e-4 relative) over the
    iterations before the recursive residual reaches the binary32 noise floor
    (h_k/h_0 > 1e-4), where the order of rounding decides nothing yet."""
    ctx, om, D, s = make(nbk, ora, args)
    niter = 60
    hist, trace, res = ctx.cg_solve(niter, "fp32a")
    ref = ora.cg(om, D, s["G"], s["f"], niter, "fp32a")
    assert res["defect_iter"] == 0 and ref.defect == 0
    win = _order_insensitive_window(ora, om, D, s, niter, ref)
    assert win >= 10
    rel = np.abs(hist[:win] - ref.hist[:win]) / ref.hist[:win]
    assert rel.max() <= 1e-4, (win, rel.max())
    # binary32 scalars; not the exactly rounded variant (R11b)
    assert (trace.astype(np.float32).astype(np.float64) == trace).all()
    hs, _, _ = ctx.cg_solve(niter, "fp32s")
    assert not np.array_equal(hist, hs)
    ctx.close()


def test_accum32_virtual_slabs_track_oracle(nbk, ora):
    """Two z-slabs: per-rank binary32 sums added in binary32 in rank order (the
    paper's single-precision all-reduce) vs the oracle with nranks = 2."""
    args = (3, 3, 4, 8, 0.1, 7, 9)
    ex, ey, ez, N, jit, sg, sr = args
    grp = nbk.Group(nbk.MeshSpec(*args), 2, "fp32")
    om = ora.Mesh(*args)
    _, _, D = ora.gll(N)
    s = ora.setup(om, want=("G", "f"))
    E2 = om.E // 2
    grp.load_arrays(D, [s["G"][:E2], s["G"][E2:]], [s["f"][:E2], s["f"][E2:]])
    hist, trace, res = grp.cg_solve(40, "fp32a")
    ref = ora.cg(om, D, s["G"], s["f"], 40, "fp32a", nranks=2)
    win = _order_insensitive_window(ora, om, D, s, 40, ref)
    assert win >= 10
    rel = np.abs(hist[:win] - ref.hist[:win]) / ref.hist[:win]
    assert rel.max() <= 1e-4, (win, rel.max())
    grp.close()


def test_accum32_rejects_jacobi(nbk):
    ctx = nbk.cg_setup(nbk.MeshSpec(2, 2, 2, 4, 0.0, 0, 1), "fp32")
    ctx.set_precond("jacobi")
    with pytest.raises(nbk.NbkError):
        ctx.cg_solve(5, "fp32a")
    ctx.close()
