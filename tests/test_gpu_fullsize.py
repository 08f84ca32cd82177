"""Full-size CG parity with the oracle: C3 (32^3, N=12,
jittered) and C5 (64^3, N=10, jittered; the bench's headline workload) in
contract mode (C10: the library ingests the oracle's D, G, f), the first 10
iterations of the T1 loop by the FP64 and by the mixed FP32 solver,
in the bench's launch configuration (one context set up with FP32 arrays, the
same kernels and graphs).  History, trace (rtz1, beta, alpha, pap, rtr) and
the solution must be bitwise equal; the true FP64 residual (C12) must match
the oracle's.

Host cost: the oracle's C5 set-up and solves need ~40 GB of host memory and a
few minutes on the GPU host's cores; the library's copy of G is 12.6 GB.
"""
import gc

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")

NITER = 10


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


def _full_size(nbk, ora, name):
    c = nbk.CONFIGS[name]
    args = c.mesh_args(1)
    ctx = nbk.cg_setup(nbk.MeshSpec(**args), "fp32")
    om = ora.Mesh(**args)
    _, _, D = ora.gll(c.N)
    s = ora.setup(om, want=("G", "f"))
    ctx.load_arrays(D, s["G"], s["f"])
    try:
        for prec in ("fp32", "fp64"):
            hist, trace, res = ctx.cg_solve(NITER, prec)
            ref = ora.cg(om, D, s["G"], s["f"], NITER, prec)
            assert bits_equal(hist, ref.hist), (name, prec)
            assert bits_equal(trace, ref.trace), (name, prec)
            xr = ref.x.astype(np.float64)
            assert bits_equal(ctx.solution(), xr), (name, prec)
            assert res["defect_iter"] == ref.defect == 0
            tr, _ = ora.true_residual(om, D, s["G"], s["f"], xr)
            assert res["true_res"] == pytest.approx(tr, rel=1e-12)
            del ref, xr
            gc.collect()
    finally:
        ctx.close()
        del s
        gc.collect()
        torch.cuda.empty_cache()


def test_c3_cg_first_iterations_bitwise(nbk, ora):
    _full_size(nbk, ora, "C3")


def test_c5_cg_first_iterations_bitwise(nbk, ora):
    _full_size(nbk, ora, "C5")
