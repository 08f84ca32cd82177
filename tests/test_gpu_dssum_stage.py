"""K_B with the tile index rows staged in shared memory (double-buffered bulk
copies, NBK_DSSUM_STAGE): the staged kernel must give the unstaged bits.

NBK_DSSUM_STAGE=2 forces staging on the small meshes the oracle can follow;
NBK_DSSUM_TILE_NODES=64 cuts C2 into ~4096 one-element tiles so that every
block owns several tiles and both buffers and both mbarrier phases cycle.
Both variables are read at set-up / graph capture, so each test builds its own
context under them.
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


@pytest.fixture
def staged(monkeypatch):
    monkeypatch.setenv("NBK_DSSUM_STAGE", "2")


def bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    assert a.dtype == b.dtype and a.shape == b.shape
    return np.array_equal(a.view(np.uint8), b.view(np.uint8))


def setup(nbk, ora, args, precision="fp32"):
    ex, ey, ez, N, jit, sg, sr = args
    spec = nbk.MeshSpec(ex, ey, ez, N, jit, sg, sr)
    ctx = nbk.cg_setup(spec, precision)
    om = ora.Mesh(ex, ey, ez, N, jit, sg, sr)
    _, _, D = ora.gll(N)
    s = ora.setup(om, want=("G", "f"))
    ctx.load_arrays(D, s["G"], s["f"])
    return ctx, om, D, s


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("args", [(3, 4, 2, 6, 0.0, 0, 0), (3, 2, 3, 2, 0.0, 0, 0),
                                  (2, 2, 3, 7, 0.1, 4, 5)])
@pytest.mark.parametrize("mask", [False, True])
def test_staged_dssum_bitwise(nbk, ora, staged, monkeypatch, dtype, args, mask):
    monkeypatch.setenv("NBK_DSSUM_TILE_NODES", "16")
    ctx, om, D, s = setup(nbk, ora, args)
    N = args[3]
    f = inputs.uniform_field((om.E, N, N, N), 31, dtype)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    fd = torch.from_numpy(np.ascontiguousarray(f)).to("cuda", tdt)
    ctx.dssum(fd, apply_mask=mask)
    ctx.sync()
    assert bits_equal(fd.cpu().numpy(), ora.dssum(om, f, apply_mask=mask))
    ctx.close()


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_staged_cg_c2_many_tiles_per_block(nbk, ora, monkeypatch, precision):
    monkeypatch.setenv("NBK_DSSUM_TILE_NODES", "64")   # auto mode stages (tiles >= 4 per block)
    monkeypatch.delenv("NBK_DSSUM_STAGE", raising=False)
    args = (16, 16, 16, 8, 0.0, 0, 1002)
    ctx, om, D, s = setup(nbk, ora, args)
    hist, trace, res = ctx.cg_solve(30, precision)
    ref = ora.cg(om, D, s["G"], s["f"], 30, precision)
    assert bits_equal(hist, ref.hist) and bits_equal(trace, ref.trace)
    assert bits_equal(ctx.solution(), ref.x.astype(np.float64))
    ctx.close()


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_staged_group_cg(nbk, ora, staged, precision):
    args = (3, 3, 4, 10, 0.1, 2005, 1005)
    ex, ey, ez, N, jit, sg, sr = args
    spec = nbk.MeshSpec(*args)
    grp = nbk.Group(spec, 2, "fp32")
    om = ora.Mesh(*args)
    _, _, D = ora.gll(N)
    s = ora.setup(om, want=("G", "f"))
    El = om.E // 2
    grp.load_arrays(D, [s["G"][r * El:(r + 1) * El] for r in range(2)],
                    [s["f"][r * El:(r + 1) * El] for r in range(2)])
    hist, trace, res = grp.cg_solve(40, precision)
    ref = ora.cg(om, D, s["G"], s["f"], 40, precision)
    assert bits_equal(hist, ref.hist) and bits_equal(trace, ref.trace)
    assert bits_equal(grp.solution(), ref.x.astype(np.float64))
    grp.close()


def test_staged_equals_unstaged_jacobi_and_single(nbk, ora, monkeypatch):
    """Jacobi PCG and the paper-literal single solver: staged == unstaged bits."""
    args = (4, 4, 4, 8, 0.1, 7, 8)
    out = []
    for mode in ("0", "2"):
        monkeypatch.setenv("NBK_DSSUM_STAGE", mode)
        monkeypatch.setenv("NBK_DSSUM_TILE_NODES", "32")
        ctx = nbk.cg_setup(nbk.MeshSpec(*args), "fp32")
        r = []
        for prec in ("fp32s", "fp64"):
            ctx.set_precond("jacobi")
            h, t, _ = ctx.cg_solve(25, prec)
            r.append((h, t, ctx.solution()))
        out.append(r)
        ctx.close()
    for a, b in zip(out[0], out[1]):
        for u, v in zip(a, b):
            assert bits_equal(u, v)
