"""Multi-rank z-slab path on one GPU: virtual slabs.

P contexts (rank r of P) of one mesh are linked in process (nbk_group_link);
the group calls run the same kernels as NCCL mode -- local dssum without the
slab-boundary planes, face pack, face merge in the canonical chain order
(lower rank's copies first), per-rank dd partials combined in rank order --
with the faces and partials shared by pointer instead of ncclSend/ncclRecv /
ncclAllGather.  The kernels of different slabs are enqueued one after the
other on one stream: no slab waits on another inside a kernel.

Everything is compared BITWISE with the oracle (which knows nothing about
slabs) and with the 1-rank library path: results must not depend on P.
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


def make_group(nbk, ora, args, P, precision="fp32", contract=True):
    ex, ey, ez, N, jit, sg, sr = args
    spec = nbk.MeshSpec(ex, ey, ez, N, jit, sg, sr)
    grp = nbk.Group(spec, P, precision)
    om = ora.Mesh(ex, ey, ez, N, jit, sg, sr)
    _, _, D = ora.gll(N)
    s = ora.setup(om, want=("G", "f"))
    if contract:
        El = om.E // P
        grp.load_arrays(D, [s["G"][r * El:(r + 1) * El] for r in range(P)],
                        [s["f"][r * El:(r + 1) * El] for r in range(P)])
    return grp, om, D, s


def slabs(a, P):
    El = a.shape[0] // P
    return [a[r * El:(r + 1) * El] for r in range(P)]


MESHES = [
    (2, 2, 4, 8, 0.0, 0, 1001),     # C1-like, 2 layers per slab at P=2
    (3, 2, 8, 5, 0.1, 9, 4),        # ragged, jittered, odd N
    (2, 3, 4, 2, 0.0, 0, 3),        # N = 2: every node on an element boundary
    (1, 1, 4, 6, 0.2, 5, 6),        # single element column
]


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("args", MESHES)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_group_ax_full_operator_bitwise(nbk, ora, P, args, dtype):
    grp, om, D, s = make_group(nbk, ora, args, P)
    N = args[3]
    u = inputs.uniform_field((om.E, N, N, N), 21, dtype)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    us = [torch.from_numpy(np.ascontiguousarray(x)).to("cuda", tdt) for x in slabs(u, P)]
    ws = [torch.empty_like(x) for x in us]
    grp.ax_apply(us, ws)
    grp.sync()
    w = np.concatenate([x.cpu().numpy() for x in ws])
    ref = ora.ax(om, D.astype(dtype), s["G"].astype(dtype), u, apply_mask=True)
    assert bits_equal(w, ref)
    grp.close()


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("mask", [False, True])
def test_group_dssum_bitwise(nbk, ora, P, mask):
    args = (3, 4, 6, 6, 0.0, 0, 0)
    grp, om, D, s = make_group(nbk, ora, args, P, contract=False)
    f = inputs.uniform_field((om.E, 6, 6, 6), 31)
    fs = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in slabs(f, P)]
    grp.dssum(fs, apply_mask=mask)
    grp.sync()
    got = np.concatenate([x.cpu().numpy() for x in fs])
    assert bits_equal(got, ora.dssum(om, f, apply_mask=mask))
    grp.close()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_group_glsc3_equals_one_rank(nbk, ora, dtype):
    args = (4, 3, 4, 8, 0.0, 0, 0)
    grp, om, D, s = make_group(nbk, ora, args, 4, contract=False)
    c = ora.multiplicity_weight(om)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    for seed in range(4):
        a = inputs.uniform_field((om.E, 8, 8, 8), seed, dtype, -3.0, 3.0)
        b = inputs.uniform_field((om.E, 8, 8, 8), seed + 50, dtype)
        ad = [torch.from_numpy(np.ascontiguousarray(x)).to("cuda", tdt) for x in slabs(a, 4)]
        bd = [torch.from_numpy(np.ascontiguousarray(x)).to("cuda", tdt) for x in slabs(b, 4)]
        assert grp.glsc3(ad, bd) == ora.glsc3(a, b, c)
    grp.close()


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("P,args", [(P, a) for P in (2, 4) for a in
                                    [(2, 2, 4, 8, 0.0, 0, 1001), (3, 3, 4, 10, 0.1, 2005, 1005),
                                     (2, 2, 8, 12, 0.1, 2003, 1003)]]
                         + [(8, (2, 2, 8, 12, 0.1, 2003, 1003)), (8, (2, 3, 8, 8, 0.0, 0, 1004))])
def test_group_cg_bitwise_vs_oracle(nbk, ora, precision, P, args):
    grp, om, D, s = make_group(nbk, ora, args, P)
    niter = 60
    hist, trace, res = grp.cg_solve(niter, precision)
    ref = ora.cg(om, D, s["G"], s["f"], niter, precision)
    assert bits_equal(hist, ref.hist)
    assert bits_equal(trace, ref.trace)
    assert bits_equal(grp.solution(), ref.x.astype(np.float64))
    tr, _ = ora.true_residual(om, D, s["G"], s["f"], ref.x.astype(np.float64))
    assert res["true_res"] == pytest.approx(tr, rel=1e-12, abs=1e-300)
    assert res["defect_iter"] == 0
    grp.close()


def test_group_independent_setup_equals_one_rank(nbk, ora):
    """Each slab's own set-up (geometry with global vertex ids, RHS with global
    node ids) equals the matching slice of the 1-rank set-up, and a P=4 solve
    from it equals the 1-rank solve bit for bit."""
    args = (3, 2, 8, 8, 0.1, 12, 13)
    spec = nbk.MeshSpec(*args)
    one = nbk.cg_setup(spec, "fp32")
    D1, G1, f1 = one.get_arrays()
    grp = nbk.Group(spec, 4, "fp32")
    for r, c in enumerate(grp.ctxs):
        Dr, Gr, fr = c.get_arrays()
        assert bits_equal(Dr, D1)
        assert bits_equal(Gr, slabs(G1, 4)[r]) and bits_equal(fr, slabs(f1, 4)[r])
        info = c.info
        assert info["e_offset"] == r * spec.E // 4 and info["face_layer"] == 3 * 2 * 64
    for prec in ("fp32", "fp64"):
        h1, t1, r1 = one.cg_solve(40, prec)
        h4, t4, r4 = grp.cg_solve(40, prec)
        assert bits_equal(h1, h4) and bits_equal(t1, t4)
        assert bits_equal(one.solution(), grp.solution())
        assert r1["true_res"] == r4["true_res"] and r1["true_res_rel"] == r4["true_res_rel"]
    one.close()
    grp.close()


def test_group_misuse_is_rejected(nbk, ora):
    spec = nbk.MeshSpec(2, 2, 4, 4)
    grp = nbk.Group(spec, 2, "fp64")
    c0 = grp.ctxs[0]
    with pytest.raises(nbk.NbkError):
        c0.cg_solve(5, "fp64")       # a virtual-slab member needs the group calls
    with pytest.raises(nbk.NbkError):
        nbk.cg_setup(nbk.MeshSpec(2, 2, 3, 4), "fp64", rank=0, nranks=2)  # ez % P != 0
    grp.close()


@pytest.mark.parametrize("cfg,P", [("C4", 2), ("C4", 4), ("C5", 2)])
def test_full_size_virtual_slabs_equal_one_rank(nbk, cfg, P):
    """BASELINE's multi-GPU configurations at full size on one GPU: the global
    problem of C4 at P GPUs (weak: 64x64x32P) and of C5 (strong: 64^3, N = 10)
    solved by one rank and by P virtual slabs, each slab with its own set-up --
    residual history, trace, true residual and solution bit for bit equal."""
    import hashlib
    c = nbk.CONFIGS[cfg]
    spec = nbk.MeshSpec(**c.mesh_args(P))
    niter = 20
    one = nbk.cg_setup(spec, "fp32")
    ref = {}
    for prec in ("fp32", "fp64"):
        h, t, r = one.cg_solve(niter, prec)
        ref[prec] = (h, t, r["true_res"], hashlib.sha256(one.solution().tobytes()).hexdigest())
    one.close()
    del one
    torch.cuda.empty_cache()
    grp = nbk.Group(spec, P, "fp32")
    for prec in ("fp32", "fp64"):
        h, t, r = grp.cg_solve(niter, prec)
        h1, t1, tr1, x1 = ref[prec]
        assert bits_equal(h, h1) and bits_equal(t, t1)
        assert r["true_res"] == tr1
        assert hashlib.sha256(grp.solution().tobytes()).hexdigest() == x1
    grp.close()
    torch.cuda.empty_cache()
