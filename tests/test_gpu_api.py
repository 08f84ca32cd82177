"""Boundary behaviour of the C ABI (include/nbk.h) that the parity suites do
not exercise: a NULL stream in nbk_dist, stream ordering of the Python
binding's asynchronous calls against torch's current stream, a loaded Jacobi
diagonal surviving a new RHS, and the emulation / Jacobi exclusion.
"""
import ctypes

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
    return a.dtype == b.dtype and a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_null_stream_context_solves(nbk, ora):
    """nbk_dist.stream == NULL: the context makes its own (blocking) stream,
    graph capture works, and the solve equals the oracle bit for bit."""
    from paper_2405_11065_b200 import nbk as B
    L = B.load()
    mesh = B.MeshSpec(2, 2, 2, 8, 0.0, 0, 1001)
    nbytes = B.workspace_bytes(mesh, "fp32")
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d = B.CDist(0, 1, 0, None, None)
    ctx = ctypes.c_void_p(None)
    B._check(L.nbk_cg_setup(ctypes.byref(mesh.c()), B.NBK_FP32, ctypes.byref(d),
                            ctypes.c_void_p(ws.data_ptr()), nbytes, ctypes.byref(ctx)))
    om = ora.Mesh(2, 2, 2, 8, 0.0, 0, 1001)
    _, _, D = ora.gll(8)
    s = ora.setup(om, want=("G", "f"))
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (D, s["G"], s["f"])]
    B._check(L.nbk_load_arrays(ctx, *[B._ptr(a) for a in arrs]), ctx)
    hist = np.zeros(101)
    res = B.CResult()
    B._check(L.nbk_cg_solve(ctx, 100, B.NBK_FP32, B._ptr(hist), None, ctypes.byref(res)), ctx)
    ref = ora.cg(om, D, s["G"], s["f"], 100, "fp32")
    assert bits_equal(hist, ref.hist)
    # asynchronous ax_apply on the context's own stream, ordered with the legacy stream
    u = torch.from_numpy(inputs.uniform_field((8, 8, 8, 8), 3)).cuda()
    w = torch.empty_like(u)
    torch.cuda.synchronize()
    B._check(L.nbk_ax_apply(ctx, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                            B.AX_DSSUM | B.AX_MASK, B.NBK_FP64), ctx)
    torch.cuda.synchronize()
    assert bits_equal(w.cpu().numpy(), ora.ax(om, D, s["G"], u.cpu().numpy(), apply_mask=True))
    L.nbk_destroy(ctx)


def test_binding_orders_streams(nbk, ora):
    """Inputs produced on torch's current stream right before the call (no
    host sync) are read after they are final; the output is ordered before the
    caller's next kernels."""
    ctx = nbk.cg_setup(nbk.MeshSpec(3, 2, 2, 8, 0.0, 0, 7), "fp32")  # private stream
    om = ora.Mesh(3, 2, 2, 8, 0.0, 0, 7)
    _, _, D = ora.gll(8)
    s = ora.setup(om, want=("G",))
    ctx.load_arrays(D, s["G"], None)
    host = inputs.uniform_field((12, 8, 8, 8), 11)
    src = torch.from_numpy(host).cuda()
    big = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
    for _ in range(3):
        torch.cuda.synchronize()
        u = torch.zeros_like(src)
        big.uniform_()                 # keep the current stream busy ...
        big.mul_(1.0001)
        u.copy_(src)                   # ... so u is written late on it
        w = torch.zeros_like(u)
        ctx.ax_apply(u, w, nbk.AX_DSSUM | nbk.AX_MASK)
        out = w.clone()                # on the current stream, after the library
        torch.cuda.synchronize()
        assert bits_equal(out.cpu().numpy(), ora.ax(om, D, s["G"], host, apply_mask=True))
    ctx.close()


def test_new_rhs_keeps_loaded_dinv(nbk, ora):
    """nbk_cg_solve_host with a new f: the operator and a loaded Jacobi
    diagonal stay in use (only h0 is refreshed)."""
    ctx = nbk.cg_setup(nbk.MeshSpec(2, 2, 2, 6, 0.1, 3, 4), "fp32")
    om = ora.Mesh(2, 2, 2, 6, 0.1, 3, 4)
    _, _, D = ora.gll(6)
    s = ora.setup(om, want=("G", "f"))
    ctx.load_arrays(D, s["G"], s["f"])
    _, dinv = ora.jacobi_dinv(om, D, s["G"])
    dinv = dinv * 0.75  # not the assembled diagonal (and still continuous)
    ctx.load_precond(dinv)
    ctx.set_precond("jacobi")
    f2 = s["f"] * 0.5
    x = np.zeros(ctx.shape)
    hist, _ = ctx.cg_solve_host(f2, 40, "fp64", x)
    ref = ora.cg(om, D, s["G"], f2, 40, "fp64", dinv=dinv)
    assert bits_equal(hist, ref.hist)
    assert bits_equal(x, ref.x)
    assert bits_equal(ctx.get_precond(), dinv)
    ctx.close()


def test_emulation_with_jacobi_rejected(nbk):
    ctx = nbk.cg_setup(nbk.MeshSpec(2, 2, 2, 4, 0.0, 0, 1), "fp32")
    ctx.set_emulation("vprec", 23, 0)
    ctx.set_precond("jacobi")
    with pytest.raises(nbk.NbkError) as ei:
        ctx.cg_solve(10, "vprec")
    from paper_2405_11065_b200 import nbk as B
    assert ei.value.status == B.NBK_EINVAL
    ctx.set_precond("none")
    ctx.cg_solve(10, "vprec")
    ctx.close()


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_batch_host_solve_equals_oracle_per_rhs(nbk, ora, prec):
    """nbk_cg_solve_host_batch: three right-hand sides of one operator, the
    copies overlapped with the solves on the library's copy streams -- every
    history and solution bitwise the oracle's for its own RHS (and the same as
    nbk_cg_solve_host)."""
    ctx = nbk.cg_setup(nbk.MeshSpec(3, 2, 2, 6, 0.1, 5, 11), "fp32")
    om = ora.Mesh(3, 2, 2, 6, 0.1, 5, 11)
    _, _, D = ora.gll(6)
    s = ora.setup(om, want=("G", "f"))
    ctx.load_arrays(D, s["G"], s["f"])
    fs = [ora.setup(ora.Mesh(3, 2, 2, 6, 0.1, 5, seed), want=("f",))["f"] for seed in (11, 12, 13)]
    fh = [torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64)).pin_memory() for f in fs]
    xh = [torch.zeros(ctx.shape, dtype=torch.float64).pin_memory() for _ in fs]
    hist, res = ctx.cg_solve_host_batch([f.numpy() for f in fh], 30, prec, [x.numpy() for x in xh])
    assert hist.shape == (3, 31) and len(res) == 3
    for k, f in enumerate(fs):
        ref = ora.cg(om, D, s["G"], f, 30, prec)
        assert bits_equal(hist[k], ref.hist), k
        assert bits_equal(xh[k].numpy(), np.asarray(ref.x, dtype=np.float64)), k   # FP32 x: exact upcast
        x1 = np.zeros(ctx.shape)
        h1, _ = ctx.cg_solve_host(f, 30, prec, x1)
        assert bits_equal(h1, hist[k]) and bits_equal(x1, xh[k].numpy()), k
    ctx.close()
