"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the library on C1 (2x2x2, N=8) and a 4^3
jittered N=10 mesh -- FP32 / FP64 / exactly rounded binary32 / binary32-
accumulating solves, Jacobi PCG, VPREC / RR emulation, virtual slabs (P = 2),
the public ax_apply / dssum / glsc3 and the host transfers.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2405_11065_b200 as nbk  # noqa: E402

torch.cuda.set_device(0)
for args in [(2, 2, 2, 8, 0.0, 0, 1001), (4, 4, 4, 10, 0.1, 2005, 1005)]:
    ctx = nbk.cg_setup(nbk.MeshSpec(*args), "fp32")
    for prec in ("fp32", "fp64", "fp32s", "fp32a"):
        h, _, r = ctx.cg_solve(12, prec)
        print(args, prec, h[-1] / h[0], r["true_res_rel"], flush=True)
    x = ctx.solution()
    ctx.set_precond("jacobi")
    for prec in ("fp32", "fp64"):
        h, _, r = ctx.cg_solve(8, prec)
        print(args, "jacobi", prec, h[-1] / h[0], flush=True)
    ctx.set_precond("none")
    if args[3] <= 8:
        ctx.set_emulation("vprec", 23, 0)
        ctx.cg_solve(5, "vprec")
        ctx.set_emulation("rr", 23, 3)
        ctx.cg_solve(5, "vprec")
    for dt in (torch.float32, torch.float64):
        u = torch.rand(ctx.shape, dtype=dt, device="cuda")
        w = torch.empty_like(u)
        ctx.ax_apply(u, w, nbk.AX_DSSUM | nbk.AX_MASK)
        ctx.dssum(w, apply_mask=True)
        g = ctx.glsc3(u, w)
        ctx.sync()
        print(args, dt, g, flush=True)
    hh, _ = ctx.cg_solve_host(x * 0.5, 6, "fp32", x)
    ctx.close()
grp = nbk.Group(nbk.MeshSpec(2, 2, 4, 6, 0.1, 3, 4), 2, "fp32")
for prec in ("fp32", "fp64", "fp32a"):
    h, _, _ = grp.cg_solve(10, prec)
    print("group", prec, h[-1] / h[0], flush=True)
us = [torch.rand(c.shape, dtype=torch.float64, device="cuda") for c in grp.ctxs]
ws = [torch.empty_like(u) for u in us]
grp.ax_apply(us, ws)
grp.sync()
grp.close()
torch.cuda.synchronize()
print("sanitize workload done")
