"""Run a few solves of one config (for ncu / sanitizer runs on the GPU box).

    python tools/run_solve.py --config C2 --precision fp32 --reps 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2405_11065_b200 as nbk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--precision", default="fp32")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--niter", type=int, default=0)
a = ap.parse_args()
cfg = nbk.CONFIGS[a.config]
ctx = nbk.cg_setup(nbk.MeshSpec(**cfg.mesh_args()), "fp32")
niter = a.niter or cfg.niter
for prec in a.precision.split(","):
    for _ in range(a.reps):
        hist, _, res = ctx.cg_solve(niter, prec, trace=False)
        print(prec, f"h_final/h0={hist[-1] / hist[0]:.3e}", f"solve_ms={res['solve_ms']:.3f}",
              f"true_res_rel={res['true_res_rel']:.3e}", flush=True)
torch.cuda.synchronize()
