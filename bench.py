#!/usr/bin/env python
"""Benchmark of the B200-native Nekbone CG hot path (arXiv 2405.11065).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl nbk|reference]

A "step" is one complete fixed-iteration CG solve (all SURVEY 8(a) rows a1-a8:
the fused p/x update + ax_e + mask, dssum, glsc3 reductions, r update, device
scalars, and the final FP64 residual check) by the mixed FP32 solver, replayed
as one CUDA graph with all inputs resident in HBM.  Default workload: C5, the
largest single-GPU configuration of BASELINE.json (64^3 hex elements, N = 10,
jittered, 200 iterations; 262 M local points, working set far above the L2).
The FP64 solver is timed the same way and reported beside it; C2-C4 are
measured briefly under `other_configs`.

--gpus N (N > 1) without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU, NCCL z-slabs).

metric = GDOF*iter/s = n_global * niter / step time (DOF = unique global GLL
nodes, reading R19).  Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CG GDOF·iter/s FP64 vs FP32 solver; ax/CG-vector HBM GB/s vs B200 peak"
UNIT = "GDOF*iter/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--impl", default="nbk", choices=["nbk", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp64", action="store_true")
    ap.add_argument("--no-accuracy", dest="accuracy", action="store_false",
                    help="skip the FP32 / paper-literal single accuracy report")
    ap.add_argument("--no-precision-study", dest="precision_study", action="store_false",
                    help="skip the VPREC sweep / MCA ensembles (NEXT-4) on C1")
    ap.add_argument("--convergence", type=int, default=4000,
                    help="iterations of the long convergence / true-residual-floor study, run on "
                         "C2 (0: skip)")
    ap.add_argument("--prof-steps", type=int, default=3,
                    help="solves replayed with CUDA events between the kernels (per-kernel times)")
    ap.add_argument("--energy-reps", type=int, default=5,
                    help="energy-to-solution repeats per solver (mean and spread, P:693-698)")
    ap.add_argument("--no-jacobi", dest="jacobi", action="store_false",
                    help="skip the Jacobi-PCG measurement beside the headline")
    ap.add_argument("--others", default="C2,C3,C4",
                    help="other configs measured briefly after the headline (1 GPU; '' = none)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


class Energy:
    """GPU energy (NVML total-energy counter, mJ) over a region (SURVEY 8(f) NEXT-3:
    energy-to-solution, the paper's third axis)."""

    def __init__(self, device_index: int):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(device_index)
        except Exception:
            self.nv = None
        self.joules = None

    def __enter__(self):
        self.e0 = self._read()
        return self

    def _read(self):
        try:
            return self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h) if self.nv else None
        except Exception:
            return None

    def __exit__(self, *a):
        e1 = self._read()
        if self.e0 is not None and e1 is not None:
            self.joules = (e1 - self.e0) / 1e3


def max_over_ranks(value: float, world: int, device="cuda") -> float:
    """Max of a per-rank number over all ranks (timings: the slowest rank)."""
    if world <= 1:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_entry(cfg_name, precision, kernel):
    """Per-launch ncu numbers of one kernel (K_A 'k_ax_fused', K_B 'k_dssum_fused',
    K_C 'k_vec_rupd') from the committed summary (profiles/ncu_summary.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d[cfg_name][precision][kernel]
    except Exception:
        return None


def ncu_traffic(cfg_name, precision, kernel="k_ax_fused"):
    e = ncu_entry(cfg_name, precision, kernel)
    return None if e is None else e["dram_bytes_per_launch"]


# ---------------------------------------------------------------- oracle
def sample_mesh_args(cfg, layers):
    """A bounded sample of a config for the CPU oracle: its first `layers`
    element layers in z as a Dirichlet box of their own (same N, element size,
    jitter and RHS generator; SplitMix64 indices of vertices and nodes are those
    of the full box for these layers)."""
    a = cfg.mesh_args(1)
    a["ez"] = min(a["ez"], layers)
    return a


def oracle_sample(cfg, precision, niter_sample, layers):
    """The oracle as it stands, timed on this host's cores on a bounded sample:
    FP64 set-up (untimed) and `niter_sample` CG iterations of the first `layers`
    element layers of the workload."""
    import oracle
    om = oracle.Mesh(**sample_mesh_args(cfg, layers))
    _, _, D = oracle.gll(cfg.N)
    s = oracle.setup(om)
    t0 = time.perf_counter()
    oracle.cg(om, D, s["G"], s["f"], niter_sample, precision)
    dt = time.perf_counter() - t0
    return om.sizes()["n_global"] * niter_sample / dt / 1e9, dt, om


def sample_layers(cfg):
    """Element layers of the oracle sample: about 1/16 of C3-C5, all of C1/C2."""
    return cfg.ez if cfg.ex * cfg.ey * cfg.ez <= 4096 else max(1, cfg.ez // 16)


def run_reference(args):
    """--impl reference: the CPU oracle (this tier's reference arm), timed as it
    stands on the host's cores; each step = 1 CG iteration (2 for small
    configs) of a bounded sample of the workload (sample_mesh_args)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2405_11065_b200.configs import CONFIGS
    import oracle
    cfg = CONFIGS[args.config]
    layers = sample_layers(cfg)
    iters = 20 if layers == cfg.ez else 1
    om = oracle.Mesh(**sample_mesh_args(cfg, layers))
    _, _, D = oracle.gll(cfg.N)
    s = oracle.setup(om)
    ng = om.sizes()["n_global"]
    for _ in range(args.warmup):
        oracle.cg(om, D, s["G"], s["f"], iters, args.precision)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.cg(om, D, s["G"], s["f"], iters, args.precision)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = ng * iters * args.steps / tot / 1e9
    cores = oracle.num_threads()
    sample = (f"{args.config} {args.precision} oracle CG on {om.ex}x{om.ey}x{om.ez} elements "
              f"(first {layers} of {cfg.ez} z-layers of the workload, N={cfg.N}, {ng} DOF), "
              f"{iters} of {cfg.niter} iterations per step (set-up untimed), OpenMP threads={cores}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak" if cfg.weak else "strong",
            "vs_baseline": None,
            "dtype": "f32" if args.precision == "fp32" else "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg, args.precision), "sample": sample,
                       "niter_per_step": iters},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_name(cfg, precision, world=1):
    solver = "mixed FP32 solver (FP64 set-up, FP64 glsc3 accumulation, FP64 final check)" \
        if precision == "fp32" else "FP64 solver"
    ez = cfg.mesh_args(world)["ez"]
    return (f"{cfg.name}: {cfg.ex}x{cfg.ey}x{ez} hex box, N={cfg.N} (p={cfg.N - 1}), "
            f"jitter={cfg.jitter}, {cfg.niter} unpreconditioned CG iterations, {solver}")


# ---------------------------------------------------------------- GPU arm
def time_solves(ctx, torch, cfg, precision, steps, warmup, flush, profile):
    """Per-step device time (CUDA events on the context stream), L2 flushed
    between steps (outside the events)."""
    import paper_2405_11065_b200 as nbk  # noqa: F401
    ctx.set_profiling(profile)
    for _ in range(warmup):
        ctx.cg_solve(cfg.niter, precision, trace=False)
    s = ctx.stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    kA, kBC = [], []
    ctx.sync()
    graph_ms = []
    for i in range(steps):
        flush.fill_(i & 0xFF)  # write 512 MiB > 126 MB L2, on the same stream
        ev[i][0].record(s)
        hist, _, res = ctx.cg_solve(cfg.niter, precision, trace=False)
        ev[i][1].record(s)
        kA.append(res["kA_ms"])
        kBC.append((res["kB_ms"], res["kC_ms"]))
        graph_ms.append(res["solve_ms"])
    ctx.sync()
    ms = [a.elapsed_time(b) for a, b in ev]
    time_solves.kBC = kBC
    return ms, kA, graph_ms, res, hist


def precision_study(nbk, torch, stream, niter=100, samples=20):
    """SURVEY 8(f) NEXT-4 on the GPU path (F4-F6), CG-loop scope, on
    the C1 mesh: VPREC sweep of the virtual precision t (final recursive and
    true residual), and `samples`-run Monte Carlo ensembles (rr and mca modes)
    at t = 23: per-iteration mean / min / max of the residual history and the
    significant bits s2 = -log2|sigma/mu|."""
    import numpy as np
    cfg = nbk.CONFIGS["C1"]
    ctx = nbk.cg_setup(nbk.MeshSpec(**cfg.mesh_args(1)), "fp64", stream=stream)
    h64, _, r64 = ctx.cg_solve(niter, "fp64", trace=False)
    out = {"workload": "C1 (2x2x2, N=8), %d iterations, unpreconditioned" % niter,
           "fp64": {"h_final_rel": float(h64[-1] / h64[0]), "true_res_rel": r64["true_res_rel"]}}
    t0 = time.perf_counter()
    sweep = {}
    for t in (3, 4, 6, 8, 10, 12, 16, 20, 23, 28, 36, 44, 52):
        ctx.set_emulation("vprec", t, 0)
        h, _, r = ctx.cg_solve(niter, "vprec", trace=False)
        sweep[t] = {"h_final_rel": float(h[-1] / h[0]), "true_res_rel": r["true_res_rel"]}
    out["vprec_sweep"] = sweep
    for mode in ("rr", "mca"):
        H = []
        for sd in range(samples):
            ctx.set_emulation(mode, 23, 1000 + sd)
            h, _, _ = ctx.cg_solve(niter, "vprec", trace=False)
            H.append(h)
        H = np.array(H)
        mu, sg = H.mean(0), H.std(0)
        s2 = -np.log2(np.maximum(sg, 1e-300) / np.abs(mu))
        ks = [k for k in (1, 10, 25, 50, 75, niter) if k <= niter]
        out[mode] = {"t": 23, "samples": samples,
                     "rel_spread_at": {k: float((H[:, k].max() - H[:, k].min()) / abs(mu[k])) for k in ks},
                     "s2_at": {k: float(s2[k]) for k in ks},
                     "mean_over_fp64_at": {k: float(mu[k] / h64[k]) for k in ks}}
    out["seconds"] = time.perf_counter() - t0
    ctx.close()
    return out


def convergence_study(ctx, niter_max):
    """Convergence beyond the fixed iteration count (NEXT-2: true-residual floor
    and iterations to 1e-10 of each solver): recursive h_k/h_0 of one long solve,
    FP64 true residual (C12) of the returned x after several lengths."""
    import numpy as np
    conv = {"niter_max": niter_max}
    for p_ in ("fp64", "fp32", "fp32s", "fp32a"):
        hh, _, rr = ctx.cg_solve(niter_max, p_, trace=False)
        rel = hh / hh[0] if hh[0] else hh
        it_to = {}
        for thr in (1e-4, 1e-6, 1e-8, 1e-10, 1e-12):
            idx = np.nonzero(rel <= thr)[0]
            it_to[f"{thr:.0e}"] = int(idx[0]) if len(idx) else None
        tr_at = {}
        for nit in sorted({n_ for n_ in (250, 500, 1000, 2000) if n_ < niter_max}):
            _, _, r2 = ctx.cg_solve(nit, p_, trace=False)
            tr_at[str(nit)] = r2["true_res_rel"]
        tr_at[str(niter_max)] = rr["true_res_rel"]
        conv[p_] = {"iters_to_recursive_rel": it_to, "recursive_rel_final": float(rel[-1]),
                    "true_res_rel_after": tr_at, "defect_iter": rr["defect_iter"]}
    return conv


def measure_other(nbk, torch, name, flush, stream, peak, steps=3, warmup=2, convergence=0):
    """Short measurement of another BASELINE config on 1 GPU (not the headline):
    FP32 and FP64 solver GDOF*iter/s, K_A roofline fraction, FP32/FP64 ratio."""
    cfg = nbk.CONFIGS[name]
    ctx = nbk.cg_setup(nbk.MeshSpec(**cfg.mesh_args(1)), "fp32", stream=stream)
    out = {"workload": workload_name(cfg, "fp32"), "n_global": ctx.n_global, "steps": steps}
    n = ctx.n_local
    with torch.cuda.stream(stream):
        for prec, s_b in (("fp32", 4), ("fp64", 8)):
            ms, _, _, res, _ = time_solves(ctx, torch, cfg, prec, steps, warmup, flush, profile=False)
            _, kA, _, _, _ = time_solves(ctx, torch, cfg, prec, 1, 1, flush, profile=True)
            ka = sum(kA) / cfg.niter
            out[prec] = {"value": ctx.n_global * cfg.niter * steps / (sum(ms) / 1e3) / 1e9,
                         "ms_per_step": sum(ms) / steps,
                         "k_ax_hbm_frac": 12 * s_b * n / (ka / 1e3) / 1e9 / peak,
                         "true_res_rel": res["true_res_rel"]}
        if convergence:
            out["convergence"] = convergence_study(ctx, convergence)
    out["speedup_fp32_vs_fp64"] = out["fp32"]["value"] / out["fp64"]["value"]
    ctx.close()
    return out


def kernel_times(torch, ctx, cfg, prec, steps, flush):
    """Per-kernel device times from a replay with CUDA events between the
    kernels of every iteration (events disable the PDL overlap)."""
    ms, kA, _, _, _ = time_solves(ctx, torch, cfg, prec, steps, 1, flush, profile=True)
    kB = sum(x[0] for x in time_solves.kBC)
    kC = sum(x[1] for x in time_solves.kBC)
    it = steps * cfg.niter
    return {"K_A_ms": sum(kA) / it, "K_B_ms": kB / it, "K_C_ms": kC / it,
            "share_K_A": sum(kA) / sum(ms)}


def kernel_report(kt, n, ng, s_b, phi, psi, peak, cfg_name, prec):
    """Algorithmic GB/s and HBM fractions of K_A / K_B / K_C (SURVEY 8(d) bytes
    per local point: 12s, phi(2s+4) + psi(s+4), 3s) plus the ncu DRAM bytes of
    the committed capture of the same kernels."""
    alg = {"K_A": 12 * s_b * n, "K_B": n * (phi * (2 * s_b + 4) + psi * (s_b + 4)), "K_C": 3 * s_b * n}
    names = {"K_A": "k_ax_fused", "K_B": "k_dssum_fused", "K_C": "k_vec_rupd"}
    out = {}
    for k in ("K_A", "K_B", "K_C"):
        t = kt[k + "_ms"] / 1e3
        e = ncu_entry(cfg_name, prec, names[k])
        out[k] = {"ms": kt[k + "_ms"], "alg_bytes": alg[k], "alg_GBps": alg[k] / t / 1e9,
                  "frac": alg[k] / t / 1e9 / peak,
                  "ncu_dram_bytes": None if e is None else e["dram_bytes_per_launch"],
                  "ncu_dram_over_alg": None if e is None else e["dram_bytes_per_launch"] / alg[k],
                  "ncu_duration_us": None if e is None else e.get("duration_us")}
    dram = [out[k]["ncu_dram_bytes"] for k in ("K_A", "K_B", "K_C")]
    out["ncu_dram_bytes_per_global_dof_iter"] = None if None in dram else sum(dram) / ng
    out["timing"] = ("CUDA events between the kernels of every iteration (profiling replay); "
                     "ncu numbers: cold-cache --set full capture of one steady-state launch")
    return out


def maybe_relaunch(args):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run (one
    rank per GPU, 127.0.0.1 rendezvous) and return its exit code."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import subprocess
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_gpu(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import paper_2405_11065_b200 as nbk
    cfg = nbk.CONFIGS[args.config]
    # z-slabs over the ranks: weak configs grow the box with N
    spec = nbk.MeshSpec(**cfg.mesh_args(world))
    stream = torch.cuda.Stream()
    nccl_id = None
    if world > 1:
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(nbk.nccl_unique_id()), dtype=torch.uint8))
        torch.distributed.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy())
    t_setup = time.perf_counter()
    ctx = nbk.cg_setup(spec, "fp32", device=local, stream=stream, rank=rank, nranks=world,
                       nccl_id=nccl_id)
    t_setup = time.perf_counter() - t_setup
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    prec = args.precision

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- timed region (headline precision; plain graph, PDL edges on) ----
    barrier()
    with torch.cuda.stream(stream), ClockSampler(local) as clk:
        ms, _, graph_ms, res, hist = time_solves(ctx, torch, cfg, prec, args.steps, args.warmup,
                                                 flush, profile=False)
        ctx.sync()
    barrier()
    tot_ms = max_over_ranks(sum(ms), world)
    ng = ctx.n_global  # global unique nodes of the whole (all-rank) box
    value = ng * cfg.niter * args.steps / (tot_ms / 1e3) / 1e9
    launches = ctx.solve_launches(cfg.niter, prec) * args.steps
    n = ctx.n_local
    info0 = ctx.info
    phi0, psi0 = info0["n_copies"] / n, info0["n_shared"] / n
    peak, peak_src = measured_peak()
    s_b = 4 if prec == "fp32" else 8

    # ---- per-kernel times (replay with events between the kernels) ----
    with torch.cuda.stream(stream):
        kt = kernel_times(torch, ctx, cfg, prec, args.prof_steps, flush)
    barrier()
    kernels = kernel_report(kt, n, ng, s_b, phi0, psi0, peak, args.config, prec)

    # ---- roofline of the dominant kernel (fused ax, K_A) ----
    bytes_ka = 12 * s_b * n  # reads r, p, x, G (9s) + writes p, x, w (3s) per local point
    ka_avg_ms = kt["K_A_ms"]
    achieved = bytes_ka / (ka_avg_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(args.config, prec),
                "kernel": "k_axl<fused> (line-owner K_A: p,x update + ax_e + mask + interior pap)",
                "algorithmic_bytes_per_launch": bytes_ka, "avg_launch_ms": ka_avg_ms,
                "share_of_step": kt["share_K_A"],
                "ncu_share_of_iteration": None,
                "timing": f"CUDA events on the context stream around each K_A launch, in a "
                          f"replay of {args.prof_steps} solves (events disable the PDL overlap)",
                "traffic_source": "profiles/ncu_summary.json (ncu --set full, same config)",
                "peak_source": peak_src}
    eA, eB, eC = (ncu_entry(args.config, prec, k) for k in ("k_ax_fused", "k_dssum_fused", "k_vec_rupd"))
    if eA and eB and eC and all(e.get("duration_us") for e in (eA, eB, eC)):
        roofline["ncu_share_of_iteration"] = eA["duration_us"] / (
            eA["duration_us"] + eB["duration_us"] + eC["duration_us"])
        roofline["events_share_of_iteration"] = kt["K_A_ms"] / (kt["K_A_ms"] + kt["K_B_ms"] + kt["K_C_ms"])

    # ---- FP64 solver beside it ----
    extra = {}
    if not args.no_fp64 and prec == "fp32":
        barrier()
        with torch.cuda.stream(stream):
            ms64, _, _, res64, _ = time_solves(ctx, torch, cfg, "fp64", args.steps,
                                               args.warmup, flush, profile=False)
            ctx.sync()
            kt64 = kernel_times(torch, ctx, cfg, "fp64", args.prof_steps, flush)
        barrier()
        v64 = ng * cfg.niter * args.steps / (max_over_ranks(sum(ms64), world) / 1e3) / 1e9
        ka64 = kt64["K_A_ms"]
        k64 = kernel_report(kt64, n, ng, 8, phi0, psi0, peak, args.config, "fp64")
        extra["fp64"] = {"value": v64, "ms_per_step": sum(ms64) / args.steps,
                         "median_step_ms": statistics.median(ms64),
                         "k_ax_avg_ms": ka64,
                         "k_ax_hbm_frac": 12 * 8 * n / (ka64 / 1e3) / 1e9 / peak,
                         "kernels": k64, "true_res_rel": res64["true_res_rel"]}
        extra["speedup_fp32_vs_fp64"] = value / v64
        d32 = kernels["ncu_dram_bytes_per_global_dof_iter"]
        d64 = k64["ncu_dram_bytes_per_global_dof_iter"]
        extra["bytes_per_dof_ncu"] = {"fp32": d32, "fp64": d64,
                                      "ratio_fp32_over_fp64": d32 / d64 if d32 and d64 else None,
                                      "note": "sum of K_A+K_B+K_C ncu DRAM bytes per launch / n_global"}
        # energy-to-solution: NVML total-energy counter over back-to-back
        # solves; `energy_reps` windows per solver, mean and standard deviation
        en = {}
        with torch.cuda.stream(stream):
            for p_ in ("fp32", "fp64"):
                ctx.cg_solve(cfg.niter, p_, trace=False)
                ctx.sync()
                per = []
                # several ranks: every rank must enqueue the same number of (collective) solves,
                # so the count comes from the rank-agreed step time, not from each rank's clock
                nfix = 0
                if world > 1:
                    step_ms = (tot_ms if p_ == "fp32" else max_over_ranks(sum(ms64), world)) / args.steps
                    nfix = max(2, int(1500.0 / step_ms) + 1)
                for _ in range(args.energy_reps):
                    nsol, t0 = 0, time.perf_counter()
                    with Energy(local) as eg:
                        while (nsol < nfix) if nfix else (time.perf_counter() - t0 < 1.5 or nsol < 2):
                            ctx.cg_solve(cfg.niter, p_, trace=False)
                            nsol += 1
                        ctx.sync()
                        dt = time.perf_counter() - t0
                    if eg.joules:
                        per.append((eg.joules / nsol, eg.joules / dt, nsol))
                if per:
                    j = [x[0] for x in per]
                    en[p_] = {"J_per_solve_mean": statistics.mean(j),
                              "J_per_solve_stdev": statistics.stdev(j) if len(j) > 1 else 0.0,
                              "avg_W_mean": statistics.mean(x[1] for x in per),
                              "windows": len(per), "solves_per_window": [x[2] for x in per]}
        if "fp32" in en and "fp64" in en:
            extra["energy"] = {**en, "fp64_over_fp32": en["fp64"]["J_per_solve_mean"] /
                               en["fp32"]["J_per_solve_mean"],
                               "energy_saving_fp32": 1 - en["fp32"]["J_per_solve_mean"] /
                               en["fp64"]["J_per_solve_mean"],
                               "note": "NVML total-energy counter, >= 1.5 s windows of back-to-back "
                                       "solves (incl. the FP64 final check), mean / stdev over "
                                       "windows (the paper: mean of 5 runs, P:693-698)"}

    # ---- accuracy of the single-precision solvers vs FP64 (P:517-522 AE / MAE; NEXT-2) ----
    if args.accuracy and world == 1:
        import numpy as np
        with torch.cuda.stream(stream):
            h, xs, rs = {}, {}, {}
            for p_ in ("fp64", "fp32", "fp32s", "fp32a"):
                h[p_], _, rs[p_] = ctx.cg_solve(cfg.niter, p_, trace=False)
                xs[p_] = ctx.solution()
            ms1, _, _, _, _ = time_solves(ctx, torch, cfg, "fp32s", min(args.steps, 3), 1, flush,
                                          profile=False)
            msa, _, _, _, _ = time_solves(ctx, torch, cfg, "fp32a", min(args.steps, 3), 1, flush,
                                          profile=False)
        acc = {}
        for p_ in ("fp32", "fp32s", "fp32a"):
            ae = np.abs(h[p_][1:] - h["fp64"][1:])
            acc[p_] = {"MAE": float(ae.mean()), "AE_max": float(ae.max()),
                       "MAE_rel_h0": float(ae.mean() / h["fp64"][0]),
                       "true_res_rel": rs[p_]["true_res_rel"],
                       "x_err_vs_fp64": float(np.abs(xs[p_] - xs["fp64"]).max() /
                                              np.abs(xs["fp64"]).max())}
        acc["fp64_true_res_rel"] = rs["fp64"]["true_res_rel"]
        acc["fp32s_value"] = ng * cfg.niter * len(ms1) / (sum(ms1) / 1e3) / 1e9
        acc["fp32a_value"] = ng * cfg.niter * len(msa) / (sum(msa) / 1e3) / 1e9
        acc["note"] = ("fp32: north_star mixed solver (FP64 inner-product accumulation); fp32s: "
                       "exactly rounded binary32 inner products and binary32 scalars (R11b); "
                       "fp32a: the paper's single-precision solver, inner products accumulated "
                       "in binary32 (R11c, P:42, P:507, P:510); AE/MAE vs the FP64 solver (P:519-522)")
        extra["accuracy"] = acc
        del xs

    # ---- Jacobi PCG beside it: same workload, z = r / diag(A) ----
    if args.jacobi:
        barrier()
        jac = {}
        with torch.cuda.stream(stream):
            ctx.set_precond("jacobi")
            for p_ in ("fp32", "fp64"):
                msj, _, _, resj, histj = time_solves(ctx, torch, cfg, p_, min(args.steps, 3), 1,
                                                     flush, profile=False)
                jac[p_] = {"value": ng * cfg.niter * len(msj) /
                           (max_over_ranks(sum(msj), world) / 1e3) / 1e9,
                           "ms_per_step": sum(msj) / len(msj),
                           "h_final_rel": float(histj[-1] / histj[0]) if histj[0] else 0.0,
                           "true_res_rel": resj["true_res_rel"]}
            ctx.set_precond("none")
        barrier()
        extra["jacobi_pcg"] = jac

    # ---- end to end through the C ABI with host buffers ----
    f_host = torch.empty(ctx.shape, dtype=torch.float64).pin_memory()
    _, _, f0 = ctx.get_arrays(G=False)
    f_host.numpy()[...] = f0
    del f0
    x_host = torch.empty(ctx.shape, dtype=torch.float64).pin_memory()
    ctx.set_profiling(False)
    for _ in range(min(args.warmup, 2)):
        ctx.cg_solve_host(f_host.numpy(), cfg.niter, prec, x_host.numpy())
    e2e_ms = []
    barrier()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.cg_solve_host(f_host.numpy(), cfg.niter, prec, x_host.numpy())
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    e2e_single = ng * cfg.niter * args.steps / (max_over_ranks(sum(e2e_ms), world) / 1e3) / 1e9
    # batched form (the call a user makes for several right-hand sides): one call over `steps`
    # RHS, each step's H2D copy and D2H copy inside the timed region, overlapped with the
    # neighbouring solves on the library's copy streams
    # (one pinned f and one pinned x buffer serve every step: each step still copies its
    # 8n bytes in and out; the D2H copies run in order, so reusing x is safe)
    f_list = [f_host.numpy()] * args.steps
    x_list = [x_host.numpy()] * args.steps
    ctx.cg_solve_host_batch(f_list[:min(2, args.steps)], cfg.niter, prec, x_list[:min(2, args.steps)])
    barrier()
    flush.fill_(0x5A)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    ctx.cg_solve_host_batch(f_list, cfg.niter, prec, x_list)
    b.record(stream)
    b.synchronize()
    batch_ms = a.elapsed_time(b)
    e2e_val = ng * cfg.niter * args.steps / (max_over_ranks(batch_ms, world) / 1e3) / 1e9
    e2e = {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 8 * n,
           "d2h_bytes_per_step": 8 * n + 8 * (cfg.niter + 1),
           "path": f"nbk_cg_solve_host_batch over {args.steps} right-hand sides (pinned host f_k -> "
                   "solve -> host x_k per step; the copies of RHS k+1 and solution k-1 overlap solve k), "
                   "CUDA events on the context stream around the call",
           "single_call_value": e2e_single,
           "single_call_path": "nbk_cg_solve_host per step (copy in, solve, copy out, serialised)"}
    del f_host, x_host, f_list, x_list

    # ---- CPU baseline: the oracle on this host, bounded sample ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        layers = sample_layers(cfg)
        iters = 40 if layers == cfg.ez else 2
        v_cpu, dt, om = oracle_sample(cfg, prec, iters, layers)
        cpu = {"value": v_cpu, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
               "sample": f"{args.config} {prec} oracle CG on {om.ex}x{om.ey}x{om.ez} elements "
                         f"(first {layers} of {cfg.ez} z-layers of the workload), {iters} of "
                         f"{cfg.niter} iterations ({dt:.1f} s; set-up untimed)"}

    # whole-iteration algorithmic bandwidth (SURVEY 8(d) B_fused model)
    b_fused = 15 * s_b + phi0 * (2 * s_b + 4) + psi0 * (s_b + 4)
    t_iter = tot_ms / args.steps / cfg.niter / 1e3
    b_fused64 = 15 * 8 + phi0 * (2 * 8 + 4) + psi0 * (8 + 4)
    model = {"B_fused_bytes_per_local_point": b_fused,
             "bytes_per_global_dof": b_fused * n / ng,
             "bytes_per_global_dof_fp64_solver": b_fused64 * n / ng,
             "bytes_per_dof_ratio_fp32_over_fp64": b_fused / b_fused64 if prec == "fp32" else 1.0,
             "iteration_GBps": b_fused * n / t_iter / 1e9,
             "iteration_hbm_frac": b_fused * n / t_iter / 1e9 / peak}

    precision = None
    if world == 1 and args.precision_study:
        precision = precision_study(nbk, torch, stream)

    others = {}
    if world == 1 and args.others:
        ctx.close()
        del ctx
        torch.cuda.empty_cache()
        for name in args.others.split(","):
            others[name] = measure_other(nbk, torch, name, flush, stream, peak,
                                         convergence=args.convergence if name == "C2" else 0)
            torch.cuda.empty_cache()

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if cfg.weak else "strong", "vs_baseline": None,
            "dtype": "f32" if prec == "fp32" else "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg, prec, world), "n_global": ng, "n_local": n,
                       "niter": cfg.niter,
                       "parallelism": "1 GPU" if world == 1 else
                       f"{world} z-slabs (NCCL face exchange + all-gather)",
                       "l2": "flushed between steps (512 MiB write, outside the events); the "
                             "per-iteration working set is far above the 126 MB L2"},
            "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clk.summary(), "true_res_rel": res["true_res_rel"],
            "h_final_rel": float(hist[-1] / hist[0]) if hist[0] else 0.0,
            "median_step_ms": statistics.median(ms), "setup_s": t_setup,
            "iteration_model": model, "kernels": kernels, **extra,
            "other_configs": others or None, "precision_tools": precision}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    rc = maybe_relaunch(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
