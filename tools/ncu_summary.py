"""Summarise ncu reports / launch lists into profiles/ (tracked).

    python tools/ncu_summary.py --round r01 \
        --rep C4:fp32:gpurun_out/prof_kax_c4.ncu-rep ... \
        --launches C2:gpurun_out/launches_c2c.csv

Writes profiles/<round>_ncu.md (human-readable) and merges per-launch DRAM
traffic of the fused ax kernel into profiles/ncu_summary.json (read by bench.py
for roofline.traffic).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_table import table  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_shared_mem", "CTA/SM limit (smem)"),
    ("launch__occupancy_limit_registers", "CTA/SM limit (regs)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw_rows(rep):
    """Header, units and rows of an ncu raw page: from a .ncu-rep (via ncu -i)
    or from the CSV `ncu -i REP --page raw --csv` wrote on the GPU box."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def stalls(h, r, top=5):
    out = []
    for i, w in enumerate(h):
        if w.startswith("smsp__pcsamp_warps_issue_stalled") and not w.endswith("not_issued"):
            try:
                out.append((float(r[i].replace(",", "")), w[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in out) or 1.0
    return [(w, v / tot) for v, w in sorted(out, reverse=True)[:top]]


def kernel_key(name):
    """Summary key of a CG-loop kernel: K_A k_ax<T, N, 1, 0>, K_B k_dssum<T, 1, 0>,
    K_C k_vec<T, V, 1, 0> (RUPD); None for the others."""
    if "k_ax<" in name and name.replace(" ", "").split(">(")[0].endswith(",1,0"):
        return "k_ax_fused"
    if "k_axl<" in name and name.replace(" ", "").replace("(int)", "").split(">(")[0].endswith(",1"):
        return "k_ax_fused"   # the line-owner K_A (nbk_axl.cuh)
    if "k_dssum<" in name and ", 1, 0>" in name:
        return "k_dssum_fused"
    if "k_vec<" in name and name.replace(" ", "").split(">(")[0].endswith(",1,0"):
        return "k_vec_rupd"
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--rep", action="append", default=[], help="CFG:PREC:path.ncu-rep")
    ap.add_argument("--launches", action="append", default=[], help="CFG:path.csv")
    ap.add_argument("--note", default="")
    ap.add_argument("--fresh", action="store_true", help="overwrite profiles/<round>_ncu.md")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    md = [f"# ncu summaries, round {a.round}", ""]
    if a.note:
        md += [a.note, ""]
    js_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    js = json.load(open(js_path)) if os.path.exists(js_path) else {}
    for spec in a.rep:
        cfg, prec, path = spec.split(":", 2)
        h, units, rows = raw_rows(path)
        md += [f"## {cfg} {prec}: `{os.path.basename(path)}` (`ncu --set full --clock-control none`)", ""]
        for r in rows:
            name = r[h.index("Kernel Name")]
            md += [f"### `{name}`", "", "| metric | value |", "|---|---|"]
            vals = {}
            for m, label in METRICS:
                if m in h:
                    v = r[h.index(m)]
                    vals[m] = v
                    md.append(f"| {label} (`{m}`) | {v} {units[h.index(m)]} |")
            md.append("| top stalls | " + ", ".join(f"{w} {100 * f:.0f}%" for w, f in stalls(h, r)) + " |")
            md.append("")
            key = kernel_key(name)
            if key:
                def b(m):
                    u = units[h.index(m)]
                    x = float(vals[m].replace(",", ""))
                    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

                def us(m):
                    u = units[h.index(m)]
                    x = float(vals[m].replace(",", ""))
                    return x * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3,
                             "second": 1e6, "s": 1e6}.get(u, 1)
                js.setdefault(cfg, {}).setdefault(prec, {})[key] = {
                    "dram_bytes_per_launch": b("dram__bytes_read.sum") + b("dram__bytes_write.sum"),
                    "dram_read_bytes": b("dram__bytes_read.sum"),
                    "dram_write_bytes": b("dram__bytes_write.sum"),
                    "duration_us": us("gpu__time_duration.sum"),
                    "source": os.path.basename(path), "round": a.round}
    for spec in a.launches:
        cfg, path = spec.split(":", 1)
        md += [f"## {cfg}: launch list `{os.path.basename(path)}` "
               "(`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
               "--clock-control none`; cold-cache, serialised: compare shares)", "",
               "| launches | mean time | DRAM read | DRAM write | kernel |", "|---|---|---|---|---|"]
        agg = table(path)
        tot = sum(v[1] for v in agg.values())
        for n, v in agg.items():
            c = v[0]
            md.append(f"| {c} | {v[1] / c / 1e3:.2f} us ({100 * v[1] / tot:.1f}% of listed) | "
                      f"{v[2] / c / 1e6:.2f} MB | {v[3] / c / 1e6:.2f} MB | `{n}` |")
        md.append("")
    with open(os.path.join(ROOT, "profiles", f"{a.round}_ncu.md"), "w" if a.fresh else "a") as fh:
        fh.write("\n".join(md) + "\n")
    with open(js_path, "w") as fh:
        json.dump(js, fh, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
