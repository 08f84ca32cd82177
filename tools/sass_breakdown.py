"""Summarise an ncu source-page SASS export (tools/gpu_kfull.sh): stall samples, executed
instructions and shared-memory wavefronts per opcode, and the top lines by samples.

    python tools/sass_breakdown.py gpurun_out/TAG/sass_C5_fp32.csv [raw.csv]
"""
import collections
import csv
import io
import sys

lines = open(sys.argv[1]).read().splitlines()
r = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = r[0]
ix = {k: i for i, k in enumerate(h)}
tot, ex, wf, wx = (collections.Counter() for _ in range(4))
seq = []
for x in r[1:]:
    if len(x) < len(h):
        continue
    op = x[ix["Source"]].strip().split()
    if not op:
        continue
    o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
    s = int(x[ix["Warp Stall Sampling (All Samples)"]] or 0)
    e = int(x[ix["Instructions Executed"]] or 0)
    w = int(x[ix["L1 Wavefronts Shared"]] or 0)
    we = int(x[ix["L1 Wavefronts Shared Excessive"]] or 0)
    tot[o] += s; ex[o] += e; wf[o] += w; wx[o] += we
    seq.append((x[ix["Address"]][-5:], x[ix["Source"]].strip()[:70], s, e, w, we))
S = sum(tot.values()) or 1
E = sum(ex.values()) or 1
print(f"samples {S}  warp instructions {E}  smem wavefronts {sum(wf.values())} (excess {sum(wx.values())})")
for o, s in tot.most_common(22):
    print(f"  {o:10s} samples {s / S * 100:5.1f}%  inst {ex[o] / E * 100:5.1f}% ({ex[o]})  wf {wf[o]} (excess {wx[o]})")
print("top lines:")
for i in sorted(sorted(range(len(seq)), key=lambda i: -seq[i][2])[:20]):
    a, src, s, e, w, we = seq[i]
    print(f"  {i:5d} {a} {s / S * 100:4.1f}% exec {e} wf {w} ex {we}  {src}")
if len(sys.argv) > 2:
    rows = list(csv.reader(io.StringIO(open(sys.argv[2]).read())))
    d = dict(zip(rows[0], rows[2]))
    st = [(k.split("stalled_")[1].split("_per")[0], float(d[k])) for k in rows[0]
          if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")]
    print("stalls per issue:", ", ".join(f"{k} {v:.2f}" for k, v in sorted(st, key=lambda x: -x[1])[:8]))
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"):
        print(f"  {k} {d.get(k)}")
