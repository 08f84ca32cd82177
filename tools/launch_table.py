"""Summarise an ncu --csv launch list: per kernel count, mean time, DRAM bytes."""
import collections
import csv
import sys


def table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per, names = collections.defaultdict(dict), {}
    for r in rows[hi + 1:]:
        per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[idi]] = r[ki]
    agg = collections.OrderedDict()
    for i in sorted(per, key=int):
        n = names[i][:70]
        d = per[i]
        a = agg.setdefault(n, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0)
        a[3] += d.get("dram__bytes_write.sum", 0)
    return agg


if __name__ == "__main__":
    for n, a in table(sys.argv[1]).items():
        c = a[0]
        gbs = (a[2] + a[3]) / c / (a[1] / c) if a[1] else 0
        print(f"{c:4d} {a[1] / c / 1e3:9.2f} us  rd {a[2] / c / 1e6:8.2f} MB  wr {a[3] / c / 1e6:8.2f} MB "
              f" {gbs:7.1f} GB/s  {n}")
