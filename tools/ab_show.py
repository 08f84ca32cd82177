"""Summarise tools/ab_lib.sh output: python tools/ab_show.py gpurun_out/TAG"""
import glob
import json
import os
import sys

d = sys.argv[1]
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    try:
        x = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(os.path.basename(f), "ERR", e)
        continue
    k = x["kernels"]
    k64 = x.get("fp64", {}).get("kernels", {})
    print(f"{os.path.basename(f):32s} fp32 {x['value']:6.2f} fp64 {x.get('fp64', {}).get('value', 0):6.2f} | "
          + " ".join(f"{n} {k[n]['ms']:.3f}" for n in ("K_A", "K_B", "K_C"))
          + " | fp64 " + " ".join(f"{n} {k64[n]['ms']:.3f}" for n in ("K_A", "K_B", "K_C") if n in k64))
