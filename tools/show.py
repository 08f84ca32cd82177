import json, sys, glob
for f in sorted(glob.glob(sys.argv[1] + "/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    r = d["roofline"]; f64 = d.get("fp64", {})
    print(f"{f.split('/')[-1]:18s} fp32 {d['value']:7.2f} ({d['ms_per_step']:8.3f} ms) kA frac {r['frac']:.3f} "
          f"kA {r['avg_launch_ms']*1e3:7.1f}us share {r['share_of_step']:.2f} | fp64 {f64.get('value', 0):6.2f} "
          f"kA64 frac {f64.get('k_ax_hbm_frac', 0):.3f} | x{d.get('speedup_fp32_vs_fp64', 0):.2f} e2e {d['e2e']['value']:.2f} clk {d['clocks']['sm_mhz']}")
