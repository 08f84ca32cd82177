"""The bench.py contract on the GPU (small config): one JSON line with the keys
the driver reads -- metric / value / unit, n_gpus, steps / warmup,
ms_per_step, roofline (bound, achieved, peak, frac, traffic), cpu_baseline
(kind oracle, cores, sample), e2e (value, h2d / d2h bytes), clocks,
gpu_launches -- and a positive, finite value.  Also the reference arm."""
import json
import math
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract_small():
    d = _run(["--config", "C2", "--steps", "3", "--warmup", "3", "--no-precision-study", "--convergence",
              "0", "--others", "", "--energy-reps", "2", "--prof-steps", "1"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "gpu_launches", "roofline", "cpu_baseline",
              "e2e", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert math.isfinite(d["value"]) and d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    # the copies are inside the timed region: end to end cannot beat the device-resident value
    assert e["value"] <= d["value"] * 1.02 and 0 < e["single_call_value"] <= d["value"] * 1.02
    assert d["clocks"]["sm_max_mhz"] and "reasons" in d["clocks"]
    assert d["config"]["workload"].startswith("C2")
    assert d["fp64"]["value"] > 0 and d["speedup_fp32_vs_fp64"] > 1.0
    assert d["accuracy"]["fp32a"]["MAE"] >= 0 and d["jacobi_pcg"]["fp32"]["value"] > 0


def test_bench_reference_arm_small():
    d = _run(["--impl", "reference", "--config", "C2", "--steps", "1", "--warmup", "0"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
