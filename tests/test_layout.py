"""The split layout of the library's CG vectors checked on
the host: the layout functions of nbk_common.cuh compiled by nvcc as host code
(no GPU needed) -- bijection, inverse, interior block first and boundary points
in natural order, the per-column and per-plane helpers."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.mark.skipif(not os.path.exists(NVCC) and shutil.which("nvcc") is None, reason="no nvcc")
def test_split_layout_bijection(tmp_path):
    exe = str(tmp_path / "sl_layout_check")
    src = os.path.join(HERE, "native", "sl_layout_check.cu")
    subprocess.run([NVCC if os.path.exists(NVCC) else "nvcc", "-std=c++17", "-o", exe, src], check=True,
                   capture_output=True, timeout=300)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stdout
    assert out.stdout.count("bad=0") == 15


@pytest.mark.skipif(not os.path.exists(NVCC) and shutil.which("nvcc") is None, reason="no nvcc")
def test_dssum_staged_tile_walk(tmp_path):
    """K_B's staged tile buffer: the flat phase-1 walk accepts exactly the slots that hold copy
    indices of the tile's nodes, at the positions phase 2 reads."""
    exe = str(tmp_path / "dssum_tile_check")
    src = os.path.join(HERE, "native", "dssum_tile_check.cu")
    subprocess.run([NVCC if os.path.exists(NVCC) else "nvcc", "-std=c++17", "-o", exe, src], check=True,
                   capture_output=True, timeout=300)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stdout
    assert "bad=0" in out.stdout and "cases=1296" in out.stdout
