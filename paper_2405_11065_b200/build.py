"""Build libnbk.so (the C-ABI CUDA library) in-tree for sm_100a with nvcc.

    python -m paper_2405_11065_b200.build [--force]

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, -fmad=false (no
contraction except the explicit __fma_rn of the canonical order, DESIGN.md
CEO-1), IEEE division / sqrt and no flush-to-zero (nvcc defaults, spelled out).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(CSRC, "libnbk.so")
# (source, object, extra flags): nbk_emu.cu is compiled once per emulation mode
SOURCES = [("nbk_capi.cu", "nbk_capi", []), ("nbk_setup.cu", "nbk_setup", []),
           ("nbk_emu.cu", "nbk_emu1", ["-DNBK_EMU_MODE=1"]),
           ("nbk_emu.cu", "nbk_emu2", ["-DNBK_EMU_MODE=2"]),
           ("nbk_emu.cu", "nbk_emu3", ["-DNBK_EMU_MODE=3"])]
HEADERS = ["nbk_common.cuh", "nbk_kernels.cuh", "nbk_axl.cuh", "nbk_kbw.cuh", "nbk_launch.cuh", "nbk_internal.h",
           "../../include/nbk.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NCCL_DIR = None
try:
    import nvidia.nccl as _nccl  # the pip NCCL torch links (one libnccl.so.2 per process)
    NCCL_DIR = os.path.dirname(_nccl.__file__) if _nccl.__file__ else list(_nccl.__path__)[0]
except Exception:  # pragma: no cover
    pass
NCCL_INC = [f"-I{os.path.join(NCCL_DIR, 'include')}"] if NCCL_DIR else []
NCCL_DEF = [f"-DNBK_NCCL_LIB=\"{os.path.join(NCCL_DIR, 'lib', 'libnccl.so.2')}\""] if NCCL_DIR else []
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-ftz=false", "-prec-div=true",
         "-prec-sqrt=true", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [src for src, _, _ in SOURCES] + HEADERS + [os.path.basename(__file__)]
    for f in deps:
        p = os.path.join(CSRC, f) if not f.endswith(".py") else os.path.join(HERE, f)
        if os.path.exists(p) and os.path.getmtime(p) > t:
            return True
    return False


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """Build libnbk.so (or, for A/B experiments, a variant at `out` with
    NBK_EXTRA_FLAGS; load it with NBK_LIB=<path>)."""
    if out is None and not force and not _stale():
        return LIB
    target = out or LIB
    objs, procs = [], []
    extra = os.environ.get("NBK_EXTRA_FLAGS", "").split()  # tuning experiments only
    for src, stem, defs in SOURCES:  # the translation units compile in parallel
        obj = os.path.join(CSRC, stem + ".o") if out is None else out + "." + stem + ".o"
        cmd = [NVCC, *ARCH, *FLAGS, *NCCL_INC, *NCCL_DEF, *defs, *extra, "-c", os.path.join(CSRC, src),
               "-o", obj]
        procs.append((stem, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    for stem, pr in procs:
        sout, err = pr.communicate()
        if pr.returncode != 0:
            sys.stderr.write(sout + err)
            raise RuntimeError(f"nvcc failed on {stem}")
        if verbose:
            sys.stderr.write(err)
        with open(os.path.join(CSRC, stem + ".ptxas.log") if out is None else out + "." + stem + ".ptxas.log", "w") as fh:
            fh.write(err)
    tmp = target + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-ldl"]
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    o = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=o))
