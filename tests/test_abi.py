"""CPU checks of the C-ABI library: it loads and exports every symbol that
include/nbk.h declares (no compute calls: no GPU here), and the build flags
that the canonical evaluation order depends on are present in the binary."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "nbk.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(nbk_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2405_11065_b200 import build
    build.build()
    return ctypes.CDLL(build.LIB)


def test_library_exports_every_declared_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    from paper_2405_11065_b200 import nbk
    assert sorted(nbk.SYMBOLS) == syms


def test_binding_loads_and_reports_version(lib):
    from paper_2405_11065_b200 import nbk
    L = nbk.load()
    assert L.nbk_version().decode().startswith("nbk")


def test_kernels_are_sm100a_and_use_no_contraction(lib):
    from paper_2405_11065_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.LIB],
                          capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for line in sass.splitlines():
        if "Function : " in line:
            cur = line.split("Function : ")[1].strip()
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    def body(prefix):
        names = [f for f in funcs if f.startswith(prefix)]
        assert len(names) == 1, (prefix, names)
        return "\n".join(funcs[names[0]])
    # the fused CG step of K_A: line-owner kernel k_axl (nbk_axl.cuh)
    fused64 = body("_ZN3nbk5k_axlIdLi10ELi1EEE")
    fused32 = body("_ZN3nbk5k_axlIfLi8ELi1EEE")
    assert "DFMA" in fused64 and "FFMA" in fused32
    # TMA 1-D bulk copies (cp.async.bulk -> UBLKCP) stage G and p in shared memory,
    # w leaves by a bulk store; r / x / p' / x' move as 16-byte vectors in slot order
    for n in (8, 10, 12):
        k32 = body(f"_ZN3nbk5k_axlIfLi{n}ELi1EEE")
        # bulk loads of G (and p where its block is staged: 9 N^3 layout), bulk store of w
        assert k32.count("UBLKCP.S.G") >= (1 if n == 10 else 2) and k32.count("UBLKCP.G.S") >= 1, n
        assert "LDG.E.128" in k32 and "STG.E.128" in k32, n
    # the plain operator (nbk_ax_apply) keeps the pencil kernel
    plain32 = body("_ZN3nbk4k_axIfLi10ELi0ELi0EE")
    assert "UBLKCP" in plain32 and "FFMA" in plain32
    # K_B: compact plan rows staged by TMA, copies gathered by cp.async (LDGSTS)
    kb32 = body("_ZN3nbk7k_dssumIfLb1ELi0EE")
    assert "UBLKCP" in kb32 and "LDGSTS" in kb32


def test_workspace_size_query_without_gpu_is_rejected_cleanly(lib):
    """Without a device the library must not fall back to CPU compute."""
    from paper_2405_11065_b200 import nbk
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(nbk.NbkError):
        nbk.Context(nbk.MeshSpec(2, 2, 2, 4), "fp64")


@pytest.mark.parametrize("args,msg", [((128, 128, 128, 12), "int32"), ((1, 1, 1, 17), "N must"),
                                      ((1, 1, 1, 1), "N must"), ((0, 2, 2, 4), ""),
                                      ((2, -1, 2, 4), "")])
def test_mesh_limits_are_validated_on_the_host(lib, args, msg):
    """Maximum / degenerate sizes: more than 2^31 local points (int32 dssum
    plan), N outside [2, 16], empty or negative boxes -- rejected with a status,
    before any device work."""
    from paper_2405_11065_b200 import nbk
    with pytest.raises(nbk.NbkError, match=msg):
        nbk.workspace_bytes(nbk.MeshSpec(*args), "fp32")


def test_largest_single_gpu_workspaces_fit_hbm(lib):
    """Workspace of the largest BASELINE configurations at one GPU (C5: 64^3,
    N = 10; C4 global at P = 8 as one rank) against 180 GB of HBM."""
    from paper_2405_11065_b200 import CONFIGS, nbk
    c5 = nbk.workspace_bytes(nbk.MeshSpec(**CONFIGS["C5"].mesh_args(1)), "fp32")
    assert c5 < 60e9
    c4p8 = nbk.workspace_bytes(nbk.MeshSpec(**CONFIGS["C4"].mesh_args(8)), "fp32")
    assert c4p8 < 180e9
