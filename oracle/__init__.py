"""CPU oracle for the Nekbone unpreconditioned-CG hot path (arXiv 2405.11065).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2405_11065_b200``) never imports it and
shares no code with it; see ``oracle/nbk_oracle.c`` for the arithmetic and the
paper passages each function follows.

This module is a thin ctypes wrapper: argument marshalling only.  ``build()``
compiles ``nbk_oracle.c`` with ``gcc -O2 -ffp-contract=off -fopenmp`` (IEEE
binary64/binary32, no contraction except explicit fma, no FTZ).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nbk_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

c_i32, c_i64, c_u64, c_dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
_p = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile the oracle shared library in-tree (gcc, no GPU needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.ora_splitmix64.restype = c_u64
        L.ora_splitmix64.argtypes = [c_u64, c_u64]
        L.ora_uniform_pm1.restype = c_dbl
        L.ora_uniform_pm1.argtypes = [c_u64, c_u64]
        L.ora_gll.restype = ctypes.c_int
        L.ora_gll.argtypes = [ctypes.c_int, _p, _p, _p]
        L.ora_sizes.restype = None
        L.ora_sizes.argtypes = [ctypes.c_int] * 4 + [_p]
        L.ora_setup.restype = ctypes.c_int
        L.ora_setup.argtypes = [ctypes.c_int] * 4 + [c_dbl, c_u64, c_u64, c_i64, c_i64] + [_p] * 7
        for nm in ("ora_ax_local64", "ora_ax_local32"):
            getattr(L, nm).restype = None
            getattr(L, nm).argtypes = [c_i64, ctypes.c_int, _p, _p, _p, _p]
        for nm in ("ora_dssum64", "ora_dssum32"):
            getattr(L, nm).restype = None
            getattr(L, nm).argtypes = [ctypes.c_int] * 4 + [_p, ctypes.c_int]
        for nm in ("ora_mask64", "ora_mask32"):
            getattr(L, nm).restype = None
            getattr(L, nm).argtypes = [ctypes.c_int] * 4 + [_p]
        for nm in ("ora_ax64", "ora_ax32"):
            getattr(L, nm).restype = None
            getattr(L, nm).argtypes = [ctypes.c_int] * 4 + [_p] * 4 + [ctypes.c_int]
        L.ora_fsum.restype = c_dbl
        L.ora_fsum.argtypes = [c_i64, _p]
        for nm in ("ora_glsc3_64", "ora_glsc3_32"):
            getattr(L, nm).restype = c_dbl
            getattr(L, nm).argtypes = [c_i64, _p, _p, _p]
        L.ora_multiplicity_weight.restype = None
        L.ora_multiplicity_weight.argtypes = [ctypes.c_int] * 4 + [_p]
        for nm in ("ora_cg64", "ora_cg32"):
            getattr(L, nm).restype = ctypes.c_int
            getattr(L, nm).argtypes = [ctypes.c_int] * 4 + [_p] * 3 + [ctypes.c_int] + [_p] * 3
        for nm in ("ora_pcg64", "ora_pcg32"):
            getattr(L, nm).restype = ctypes.c_int
            getattr(L, nm).argtypes = [ctypes.c_int] * 4 + [_p] * 4 + [ctypes.c_int] + [_p] * 3
        L.ora_cg32s.restype = ctypes.c_int
        L.ora_cg32s.argtypes = [ctypes.c_int] * 4 + [_p] * 4 + [ctypes.c_int] + [_p] * 3
        L.ora_glsc3_32s.restype = ctypes.c_float
        L.ora_glsc3_32s.argtypes = [c_i64, _p, _p, _p]
        L.ora_cg32a.restype = ctypes.c_int
        L.ora_cg32a.argtypes = [ctypes.c_int] * 4 + [_p] * 4 + [ctypes.c_int] * 2 + [_p] * 3
        L.ora_glsc3_32a_p.restype = ctypes.c_float
        L.ora_glsc3_32a_p.argtypes = [c_i64, _p, _p, _p, ctypes.c_int]
        L.ora_fsum32.restype = ctypes.c_float
        L.ora_fsum32.argtypes = [c_i64, _p]
        L.ora_vprec_round.restype = c_dbl
        L.ora_vprec_round.argtypes = [c_dbl, ctypes.c_int]
        L.ora_cgvp.restype = ctypes.c_int
        L.ora_cgvp.argtypes = [ctypes.c_int] * 4 + [_p] * 3 + [ctypes.c_int] * 2 + [_p] * 3
        L.ora_cgpm.restype = ctypes.c_int
        L.ora_cgpm.argtypes = ([ctypes.c_int] * 4 + [_p] * 3 + [ctypes.c_int] * 2 + [c_u64] +
                               [ctypes.c_int] + [_p] * 3)
        L.ora_jacobi_dinv.restype = None
        L.ora_jacobi_dinv.argtypes = [ctypes.c_int] * 4 + [_p] * 4
        L.ora_true_residual.restype = c_dbl
        L.ora_true_residual.argtypes = [ctypes.c_int] * 4 + [_p] * 5
        L.ora_num_threads.restype = ctypes.c_int
        L.ora_num_threads.argtypes = []
        _lib = L
    return _lib


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Mesh:
    """Box of ex*ey*ez hexahedra, N GLL points per direction (reading R1/R5)."""
    ex: int
    ey: int
    ez: int
    N: int
    jitter: float = 0.0
    seed_geom: int = 0
    seed_rhs: int = 0

    @property
    def E(self) -> int:
        return self.ex * self.ey * self.ez

    @property
    def dims(self):
        return (self.ex, self.ey, self.ez, self.N)

    def sizes(self) -> dict:
        out = np.zeros(4, dtype=np.int64)
        lib().ora_sizes(self.ex, self.ey, self.ez, self.N, _ptr(out))
        return dict(n_local=int(out[0]), n_global=int(out[1]), n_interior=int(out[2]),
                    n_shared=int(out[3]))


def splitmix64(seed: int, i: int) -> int:
    return int(lib().ora_splitmix64(seed & (2**64 - 1), i))


def uniform_pm1(seed: int, i: int) -> float:
    return float(lib().ora_uniform_pm1(seed & (2**64 - 1), i))


def gll(N: int):
    """GLL nodes, weights and derivative matrix D[a, b] = l_b'(xi_a)."""
    xi = np.zeros(N)
    rho = np.zeros(N)
    D = np.zeros((N, N))
    rc = lib().ora_gll(N, _ptr(xi), _ptr(rho), _ptr(D))
    if rc:
        raise ValueError(f"ora_gll failed ({rc})")
    return xi, rho, D


def setup(mesh: Mesh, e0: int = 0, e1: int | None = None, want=("G", "f")):
    """FP64 set-up arrays for elements [e0, e1): dict of numpy arrays."""
    e1 = mesh.E if e1 is None else e1
    E = e1 - e0
    out = {}
    shapes = {"G": ((E, 6, mesh.N, mesh.N, mesh.N), np.float64),
              "f": ((E, mesh.N, mesh.N, mesh.N), np.float64),
              "mass": ((E, mesh.N, mesh.N, mesh.N), np.float64),
              "gid": ((E, mesh.N, mesh.N, mesh.N), np.int64),
              "mult": ((E, mesh.N, mesh.N, mesh.N), np.int32),
              "mask": ((E, mesh.N, mesh.N, mesh.N), np.uint8),
              "xyz": ((E, 3, mesh.N, mesh.N, mesh.N), np.float64)}
    for k in want:
        shp, dt = shapes[k]
        out[k] = np.zeros(shp, dtype=dt)
    rc = lib().ora_setup(mesh.ex, mesh.ey, mesh.ez, mesh.N, float(mesh.jitter),
                         mesh.seed_geom & (2**64 - 1), mesh.seed_rhs & (2**64 - 1), e0, e1,
                         *[_ptr(out.get(k)) for k in ("G", "f", "mass", "gid", "mult", "mask", "xyz")])
    if rc:
        raise ValueError(f"ora_setup failed ({rc})")
    return out


def multiplicity_weight(mesh: Mesh) -> np.ndarray:
    c = np.zeros((mesh.E, mesh.N, mesh.N, mesh.N))
    lib().ora_multiplicity_weight(*mesh.dims, _ptr(c))
    return c


def ax_local(D, G, u):
    """Per-element ax_e = D^T G D u_e in the canonical order (C1-C3)."""
    u = np.ascontiguousarray(u)
    w = np.empty_like(u)
    E, N = u.shape[0], u.shape[-1]
    if u.dtype == np.float64:
        lib().ora_ax_local64(E, N, _ptr(np.ascontiguousarray(D, np.float64)),
                             _ptr(np.ascontiguousarray(G, np.float64)), _ptr(u), _ptr(w))
    elif u.dtype == np.float32:
        lib().ora_ax_local32(E, N, _ptr(np.ascontiguousarray(D, np.float32)),
                             _ptr(np.ascontiguousarray(G, np.float32)), _ptr(u), _ptr(w))
    else:
        raise TypeError(u.dtype)
    return w


def dssum(mesh: Mesh, w, apply_mask: bool = False):
    w = np.array(w, copy=True, order="C")
    fn = lib().ora_dssum64 if w.dtype == np.float64 else lib().ora_dssum32
    fn(*mesh.dims, _ptr(w), int(apply_mask))
    return w


def mask(mesh: Mesh, w):
    w = np.array(w, copy=True, order="C")
    fn = lib().ora_mask64 if w.dtype == np.float64 else lib().ora_mask32
    fn(*mesh.dims, _ptr(w))
    return w


def ax(mesh: Mesh, D, G, u, apply_mask: bool = True):
    """w = mask(dssum(ax_e(u)))  (T1 line 5)."""
    return dssum(mesh, ax_local(D, G, u), apply_mask=apply_mask)


def fsum(t) -> float:
    t = np.ascontiguousarray(t, dtype=np.float64)
    return float(lib().ora_fsum(t.size, _ptr(t)))


def glsc3_single(a, b, c) -> float:
    """Paper-literal binary32 glsc3 (NEXT-2): RN32 of the exact sum of RN32(a b) c."""
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    c = np.ascontiguousarray(c, dtype=np.float64)
    return float(lib().ora_glsc3_32s(a.size, _ptr(a), _ptr(b), _ptr(c)))


def glsc3_accum32(a, b, c, nranks: int = 1) -> float:
    """The paper's binary32 glsc3 (NEXT-2, R11c): sequential binary32
    accumulation of RN32(RN32(a b) c) per rank (contiguous ranges), then the
    per-rank sums added in binary32 in rank order."""
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    c = np.ascontiguousarray(c, dtype=np.float64)
    return float(lib().ora_glsc3_32a_p(a.size, _ptr(a), _ptr(b), _ptr(c), int(nranks)))


def fsum32(t) -> float:
    """RN32 of the exact sum of binary64 terms."""
    t = np.ascontiguousarray(t, dtype=np.float64)
    return float(lib().ora_fsum32(t.size, _ptr(t)))


def glsc3(a, b, c) -> float:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    c = np.ascontiguousarray(c, dtype=np.float64)
    assert a.dtype == b.dtype and a.size == b.size == c.size
    fn = lib().ora_glsc3_64 if a.dtype == np.float64 else lib().ora_glsc3_32
    return float(fn(a.size, _ptr(a), _ptr(b), _ptr(c)))


@dataclass
class CgResult:
    x: np.ndarray
    hist: np.ndarray   # h_0..h_niter
    trace: np.ndarray  # (niter, 5): rtz1, beta, alpha, pap, rtr
    defect: int


def vprec_round(x: float, t: int) -> float:
    """VPREC rounding of a binary64 value to t mantissa bits (RN, ties to even)."""
    return float(lib().ora_vprec_round(float(x), int(t)))


def cg_vprec(mesh: Mesh, D, G, f, niter: int, t: int) -> CgResult:
    """VPREC-emulated CG (NEXT-4): binary64 loop, every
    operation of the CG kernels rounded to t mantissa bits."""
    D = np.ascontiguousarray(D, np.float64)
    G = np.ascontiguousarray(G, np.float64)
    f = np.ascontiguousarray(f, np.float64)
    hist = np.zeros(niter + 1)
    trace = np.zeros((niter, 5))
    x = np.zeros_like(f)
    rc = lib().ora_cgvp(*mesh.dims, _ptr(D), _ptr(G), _ptr(f), int(t), niter, _ptr(x), _ptr(hist),
                        _ptr(trace))
    return CgResult(x=x, hist=hist, trace=trace, defect=int(rc))


EMU = {"vprec": 1, "rr": 2, "mca": 3}


def cg_emulated(mesh: Mesh, D, G, f, niter: int, mode: str, t: int, seed: int = 0) -> CgResult:
    """Precision-emulated CG (NEXT-4): 'vprec' (every operation rounded to t
    bits), 'rr' (random rounding of every result at virtual precision t) or
    'mca' (operands and results perturbed); seed selects the RR / MCA sample."""
    D = np.ascontiguousarray(D, np.float64)
    G = np.ascontiguousarray(G, np.float64)
    f = np.ascontiguousarray(f, np.float64)
    hist = np.zeros(niter + 1)
    trace = np.zeros((niter, 5))
    x = np.zeros_like(f)
    rc = lib().ora_cgpm(*mesh.dims, _ptr(D), _ptr(G), _ptr(f), EMU[mode], int(t),
                        seed & (2**64 - 1), niter, _ptr(x), _ptr(hist), _ptr(trace))
    return CgResult(x=x, hist=hist, trace=trace, defect=int(rc))


def jacobi_dinv(mesh: Mesh, D, G):
    """Jacobi preconditioner data (NEXT-1): the assembled diagonal d
    of the stiffness operator (masked entries 1) and dinv = 1/d, FP64, local storage."""
    D = np.ascontiguousarray(D, np.float64)
    G = np.ascontiguousarray(G, np.float64)
    d = np.zeros((mesh.E, mesh.N, mesh.N, mesh.N))
    dinv = np.zeros_like(d)
    lib().ora_jacobi_dinv(*mesh.dims, _ptr(D), _ptr(G), _ptr(d), _ptr(dinv))
    return d, dinv


def cg(mesh: Mesh, D, G, f, niter: int, precision: str = "fp64", dinv=None,
       nranks: int = 1) -> CgResult:
    """Fixed-iteration CG (T1).  precision 'fp64', 'fp32' (mixed: FP64 set-up
    data rounded once to binary32, FP64 accumulation of glsc3), 'fp32s'
    (binary32 scalars, exactly rounded binary32 inner products, R11b) or
    'fp32a' (the paper's single-precision solver: binary32 accumulation of the
    inner products per rank, binary32 all-reduce in rank order over `nranks`
    z-slabs, binary32 scalars; R11c).  dinv (FP64 local array) selects Jacobi
    PCG: z = r * dinv (dinv rounded to the loop's precision), rtz1 = glsc3(r, c, z)."""
    D = np.ascontiguousarray(D, np.float64)
    G = np.ascontiguousarray(G, np.float64)
    f = np.ascontiguousarray(f, np.float64)
    hist = np.zeros(niter + 1)
    trace = np.zeros((niter, 5))
    L = lib()
    if precision == "fp32a":  # the paper's single-precision solver (NEXT-2, R11c)
        di = None if dinv is None else np.ascontiguousarray(dinv, np.float64)
        x = np.zeros(f.shape, np.float32)
        rc = L.ora_cg32a(*mesh.dims, _ptr(D), _ptr(G), _ptr(f), _ptr(di), int(nranks), niter,
                         _ptr(x), _ptr(hist), _ptr(trace))
        return CgResult(x=x, hist=hist, trace=trace, defect=int(rc))
    if precision == "fp32s":  # binary32 scalars, exactly rounded binary32 glsc3 (R11b)
        di = None if dinv is None else np.ascontiguousarray(dinv, np.float64)
        x = np.zeros(f.shape, np.float32)
        rc = L.ora_cg32s(*mesh.dims, _ptr(D), _ptr(G), _ptr(f), _ptr(di), niter, _ptr(x),
                         _ptr(hist), _ptr(trace))
        return CgResult(x=x, hist=hist, trace=trace, defect=int(rc))
    if dinv is not None:
        di = np.ascontiguousarray(dinv, np.float64)
        if precision == "fp64":
            x = np.zeros_like(f)
            rc = L.ora_pcg64(*mesh.dims, _ptr(D), _ptr(G), _ptr(f), _ptr(di), niter, _ptr(x),
                             _ptr(hist), _ptr(trace))
        elif precision == "fp32":
            x = np.zeros(f.shape, np.float32)
            rc = L.ora_pcg32(*mesh.dims, _ptr(D), _ptr(G), _ptr(f), _ptr(di), niter, _ptr(x),
                             _ptr(hist), _ptr(trace))
        else:
            raise ValueError(precision)
    elif precision == "fp64":
        x = np.zeros_like(f)
        rc = L.ora_cg64(*mesh.dims, _ptr(D), _ptr(G), _ptr(f), niter, _ptr(x), _ptr(hist),
                        _ptr(trace))
    elif precision == "fp32":
        x = np.zeros(f.shape, np.float32)
        rc = L.ora_cg32(*mesh.dims, _ptr(D), _ptr(G), _ptr(f), niter, _ptr(x), _ptr(hist),
                        _ptr(trace))
    else:
        raise ValueError(precision)
    return CgResult(x=x, hist=hist, trace=trace, defect=int(rc))


def true_residual(mesh: Mesh, D, G, f, x):
    """Final FP64 check (C12): (||f - A x64||_c, h0)."""
    x64 = np.ascontiguousarray(x, dtype=np.float64)
    h0 = ctypes.c_double(0.0)
    r = lib().ora_true_residual(*mesh.dims, _ptr(np.ascontiguousarray(D, np.float64)),
                                _ptr(np.ascontiguousarray(G, np.float64)),
                                _ptr(np.ascontiguousarray(f, np.float64)), _ptr(x64),
                                ctypes.cast(ctypes.pointer(h0), ctypes.c_void_p))
    return float(r), float(h0.value)


def num_threads() -> int:
    return int(lib().ora_num_threads())
