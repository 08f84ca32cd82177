"""Thin Python binding of libnbk.so (include/nbk.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels.  PyTorch is used
for device memory (the caller-owned workspace and field tensors) and streams.
There is no CPU fallback: if ``csrc/libnbk.so`` is missing or no CUDA device is
present, the calls raise.

Names follow the north_star boundary: ``cg_setup``, ``ax_apply``, ``dssum``,
``glsc3``, ``cg_solve``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "csrc", "libnbk.so")
if os.environ.get("NBK_LIB"):  # A/B experiments: a variant build (build.py --out)
    LIB_PATH = os.path.abspath(os.environ["NBK_LIB"])

NBK_OK, NBK_EINVAL, NBK_EDEFECT, NBK_ECUDA, NBK_ENCCL, NBK_ENOMEM, NBK_ESTATE = 0, 2, 3, 4, 5, 6, 7
NBK_FP64, NBK_FP32 = 0, 1
AX_LOCAL, AX_DSSUM, AX_MASK = 0, 1, 2
NBK_FP32S, NBK_VPREC, NBK_FP32A = 2, 3, 4
PREC = {"fp64": NBK_FP64, "fp32": NBK_FP32, "fp32s": NBK_FP32S, "vprec": NBK_VPREC,
        "fp32a": NBK_FP32A}
PRECOND = {"none": 0, "jacobi": 1}
EMU = {"vprec": 1, "rr": 2, "mca": 3}

# every symbol include/nbk.h declares
SYMBOLS = ["nbk_workspace_bytes", "nbk_partition", "nbk_nccl_unique_id", "nbk_cg_setup",
           "nbk_load_arrays", "nbk_get_arrays", "nbk_ax_apply", "nbk_dssum", "nbk_glsc3",
           "nbk_cg_solve", "nbk_cg_solve_host", "nbk_cg_solve_host_batch", "nbk_get_solution", "nbk_solution_ptr",
           "nbk_set_emulation", "nbk_set_vprec", "nbk_set_precond", "nbk_load_precond", "nbk_get_precond", "nbk_set_profiling",
           "nbk_query", "nbk_solve_launches", "nbk_group_link",
           "nbk_group_ax_apply", "nbk_group_dssum", "nbk_group_glsc3", "nbk_group_cg_solve",
           "nbk_last_error", "nbk_version", "nbk_destroy"]


class NbkError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libnbk status {status}: {msg}")
        self.status = status


class CMesh(ctypes.Structure):
    _fields_ = [("ex", ctypes.c_int32), ("ey", ctypes.c_int32), ("ez", ctypes.c_int32),
                ("N", ctypes.c_int32), ("jitter", ctypes.c_double),
                ("seed_geom", ctypes.c_uint64), ("seed_rhs", ctypes.c_uint64)]


class CDist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("device", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("nccl_id", ctypes.c_void_p)]


class CInfo(ctypes.Structure):
    _fields_ = [("n_local", ctypes.c_int64), ("n_global", ctypes.c_int64),
                ("e_local", ctypes.c_int64), ("e_offset", ctypes.c_int64),
                ("n_shared", ctypes.c_int64), ("n_copies", ctypes.c_int64),
                ("N", ctypes.c_int32), ("has_fp32", ctypes.c_int32),
                ("face_layer", ctypes.c_int64), ("face_nodes", ctypes.c_int64)]


class CResult(ctypes.Structure):
    _fields_ = [("true_res", ctypes.c_double), ("true_res_rel", ctypes.c_double),
                ("defect_iter", ctypes.c_int32), ("niter", ctypes.c_int32),
                ("solve_ms", ctypes.c_float), ("kA_ms", ctypes.c_float),
                ("kB_ms", ctypes.c_float), ("kC_ms", ctypes.c_float)]


_lib = None


def load() -> ctypes.CDLL:
    """Load libnbk.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -m paper_2405_11065_b200.build` (no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    P = ctypes.POINTER
    sig = {
        "nbk_workspace_bytes": [P(CMesh), ctypes.c_int, P(CDist), P(ctypes.c_size_t)],
        "nbk_partition": [P(CMesh), P(CDist), P(CInfo)],
        "nbk_nccl_unique_id": [vp],
        "nbk_group_link": [P(vp), i32],
        "nbk_group_ax_apply": [P(vp), i32, P(vp), P(vp), i32, ctypes.c_int],
        "nbk_group_dssum": [P(vp), i32, P(vp), i32, ctypes.c_int],
        "nbk_group_glsc3": [P(vp), i32, P(vp), P(vp), ctypes.c_int, P(ctypes.c_double)],
        "nbk_group_cg_solve": [P(vp), i32, i32, ctypes.c_int, vp, vp, P(CResult)],
        "nbk_cg_setup": [P(CMesh), ctypes.c_int, P(CDist), vp, ctypes.c_size_t, P(vp)],
        "nbk_load_arrays": [vp, vp, vp, vp],
        "nbk_get_arrays": [vp, vp, vp, vp],
        "nbk_ax_apply": [vp, vp, vp, i32, ctypes.c_int],
        "nbk_dssum": [vp, vp, i32, ctypes.c_int],
        "nbk_glsc3": [vp, vp, vp, ctypes.c_int, P(ctypes.c_double)],
        "nbk_cg_solve": [vp, i32, ctypes.c_int, vp, vp, P(CResult)],
        "nbk_cg_solve_host": [vp, vp, i32, ctypes.c_int, vp, vp, P(CResult)],
        "nbk_cg_solve_host_batch": [vp, i32, P(vp), i32, ctypes.c_int, P(vp), vp, P(CResult)],
        "nbk_get_solution": [vp, vp],
        "nbk_solution_ptr": [vp, ctypes.c_int, P(vp)],
        "nbk_set_profiling": [vp, i32],
        "nbk_set_precond": [vp, i32],
        "nbk_set_vprec": [vp, i32],
        "nbk_set_emulation": [vp, i32, i32, ctypes.c_uint64],
        "nbk_load_precond": [vp, vp],
        "nbk_get_precond": [vp, vp],
        "nbk_query": [vp, P(CInfo)],
        "nbk_solve_launches": [vp, i32, ctypes.c_int, P(i64)],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.nbk_last_error.argtypes = [vp]
    L.nbk_last_error.restype = ctypes.c_char_p
    L.nbk_version.argtypes = []
    L.nbk_version.restype = ctypes.c_char_p
    L.nbk_destroy.argtypes = [vp]
    L.nbk_destroy.restype = None
    _lib = L
    return L


def _check(st: int, ctx=None, ok=(NBK_OK,)):
    if st not in ok:
        msg = load().nbk_last_error(ctx).decode()
        raise NbkError(st, msg)
    return st


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"] and a.dtype == np.float64
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass(frozen=True)
class MeshSpec:
    ex: int
    ey: int
    ez: int
    N: int
    jitter: float = 0.0
    seed_geom: int = 0
    seed_rhs: int = 0

    def c(self) -> CMesh:
        return CMesh(self.ex, self.ey, self.ez, self.N, float(self.jitter),
                     self.seed_geom & (2**64 - 1), self.seed_rhs & (2**64 - 1))

    @property
    def E(self) -> int:
        return self.ex * self.ey * self.ez


def workspace_bytes(mesh: MeshSpec, precision: str = "fp32", nranks: int = 1, rank: int = 0) -> int:
    out = ctypes.c_size_t(0)
    d = CDist(rank, nranks, 0, None, None)
    _check(load().nbk_workspace_bytes(ctypes.byref(mesh.c()), PREC[precision], ctypes.byref(d),
                                      ctypes.byref(out)))
    return int(out.value)


def partition(mesh: MeshSpec, nranks: int = 1, rank: int = 0) -> dict:
    """Slab partition of the mesh for one rank (host only; no device needed)."""
    info = CInfo()
    d = CDist(rank, nranks, 0, None, None)
    _check(load().nbk_partition(ctypes.byref(mesh.c()), ctypes.byref(d), ctypes.byref(info)))
    return {k: getattr(info, k) for k, _ in CInfo._fields_}


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0; broadcast it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().nbk_nccl_unique_id(buf))
    return buf.raw


class Context:
    """cg_setup(mesh, N, precision): a device-resident problem (one per GPU).

    nranks > 1: this context owns z-slab `rank`.  With `nccl_id` (128 bytes from
    nccl_unique_id() on rank 0) the set-up and every call are collective over
    NCCL; without it the context is a virtual slab to be linked with Group."""

    def __init__(self, mesh: MeshSpec, precision: str = "fp32", device: int = 0, stream=None,
                 rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None):
        import torch
        self.torch = torch
        if not torch.cuda.is_available():
            raise NbkError(NBK_ECUDA, "no CUDA device: libnbk has no CPU fallback")
        self.lib = load()
        self.mesh = mesh
        self.rank, self.nranks = rank, nranks
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.device)
        nbytes = workspace_bytes(mesh, precision, nranks, rank)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self._ctx = ctypes.c_void_p(None)
        self._id = None if nccl_id is None else ctypes.create_string_buffer(bytes(nccl_id), 128)
        d = CDist(rank, nranks, device, ctypes.c_void_p(self.stream.cuda_stream),
                  None if self._id is None else ctypes.cast(self._id, ctypes.c_void_p))
        _check(self.lib.nbk_cg_setup(ctypes.byref(mesh.c()), PREC[precision], ctypes.byref(d),
                                     ctypes.c_void_p(self.workspace.data_ptr()), nbytes,
                                     ctypes.byref(self._ctx)))
        info = CInfo()
        _check(self.lib.nbk_query(self._ctx, ctypes.byref(info)), self._ctx)
        self.info = {k: getattr(info, k) for k, _ in CInfo._fields_}
        self.n_local = info.n_local
        self.n_global = info.n_global
        self.N = mesh.N
        self.shape = (info.e_local, mesh.N, mesh.N, mesh.N)

    # ------------------------------------------------------------------
    def close(self):
        if self._ctx:
            self.lib.nbk_destroy(self._ctx)
            self._ctx = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        self.stream.synchronize()

    def _dev(self, t, dtype):
        assert t.is_cuda and t.is_contiguous() and t.dtype == dtype and t.numel() == self.n_local
        return ctypes.c_void_p(t.data_ptr())

    @staticmethod
    def _prec_of(t):
        import torch
        return "fp64" if t.dtype == torch.float64 else "fp32"

    # ---------------------------------------------------------------- ABI
    def load_arrays(self, D=None, G=None, f=None):
        """Parity path (C10): ingest host FP64 arrays (e.g. the oracle's)."""
        arrs = [None if a is None else np.ascontiguousarray(a, dtype=np.float64) for a in (D, G, f)]
        _check(self.lib.nbk_load_arrays(self._ctx, *[_ptr(a) for a in arrs]), self._ctx)

    def get_arrays(self, G: bool = True):
        """The context's FP64 set-up data (D, G, f); G=False skips the 48 B/pt G."""
        N = self.N
        D = np.zeros((N, N))
        Ga = np.zeros((self.shape[0], 6, N, N, N)) if G else None
        f = np.zeros(self.shape)
        _check(self.lib.nbk_get_arrays(self._ctx, _ptr(D), _ptr(Ga), _ptr(f)), self._ctx)
        return D, Ga, f

    def _enter(self):
        """Order the context stream after the caller's current stream (the
        tensors passed in may still be being produced there)."""
        cur = self.torch.cuda.current_stream(self.device)
        if cur != self.stream:
            self.stream.wait_stream(cur)
        return cur

    def _leave(self, cur, *tensors):
        """Order the caller's stream after the library's work on `tensors`."""
        if cur != self.stream:
            cur.wait_stream(self.stream)
            for t in tensors:
                t.record_stream(self.stream)

    def ax_apply(self, u, w, flags: int = AX_DSSUM | AX_MASK):
        prec = self._prec_of(u)
        cur = self._enter()
        _check(self.lib.nbk_ax_apply(self._ctx, self._dev(u, u.dtype), self._dev(w, u.dtype),
                                     flags, PREC[prec]), self._ctx)
        self._leave(cur, u, w)
        return w

    def dssum(self, f, apply_mask: bool = False):
        prec = self._prec_of(f)
        cur = self._enter()
        _check(self.lib.nbk_dssum(self._ctx, self._dev(f, f.dtype), int(apply_mask), PREC[prec]),
               self._ctx)
        self._leave(cur, f)
        return f

    def glsc3(self, a, b, single: bool = False) -> float:
        prec = self._prec_of(a)
        if single:
            prec = "fp32s"
        out = ctypes.c_double(0.0)
        self._enter()  # synchronous call: nothing to order afterwards
        _check(self.lib.nbk_glsc3(self._ctx, self._dev(a, a.dtype), self._dev(b, a.dtype),
                                  PREC[prec], ctypes.byref(out)), self._ctx)
        return float(out.value)

    def set_vprec(self, t: int):
        """Mantissa bits of the VPREC-emulated solver (cg_solve(..., 'vprec'))."""
        _check(self.lib.nbk_set_vprec(self._ctx, int(t)), self._ctx)

    def set_emulation(self, mode: str, t: int, seed: int = 0):
        """Emulation of cg_solve(..., 'vprec'): mode 'vprec', 'rr' or 'mca' at
        virtual precision t; seed selects the RR / MCA sample."""
        _check(self.lib.nbk_set_emulation(self._ctx, EMU[mode], int(t), seed & (2**64 - 1)),
               self._ctx)

    def set_precond(self, precond: str):
        """'none' (z = r, the default) or 'jacobi' (z = r / diag(A))."""
        _check(self.lib.nbk_set_precond(self._ctx, PRECOND[precond]), self._ctx)

    def load_precond(self, dinv):
        """Parity path: use the host array dinv (FP64, local storage) as 1/diag(A)."""
        a = np.ascontiguousarray(dinv, dtype=np.float64)
        _check(self.lib.nbk_load_precond(self._ctx, _ptr(a)), self._ctx)

    def get_precond(self) -> np.ndarray:
        out = np.zeros(self.shape)
        _check(self.lib.nbk_get_precond(self._ctx, _ptr(out)), self._ctx)
        return out

    def set_profiling(self, on: bool):
        _check(self.lib.nbk_set_profiling(self._ctx, int(on)), self._ctx)

    def cg_solve(self, niter: int, precision: str = "fp32", trace: bool = True):
        hist = np.zeros(niter + 1)
        tr = np.zeros((niter, 5)) if trace else None
        res = CResult()
        st = self.lib.nbk_cg_solve(self._ctx, niter, PREC[precision], _ptr(hist),
                                   _ptr(tr) if trace else None, ctypes.byref(res))
        _check(st, self._ctx, ok=(NBK_OK, NBK_EDEFECT))
        out = {k: getattr(res, k) for k, _ in CResult._fields_}
        return hist, tr, out

    def cg_solve_host(self, f_host, niter: int, precision: str = "fp32", x_host=None):
        hist = np.zeros(niter + 1)
        res = CResult()
        fh = None if f_host is None else np.ascontiguousarray(f_host, dtype=np.float64)
        st = self.lib.nbk_cg_solve_host(self._ctx, _ptr(fh), niter, PREC[precision],
                                        _ptr(x_host), _ptr(hist), ctypes.byref(res))
        _check(st, self._ctx, ok=(NBK_OK, NBK_EDEFECT))
        return hist, {k: getattr(res, k) for k, _ in CResult._fields_}

    def cg_solve_host_batch(self, f_hosts, niter: int, precision: str = "fp32", x_hosts=None):
        """nbk_cg_solve_host_batch: RHS f_hosts[k] -> solution x_hosts[k] (host arrays,
        pinned for overlapped copies); returns (hist[nrhs, niter+1], [result dicts])."""
        k = len(f_hosts)
        fs = [np.ascontiguousarray(f, dtype=np.float64) for f in f_hosts]
        fp = (ctypes.c_void_p * k)(*[_ptr(f) for f in fs])
        xp = None
        if x_hosts is not None:
            xp = (ctypes.c_void_p * k)(*[_ptr(x) for x in x_hosts])
        hist = np.zeros((k, niter + 1))
        res = (CResult * k)()
        st = self.lib.nbk_cg_solve_host_batch(self._ctx, k, fp, niter, PREC[precision], xp, _ptr(hist), res)
        _check(st, self._ctx, ok=(NBK_OK, NBK_EDEFECT))
        return hist, [{n: getattr(r, n) for n, _ in CResult._fields_} for r in res]

    def solution(self) -> np.ndarray:
        x = np.zeros(self.shape)
        _check(self.lib.nbk_get_solution(self._ctx, _ptr(x)), self._ctx)
        return x

    def solution_ptr(self, precision: str) -> int:
        p = ctypes.c_void_p(None)
        _check(self.lib.nbk_solution_ptr(self._ctx, PREC[precision], ctypes.byref(p)), self._ctx)
        return int(p.value)

    def solve_launches(self, niter: int, precision: str) -> int:
        n = ctypes.c_int64(0)
        _check(self.lib.nbk_solve_launches(self._ctx, niter, PREC[precision], ctypes.byref(n)),
               self._ctx)
        return int(n.value)


def cg_setup(mesh: MeshSpec, precision: str = "fp32", device: int = 0, stream=None,
             rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None) -> Context:
    return Context(mesh, precision, device, stream, rank, nranks, nccl_id)


class Group:
    """Virtual slabs: P contexts (rank r of P) of one mesh on one device and
    stream, linked in process (nbk_group_link) and driven together; the same
    kernels as NCCL mode run with faces / partials shared by pointer."""

    def __init__(self, mesh: MeshSpec, P: int, precision: str = "fp32", device: int = 0,
                 stream=None):
        import torch
        self.torch = torch
        self.lib = load()
        self.P = P
        self.stream = stream if stream is not None else torch.cuda.Stream(device=device)
        self.ctxs = [Context(mesh, precision, device, self.stream, rank=r, nranks=P)
                     for r in range(P)]
        self._arr = (ctypes.c_void_p * P)(*[c._ctx.value for c in self.ctxs])
        _check(self.lib.nbk_group_link(self._arr, P), self.ctxs[0]._ctx)
        self.n_global = self.ctxs[0].n_global

    def close(self):
        for c in self.ctxs:
            c.close()

    def sync(self):
        self.stream.synchronize()

    def _ptrs(self, ts):
        assert len(ts) == self.P
        return (ctypes.c_void_p * self.P)(*[t.data_ptr() for t in ts])

    def load_arrays(self, D, G_slabs, f_slabs):
        for c, G, f in zip(self.ctxs, G_slabs, f_slabs):
            c.load_arrays(D, G, f)

    def ax_apply(self, us, ws, flags: int = AX_DSSUM | AX_MASK):
        prec = Context._prec_of(us[0])
        cur = self.ctxs[0]._enter()
        _check(self.lib.nbk_group_ax_apply(self._arr, self.P, self._ptrs(us), self._ptrs(ws),
                                           flags, PREC[prec]), self.ctxs[0]._ctx)
        self.ctxs[0]._leave(cur, *us, *ws)
        return ws

    def dssum(self, fs, apply_mask: bool = False):
        prec = Context._prec_of(fs[0])
        cur = self.ctxs[0]._enter()
        _check(self.lib.nbk_group_dssum(self._arr, self.P, self._ptrs(fs), int(apply_mask),
                                        PREC[prec]), self.ctxs[0]._ctx)
        self.ctxs[0]._leave(cur, *fs)
        return fs

    def glsc3(self, a_s, b_s) -> float:
        prec = Context._prec_of(a_s[0])
        out = ctypes.c_double(0.0)
        self.ctxs[0]._enter()
        _check(self.lib.nbk_group_glsc3(self._arr, self.P, self._ptrs(a_s), self._ptrs(b_s),
                                        PREC[prec], ctypes.byref(out)), self.ctxs[0]._ctx)
        return float(out.value)

    def cg_solve(self, niter: int, precision: str = "fp32", trace: bool = True):
        hist = np.zeros(niter + 1)
        tr = np.zeros((niter, 5)) if trace else None
        res = CResult()
        st = self.lib.nbk_group_cg_solve(self._arr, self.P, niter, PREC[precision], _ptr(hist),
                                         _ptr(tr) if trace else None, ctypes.byref(res))
        _check(st, self.ctxs[0]._ctx, ok=(NBK_OK, NBK_EDEFECT))
        return hist, tr, {k: getattr(res, k) for k, _ in CResult._fields_}

    def solution(self) -> np.ndarray:
        return np.concatenate([c.solution() for c in self.ctxs], axis=0)

    # (precision emulation runs on one rank: Group has no set_emulation)

    def set_precond(self, precond: str):
        for c in self.ctxs:
            c.set_precond(precond)

    def load_precond(self, dinv_slabs):
        for c, d in zip(self.ctxs, dinv_slabs):
            c.load_precond(d)


def version() -> str:
    return load().nbk_version().decode()
