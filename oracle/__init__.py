"""CPU oracle for the RK4 + 2SHOC NLSE step — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1109_1027_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle.c`` (plain C, IEEE double, no FMA contraction); this
module is ctypes marshalling.  See ``oracle.h`` for the paper passage each function
follows and DESIGN.md §3 for the readings of the paper it adopts.

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_pins.py`` (paper tables, closed forms, brute force) except the
Laplacian-zero boundary rule, whose only pins are closed forms (P14-type quartic test,
linearity/gauge properties): the paper prints no Laplacian-zero value
("parity unpinned by the paper" for that reading; R9).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]

BC = {"dirichlet": 0, "lapzero": 1, "msd": 2}
SCHEME = {"2shoc": 0, "cd": 1}


class _Problem(ctypes.Structure):
    _fields_ = [
        ("dims", ctypes.c_int),
        ("n", ctypes.c_int64 * 3),
        ("h", ctypes.c_double * 3),
        ("a", ctypes.c_double),
        ("s", ctypes.c_double),
        ("V", ctypes.c_void_p),
        ("bc", ctypes.c_int),
        ("scheme", ctypes.c_int),
    ]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    hdr = os.path.join(_HERE, "oracle.h")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(os.path.getmtime(src), os.path.getmtime(hdr)):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO, src, "-lm"])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.POINTER(_Problem)
        for name in ("orc_laplacian", "orc_rhs"):
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [P, ctypes.c_void_p, ctypes.c_void_p]
        lib.orc_rk4.restype = ctypes.c_int
        lib.orc_rk4.argtypes = [P, ctypes.c_void_p, ctypes.c_double, ctypes.c_int64]
        lib.orc_N_minmax.restype = ctypes.c_int
        lib.orc_N_minmax.argtypes = [P, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        lib.orc_kmax_from_N.restype = ctypes.c_double
        lib.orc_kmax_from_N.argtypes = [ctypes.c_int, ctypes.c_double * 3, ctypes.c_double, ctypes.c_double, ctypes.c_double]
        lib.orc_kmax.restype = ctypes.c_double
        lib.orc_kmax.argtypes = [P, ctypes.c_void_p]
        lib.orc_table2_G.restype = ctypes.c_int
        lib.orc_table2_G.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        lib.orc_set_threads.restype = ctypes.c_int
        lib.orc_set_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


class Problem:
    """Grid + NLSE parameters for the oracle.  ``V`` is a float64 array of the grid's
    shape (materialised potential) or None for V = 0."""

    def __init__(self, dims, n, h, a, s, V=None, bc="dirichlet", scheme="2shoc"):
        self.dims = int(dims)
        self.n = [int(v) for v in list(n)[:dims]] + [1] * (3 - dims)
        self.h = [float(v) for v in list(h)[:dims]] + [1.0] * (3 - dims)
        self.a, self.s = float(a), float(s)
        self.shape = tuple(self.n[d] for d in reversed(range(dims)))
        self.V = None if V is None else np.ascontiguousarray(V, dtype=np.float64).reshape(self.shape)
        self.bc = bc
        self.scheme = scheme

    def _c(self):
        p = _Problem()
        p.dims = self.dims
        for d in range(3):
            p.n[d] = self.n[d]
            p.h[d] = self.h[d]
        p.a, p.s = self.a, self.s
        p.V = None if self.V is None else self.V.ctypes.data
        p.bc = BC[self.bc]
        p.scheme = SCHEME[self.scheme]
        return p

    def _field(self, psi):
        arr = np.ascontiguousarray(np.asarray(psi, dtype=np.complex128).reshape(self.shape))
        return arr


def laplacian(P: Problem, psi) -> np.ndarray:
    x = P._field(psi)
    out = np.empty_like(x)
    p = P._c()
    if _load().orc_laplacian(ctypes.byref(p), x.ctypes.data, out.ctypes.data):
        raise ValueError("oracle: invalid problem")
    return out


def rhs(P: Problem, psi) -> np.ndarray:
    x = P._field(psi)
    out = np.empty_like(x)
    p = P._c()
    if _load().orc_rhs(ctypes.byref(p), x.ctypes.data, out.ctypes.data):
        raise ValueError("oracle: invalid problem")
    return out


def rk4(P: Problem, psi, dt: float, nsteps: int) -> np.ndarray:
    x = P._field(psi).copy()
    p = P._c()
    if _load().orc_rk4(ctypes.byref(p), x.ctypes.data, float(dt), int(nsteps)):
        raise ValueError("oracle: invalid problem / dt / nsteps")
    return x


def N_minmax(P: Problem, psi):
    x = P._field(psi)
    lo, hi = ctypes.c_double(), ctypes.c_double()
    p = P._c()
    if _load().orc_N_minmax(ctypes.byref(p), x.ctypes.data, ctypes.byref(lo), ctypes.byref(hi)):
        raise ValueError("oracle: invalid problem")
    return lo.value, hi.value


def kmax_from_N(dims, h, a, nmin, nmax) -> float:
    hh = [float(v) for v in list(h)[:dims]] + [1.0] * (3 - dims)
    return _load().orc_kmax_from_N(int(dims), (ctypes.c_double * 3)(*hh), float(a), float(nmin), float(nmax))


def kmax(P: Problem, psi) -> float:
    x = P._field(psi)
    p = P._c()
    return _load().orc_kmax(ctypes.byref(p), x.ctypes.data)


def table2_G(d: int):
    buf = (ctypes.c_int * 20)()
    n = _load().orc_table2_G(int(d), buf)
    return [buf[i] for i in range(n)]


# ----------------------------------------------------------------------------------
# Workload plumbing (icgen configs -> oracle Problem).  No method arithmetic here.

def problem_from_work(work: dict, scheme: str = "2shoc", lo=None, cnt=None) -> Problem:
    """Oracle Problem for a workload dict (icgen.configs), optionally on a crop box."""
    import icgen

    g = work["grid"]
    dims = g["dims"]
    if lo is None:
        lo = [0, 0, 0]
        cnt = list(g["n"])
    lo = list(lo) + [0] * (3 - len(lo))
    cnt = list(cnt) + [1] * (3 - len(cnt))
    V = None
    if work["V"]["kind"] in ("harmonic", "array"):
        V = icgen.harmonic(g, work["V"]["w"], work["V"]["c"], lo=lo, cnt=cnt)
    return Problem(dims, cnt[:dims], g["h"][:dims], work["a"], work["s"], V, work["bc"], scheme)


def set_threads(n: int = 0) -> int:
    """OpenMP threads of the oracle's point loops (n > 0 sets them); returns the count in effect."""
    return int(_load().orc_set_threads(int(n)))
