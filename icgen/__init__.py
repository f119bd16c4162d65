"""Seeded synthetic input generator (initial states Psi0, potentials V).

Input generation only — this package holds none of the 2SHOC/RK4 arithmetic, so it
may serve both the CPU oracle (``oracle/``) and the harness that drives the CUDA
library (``tests/``, ``bench.py``).  The C implementation is ``icgen.c``; this
module is ctypes marshalling plus the workload table in ``configs.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libicgen.so")

ICG_NOISE, ICG_BRIGHT_SECH, ICG_DARK_TANH, ICG_TF_VORTEX2D = 0, 1, 2, 3
ICG_TF_RING3D, ICG_GAUSS_NOISE, ICG_GAUSS_EXACT, ICG_SMOOTH_NOISE = 4, 5, 6, 7
ICG_DARK_MOVING = 8


class _Spec(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("dims", ctypes.c_int),
        ("n", ctypes.c_int64 * 3),
        ("xmin", ctypes.c_double * 3),
        ("h", ctypes.c_double * 3),
        ("seed", ctypes.c_uint64),
        ("p", ctypes.c_double * 8),
    ]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "icgen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "icgen.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", _SO, src, "-lm"]
        )
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.icg_uniform.restype = ctypes.c_double
        lib.icg_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]
        for fn in (lib.icg_fill_c128, lib.icg_fill_c64):
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.POINTER(_Spec), ctypes.c_int64 * 3, ctypes.c_int64 * 3, ctypes.c_void_p]
        lib.icg_harmonic.restype = ctypes.c_int
        lib.icg_harmonic.argtypes = [
            ctypes.c_int, ctypes.c_double * 3, ctypes.c_double * 3, ctypes.c_double * 3,
            ctypes.c_double * 3, ctypes.c_int64 * 3, ctypes.c_int64 * 3, ctypes.c_void_p,
        ]
        _lib = lib
    return _lib


def uniform(seed: int, stream: int, idx: int) -> float:
    return _load().icg_uniform(seed, stream, idx)


def _spec(ic: dict, grid: dict) -> _Spec:
    s = _Spec()
    s.kind = ic["kind"]
    s.dims = grid["dims"]
    n = list(grid["n"]) + [1] * (3 - len(grid["n"]))
    xmin = list(grid["xmin"]) + [0.0] * (3 - len(grid["xmin"]))
    h = list(grid["h"]) + [1.0] * (3 - len(grid["h"]))
    for d in range(3):
        s.n[d], s.xmin[d], s.h[d] = int(n[d]), float(xmin[d]), float(h[d])
    s.seed = int(ic.get("seed", 1))
    p = list(ic.get("p", [])) + [0.0] * (8 - len(ic.get("p", [])))
    for i in range(8):
        s.p[i] = float(p[i])
    return s


def _box(grid, lo, cnt):
    n = list(grid["n"]) + [1] * (3 - len(grid["n"]))
    lo = [0, 0, 0] if lo is None else list(lo) + [0] * (3 - len(lo))
    cnt = [n[d] - lo[d] for d in range(3)] if cnt is None else list(cnt) + [1] * (3 - len(cnt))
    return lo, cnt


def fill(ic: dict, grid: dict, dtype=np.complex128, lo=None, cnt=None, out=None) -> np.ndarray:
    """Psi0 over the box [lo, lo+cnt) (x,y,z order) of the global grid.

    Returns an array of shape (cnt_z, cnt_y, cnt_x) squeezed to ``dims`` axes, or
    fills ``out`` (a C-contiguous complex numpy array, or anything exposing
    ``data_ptr()`` with enough complex elements of ``dtype``)."""
    lib = _load()
    lo, cnt = _box(grid, lo, cnt)
    shape = tuple(int(c) for c in (cnt[2], cnt[1], cnt[0])[3 - grid["dims"]:])
    dtype = np.dtype(dtype)
    if out is None:
        arr = np.empty(shape, dtype=dtype)
        ptr = arr.ctypes.data
    elif isinstance(out, np.ndarray):
        arr = out
        assert arr.dtype == dtype and arr.flags.c_contiguous and arr.size == int(np.prod(cnt))
        ptr = arr.ctypes.data
    else:  # torch tensor (pinned host memory)
        arr = out
        ptr = out.data_ptr()
    spec = _spec(ic, grid)
    fn = lib.icg_fill_c128 if dtype == np.complex128 else lib.icg_fill_c64
    rc = fn(ctypes.byref(spec), (ctypes.c_int64 * 3)(*lo), (ctypes.c_int64 * 3)(*cnt), ctypes.c_void_p(ptr))
    if rc != 0:
        raise ValueError("icgen: bad box or spec")
    return arr


def harmonic(grid: dict, w, c=(0.0, 0.0, 0.0), lo=None, cnt=None) -> np.ndarray:
    """Materialise V = sum_d w_d (x_d - c_d)^2 in double over a box."""
    lib = _load()
    lo, cnt = _box(grid, lo, cnt)
    dims = grid["dims"]
    shape = tuple(int(v) for v in (cnt[2], cnt[1], cnt[0])[3 - dims:])
    V = np.empty(shape, dtype=np.float64)
    xmin = list(grid["xmin"]) + [0.0] * (3 - len(grid["xmin"]))
    h = list(grid["h"]) + [1.0] * (3 - len(grid["h"]))
    w = list(w) + [0.0] * (3 - len(w))
    c = list(c) + [0.0] * (3 - len(c))
    rc = lib.icg_harmonic(
        dims, (ctypes.c_double * 3)(*xmin), (ctypes.c_double * 3)(*h), (ctypes.c_double * 3)(*w),
        (ctypes.c_double * 3)(*c), (ctypes.c_int64 * 3)(*lo), (ctypes.c_int64 * 3)(*cnt),
        ctypes.c_void_p(V.ctypes.data),
    )
    if rc != 0:
        raise ValueError("icgen: bad harmonic box")
    return V
