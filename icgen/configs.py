"""Workload table: BASELINE.json configs C1-C5 and the paper's accuracy experiments,
as concrete seeded synthetic inputs (SURVEY.md §8(d) "Concrete inputs").

A workload is a plain dict: the grid, the NLSE parameters (a, s, V), the boundary
condition, the step count and the dt rule.  Nothing here evaluates the method; dt
is derived later from the stability bound (PAPER.md `kdfull`) by
whichever side (oracle or CUDA library) runs the workload.

No public dataset is involved: the paper's workloads are closed-form fields
 and BASELINE.json's C1-C5 are synthetic fields of the same family.
"""
from __future__ import annotations

import copy

from . import (ICG_BRIGHT_SECH, ICG_DARK_MOVING, ICG_DARK_TANH, ICG_GAUSS_EXACT, ICG_GAUSS_NOISE,
               ICG_NOISE, ICG_SMOOTH_NOISE, ICG_TF_RING3D, ICG_TF_VORTEX2D)

DIRICHLET, LAPZERO = "dirichlet", "lapzero"


def grid_inclusive(lo, hi, n):
    """Endpoints on the grid: h = (hi - lo)/(n - 1)."""
    dims = len(n)
    return {
        "dims": dims,
        "n": [int(v) for v in n] + [1] * (3 - dims),
        "xmin": [float(v) for v in lo] + [0.0] * (3 - dims),
        "h": [(hi[d] - lo[d]) / (n[d] - 1) for d in range(dims)] + [1.0] * (3 - dims),
    }


def grid_centred(n, h):
    dims = len(n)
    return {
        "dims": dims,
        "n": [int(v) for v in n] + [1] * (3 - dims),
        "xmin": [-(n[d] - 1) / 2.0 * h for d in range(dims)] + [0.0] * (3 - dims),
        "h": [float(h)] * dims + [1.0] * (3 - dims),
    }


def _w(name, grid, a, s, V, bc, steps, dtypes, dt_rule, ic, **extra):
    d = {"name": name, "grid": grid, "a": float(a), "s": float(s), "V": V, "bc": bc,
         "steps": int(steps), "dtypes": list(dtypes), "dt_rule": dt_rule, "ic": ic}
    d.update(extra)
    return d


V_NONE = {"kind": "none"}


def V_harm(w, dims):
    return {"kind": "harmonic", "w": [float(w)] * dims + [0.0] * (3 - dims), "c": [0.0, 0.0, 0.0]}


def C1():
    """1D bright soliton, c128, N=1024 on [-20,20], a=1, s=1, Dirichlet, 2000 steps,
    dt = 0.4 kmax; exact solution sqrt2 sech(x) e^{it}."""
    g = grid_inclusive([-20.0], [20.0], [1024])
    return _w("C1_bright_soliton_1d", g, 1.0, 1.0, V_NONE, DIRICHLET, 2000, ["c128"],
              ("kmax_frac", 0.4), {"kind": ICG_BRIGHT_SECH, "p": [2 ** 0.5, 1.0, 0.0]})


def C2():
    """1D dark soliton, N=2^22 on [-200,200], a=1, s=-1, Laplacian-zero, 500 steps."""
    g = grid_inclusive([-200.0], [200.0], [1 << 22])
    return _w("C2_dark_soliton_1d", g, 1.0, -1.0, V_NONE, LAPZERO, 500, ["c128", "c64"],
              ("kmax_frac", 0.8), {"kind": ICG_DARK_TANH, "p": [1e-3], "seed": 1})


def C3():
    """2D vortex lattice in a harmonic trap, 8192^2 on [-12,12]^2, c128, Dirichlet."""
    g = grid_inclusive([-12.0, -12.0], [12.0, 12.0], [8192, 8192])
    return _w("C3_vortex_lattice_2d", g, 0.5, -1.0, V_harm(0.5, 2), DIRICHLET, 200, ["c128"],
              ("kmax_frac", 0.8),
              {"kind": ICG_TF_VORTEX2D, "p": [20.0, 0.5, 4, -3.0, 6.0], "seed": 1})


def C4(n=768):
    """3D vortex ring, 768^3 on [-8,8]^3, c64, a=0.5, s=-1, V=r^2/2, Dirichlet, 100 steps."""
    g = grid_inclusive([-8.0] * 3, [8.0] * 3, [n] * 3)
    return _w("C4_vortex_ring_3d", g, 0.5, -1.0, V_harm(0.5, 3), DIRICHLET, 100, ["c64"],
              ("kmax_frac", 0.8),
              {"kind": ICG_TF_RING3D, "p": [15.0, 0.5, 3.0, 1e-3], "seed": 1})


def C5(n=(1536, 1536, 1536)):
    """3D Gaussian + noise, centred h=0.05, a=1, s=1, Laplacian-zero, 50 steps.
    (S) strong: 1536^3; (W) weak: 768 x 768 x 192P."""
    g = grid_centred(list(n), 0.05)
    return _w("C5_gaussian_3d", g, 1.0, 1.0, V_NONE, LAPZERO, 50, ["c64", "c128"],
              ("kmax_frac", 0.8), {"kind": ICG_GAUSS_NOISE, "p": [4.0, 0.01], "seed": 1})


def C5W(P=1):
    w = C5((768, 768, 192 * P))
    w["name"] = f"C5W_gaussian_3d_P{P}"
    return w


def EXP_GAUSS(dims, h, t_end=10.0):
    """PAPER.md Exp. 2/3: linear (s=0) Gaussian in V = r^2/a, a=1,
    Dirichlet on [-6,6]^d, k = 1e-3 (2D) / 5e-4 (3D), t = 10."""
    n = int(round(12.0 / h)) + 1
    g = grid_inclusive([-6.0] * dims, [6.0] * dims, [n] * dims)
    k = 1e-3 if dims == 2 else 5e-4
    steps = int(round(t_end / k))
    return _w(f"EXP{dims}_gauss_h{h}", g, 1.0, 0.0, V_harm(1.0, dims), DIRICHLET, steps,
              ["c128"], ("fixed", k), {"kind": ICG_GAUSS_EXACT, "p": [1.0, float(dims), 0.0]})


def EXP_DARK(h, lo=-25.5, hi=31.0, t_end=10.0):
    """PAPER.md Exp. 1: co-moving dark soliton `1dmds` with s = -1, a = 1,
    c = 0.5, Omega = -1, MSD boundary, k = 5e-4, t = 10.  Domain: reading R5 ([-25.5, 31];
    the paper says only 'large enough')."""
    n = int(round((hi - lo) / h)) + 1
    g = grid_inclusive([lo], [hi], [n])
    k = 5e-4
    return _w(f"EXP1_dark_h{h}", g, 1.0, -1.0, V_NONE, "msd", int(round(t_end / k)), ["c128"], ("fixed", k),
              {"kind": ICG_DARK_MOVING, "p": [0.5, -1.0, 1.0, -1.0, 0.0]})


def SMALL(dims, n, bc, dtype="c128", V="harmonic", noise=1e-2, seed=7, a=0.7, s=-0.9,
          steps=10, h=None):
    """Small ragged test grids for GPU<->oracle parity (nonzero noisy boundary values,
    anisotropic spacing allowed)."""
    nn = list(n)
    if h is None:
        h = [0.11, 0.13, 0.17][:dims]
    g = {"dims": dims, "n": nn + [1] * (3 - dims),
         "xmin": [-(nn[d] - 1) / 2.0 * h[d] for d in range(dims)] + [0.0] * (3 - dims),
         "h": list(h) + [1.0] * (3 - dims)}
    if V == "harmonic":
        Vd = {"kind": "harmonic", "w": [0.4, 0.3, 0.2][:dims] + [0.0] * (3 - dims),
              "c": [0.05, -0.07, 0.03]}
    elif V == "array":
        Vd = {"kind": "array", "w": [0.4, 0.3, 0.2][:dims] + [0.0] * (3 - dims),
              "c": [0.05, -0.07, 0.03]}
    else:
        Vd = V_NONE
    return _w(f"SMALL{dims}d_{'x'.join(map(str, nn))}_{bc}_{dtype}", g, a, s, Vd, bc, steps,
              [dtype], ("kmax_frac", 0.8),
              {"kind": ICG_SMOOTH_NOISE, "p": [noise, 0.02], "seed": seed})


def NOISE(dims, n, bc, amp=1.0, seed=3, a=1.0, s=-1.0):
    g = {"dims": dims, "n": list(n) + [1] * (3 - dims), "xmin": [0.0] * 3,
         "h": [0.1, 0.12, 0.15][:dims] + [1.0] * (3 - dims)}
    return _w("NOISE", g, a, s, V_NONE, bc, 1, ["c128"], ("kmax_frac", 0.8),
              {"kind": ICG_NOISE, "p": [amp, 0.0, 0.0], "seed": seed})


def crop(work: dict, lo, cnt) -> dict:
    """Same workload restricted to the box [lo, lo+cnt): coordinates and RNG indices are
    those of the global grid (icgen indexes noise by the global linear index)."""
    w = copy.deepcopy(work)
    g = w["grid"]
    w["crop"] = {"lo": list(lo), "cnt": list(cnt), "global_n": list(g["n"])}
    return w


ALL = {"C1": C1, "C2": C2, "C3": C3, "C4": C4, "C5": C5}
