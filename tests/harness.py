"""Test-side helpers: run a workload through the CUDA library and through the oracle on the
same seeded inputs.  (Test infrastructure: the only place both sides meet.)"""
from __future__ import annotations

import numpy as np

import icgen
import oracle

NP = {"c64": np.complex64, "c128": np.complex128}
TOL = {"c64": 1e-5, "c128": 1e-12}  # north star: max relative L2 after the stated steps


def torch_dtype(dt):
    import torch

    return torch.complex64 if dt == "c64" else torch.complex128


def psi0_host(work, dtype, lo=None, cnt=None):
    """Psi0 as the GPU sees it (rounded to complex64 for c64 runs, reading R19)."""
    return icgen.fill(work["ic"], work["grid"], dtype=NP[dtype], lo=lo, cnt=cnt)


def oracle_kmax_full(work, dtype, slab=64):
    """kmax of the whole grid from the oracle, computed slab by slab (min/max fold is exact)."""
    g = work["grid"]
    dims = g["dims"]
    nslow = g["n"][dims - 1]
    lo_all, hi_all = np.inf, -np.inf
    for z0 in range(0, nslow, slab):
        nz = min(slab, nslow - z0)
        lo = [0, 0, 0]
        cnt = list(g["n"])
        lo[dims - 1] = z0
        cnt[dims - 1] = nz
        psi = psi0_host(work, dtype, lo, cnt).astype(np.complex128)
        P = oracle.problem_from_work(work, lo=lo, cnt=cnt)
        a, b = oracle.N_minmax(P, psi)
        lo_all, hi_all = min(lo_all, a), max(hi_all, b)
    return oracle.kmax_from_N(dims, g["h"][:dims], work["a"], lo_all, hi_all)


def V_array_device(work, dtype):
    import torch

    V = icgen.harmonic(work["grid"], work["V"]["w"], work["V"]["c"])
    return torch.from_numpy(V.astype(np.float32 if dtype == "c64" else np.float64)).cuda()


def gpu_solver(work, dtype, variant=0, scheme="2shoc"):
    import paper_1109_1027_b200 as nl

    Varr = V_array_device(work, dtype) if work["V"]["kind"] == "array" else None
    S = nl.solver_from_work(work, dtype, V_array=Varr)
    if scheme != "2shoc":
        S.set_scheme(scheme)
    if variant:
        S.set_variant(variant)
    S._varr = Varr
    return S


def oracle_problem(work, lo=None, cnt=None, scheme="2shoc"):
    return oracle.problem_from_work(work, scheme=scheme, lo=lo, cnt=cnt)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def crop_box(work, target_lo, target_cnt, nsteps):
    """Dependency cone: after n steps a value depends only on Psi0 within L1 distance 8n
    (4 stages x radius 2; the face rule's tangential taps are at L1 distance 2 too)."""
    g = work["grid"]
    m = 8 * nsteps
    lo, cnt = [], []
    for d in range(3):
        if d >= g["dims"]:
            lo.append(0)
            cnt.append(1)
            continue
        a = max(0, target_lo[d] - m)
        b = min(g["n"][d], target_lo[d] + target_cnt[d] + m)
        lo.append(a)
        cnt.append(b - a)
    return lo, cnt


def sl(dims, lo, cnt):
    """numpy slice (z, y, x order) of box [lo, lo+cnt)."""
    s = [slice(lo[d], lo[d] + cnt[d]) for d in range(dims)]
    return tuple(reversed(s))
