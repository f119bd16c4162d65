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


def oracle_crop_rk4(work, dtype, tlo, tcnt, dt, nsteps, segments=10):
    """The oracle's Psi after nsteps on the target box [tlo, tlo+tcnt), from runs on shrinking
    dependency-cone crops.  A crop with margin m around the target (true global faces kept
    where the target is closer than m to them) is exact at depth >= 8 t from its artificial
    faces after t steps (4 stages x radius 2, reading R8's tangential taps included), so
    after a segment of c steps it is cut to margin 8 (nsteps - t - c) and continued.  Every
    value inside the target is the full-grid oracle's, bit for bit (the oracle arithmetic is
    unchanged; only points that can no longer influence the target are dropped)."""
    dims = work["grid"]["dims"]
    seg = max(1, -(-nsteps // segments))
    lo, cnt = crop_box(work, tlo, tcnt, nsteps)
    psi = psi0_host(work, dtype, lo, cnt).astype(np.complex128)
    t = 0
    while t < nsteps:
        c = min(seg, nsteps - t)
        psi = oracle.rk4(oracle_problem(work, lo, cnt), psi, dt, c)
        t += c
        nlo, ncnt = crop_box(work, tlo, tcnt, nsteps - t)
        rel = [nlo[d] - lo[d] for d in range(3)]
        psi = np.ascontiguousarray(psi[sl(dims, rel, ncnt)])
        lo, cnt = nlo, ncnt
    return psi


def gpu_field(work, dtype, slab=64, with_kmax=False):
    """Psi0 of the whole grid on the device, generated slab by slab on the host, so that
    1536^3 fields never need a whole copy in host memory.  with_kmax: also return the
    oracle's k_max of the whole grid, folded from the same host slabs (min/max is exact)."""
    import torch

    g = work["grid"]
    dims = g["dims"]
    shape = tuple(reversed(g["n"][:dims]))
    out = torch.empty(shape, dtype=torch_dtype(dtype), device="cuda")
    lo_all, hi_all = np.inf, -np.inf
    nslow = g["n"][dims - 1]
    for z0 in range(0, nslow, slab):
        lo = [0, 0, 0]
        cnt = list(g["n"])
        lo[dims - 1] = z0
        cnt[dims - 1] = min(slab, nslow - z0)
        h = psi0_host(work, dtype, lo, cnt)
        out[z0:z0 + cnt[dims - 1]].copy_(torch.from_numpy(h.reshape((cnt[dims - 1],) + shape[1:])))
        if with_kmax:
            a, b = oracle.N_minmax(oracle.problem_from_work(work, lo=lo, cnt=cnt), h.astype(np.complex128))
            lo_all, hi_all = min(lo_all, a), max(hi_all, b)
    if with_kmax:
        return out, oracle.kmax_from_N(dims, g["h"][:dims], work["a"], lo_all, hi_all)
    return out


def compare(got, want, tol, what=""):
    """Relative L2 (the north star's measure) and the per-element max norm relative to the
    box's largest |Psi| (catches errors confined to a few points, e.g. a wrong ghost on one
    tile edge); both must be <= tol.  Each comparison is appended to $PARITY_LOG (JSON lines)
    when that is set, so the margins can be reported."""
    import os

    node = os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0]
    what = what or node
    got = np.asarray(got, dtype=np.complex128)
    want = np.asarray(want, dtype=np.complex128)
    if not np.any(want):
        # a region where the oracle is exactly zero (e.g. outside C3's Thomas-Fermi support):
        # relative measures are undefined, the GPU must be exactly zero too
        assert not np.any(got), (what, "oracle is zero here, GPU is not")
        what += " (zero region: exact)"
    rel = rel_l2(got, want)
    mx = float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))
    import json

    path = os.environ.get("PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"what": what, "rel_l2": rel, "max_rel": mx, "tol": tol, "points": int(want.size)}) + "\n")
    assert rel <= tol and mx <= tol, (what, rel, mx, tol)
    return rel, mx
