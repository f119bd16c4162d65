"""Seeded random sweep of small problems through the CUDA library against the oracle: random
dims / sizes around tile multiples / BC / potential kind / dtype / variant / scheme, combined
with random execution-path options (lean steps, tile schedule, z-chunks, short end chunks,
CUDA graph, check_every, caller-owned workspace, padded layout, loopback slabs with either
exchange).  One JSON line per case; exits 1 if any case exceeds the north-star tolerance, or,
under the range-checked build (NLSE_LIB=.../libnlse2shoc_checked.so), if any store of the
2D/3D stage kernels fell outside its buffer.
  python scripts/fuzz_parity.py [ncases] [seed]"""
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import harness as H
import oracle
import paper_1109_1027_b200 as nl
from icgen import configs

ncases = int(sys.argv[1]) if len(sys.argv) > 1 else 120
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
torch.cuda.set_device(0)
TILE = {"c64": (64, 24), "c128": (32, 32)}
bad = 0
for case in range(ncases):
    dims = rng.choice([1, 2, 2, 3, 3, 3])
    dtype = rng.choice(["c64", "c128"])
    TX, TY = TILE[dtype]
    if dims == 1:
        n = (rng.choice([5, 9, 300, 5000, 16385 + rng.randrange(3000), 40000 + rng.randrange(999)]),)
    elif dims == 2:
        n = (rng.choice([5, 7, 130, 511, 512, 513, 1037, 2100]) + rng.randrange(3), rng.choice([5, 6, 9, 33, 70]))
    else:
        n = (rng.choice([5, 33, TX - 1, TX, TX + 1, 2 * TX - 1, 2 * TX + 2, 131]), rng.choice([5, 7, TY - 1, TY + 1, 2 * TY, 2 * TY + 1, 51]),
             rng.choice([5, 6, 9, 13, 20, 35]))
    bc = rng.choice(["dirichlet", "lapzero"])
    V = rng.choice(["harmonic", "array", "none"])
    scheme = rng.choice(["2shoc", "2shoc", "2shoc", "cd"])
    variant = rng.choice([0, 0, 0, 2, 5, 6, 1, 3, 4])
    if scheme == "cd" and variant in (1, 3):
        variant = 0
    if variant == 4 and (dims == 1 or min(n) < 6):
        variant = 0
    aniso = rng.random() < 0.6
    w = configs.SMALL(dims, n, bc, dtype=dtype, V=V, noise=rng.choice([1e-2, 0.1]), seed=rng.randrange(1, 99),
                      h=None if aniso else [0.12] * dims)
    nslow = n[-1]
    shard = None
    if dims >= 2 and variant in (0, 2, 5, 6) and nslow >= 9 and rng.random() < 0.3:
        shard = {"loopback": rng.choice([2, 3])}
    opts = {}
    if rng.random() < 0.5:
        opts = {k: v for k, v in {"lean_steps": rng.choice([0, 1, 2, 3]), "tile_schedule": rng.choice([0, 1]),
                                  "zchunks": rng.choice([0, 1, 3, 7]), "tail_chunks": rng.choice([0, 1]),
                                  "cuda_graph": rng.choice([0, 1]), "reverse_order": rng.choice([0, 1]),
                                  "fused_exchange": rng.choice([0, 1]), "overlap": rng.choice([0, 1])}.items()
                if rng.random() < 0.5}
    extra = rng.choice(["", "", "workspace", "padded", "check_every"])
    if shard and extra == "workspace":
        extra = ""
    nsteps = rng.choice([1, 3, 6])
    psi = H.psi0_host(w, dtype)
    P = H.oracle_problem(w, scheme=scheme)
    dt = 0.8 * oracle.kmax(P, psi.astype(np.complex128)) if scheme == "2shoc" else None
    Varr = H.V_array_device(w, dtype) if V == "array" else None
    S = nl.solver_from_work(w, dtype, V_array=Varr, shard=shard)
    if scheme != "2shoc":
        S.set_scheme(scheme)
    if variant:
        S.set_variant(variant)
    for k, v in opts.items():
        S.set_option(k, v)
    g = torch.from_numpy(psi).cuda()
    if dt is None:
        dt = 0.8 * S.stability_bound(g)
    keep = None
    if extra == "workspace":
        keep = torch.empty(S.stage_workspace_bytes, dtype=torch.uint8, device="cuda")
        S.set_workspace(keep)
    if extra == "check_every":
        S.set_option("check_every", 2)
    if extra == "padded":
        pitch, _ = S.padded_layout
        gp = torch.zeros(tuple(psi.shape[:-1]) + (pitch[0],), dtype=g.dtype, device="cuda")
        gp[..., :psi.shape[-1]] = g
        S.rk4_padded(gp, dt, nsteps)
        g = gp[..., :psi.shape[-1]].contiguous()
    else:
        S.rk4(g, dt, nsteps)
    torch.cuda.synchronize()
    got = g.cpu().numpy()
    ref = oracle.rk4(P, psi.astype(np.complex128), dt, nsteps)
    den = np.linalg.norm(ref)
    rel = float(np.linalg.norm(got - ref) / den) if den > 0 else float(np.abs(got).max())
    ok = bool(np.isfinite(got).all() and rel <= H.TOL[dtype])
    bad += not ok
    print(json.dumps({"case": case, "dims": dims, "n": n, "dtype": dtype, "bc": bc, "V": V, "scheme": scheme,
                      "variant": variant, "shard": shard, "opts": opts, "extra": extra, "steps": nsteps,
                      "rel_l2": rel, "ok": ok}), flush=True)
    S.close()
viol = int(nl._lib.lib().nlse2shoc_checked_violations())  # -1: not the range-checked build
print(json.dumps({"cases": ncases, "failed": bad, "checked_violations": viol}))
sys.exit(1 if bad or viol > 0 else 0)
