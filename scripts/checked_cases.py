"""One small call of every kernel family (fused 2D/3D incl. lean / face-lean / general steps,
1D resident / tile / stream / MSD, two-kernel single- and multi-storage, stage pairs, CD,
loopback shards with the fused exchange).  Run against the checked build
(NLSE_LIB=paper_1109_1027_b200/libnlse2shoc_checked.so): it prints the number of out-of-range
stores the range checks caught; tests/test_gpu_checked.py requires 0.  (compute-sanitizer is
closed on the GPU pool, so these checks stand in for memcheck's store coverage.)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import icgen
import paper_1109_1027_b200 as nl
from icgen import configs

torch.cuda.set_device(0)


def run(dims, n, bc, dtype, V="harmonic", variant=0, shard=None, steps=2, lap=True, scheme=None, opts=()):
    w = configs.SMALL(dims, n, bc, dtype=dtype, V=V, noise=0.05)
    Varr = None
    if V == "array":
        Vh = icgen.harmonic(w["grid"], w["V"]["w"], w["V"]["c"])
        Varr = torch.from_numpy(Vh.astype(np.float32 if dtype == "c64" else np.float64)).cuda()
    S = nl.solver_from_work(w, dtype, V_array=Varr, shard=shard)
    if scheme:
        S.set_scheme(scheme)
    if variant:
        S.set_variant(variant)
    for k, v in opts:
        S.set_option(k, v)
    psi = torch.from_numpy(icgen.fill(w["ic"], w["grid"], dtype=np.complex64 if dtype == "c64" else np.complex128)).cuda()
    k = S.stability_bound(psi)
    S.rk4(psi, 0.5 * k, steps)
    if lap:
        S.laplacian(psi)
    torch.cuda.synchronize()
    S.close()
    print(f"ok {dims}D {n} {bc} {dtype} V={V} variant={variant} shard={shard} opts={opts}", flush=True)


# fused 3D (c64 tiles 64x24, c128 32x32): interior lean, face lean and general steps
run(3, (131, 51, 12), "dirichlet", "c64")
run(3, (131, 51, 12), "lapzero", "c64", variant=2)
run(3, (70, 67, 10), "dirichlet", "c128", variant=6)
run(3, (70, 67, 10), "lapzero", "c128", V="array")
run(3, (131, 51, 12), "dirichlet", "c64", opts=(("lean_steps", 0),))
# fused 2D (row tiles), odd-N_x complex64 staging
run(2, (2100, 9), "dirichlet", "c64")
run(2, (1037, 10), "lapzero", "c128", V="array")
run(2, (301, 12), "dirichlet", "c64")
# 1D: resident, tile, stream kernels, MSD
run(1, (1001,), "dirichlet", "c128", steps=4)
run(1, (5000,), "dirichlet", "c64", opts=(("resident_1d", 0),))
run(1, (20000,), "lapzero", "c128", opts=(("resident_1d", 0),))
w = configs.EXP_DARK(0.25)
S = nl.solver_from_work(w, "c128")
psi = torch.from_numpy(icgen.fill(w["ic"], w["grid"])).cuda()
S.rk4(psi, 5e-4, 4)
torch.cuda.synchronize()
S.close()
print("ok 1D MSD", flush=True)
# two-kernel (single- and multi-storage), stage pairs, CD scheme
run(3, (40, 30, 12), "dirichlet", "c64", variant=1)
run(3, (40, 30, 12), "lapzero", "c128", variant=3)
run(2, (300, 20), "dirichlet", "c128", variant=3)
run(3, (70, 40, 12), "dirichlet", "c64", variant=4)
run(2, (2100, 12), "lapzero", "c128", variant=4)
run(3, (40, 30, 12), "dirichlet", "c64", scheme="cd")
# sharded decomposition (loopback: halo copies, seam tensor maps, edge-first overlap)
run(3, (70, 30, 24), "dirichlet", "c64", shard={"loopback": 3})
run(3, (40, 33, 20), "lapzero", "c128", shard={"loopback": 2}, variant=1)
run(2, (600, 40), "dirichlet", "c64", shard={"loopback": 4})
run(3, (131, 51, 40), "lapzero", "c64", shard={"loopback": 8}, steps=3)
run(3, (70, 67, 30), "dirichlet", "c128", shard={"loopback": 3}, variant=6, steps=3)
run(3, (70, 30, 24), "dirichlet", "c64", shard={"loopback": 3}, opts=(("fused_exchange", 0),))
from paper_1109_1027_b200 import _lib

L = _lib.lib()
v = L.nlse2shoc_checked_violations() if hasattr(L, "nlse2shoc_checked_violations") else -1
print(f"library {L.nlse2shoc_version().decode()}", flush=True)
print(f"violations {v}", flush=True)
