"""One small call of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): scripts/sanitize.sh runs this under each tool.  No oracle: the
sanitizer checks memory and synchronisation, parity is tests/'s job."""
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
print("all cases done", flush=True)
