"""One config, N RK4 steps with the given options (no CUDA graph, so every stage launch is a
plain kernel launch): the command profiled by ncu for launch lists.
  python scripts/one_step.py C4 c64 [steps] [opt=val ...]   (loopback=P: virtual slabs)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import icgen
import paper_1109_1027_b200 as nl
from icgen import configs

name, dtype = sys.argv[1], sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = {"C5W": lambda: configs.C5W(1), "C5S": configs.C5}.get(name, configs.ALL.get(name))()
g = w["grid"]
dims = g["dims"]
shape = tuple(reversed(g["n"][:dims]))
tdt = torch.complex64 if dtype == "c64" else torch.complex128
psi = torch.empty(shape, dtype=tdt, device="cuda")
nslow = g["n"][dims - 1]
for z0 in range(0, nslow, 64):
    lo, cnt = [0, 0, 0], list(g["n"])
    lo[dims - 1], cnt[dims - 1] = z0, min(64, nslow - z0)
    h = icgen.fill(w["ic"], g, dtype=np.complex64 if dtype == "c64" else np.complex128, lo=lo, cnt=cnt)
    psi[z0:z0 + cnt[dims - 1]].copy_(torch.from_numpy(h.reshape((cnt[dims - 1],) + shape[1:])))
kvs = [kv.split("=") for kv in sys.argv[4:]]
shard = {"loopback": int(v) for k, v in kvs if k == "loopback"} or None
S = nl.solver_from_work(w, dtype, shard=shard)
S.set_option("cuda_graph", 0)
for k, v in kvs:
    if k == "loopback":
        continue
    if k == "variant":
        S.set_variant(int(v))
    else:
        S.set_option(k, int(v))
dt = 0.8 * S.stability_bound(psi)
S.rk4(psi, dt, steps)
torch.cuda.synchronize()
print("done", name, dtype, steps, sys.argv[4:])
