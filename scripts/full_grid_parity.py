"""A config at its stated step count on its WHOLE grid against the oracle's whole-grid run
(the driver's suite checks C3 / C4 / C5W on dependency-cone crop boxes, which are the
whole-grid oracle's values bit for bit inside each box; this gives the global numbers).
  python scripts/full_grid_parity.py C3 c128 | C5W c64 | C5W c128 | C4 c64
Needs host memory for 7 complex128 fields of the grid (C4: ~54 GB) and minutes of oracle time,
so it runs under gpurun, not in the test suite; writes gpurun_out/full_parity_<cfg>_<dtype>.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import harness as H
import oracle
from icgen import configs

name, dtype = sys.argv[1], sys.argv[2]
torch.cuda.set_device(0)
w = {"C5W": lambda: configs.C5W(1)}.get(name, configs.ALL.get(name))()
tol = H.TOL[dtype]
t0 = time.time()
g, kmax = H.gpu_field(w, dtype, with_kmax=True)
dt = 0.8 * kmax
S = H.gpu_solver(w, dtype)
S.rk4(g, dt, w["steps"])
torch.cuda.synchronize()
got = g.cpu().numpy()
S.close()
del g
torch.cuda.empty_cache()
t_gpu = time.time() - t0
psi = H.psi0_host(w, dtype).astype(np.complex128)
t1 = time.time()
ref = oracle.rk4(H.oracle_problem(w), psi, dt, w["steps"])
t_orc = time.time() - t1
del psi
d = np.abs(got.astype(np.complex128) - ref)
out = {"config": f"{w['name']} {'x'.join(map(str, w['grid']['n'][:w['grid']['dims']]))} {dtype}, {w['bc']}, "
                 f"{w['steps']} steps, dt = 0.8 kmax (oracle, whole grid)",
       "dt": dt, "kmax": kmax, "points": int(ref.size),
       "rel_l2": float(np.sqrt((d ** 2).sum() / (np.abs(ref) ** 2).sum())),
       "max_abs": float(d.max()), "max_rel_to_max": float(d.max() / np.abs(ref).max()),
       "tol": tol, "oracle_seconds": t_orc, "oracle_threads": oracle.set_threads(0), "gpu_phase_seconds": t_gpu}
out["pass"] = bool(out["rel_l2"] <= tol and out["max_rel_to_max"] <= tol)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/full_parity_{name}_{dtype}.json", "w"), indent=1)
print(json.dumps(out))
sys.exit(0 if out["pass"] else 1)
