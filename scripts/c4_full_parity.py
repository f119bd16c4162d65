"""C4 at its stated 100 steps on the WHOLE 768^3 grid against the oracle's whole-grid run
("one full-grid 100-step oracle comparison ... recorded in profiles/r02/").
The oracle needs ~54 GB of host memory and ~20 min on 16 cores, too long for the driver's
test step, so it runs here (under gpurun) and writes gpurun_out/c4_full_parity.json."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import harness as H
import oracle
from icgen import configs

torch.cuda.set_device(0)
w = configs.C4()
t0 = time.time()
g, kmax = H.gpu_field(w, "c64", with_kmax=True)
dt = 0.8 * kmax
S = H.gpu_solver(w, "c64")
S.rk4(g, dt, w["steps"])
torch.cuda.synchronize()
got = g.cpu().numpy()
S.close()
del g
torch.cuda.empty_cache()
t_gpu = time.time() - t0
psi = H.psi0_host(w, "c64").astype(np.complex128)
t1 = time.time()
ref = oracle.rk4(H.oracle_problem(w), psi, dt, w["steps"])
t_orc = time.time() - t1
del psi
d = np.abs(got.astype(np.complex128) - ref)
out = {"config": "C4 768^3 complex64, Dirichlet, 100 steps, dt = 0.8 kmax (oracle, whole grid)",
       "dt": dt, "kmax": kmax, "points": int(ref.size),
       "rel_l2": float(np.sqrt((d ** 2).sum() / (np.abs(ref) ** 2).sum())),
       "max_abs": float(d.max()), "max_rel_to_max": float(d.max() / np.abs(ref).max()),
       "tol": 1e-5, "oracle_seconds": t_orc, "oracle_threads": oracle.set_threads(0), "gpu_phase_seconds": t_gpu}
out["pass"] = out["rel_l2"] <= 1e-5 and out["max_rel_to_max"] <= 1e-5
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/c4_full_parity.json", "w"), indent=1)
print(json.dumps(out))
