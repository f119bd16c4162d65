"""Timing sweep of library variants on the C4 grid (768^3 c64, Dirichlet, harmonic V):
random smooth-ish input, dt from the library's bound, 20 RK4 steps, CUDA events."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1109_1027_b200 as nl
from icgen import configs
w = configs.C4()
S = nl.solver_from_work(w, "c64")
n = 768
torch.manual_seed(0)
psi = (torch.randn(n, n, n, dtype=torch.complex64, device="cuda") * 0.01 + 1.0)
dt = 0.8 * S.stability_bound(psi)
S.rk4(psi, dt, 3)
torch.cuda.synchronize()
res = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); S.rk4(psi, dt, 20); e1.record(); torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 20)
ms = min(res)
print(json.dumps({"lib": os.environ.get("NLSE_LIB", "default"), "ms_per_step": ms, "pt_steps_s": n**3 / ms * 1e3,
                  "finite": bool(torch.isfinite(torch.view_as_real(psi)).all())}))
