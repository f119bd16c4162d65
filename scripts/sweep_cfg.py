"""Time nlse2shoc_rk4 on one BASELINE config with whatever library NLSE_LIB points at
(sweeps over compile-time presets): smooth random input, dt from the library's bound,
best of 3 x K steps, CUDA events.  python scripts/sweep_cfg.py C3 c128 [K]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1109_1027_b200 as nl
from icgen import configs

name, dtype = sys.argv[1], sys.argv[2]
K = int(sys.argv[3]) if len(sys.argv) > 3 else 20
w = {"C5W": lambda: configs.C5W(1)}.get(name, configs.ALL.get(name))()
g = w["grid"]
dims = g["dims"]
shape = tuple(reversed(g["n"][:dims]))
S = nl.solver_from_work(w, dtype)
variant = int(os.environ.get("NLSE_VARIANT", "0"))
if variant:
    S.set_variant(variant)
torch.manual_seed(0)
tdt = torch.complex64 if dtype == "c64" else torch.complex128
psi = torch.randn(shape, dtype=tdt, device="cuda") * 0.01 + 1.0
dt = 0.5 * S.stability_bound(psi)
S.rk4(psi, dt, 3)
torch.cuda.synchronize()
res = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); S.rk4(psi, dt, K); e1.record(); torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / K)
ms = min(res)
n = 1
for v in shape: n *= v
print(json.dumps({"lib": os.path.basename(os.environ.get("NLSE_LIB", "default")), "config": name, "dtype": dtype, "variant": variant,
                  "ms_per_step": round(ms, 4), "pt_steps_s": n / ms * 1e3,
                  "finite": bool(torch.isfinite(torch.view_as_real(psi)).all())}))
