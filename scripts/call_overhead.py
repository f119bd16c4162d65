"""Per-call fixed cost of nlse2shoc_rk4 on C4: device time of rk4(K) for several K, first call
(captures + instantiates the step graph) and repeated call (replays the cached graph)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1109_1027_b200 as nl
from icgen import configs

torch.cuda.set_device(0)
w = configs.C4()
S = nl.solver_from_work(w, "c64")
torch.manual_seed(0)
psi = torch.randn(768, 768, 768, dtype=torch.complex64, device="cuda") * 0.01 + 1.0
for K in (4, 20, 100):
    for rep in ("first", "cached"):
        dt = 1e-5 * (1 + K) if rep == "first" else dt
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        e0.record()
        S.rk4(psi, dt, K)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"K": K, "call": rep, "ms_per_step": e0.elapsed_time(e1) / K}), flush=True)
