"""Soak run: thousands of consecutive RK4 steps (tens of thousands of stage launches through
the dynamic tile-schedule counters, the cached step graph and, for loopback slabs, the fused
exchange's arrival counters and epochs) — one call of N steps must equal two calls of N/2 to
the bit, stay finite and, for loopback slabs, raise no wait timeout.
  python scripts/soak.py [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import icgen
import paper_1109_1027_b200 as nl
from icgen import configs

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
torch.cuda.set_device(0)
for name, w, dtype, shard in [("C5W", configs.C5W(1), "c64", None), ("C5W", configs.C5W(1), "c64", {"loopback": 4}),
                              ("C3/4", configs.SMALL(2, (4096, 2048), "dirichlet", dtype="c128"), "c128", {"loopback": 3}),
                              ("C2", configs.C2(), "c128", None)]:
    g = w["grid"]
    dims = g["dims"]
    psi0 = torch.from_numpy(icgen.fill(w["ic"], g, dtype=np.complex64 if dtype == "c64" else np.complex128)).cuda()
    S = nl.solver_from_work(w, dtype, shard=shard)
    dt = 0.5 * S.stability_bound(psi0)
    a, b = psi0.clone(), psi0.clone()
    t0 = time.time()
    S.rk4(a, dt, N)
    torch.cuda.synchronize()
    t1 = time.time() - t0
    S.rk4(b, dt, N // 2)
    S.rk4(b, dt, N - N // 2)
    torch.cuda.synchronize()
    out = {"config": name, "dtype": dtype, "shard": shard, "steps": N, "seconds_one_call": round(t1, 3),
           "finite": bool(torch.isfinite(torch.view_as_real(a)).all()), "bitwise_equal_split": bool(torch.equal(a, b)),
           "exchange_timeouts": S.exchange_timeouts if shard else 0, "launches": S.last_launch_count}
    print(json.dumps(out), flush=True)
    S.close()
    del a, b, psi0
    torch.cuda.empty_cache()
