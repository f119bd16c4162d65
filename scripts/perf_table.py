"""Per-config single-GPU timing of nlse2shoc_rk4 (BASELINE.json configs C1-C5; informational,
the bench line is C4).  Input: the config's own Psi0 from icgen for configs up to 768^3, a
device-side smooth field for 1536^3 (values do not change the timing); dt = 0.8 kmax (C1: 0.4)
from the library's own bound.  CUDA events around one nlse2shoc_rk4 call of K steps."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import icgen
import paper_1109_1027_b200 as nl
from icgen import configs

def run(work, dtype, steps, variant=0, synthetic=False):
    g = work["grid"]; dims = g["dims"]
    shape = tuple(reversed(g["n"][:dims]))
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    if synthetic:
        psi = (torch.randn(shape, dtype=tdt, device="cuda") * 0.01 + 0.5)
    else:
        host = torch.empty(shape, dtype=tdt, pin_memory=True)
        icgen.fill(work["ic"], g, dtype=np.complex64 if dtype == "c64" else np.complex128, out=host.numpy())
        psi = host.cuda()
    S = nl.solver_from_work(work, dtype)
    if variant: S.set_variant(variant)
    frac = work["dt_rule"][1] if work["dt_rule"][0] == "kmax_frac" else None
    dt = frac * S.stability_bound(psi) if frac else work["dt_rule"][1]
    S.rk4(psi, dt, steps); torch.cuda.synchronize()  # warm-up with the timed dt and buffer (cached graph)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); S.rk4(psi, dt, steps); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    npts = int(np.prod(g["n"][:dims]))
    S_b = 8 if dtype == "c64" else 16
    r = {"config": work["name"], "dtype": dtype, "variant": {0: "fused", 1: "two_kernel", 4: "stage_pairs"}[variant], "grid": g["n"][:dims],
         "steps": steps, "ms_per_step": ms / steps, "pt_steps_s": npts * steps / ms * 1e3,
         "alg_GBs_12S": npts * steps * 12 * S_b / ms / 1e6, "alg_GBs_16S": npts * steps * 16 * S_b / ms / 1e6,
         "launches": S.last_launch_count}
    S.close(); del psi; torch.cuda.empty_cache()
    return r

only = sys.argv[1:] 
jobs = [("C1", configs.C1(), "c128", 2000, False), ("C2", configs.C2(), "c128", 200, False), ("C2", configs.C2(), "c64", 200, False),
        ("C3", configs.C3(), "c128", 40, False), ("C4", configs.C4(), "c64", 50, False),
        ("C5W", configs.C5W(1), "c64", 50, False), ("C5W", configs.C5W(1), "c128", 50, False),
        ("C5S", configs.C5(), "c64", 10, True), ("C4-2k", configs.C4(), "c64", 20, False),
        ("C4-pairs", configs.C4(), "c64", 20, False), ("C3-pairs", configs.C3(), "c128", 20, False)]
for name, w, dt, steps, syn in jobs:
    if only and name not in only: continue
    try:
        v = 1 if name.endswith("2k") else (4 if name.endswith("pairs") else 0)
        print(json.dumps(run(w, dt, steps, v, syn)), flush=True)
    except Exception as e:
        print(json.dumps({"config": name, "dtype": dt, "error": str(e)[:300]}), flush=True)
