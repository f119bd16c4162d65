"""Kernel timeline of a live nlse2shoc_rk4 call (CUPTI through torch.profiler, no ncu replay,
no cache flush): per-kernel durations and the idle gaps between consecutive kernels, to
compare with the serialised ncu launch list.
  python scripts/timeline.py C4 c64 [steps] [opt=val ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import icgen
import paper_1109_1027_b200 as nl
from icgen import configs

name, dtype = sys.argv[1], sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
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
S = nl.solver_from_work(w, dtype)
for kv in sys.argv[4:]:
    k, v = kv.split("=")
    S.set_variant(int(v)) if k == "variant" else S.set_option(k, int(v))
dt = 0.8 * S.stability_bound(psi)
S.rk4(psi, dt, steps)  # warm-up: instantiates the step graph
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); S.rk4(psi, dt, steps); e1.record(); torch.cuda.synchronize()
plain_ms = e0.elapsed_time(e1) / steps
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    S.rk4(psi, dt, steps)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "kernel" in e.name]
ev.sort(key=lambda e: e.time_range.start)
per = {}
gaps = []
for i, e in enumerate(ev):
    key = e.name.split("(")[0][-44:]
    per.setdefault(key, []).append(e.time_range.end - e.time_range.start)
    if i:
        gaps.append(e.time_range.start - ev[i - 1].time_range.end)
span = (ev[-1].time_range.end - ev[0].time_range.start) / steps
out = {"config": name, "dtype": dtype, "steps": steps, "opts": sys.argv[4:], "ms_per_step_events": plain_ms,
       "us_per_step_profiled_span": span, "kernels": {k: {"n": len(v), "avg_us": sum(v) / len(v)} for k, v in per.items()},
       "sum_kernel_us_per_step": sum(sum(v) for v in per.values()) / steps,
       "gap_us_avg": sum(gaps) / max(1, len(gaps)), "gap_us_max": max(gaps) if gaps else 0, "n_kernels": len(ev)}
print(json.dumps(out))
