"""A/B timing of execution-path options on the BASELINE configs (same library, same input):
  python scripts/ab_options.py C4:c64 C5W:c128 ... -- tile_schedule=0 tile_schedule=1
Each option set runs REPS x K steps (CUDA events, best and median per step), interleaved
across sets so that clock drift hits every set alike.  One JSON line per (config, set)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import icgen
import paper_1109_1027_b200 as nl
from icgen import configs

args = sys.argv[1:]
cut = args.index("--") if "--" in args else len(args)
cfgs, sets = args[:cut], [s.split(",") for s in args[cut + 1:]] or [[]]
K = int(os.environ.get("AB_STEPS", "20"))
REPS = int(os.environ.get("AB_REPS", "3"))
torch.cuda.set_device(0)


def work_of(name):
    return {"C5W": lambda: configs.C5W(1), "C5S": configs.C5}.get(name, configs.ALL.get(name))()


for cfg in cfgs:
    name, dtype = cfg.split(":")
    w = work_of(name)
    g = w["grid"]
    dims = g["dims"]
    shape = tuple(reversed(g["n"][:dims]))
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    psi0 = torch.empty(shape, dtype=tdt, device="cuda")
    nslow = g["n"][dims - 1]
    for z0 in range(0, nslow, 64):
        lo, cnt = [0, 0, 0], list(g["n"])
        lo[dims - 1], cnt[dims - 1] = z0, min(64, nslow - z0)
        h = icgen.fill(w["ic"], g, dtype=np.complex64 if dtype == "c64" else np.complex128, lo=lo, cnt=cnt)
        psi0[z0:z0 + cnt[dims - 1]].copy_(torch.from_numpy(h.reshape((cnt[dims - 1],) + shape[1:])))
    solvers = []
    for st in sets:
        kvs = dict(kv.split("=") for kv in st if kv)
        shard = {"loopback": int(kvs.pop("loopback"))} if "loopback" in kvs else None
        S = nl.solver_from_work(w, dtype, shard=shard)
        for k, v in kvs.items():
            if k == "variant":
                S.set_variant(int(v))
            elif hasattr(nl._lib.lib(), "nlse2shoc_set_option"):
                S.set_option(k, int(v))
        solvers.append(S)
    dt = 0.8 * solvers[0].stability_bound(psi0)
    psi = psi0.clone()
    times = [[] for _ in sets]
    outs = []
    for i, S in enumerate(solvers):
        S.rk4(psi, dt, K)  # same dt and buffer as the timed calls: their step graph is cached
    for rep in range(REPS):
        for i, S in enumerate(solvers):
            psi.copy_(psi0)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            S.rk4(psi, dt, K)
            e1.record()
            torch.cuda.synchronize()
            times[i].append(e0.elapsed_time(e1) / K)
            if rep == 0:
                outs.append(psi.clone() if psi.numel() * psi.element_size() < 8 << 30 else None)
    npts = int(np.prod(shape))
    for i, st in enumerate(sets):
        same = None
        if outs[0] is not None and outs[i] is not None:
            same = bool(torch.equal(torch.view_as_real(outs[i]), torch.view_as_real(outs[0])))
        print(json.dumps({"config": name, "dtype": dtype, "set": ",".join(st) or "default",
                          "ms_best": round(min(times[i]), 4), "ms_median": round(statistics.median(times[i]), 4),
                          "pt_steps_s": npts / min(times[i]) * 1e3, "bitwise_equal_to_first": same}), flush=True)
    for S in solvers:
        S.close()
    del psi, psi0, outs
    torch.cuda.empty_cache()
