"""Single-GPU proxy for the multi-GPU scaling curve: the same grid run as
one slab and as P = 2, 4, 8 virtual slabs of the loopback handle (the sharded code path: edge
/ interior split, seam tensor maps, halo copies, graph-captured edge-first step).  With P
GPUs each rank runs one slab, so T_P ~ T_loop(P) / P plus the NVLink halo time that the
edge-first schedule overlaps; the predicted efficiencies are
  strong (C4):  E_P ~ T_1 / T_loop(P)
  weak  (C5W):  E_P ~ T_1(768x768x192) / (T_loop(P) / P)  with the grid 768 x 768 x 192P
and the halo bytes per stage (2 planes each way) are reported for the NVLink estimate.
Writes one JSON line per (workload, P) to stdout."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import icgen
import paper_1109_1027_b200 as nl
from icgen import configs

torch.cuda.set_device(0)
K = int(os.environ.get("PROXY_STEPS", "20"))


def timed(work, dtype, shard, K):
    S = nl.solver_from_work(work, dtype, shard=shard)
    g = work["grid"]
    psi = torch.empty(tuple(reversed(g["n"][:3])), dtype=torch.complex64 if dtype == "c64" else torch.complex128,
                      device="cuda")
    for z0 in range(0, g["n"][2], 64):
        c = min(64, g["n"][2] - z0)
        h = icgen.fill(work["ic"], g, dtype=np.complex64 if dtype == "c64" else np.complex128, lo=[0, 0, z0],
                       cnt=[g["n"][0], g["n"][1], c])
        psi[z0:z0 + c].copy_(torch.from_numpy(h))
    dt = 0.8 * S.stability_bound(psi)
    S.rk4(psi, dt, K)  # warm-up with the timed call's dt and buffer: its step graph is cached
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S.rk4(psi, dt, K)
    e1.record()
    torch.cuda.synchronize()
    launches = S.last_launch_count
    S.close()
    del psi
    torch.cuda.empty_cache()
    return e0.elapsed_time(e1) / K, launches


for dtype in ("c64",):
    w = configs.C4()
    t1, l1 = timed(w, dtype, None, K)
    print(json.dumps({"workload": "C4", "dtype": dtype, "P": 1, "ms_per_step": t1, "launches_per_step": l1 / K}),
          flush=True)
    for P in (2, 4, 8):
        tp, lp = timed(w, dtype, {"loopback": P}, K)
        halo = 2 * 2 * 768 * 768 * 8  # bytes per stage per interior rank, both directions
        print(json.dumps({"workload": "C4", "dtype": dtype, "P": P, "ms_per_step_all_slabs": tp,
                          "launches_per_step": lp / K, "overhead_vs_single": tp / t1 - 1,
                          "predicted_strong_efficiency": t1 / tp,
                          "halo_bytes_per_stage_per_rank": halo,
                          "halo_us_at_900GBs": halo / 900e9 * 1e6,
                          "stage_us_per_rank_predicted": tp / 4 / P * 1e3}), flush=True)
for dtype in ("c64", "c128"):
    t1, _ = timed(configs.C5W(1), dtype, None, K)
    print(json.dumps({"workload": "C5W", "dtype": dtype, "P": 1, "ms_per_step": t1}), flush=True)
    for P in (2, 4, 8):
        tp, lp = timed(configs.C5W(P), dtype, {"loopback": P}, K)
        print(json.dumps({"workload": "C5W", "dtype": dtype, "P": P, "ms_per_step_all_slabs": tp,
                          "launches_per_step": lp / K, "predicted_weak_efficiency": t1 / (tp / P)}), flush=True)
