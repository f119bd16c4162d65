#!/usr/bin/env python
"""Measured counterpart of the paper's cost Tables 3-5.

The paper counts operations and storage of the Laplacian and of one RK4 step for the
non-compact scheme and the 2SHOC single-storage ("1X") and multi-storage ("2X"/"3X") forms.
Here each realisation in the library is timed on one B200 at a paper-sized workload:

  fused-12  variant 0: one kernel per stage, wide 2SHOC form (= the non-compact stencil in the
            interior), carried-sum combine (12 field transfers per point-step)
  fused-13  variant 5: as fused-12 with the write-light combine (13 transfers)
  fused-13r variant 6: as fused-12 with the reconstructed accumulator (13 transfers)
  fused-16  variant 2: as fused-12 with the explicit accumulator (16 transfers)
  2k-1X     variant 1: the paper's single-storage two-step scheme, D stored (`2d2shocs1/2`)
  2k-MS     variant 3: the paper's multi-storage scheme, D_d per axis stored (`*2shocMs1/2`)
  CD        scheme CD through fused-12 (`uttmp`, the 2nd-order comparison scheme)
  pairs     variant 4: two stages per pass (temporal blocking, stage_pair.cuh)

  python scripts/cost_tables.py                 # timing -> JSON lines on stdout
  python scripts/cost_tables.py --ncu           # 1 Laplacian + 1 RK4 step per row (run under ncu)
  python scripts/cost_tables.py --parse launches.csv order.json   # dram bytes per row

Storage = (Psi + the handle's workspace) / (N x bytes per point), the paper's "kN" column.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

ROWS = [("fused-12", 0, "2shoc"), ("fused-13", 5, "2shoc"), ("fused-13r", 6, "2shoc"), ("fused-16", 2, "2shoc"), ("2k-1X", 1, "2shoc"),
        ("2k-MS", 3, "2shoc"), ("CD", 0, "cd"), ("pairs", 4, "2shoc")]

# paper's static counts (Tables 3-5): (Laplacian ops, Laplacian storage, RK4 ops, RK4 storage)
PAPER = {
    1: {"non-compact": (7, 1, 69, 5), "2SHOC": (8, 2, 73, 6)},
    2: {"non-compact": (9, 1, 77, 5), "2SHOC 2X": (15, 3, 101, 7), "2SHOC 1X": (19, 2, 117, 6)},
    3: {"non-compact": (14, 1, 97, 5), "2SHOC 3X": (22, 4, 129, 8), "2SHOC 1X": (31, 2, 165, 6)},
}


def workloads():
    from icgen import configs

    return [(1, "C2 2^22 c128", configs.C2(), "c128"), (2, "C3 8192^2 c128", configs.C3(), "c128"),
            (3, "C4 768^3 c64", configs.C4(), "c64")]


def rows_for(dims):
    return [r for r in ROWS if not (dims == 1 and r[1] in (3, 4, 6))]  # 1D: MS == 1X; pairs 2D/3D


def run(ncu: bool, steps: int, reps: int, only):
    import numpy as np
    import torch

    import harness as H

    order = []
    for dims, wname, w, dtype in workloads():
        if only and dims not in only:
            continue
        g = w["grid"]
        npts = int(np.prod(g["n"]))
        S_b = 16 if dtype == "c128" else 8
        psi_h = H.psi0_host(w, dtype)
        for name, variant, scheme in rows_for(dims):
            S = H.gpu_solver(w, dtype, variant=variant, scheme=scheme)
            psi = torch.from_numpy(psi_h).cuda()
            L = torch.empty_like(psi)
            dt = 0.8 * S.stability_bound(psi)
            st = torch.cuda.current_stream()
            if ncu:
                S.laplacian(psi, out=L)
                nl = S.last_launch_count
                S.rk4(psi, dt, 1)
                nr = S.last_launch_count
                torch.cuda.synchronize()
                order.append({"dims": dims, "row": name, "lap_launches": nl, "rk4_launches": nr, "npts": npts})
                del S, psi, L
                torch.cuda.empty_cache()
                continue
            for _ in range(2):
                S.laplacian(psi, out=L)
            S.rk4(psi, dt, steps)  # same dt and buffer as the timed call: its step graph is cached
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            torch.cuda.synchronize()
            e[0].record(st)
            for _ in range(reps):
                S.laplacian(psi, out=L)
            e[1].record(st)
            e[2].record(st)
            S.rk4(psi, dt, steps)
            e[3].record(st)
            torch.cuda.synchronize()
            t_lap = e[0].elapsed_time(e[1]) / reps
            t_step = e[2].elapsed_time(e[3]) / steps
            ok = bool(torch.isfinite(torch.view_as_real(psi)).all())
            print(json.dumps({
                "dims": dims, "workload": wname, "row": name, "variant": variant, "scheme": scheme,
                "npts": npts, "bytes_per_pt": S_b,
                "storage_N": round(1 + S.workspace_bytes / (npts * S_b), 2),
                "lap_ms": round(t_lap, 4), "step_ms": round(t_step, 4),
                "pt_steps_per_s": npts / (t_step * 1e-3), "lap_pts_per_s": npts / (t_lap * 1e-3),
                "finite": ok,
            }), flush=True)
            del S, psi, L
            torch.cuda.empty_cache()
    if ncu:
        print("ORDER " + json.dumps(order), flush=True)


def parse(csv_path, order_path):
    """Assign the ncu launch list (in launch order) to the rows of order.json."""
    order = json.load(open(order_path))
    rows = list(csv.reader(open(csv_path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d[int(r[idi])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[idi])] = r[ki].split("(")[0]
    ids = sorted(d)
    # launches that are not the library's (torch fills, reductions) are skipped by name
    ids = [i for i in ids if any(k in names[i] for k in ("stage", "two_", "line", "resident", "pair"))]
    pos = 0
    out = []
    for o in order:
        # the stability bound's reduce_N kernel is filtered out; laplacian, then one RK4 step
        lap = ids[pos:pos + o["lap_launches"]]
        pos += o["lap_launches"]
        rk = ids[pos:pos + o["rk4_launches"]]
        pos += o["rk4_launches"]

        def tot(sel, m):
            return sum(d[i].get(m, 0.0) for i in sel)

        n = o["npts"]
        out.append({
            **o,
            "lap_dram_B_per_pt": (tot(lap, "dram__bytes_read.sum") + tot(lap, "dram__bytes_write.sum")) / n,
            "step_dram_B_per_pt": (tot(rk, "dram__bytes_read.sum") + tot(rk, "dram__bytes_write.sum")) / n,
            "lap_ncu_ms": tot(lap, "gpu__time_duration.sum") / 1e6,
            "step_ncu_ms": tot(rk, "gpu__time_duration.sum") / 1e6,
            "kernels": sorted({names[i] for i in lap + rk}),
        })
    for r in out:
        print(json.dumps(r))


def report(time_path, ncu_path, peaks_path):
    """Markdown table from the timing JSON lines and the parsed ncu JSON lines."""
    T = [json.loads(l) for l in open(time_path)]
    Nc = {(r["dims"], r["row"]): r for r in map(json.loads, open(ncu_path))}
    pk = json.load(open(peaks_path))["hbm_gbs"]
    out = ["| dims | workload | realisation | storage (N) | Laplacian ms | RK4 step ms | pt-steps/s | DRAM B/pt Lap | "
           "DRAM B/pt step | step GB/s (DRAM) | frac of HBM |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in T:
        n = Nc[(r["dims"], r["row"])]
        gbs = n["step_dram_B_per_pt"] * r["npts"] / (r["step_ms"] * 1e-3) / 1e9
        out.append(f"| {r['dims']} | {r['workload']} | {r['row']} | {r['storage_N']} | {r['lap_ms']:.3f} | "
                   f"{r['step_ms']:.3f} | {r['pt_steps_per_s']:.3e} | {n['lap_dram_B_per_pt']:.1f} | "
                   f"{n['step_dram_B_per_pt']:.1f} | {gbs:.0f} | {gbs / pk:.2f} |")
    out += ["", "Paper's static counts (Tables 3-5): Laplacian ops / storage, RK4 ops / storage", "",
            "| dims | scheme | Lap ops | Lap storage | RK4 ops | RK4 storage |", "|---|---|---|---|---|---|"]
    for d, rows in PAPER.items():
        for k, v in rows.items():
            out.append(f"| {d} | {k} | {v[0]} | {v[1]}N | {v[2]} | {v[3]}N |")
    print("\n".join(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--parse", nargs=2)
    ap.add_argument("--report", nargs=3, metavar=("TIME_JSONL", "NCU_JSONL", "PEAKS_JSON"))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--dims", type=int, nargs="*")
    a = ap.parse_args()
    if a.report:
        report(*a.report)
    elif a.parse:
        parse(*a.parse)
    else:
        run(a.ncu, a.steps, a.reps, a.dims)


if __name__ == "__main__":
    main()
