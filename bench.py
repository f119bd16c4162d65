#!/usr/bin/env python
"""Benchmark: grid-point RK4 steps/s of the 2SHOC NLSE step (BASELINE.json metric).

Workload (N=1): C4 — 3D vortex ring, 768^3, complex64, Dirichlet, V = r^2/2 (BASELINE.json
configs[3]), the configuration the north star's >=70%-of-roofline target binds.  One bench
"step" = one full RK4 step (4 fused stage launches) over the whole grid.  N>1: the same
768^3 grid z-slab sharded over N ranks (strong scaling, per-stage 2-plane NCCL halo).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Timing: W untimed warm-up steps, then K steps inside one nlse2shoc_rk4 call bracketed by a
barrier + cuda synchronize, CUDA events on the launching stream, max over ranks.  Every
field (3.4 GiB) is far larger than L2 (126 MB), so no L2 flush is needed.
`--impl reference` times the CPU oracle on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-point RK4 steps/s (2SHOC NLSE)"
UNIT = "pt-steps/s"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return int(os.environ.get("RANK", "0")), ws, int(os.environ.get("LOCAL_RANK", "0"))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def profile_traffic():
    p = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu):
        self.gpu, self.proc = gpu, None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sms.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sms:
            return None
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sms)}


def oracle_sample(work, steps_per_call, box=96):
    """Time the CPU oracle on a centred box of the workload (bounded sample)."""
    import numpy as np

    import icgen
    import oracle

    g = work["grid"]
    n = g["n"]
    lo = [max(0, (n[d] - box) // 2) if d < g["dims"] else 0 for d in range(3)]
    cnt = [min(box, n[d]) if d < g["dims"] else 1 for d in range(3)]
    psi = icgen.fill(work["ic"], g, dtype=np.complex64, lo=lo, cnt=cnt).astype(np.complex128)
    P = oracle.problem_from_work(work, lo=lo, cnt=cnt)
    dt = 0.8 * oracle.kmax(P, psi)
    t0 = time.perf_counter()
    oracle.rk4(P, psi, dt, steps_per_call)
    t = time.perf_counter() - t0
    pts = int(np.prod([cnt[d] for d in range(g["dims"])]))
    return pts, t, f"C4 centred {'x'.join(str(c) for c in cnt[:g['dims']])} box, {steps_per_call} RK4 step(s), oracle in double"


def cores():
    """OpenMP threads the oracle actually runs with."""
    import oracle

    return oracle.set_threads(0)


def host_info():
    """CPU model, sockets and logical CPUs of the box the oracle runs on."""
    model, sockets = None, set()
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name") and model is None:
                model = ln.split(":", 1)[1].strip()
            elif ln.startswith("physical id"):
                sockets.add(ln.split(":", 1)[1].strip())
    except OSError:
        pass
    return {"cpu_model": model, "sockets": len(sockets) or None, "nproc": os.cpu_count()}


def cpu_baseline_line(work, box):
    """The oracle on all host cores (box^3 sample) and on one core (a smaller sample)."""
    import oracle

    nth = oracle.set_threads(0)
    pts, tcpu, desc = oracle_sample(work, 1, box=box)
    oracle.set_threads(1)
    p1, t1, d1 = oracle_sample(work, 1, box=max(16, box // 2))
    oracle.set_threads(nth)
    return {"value": pts / tcpu, "unit": UNIT, "cores": nth, "kind": "oracle", "sample": desc,
            "value_1core": p1 / t1, "sample_1core": d1, **host_info()}


def run_reference(args):
    rank, ws, _ = dist_env()
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo", init_method="env://")
        if rank != 0:
            dist.barrier()
            dist.destroy_process_group()
            return
    from icgen import configs

    work = configs.C4()
    box = int(os.environ.get("NLSE_REF_BOX", "96"))
    for _ in range(args.warmup):
        oracle_sample(work, 1, box=min(box, 48))
    tot_pts, tot_t, desc = 0, 0.0, ""
    for _ in range(args.steps):
        pts, t, desc = oracle_sample(work, 1, box=box)
        tot_pts += pts
        tot_t += t
    value = tot_pts / tot_t
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "C4_vortex_ring_3d (BASELINE configs[3]) sample", "grid": [768, 768, 768],
                       "sample": desc},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "oracle", "sample": desc,
                             **host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


def run_ours(args):
    import numpy as np
    import torch

    import paper_1109_1027_b200 as nl
    from icgen import configs

    rank, ws, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    shard = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(nl.nlse2shoc_get_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        shard = {"uid": bytes(uid.cpu().numpy().tobytes()), "rank": rank, "nranks": ws}

    import icgen

    work = configs.C4()
    dtype = "c64"
    S = nl.solver_from_work(work, dtype, shard=shard)
    g = work["grid"]
    npts_global = int(np.prod(g["n"][:3]))
    lshape = S.local_shape
    lo = [0, 0, S.z0]
    cnt = [g["n"][0], g["n"][1], S.nz]
    host = torch.empty(lshape, dtype=torch.complex64, pin_memory=True)
    icgen.fill(work["ic"], g, dtype=np.complex64, lo=lo, cnt=cnt, out=host.numpy())
    psi = host.cuda()
    kmax = S.stability_bound(psi)
    dt = 0.8 * kmax

    def barrier():
        if dist is not None:
            dist.barrier()

    stream = torch.cuda.current_stream()
    # warm-up
    S.rk4(psi, dt, max(args.warmup, 1))
    torch.cuda.synchronize()
    barrier()
    # timed: K RK4 steps in one public call
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        S.rk4(psi, dt, args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = S.last_launch_count
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = npts_global * args.steps / (ms / 1e3)

    # end-to-end through the public API with HOST buffers: H2D(Psi0) + rk4(K) + D2H(Psi)
    out_host = torch.empty(lshape, dtype=torch.complex64, pin_memory=True)  # empty_like would not pin
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    f0.record(stream)
    psi.copy_(host, non_blocking=True)
    S.rk4(psi, dt, args.steps)
    out_host.copy_(psi, non_blocking=True)
    f1.record(stream)
    torch.cuda.synchronize()
    ems = f0.elapsed_time(f1)
    te = torch.tensor([ems], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    ems = float(te.item())
    nbytes = host.numel() * host.element_size() * ws

    S_bytes = 8
    # the fused default's own minimum traffic: 13 complex transfers per point-step
    # (write-light form, stages 2 / 3 / 3 / 5); SURVEY §8(d) counts 16 for the
    # explicit-accumulator form, reported beside it as achieved_16S_equiv
    transfers = 13
    alg_bytes_per_launch = transfers / 4 * S_bytes * npts_global / ws
    launch_ms = ms / (4 * args.steps)
    achieved = alg_bytes_per_launch / (launch_ms / 1e3) / 1e9
    peak, peak_kind = peaks()
    tr = profile_traffic()
    traffic = None
    if tr and tr.get("workload") == "C4" and tr.get("dram_bytes_per_point_stage"):
        traffic = tr["dram_bytes_per_point_stage"] * npts_global / ws
    clocks = clk.summary()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c64 (fp32 pairs)", "data": "synthetic",
            "config": {"workload": "C4_vortex_ring_3d (BASELINE configs[3])", "grid": g["n"][:3],
                       "bc": "dirichlet", "V": "harmonic 0.5 r^2", "dt": dt, "kmax": kmax,
                       "parallelism": f"z-slab x{ws}" if ws > 1 else "single GPU",
                       "l2": "inputs (3.4 GiB per field) >> L2 (126 MB); no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "alg_bytes_per_point_step": transfers * S_bytes,
                         "achieved_16S_equiv": achieved * 16 / transfers,
                         "frac_of_8TBs": achieved / 8000.0,
                         "kernel": "stage_stream_kernel<3,float,*> (avg over the 4 stage launches)"},
            "e2e": {"value": npts_global * args.steps / (ems / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": nbytes / args.steps, "d2h_bytes_per_step": nbytes / args.steps,
                    "note": "per job of K steps: H2D(Psi0 pinned) + nlse2shoc_rk4(K) + D2H(Psi)"},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_line(work, int(os.environ.get("NLSE_REF_BOX", "96")))
        print(json.dumps(line), flush=True)
    S.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
