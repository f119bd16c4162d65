#!/usr/bin/env python
"""Benchmark: grid-point RK4 steps/s of the 2SHOC NLSE step (BASELINE.json metric).

Workload (default, N=1): C4 — 3D vortex ring, 768^3, complex64, Dirichlet, V = r^2/2
(BASELINE.json configs[3]), the configuration the north star's >=70%-of-roofline target
binds.  One bench "step" = one full RK4 step (4 fused stage launches) over the whole grid.
N>1: the same 768^3 grid z-slab sharded over N ranks (strong scaling, per-stage 2-plane NCCL
halo).  --workload C5W: the weak-scaling config (768 x 768 x 192 per GPU, 768 x 768 x 192N
in all, Laplacian-zero Gaussian, BASELINE configs[4]); C5S (1536^3, strong), C3 (8192^2
c128) and C2 (2^22, 1D) are the other parity configs, for the perf table.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload C4|C5W|C5S|C3|C2] [--dtype c64|c128]

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
WORKLOADS = {"C4": "C4_vortex_ring_3d (BASELINE configs[3])",
             "C5W": "C5W_gaussian_3d weak scaling 768x768x192 per GPU (BASELINE configs[4])",
             "C5S": "C5S_gaussian_3d 1536^3 (BASELINE configs[4])",
             "C3": "C3_vortex_lattice_2d 8192^2 (BASELINE configs[2])",
             "C2": "C2_dark_soliton_1d 2^22 (BASELINE configs[1])"}
KERNEL = {3: "stage_stream_kernel<3,{},*> (avg over the 4 stage launches)",
          2: "stage_stream_kernel<2,{},*> (avg over the 4 stage launches)",
          1: "line kernels <{}> (avg over the 4 stage launches)"}
UNIT = "pt-steps/s"
DTYPE_DEFAULT = {"C3": "c128", "C2": "c128"}


def workload(wl, ws):
    from icgen import configs

    return {"C4": configs.C4, "C5W": lambda: configs.C5W(ws), "C5S": configs.C5, "C3": configs.C3,
            "C2": configs.C2}[wl]()


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


def oracle_sample(work, steps_per_call, box=96, dtype="c64"):
    """Time the CPU oracle on a centred box of the workload (bounded sample; box = edge length
    in 3D, scaled to the same point count in 2D / 1D)."""
    import numpy as np

    import icgen
    import oracle

    g = work["grid"]
    n = g["n"]
    box = int(round(box ** (3.0 / g["dims"])))
    lo = [max(0, (n[d] - box) // 2) if d < g["dims"] else 0 for d in range(3)]
    cnt = [min(box, n[d]) if d < g["dims"] else 1 for d in range(3)]
    psi = icgen.fill(work["ic"], g, dtype=np.complex64 if dtype == "c64" else np.complex128, lo=lo,
                     cnt=cnt).astype(np.complex128)
    P = oracle.problem_from_work(work, lo=lo, cnt=cnt)
    dt = 0.8 * oracle.kmax(P, psi)
    t0 = time.perf_counter()
    oracle.rk4(P, psi, dt, steps_per_call)
    t = time.perf_counter() - t0
    pts = int(np.prod([cnt[d] for d in range(g["dims"])]))
    name = work["name"].split("_")[0]
    return pts, t, f"{name} centred {'x'.join(str(c) for c in cnt[:g['dims']])} box, {steps_per_call} RK4 step(s), oracle in double"


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


def calibrated_sample(work, box, seconds, max_steps=1000):
    """Oracle sample of about `seconds` of CPU work: a 3-step call on the box to estimate the
    rate, then as many steps (2 ... max_steps) in one call as fit the budget."""
    oracle_sample(work, 1, box=box)  # first touch: thread pool, page faults
    _, t3, _ = oracle_sample(work, 3, box=box)
    steps = int(min(max_steps, max(2, round(seconds / max(t3 / 3, 1e-6)))))
    pts, t, desc = oracle_sample(work, steps, box=box)
    return pts * steps, t, desc


def cpu_baseline_line(work, box):
    """The oracle as it stands on all host cores (a bounded sample of the workload: a centred
    box^3 box for about 12 s of CPU work) and on one core (a smaller box, about 4 s)."""
    import oracle

    nth = oracle.set_threads(0)
    pts, tcpu, desc = calibrated_sample(work, box, 12.0)
    oracle.set_threads(1)
    p1, t1, d1 = calibrated_sample(work, max(16, box // 2), 4.0)
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
    wl = args.workload
    work = workload(wl, ws)
    dtype = args.dtype or DTYPE_DEFAULT.get(wl, "c64")
    # one bench step of the reference arm = one oracle call of REF_STEPS RK4 steps on a centred
    # box^3 box of the workload (a bounded sample: about a second of CPU work per bench step)
    box = int(os.environ.get("NLSE_REF_BOX", "128"))
    ref_steps = int(os.environ.get("NLSE_REF_STEPS", "32"))
    for _ in range(args.warmup):
        oracle_sample(work, 1, box=min(box, 48), dtype=dtype)
    tot_pts, tot_t, desc = 0, 0.0, ""
    for _ in range(args.steps):
        pts, t, desc = oracle_sample(work, ref_steps, box=box, dtype=dtype)
        tot_pts += pts * ref_steps
        tot_t += t
    value = tot_pts / tot_t
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True,
            "scaling": "weak" if wl == "C5W" else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOADS[wl] + " sample", "grid": work["grid"]["n"][:work["grid"]["dims"]],
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

    wl = args.workload
    work = workload(wl, ws)
    dtype = args.dtype or DTYPE_DEFAULT.get(wl, "c64")
    if work["grid"]["dims"] == 1 and ws > 1:
        raise SystemExit("1D configs are replicas only (DESIGN.md §8): run --gpus 1")
    S = nl.solver_from_work(work, dtype, shard=shard)
    exchange = args.exchange
    if ws > 1 and exchange == "fused":
        try:
            S.connect_peers()  # halo exchange fused into the stage kernels over CUDA IPC / NVLink
        except Exception as e:  # no peer mapping: the NCCL exchange (validated below)
            exchange = f"nccl (connect_peers failed: {str(e)[:120]})"
    ctype = torch.complex64 if dtype == "c64" else torch.complex128
    g = work["grid"]
    npts_global = int(np.prod(g["n"][:3]))
    lshape = S.local_shape
    dims = g["dims"]
    lo = [0, 0, 0]
    cnt = list(g["n"])
    if dims >= 2:
        lo[dims - 1], cnt[dims - 1] = S.z0, S.nz
    host = torch.empty(lshape, dtype=ctype, pin_memory=True)
    icgen.fill(work["ic"], g, dtype=np.complex64 if dtype == "c64" else np.complex128, lo=lo, cnt=cnt,
               out=host.numpy())
    psi = host.cuda()
    kmax = S.stability_bound(psi)
    dt = 0.8 * kmax
    if ws > 1 and exchange == "fused":
        # the fused exchange must reproduce the NCCL exchange bit for bit on every rank (and no
        # arrival wait may have timed out), else the timed run uses the NCCL exchange
        a, b = psi.clone(), psi.clone()
        S.rk4(a, dt, 2)
        S.set_option("fused_exchange", 0)
        S.rk4(b, dt, 2)
        S.set_option("fused_exchange", 1)
        ok = torch.tensor([1 if (torch.equal(torch.view_as_real(a), torch.view_as_real(b))
                                 and S.exchange_timeouts == 0) else 0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            S.set_option("fused_exchange", 0)
            exchange = "nccl (fused exchange failed its bitwise check against NCCL)"
        del a, b

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
    out_host = torch.empty(lshape, dtype=ctype, pin_memory=True)  # empty_like would not pin
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

    S_bytes = 8 if dtype == "c64" else 16
    # Roofline: the algorithmic bytes are 16 S per point-step (the minimum with
    # every stage result stored); the fused default moves 12 S (carried-sum form),
    # so its 16 S rate can exceed the copy bandwidth.  Reported beside it: the 12 S rate and
    # the DRAM-counter rate (ncu bytes of the same kernels, profiles/roofline_traffic.json).
    pts_local = npts_global / ws
    launch_ms = ms / (4 * args.steps)  # the 4 stage launches of a step (device time per launch)
    achieved = 16 / 4 * S_bytes * pts_local / (launch_ms / 1e3) / 1e9
    peak, peak_kind = peaks()
    tr = profile_traffic()
    traffic = None
    key = f"{wl}_{dtype}"
    if tr and tr.get("workload") in (wl, key) and tr.get("dram_bytes_per_point_stage"):
        traffic = tr["dram_bytes_per_point_stage"] * pts_local
    elif tr and key in tr.get("workloads", {}):
        traffic = tr["workloads"][key]["dram_bytes_per_point_stage"] * pts_local
    clocks = clk.summary()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if wl == "C5W" else "strong", "vs_baseline": None,
            "dtype": "c64 (fp32 pairs)" if dtype == "c64" else "c128 (fp64 pairs)", "data": "synthetic",
            "config": {"workload": WORKLOADS[wl], "grid": g["n"][:dims], "bc": work["bc"],
                       "V": work["V"]["kind"], "dt": dt, "kmax": kmax,
                       "parallelism": f"z-slab x{ws}, {exchange} halo exchange" if ws > 1 else "single GPU",
                       "l2": f"inputs ({host.numel() * host.element_size() / 2**30:.2f} GiB per field per GPU) vs "
                             "L2 126 MB: no flush" + (" (C2: fields comparable to L2, DRAM bytes can fall "
                                                      "below algorithmic)" if wl == "C2" else "")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "alg_bytes_per_point_step": 16 * S_bytes,
                         "alg_bytes_note": "SURVEY 8(d) 16 S per point-step; the carried-sum default moves 12 S",
                         "achieved_12S": achieved * 12 / 16, "frac_12S": achieved * 12 / 16 / peak,
                         "dram_achieved": (traffic / (launch_ms / 1e3) / 1e9) if traffic else None,
                         "dram_frac": (traffic / (launch_ms / 1e3) / 1e9 / peak) if traffic else None,
                         "frac_of_8TBs": achieved / 8000.0,
                         "kernel": KERNEL[dims].format("float" if dtype == "c64" else "double")},
            "e2e": {"value": npts_global * args.steps / (ems / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": nbytes / args.steps, "d2h_bytes_per_step": nbytes / args.steps,
                    "note": "per job of K steps: H2D(Psi0 pinned) + nlse2shoc_rk4(K) + D2H(Psi)"},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if ws == 1 and not args.no_cpu_baseline and wl == "C4":
            line["cpu_baseline"] = cpu_baseline_line(work, int(os.environ.get("NLSE_REF_BOX", "128")))
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
    ap.add_argument("--workload", default="C4", choices=["C4", "C5W", "C5S", "C3", "C2"])
    ap.add_argument("--dtype", default=None, choices=["c64", "c128"])
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="N>1: halo exchange fused into the stage kernels (peer stores + counters) or NCCL send/recv")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
