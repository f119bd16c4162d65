"""Multi-process (gloo, CPU) coverage of the z-slab sharding protocol.

Each rank owns the slab nlse2shoc_split gives it, exchanges its two edge planes with its
neighbours before every RK4 stage (the library's per-stage 2-plane halo), and evaluates F on
its halo-extended slab with the CPU oracle.  Two halo planes make F exact on the whole slab
(the 13-point star reaches 2 planes), so the sharded run must reproduce the single-domain
run; the stage combine uses the library's Psi-space accumulator algebra, so the comparison
is against the same algebra on the whole grid (bitwise), and against the oracle's RK4
listing to rounding.
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _grid_rhs(oracle, work, lo, cnt, psi):
    P = oracle.problem_from_work(work, lo=lo, cnt=cnt)
    return oracle.rhs(P, psi)


def _psi_space_rk4(F, psi, dt, nsteps):
    """Whole-grid RK4 in the library's accumulator form."""
    for _ in range(nsteps):
        K = F(psi)
        acc = psi + (dt / 6) * K
        TA = psi + (dt / 2) * K
        K = F(TA)
        acc = acc + (dt / 3) * K
        TB = psi + (dt / 2) * K
        K = F(TB)
        acc = acc + (dt / 3) * K
        TA = psi + dt * K
        K = F(TA)
        psi = acc + (dt / 6) * K
    return psi


def _worker(rank, world, port, work, dt, nsteps, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import icgen
    import oracle
    import paper_1109_1027_b200 as nl

    g = work["grid"]
    NZ = g["n"][2]
    z0, nz = nl.nlse2shoc_split(NZ, world, rank)
    psi = icgen.fill(work["ic"], g, lo=[0, 0, z0], cnt=[g["n"][0], g["n"][1], nz])
    lo_face, hi_face = z0 == 0, z0 + nz == NZ

    def halo(x):
        """2 planes from each neighbour (the library's ncclSend/ncclRecv pairs)."""
        lo = np.empty((2,) + x.shape[1:], x.dtype)
        hi = np.empty((2,) + x.shape[1:], x.dtype)
        ops = []
        if not lo_face:
            ops += [dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(x[:2])), rank - 1),
                    dist.P2POp(dist.irecv, torch.from_numpy(lo), rank - 1)]
        if not hi_face:
            ops += [dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(x[-2:])), rank + 1),
                    dist.P2POp(dist.irecv, torch.from_numpy(hi), rank + 1)]
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        return lo, hi

    def F(x):
        lo, hi = halo(x)
        parts, zlo, zc = [x], z0, nz
        if not lo_face:
            parts.insert(0, lo)
            zlo -= 2
            zc += 2
        if not hi_face:
            parts.append(hi)
            zc += 2
        ext = np.concatenate(parts, axis=0)
        Fe = _grid_rhs(oracle, work, [0, 0, zlo], [g["n"][0], g["n"][1], zc], ext)
        return Fe[z0 - zlo: z0 - zlo + nz]

    out = _psi_space_rk4(F, psi, dt, nsteps)
    out_q.put((rank, z0, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("bc", ["dirichlet", "lapzero"])
def test_gloo_slab_sharding_matches_single_domain(world, bc):
    import icgen
    import oracle
    from icgen import configs

    work = configs.SMALL(3, (11, 9, 16), bc, noise=0.05)
    P = oracle.problem_from_work(work)
    psi0 = icgen.fill(work["ic"], work["grid"])
    dt = 0.8 * oracle.kmax(P, psi0)
    nsteps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000) + world * 7 + (bc == "lapzero")
    procs = [ctx.Process(target=_worker, args=(r, world, port, work, dt, nsteps, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    parts.sort(key=lambda t: t[1])
    got = np.concatenate([t[2] for t in parts], axis=0)
    whole = _psi_space_rk4(lambda x: oracle.rhs(P, x), psi0, dt, nsteps)
    assert np.array_equal(got, whole)  # same per-point arithmetic, halos are exact copies
    ref = oracle.rk4(P, psi0, dt, nsteps)  # the paper's listing: equal to rounding
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-13


def test_bench_reference_arm_multirank_prints_once():
    """`bench.py --impl reference` under torchrun: rank 0 alone runs and prints one line."""
    env = dict(os.environ, NLSE_REF_BOX="24", OMP_NUM_THREADS="2")
    r = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
         "127.0.0.1", "--master-port", str(31000 + os.getpid() % 1000), os.path.join(ROOT, "bench.py"), "--impl",
         "reference", "--gpus", "2", "--steps", "2", "--warmup", "1"],
        capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json

    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def _peer_worker(rank, ws, port, q):
    import torch.distributed as dist

    import paper_1109_1027_b200 as nl

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    mine = bytes([rank]) * 64
    q.put((rank, nl.gather_peer_handles(mine)))
    dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_gather_peer_handles_gloo(ws):
    """Host side of the fused exchange (nlse2shoc_connect_peers): the all-gathered IPC handles
    give each rank exactly its z-neighbours (None at the global faces)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29650 + ws
    ps = [ctx.Process(target=_peer_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(ws))
    for p in ps:
        p.join(timeout=60)
    for r in range(ws):
        lo, hi = got[r]
        assert lo == (bytes([r - 1]) * 64 if r > 0 else None)
        assert hi == (bytes([r + 1]) * 64 if r < ws - 1 else None)
