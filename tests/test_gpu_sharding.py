"""Sharded path on one GPU (SURVEY §4 T3'): the loopback handle splits the slowest axis into
virtual slabs exactly like the NCCL shards (nlse2shoc_split), exchanges 2-plane halos by
device copies and runs the same kernels.  The step has no reductions and halos are exact
copies, so results must be BITWISE equal to the single-slab handle."""
import numpy as np
import pytest

from icgen import configs

import harness as H

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _run(work, dtype, shard, variant, nsteps, dt, psi0, lap=False):
    import paper_1109_1027_b200 as nl

    Varr = H.V_array_device(work, dtype) if work["V"]["kind"] == "array" else None
    S = nl.solver_from_work(work, dtype, V_array=Varr, shard=shard)
    if variant:
        S.set_variant(variant)
    g = torch.from_numpy(psi0).cuda()
    if lap:
        out = S.laplacian(g).cpu().numpy()
    else:
        S.rk4(g, dt, nsteps)
        out = g.cpu().numpy()
    k = S.stability_bound(torch.from_numpy(psi0).cuda())
    S.close()
    return out, k


CASES = [
    (3, (37, 19, 23), "dirichlet", "c64", "harmonic"),
    (3, (40, 33, 31), "lapzero", "c128", "none"),
    (3, (21, 18, 29), "dirichlet", "c128", "array"),
    (2, (70, 61), "dirichlet", "c128", "harmonic"),
    (2, (531, 17), "lapzero", "c64", "none"),
]


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 5, 6])
@pytest.mark.parametrize("nslabs", [2, 3, 7])
@pytest.mark.parametrize("dims,n,bc,dtype,V", CASES)
def test_loopback_bitwise_equal(dims, n, bc, dtype, V, nslabs, variant):
    w = configs.SMALL(dims, n, bc, dtype=dtype, V=V, noise=0.05)
    psi0 = H.psi0_host(w, dtype)
    ref, k1 = _run(w, dtype, None, variant, 6, 1e-4, psi0)
    got, kP = _run(w, dtype, {"loopback": nslabs}, variant, 6, 1e-4, psi0)
    assert np.array_equal(got.view(np.uint8), ref.view(np.uint8))
    assert kP == k1
    lref, _ = _run(w, dtype, None, variant, 0, 1.0, psi0, lap=True)
    lgot, _ = _run(w, dtype, {"loopback": nslabs}, variant, 0, 1.0, psi0, lap=True)
    assert np.array_equal(lgot.view(np.uint8), lref.view(np.uint8))


def test_loopback_C4_full_size_matches_single_gpu():
    """C4's 768^3 grid with its own Psi0, split like an 8-GPU run (96 planes per slab, halo
    exchange fused into the stage kernels), at its stated 100 steps: bitwise equal to the
    single slab, which matches the oracle's whole-grid run to 2.8e-7
    (profiles/r02/c4_full_100_steps_parity.json); no arrival wait may time out."""
    import paper_1109_1027_b200 as nl

    w = configs.C4()
    g, kmax = H.gpu_field(w, "c64", with_kmax=True)
    dt = 0.8 * kmax
    a = g.clone()
    S1 = H.gpu_solver(w, "c64")
    S1.rk4(a, dt, w["steps"])
    S1.close()
    S8 = nl.solver_from_work(w, "c64", shard={"loopback": 8})
    S8.rk4(g, dt, w["steps"])
    assert torch.equal(torch.view_as_real(a), torch.view_as_real(g))
    assert S8.exchange_timeouts == 0
    S8.close()


def test_nccl_sharded_handle_single_rank():
    """The real NCCL path: a one-rank communicator (no neighbours, so no exchange) must give
    exactly the single-GPU result; exercises ncclGetUniqueId / ncclCommInitRank."""
    import paper_1109_1027_b200 as nl

    w = configs.SMALL(3, (40, 33, 31), "dirichlet", dtype="c64", V="harmonic", noise=0.05)
    psi0 = H.psi0_host(w, "c64")
    ref, _ = _run(w, "c64", None, 0, 4, 1e-4, psi0)
    uid = nl.nlse2shoc_get_unique_id()
    assert len(uid) == 128
    got, _ = _run(w, "c64", {"uid": uid, "rank": 0, "nranks": 1}, 0, 4, 1e-4, psi0)
    assert np.array_equal(got.view(np.uint8), ref.view(np.uint8))


@pytest.mark.parametrize("nslabs", [2, 3, 8])
@pytest.mark.parametrize("dims,n,bc,dtype,V", [
    (3, (37, 19, 48), "dirichlet", "c64", "harmonic"), (3, (40, 33, 41), "lapzero", "c128", "none"),
    (3, (21, 18, 50), "dirichlet", "c128", "array"), (2, (70, 64), "lapzero", "c64", "harmonic")])
def test_loopback_matches_oracle(dims, n, bc, dtype, V, nslabs):
    """The sharded decomposition against the oracle itself (not only against the single
    slab): seams of every slab, the overlapped edge-first schedule (>= 8 planes per slab for
    P = 2, 3), 10 steps at 0.8 k_max."""
    import oracle

    w = configs.SMALL(dims, n, bc, dtype=dtype, V=V, noise=0.05)
    psi0 = H.psi0_host(w, dtype)
    P = H.oracle_problem(w)
    dt = 0.8 * oracle.kmax(P, psi0.astype(np.complex128))
    got, _ = _run(w, dtype, {"loopback": nslabs}, 0, 10, dt, psi0)
    ref = oracle.rk4(P, psi0.astype(np.complex128), dt, 10)
    H.compare(got, ref, H.TOL[dtype], f"loopback P={nslabs} {dims}D {bc} {dtype} {V} 10 steps")


def test_loopback_C4_seams_match_oracle():
    """C4 768^3 split like an 8-GPU run: boxes straddling the seams z = 96, 384 and 672 (at a
    global corner, in the ring core, at an x-face) after 10 steps against oracle crops."""
    import paper_1109_1027_b200 as nl

    w = configs.C4()
    g, kmax = H.gpu_field(w, "c64", with_kmax=True)
    dt = 0.8 * kmax
    S8 = nl.solver_from_work(w, "c64", shard={"loopback": 8})
    S8.rk4(g, dt, 10)
    T = [([0, 0, 88], [16, 16, 16]), ([376, 370, 376], [16, 20, 16]), ([0, 400, 664], [12, 16, 16])]
    got = [g[H.sl(3, a, b)].cpu().numpy() for a, b in T]
    S8.close()
    del g
    torch.cuda.empty_cache()
    for (tlo, tcnt), gb in zip(T, got):
        want = H.oracle_crop_rk4(w, "c64", tlo, tcnt, dt, 10)
        H.compare(gb, want, 1e-5, f"C4 loopback P=8 10 steps, seam box {tlo}+{tcnt}")


@pytest.mark.parametrize("variant", [0, 2, 5, 6])
@pytest.mark.parametrize("nslabs", [2, 3, 8])
def test_fused_exchange_bitwise_and_one_launch_per_stage(nslabs, variant):
    """Halo exchange fused into the stage kernels (loopback slabs are each other's peers): the
    edge planes are stored straight into the neighbours' halo buffers and counted there, so a
    step is 4 launches per slab and nothing else, bitwise equal to the NCCL-style exchange
    (option FUSED_EXCHANGE = 0) and to the single slab; across calls the device-side epochs
    keep the arrival counters consistent (second call, cached graph)."""
    import paper_1109_1027_b200 as nl

    w = configs.SMALL(3, (70, 33, 48), "dirichlet", dtype="c64", V="harmonic", noise=0.05)
    psi0 = H.psi0_host(w, "c64")
    res = {}
    for fused in (1, 0):
        S = nl.solver_from_work(w, "c64", shard={"loopback": nslabs})
        if variant:
            S.set_variant(variant)
        S.set_option("fused_exchange", fused)
        g = torch.from_numpy(psi0).cuda()
        S.rk4(g, 1e-4, 3)
        S.rk4(g, 1e-4, 3)
        if fused:
            assert S.last_launch_count == 4 * nslabs * 3
            assert S.exchange_timeouts == 0
        res[fused] = g.cpu()
        S.close()
    ref, _ = _run(w, "c64", None, variant, 6, 1e-4, psi0)
    assert torch.equal(res[1], res[0])
    assert np.array_equal(res[1].numpy().view(np.uint8), ref.view(np.uint8))


def test_loopback_C5W_weak_P2_stated_steps_match_oracle():
    """C5's weak-scaling configuration at P = 2 (768 x 768 x 384, the z-slab seam at 192) run
    sharded with the fused exchange for its stated 50 steps: a box across the seam at a global
    x-y corner and one at the far corner, against oracle crops (margin 400; a box at the
    Gaussian's centre would need ~2 min of oracle time, C5W(P=1) covers it)."""
    import paper_1109_1027_b200 as nl

    w = configs.C5W(2)
    g, kmax = H.gpu_field(w, "c64", with_kmax=True)
    dt = 0.8 * kmax
    S = nl.solver_from_work(w, "c64", shard={"loopback": 2})
    S.rk4(g, dt, w["steps"])
    assert S.exchange_timeouts == 0
    T = [([0, 0, 184], [16, 16, 16]), ([752, 0, 368], [16, 16, 16])]
    got = [g[H.sl(3, a, b)].cpu().numpy() for a, b in T]
    S.close()
    del g
    torch.cuda.empty_cache()
    for (tlo, tcnt), gb in zip(T, got):
        want = H.oracle_crop_rk4(w, "c64", tlo, tcnt, dt, w["steps"])
        H.compare(gb, want, 1e-5, f"C5W(P=2) loopback fused 50 steps, box {tlo}+{tcnt}")
