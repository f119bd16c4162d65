"""GPU <-> oracle parity through the C-ABI (needs a B200).

Tolerances (north star, written here): max relative L2 <= 1e-12 for complex128 and
<= 1e-5 for complex64 after the stated steps; the oracle runs in double from the same
(float-rounded for c64) seeded input (reading R19).
"""
import math

import numpy as np
import pytest

import oracle
from icgen import configs

import harness as H

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


SHAPES = {
    1: [(5,), (7,), (37,), (1001,)],
    2: [(5, 5), (7, 6), (37, 13), (530, 9), (1030, 7)],
    3: [(5, 5, 5), (7, 6, 5), (37, 19, 9), (70, 35, 11), (130, 17, 7)],
}


def _small(dims, n, bc, dtype, V, aniso=True):
    h = [0.11, 0.13, 0.17][:dims] if aniso else [0.12] * dims
    return configs.SMALL(dims, n, bc, dtype=dtype, V=V, h=h)


CASES = []
for dims in (1, 2, 3):
    for i, n in enumerate(SHAPES[dims]):
        for dtype in ("c64", "c128"):
            for bc in ("dirichlet", "lapzero"):
                V = ["harmonic", "array", "none"][(i + (bc == "lapzero")) % 3]
                CASES.append((dims, n, dtype, bc, V))


@pytest.mark.parametrize("variant", [0, 1, 3])
@pytest.mark.parametrize("dims,n,dtype,bc,V", CASES)
def test_laplacian_parity(dims, n, dtype, bc, V, variant):
    w = _small(dims, n, bc, dtype, V, aniso=(variant != 1 or dims != 2))
    S = H.gpu_solver(w, dtype, variant)
    psi = H.psi0_host(w, dtype)
    L = S.laplacian(_dev(psi))
    torch.cuda.synchronize()
    Lo = oracle.laplacian(H.oracle_problem(w), psi.astype(np.complex128))
    tol = 1e-12 if dtype == "c128" else 1e-5
    H.compare(L.cpu().numpy(), Lo, tol, "")


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("dims,n,dtype,bc,V", CASES[::2])
def test_rk4_parity_10_steps(dims, n, dtype, bc, V, variant):
    if variant == 4 and dims == 1:
        pytest.skip("stage pairs: 2D/3D only")
    w = _small(dims, n, bc, dtype, V)
    S = H.gpu_solver(w, dtype, variant)
    psi = H.psi0_host(w, dtype)
    P = H.oracle_problem(w)
    dt = 0.8 * oracle.kmax(P, psi.astype(np.complex128))
    g = _dev(psi)
    S.rk4(g, dt, 10)
    torch.cuda.synchronize()
    ref = oracle.rk4(P, psi.astype(np.complex128), dt, 10)
    H.compare(g.cpu().numpy(), ref, H.TOL[dtype], "")


@pytest.mark.parametrize("dims,n,dtype,bc,V", [c for c in CASES if c[2] == "c128"][::3])
def test_stability_bound_matches_oracle(dims, n, dtype, bc, V):
    w = _small(dims, n, bc, dtype, V)
    S = H.gpu_solver(w, dtype)
    psi = H.psi0_host(w, dtype)
    k = S.stability_bound(_dev(psi))
    ko = oracle.kmax(H.oracle_problem(w), psi)
    assert abs(k - ko) <= 1e-13 * ko


def test_fused_and_two_kernel_agree_3d():
    w = _small(3, (70, 35, 11), "dirichlet", "c128", "harmonic", aniso=False)
    psi = H.psi0_host(w, "c128")
    outs = []
    for v in (0, 1, 2):
        S = H.gpu_solver(w, "c128", v)
        g = _dev(psi)
        S.rk4(g, 1e-4, 5)
        outs.append(g.cpu().numpy())
    H.compare(outs[0], outs[1], 1e-13, "")
    H.compare(outs[0], outs[2], 1e-13, "")


def test_edge_cases_and_errors():
    import paper_1109_1027_b200 as nl

    w = _small(3, (9, 8, 7), "dirichlet", "c64", "harmonic")
    S = H.gpu_solver(w, "c64")
    psi = _dev(H.psi0_host(w, "c64"))
    before = psi.clone()
    S.rk4(psi, 1e-3, 0)  # nsteps = 0 is a no-op
    assert torch.equal(psi, before)
    with pytest.raises(nl.NLSE2SHOCError):
        S.rk4(psi, -1.0, 1)
    with pytest.raises(nl.NLSE2SHOCError):
        S.rk4(psi, float("nan"), 1)
    with pytest.raises(nl.NLSE2SHOCError):
        S.laplacian(psi, out=psi)
    flat = torch.zeros(psi.numel() + 1, dtype=psi.dtype, device="cuda")
    with pytest.raises(nl.NLSE2SHOCError):  # 8-byte aligned only
        S.rk4(flat[1:].view(psi.shape), 1e-3, 1)
    bad = psi.clone()
    bad.view(-1)[17] = complex(float("nan"), 0.0)
    with pytest.raises(nl.NLSE2SHOCError):
        S.check_finite(bad)
    S.check_finite(psi)


@pytest.mark.parametrize("variant,n,dtype", [(0, (37, 19, 9), "c128"), (5, (37, 19, 9), "c128"), (6, (37, 19, 9), "c64"),
                                              (0, (131, 51, 12), "c64"), (0, (70, 67, 10), "c128")])
def test_dirichlet_boundary_values_are_bit_exact(variant, n, dtype):
    """`dbc_ut`: Psi_t,b = 0, so boundary values never change, to the bit (the default
    carried-sum form returns T_C,b = Psi_b at boundary points; grids with face-lean tiles too)."""
    w = _small(3, n, "dirichlet", dtype, "harmonic")
    S = H.gpu_solver(w, dtype, variant)
    psi = H.psi0_host(w, dtype)
    g = _dev(psi)
    S.rk4(g, 1e-4, 7)
    out = g.cpu().numpy()
    m = np.ones(psi.shape, bool)
    m[1:-1, 1:-1, 1:-1] = False
    assert np.array_equal(out[m], psi[m])


@pytest.mark.parametrize("variant", [0, 2, 4, 5, 6])
@pytest.mark.parametrize("dims,n,dtype,bc,V", [c for c in CASES if c[0] > 1][1::3])
def test_rk4_parity_isotropic(dims, n, dtype, bc, V, variant):
    """Equal spacing on every axis selects the kernels' summed-neighbour stencil form."""
    if variant == 4 and min(n) < 6:
        pytest.skip("tiny grid")
    w = _small(dims, n, bc, dtype, V, aniso=False)
    S = H.gpu_solver(w, dtype, variant)
    psi = H.psi0_host(w, dtype)
    P = H.oracle_problem(w)
    dt = 0.8 * oracle.kmax(P, psi.astype(np.complex128))
    g = _dev(psi)
    S.rk4(g, dt, 10)
    ref = oracle.rk4(P, psi.astype(np.complex128), dt, 10)
    H.compare(g.cpu().numpy(), ref, H.TOL[dtype], "")


@pytest.mark.parametrize("dims,n,aniso", [(1, (3000,), True), (2, (300, 70), False), (2, (300, 70), True),
                                          (3, (80, 40, 20), False), (3, (80, 40, 20), True)])
@pytest.mark.parametrize("bc", ["dirichlet", "lapzero"])
@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 5])
def test_constant_field_is_stationary_to_the_bit(dims, n, aniso, bc, variant):
    """s = 0, V = 0, Psi = const: the exact Laplacian is 0, so Psi_t = 0 and RK4 must return
    Psi unchanged.  The stencil is written with the centre inside each difference (lap5 /
    lap_wide), so with weights rounded to fp32 it still annihilates constants exactly; the
    separate -30 g0 form left an O(eps) frequency shift per step (C2 c64 drifted 5.8e-5 in 500
    steps)."""
    if variant == 4 and dims == 1:
        pytest.skip("stage pairs: 2D/3D only")
    w = _small(dims, n, bc, "c64", "none", aniso=aniso)
    w["s"] = 0.0
    S = H.gpu_solver(w, "c64", variant)
    g = torch.full(tuple(reversed(n)), complex(0.6, -0.8), dtype=torch.complex64, device="cuda")
    g0 = g.clone()
    S.rk4(g, 0.5 * S.stability_bound(g), 50)
    assert torch.equal(g, g0)
    assert torch.count_nonzero(S.laplacian(g0)) == 0


@pytest.mark.parametrize("variant", [0, 2, 4])
@pytest.mark.parametrize("dims,n,dtype", [
    (3, (129, 49, 9), "c64"),    # x0 + TX = nx - 1 and y0 + TY = ny - 1 (64 x 24 tiles)
    (3, (97, 65, 9), "c128"),    # the same for 32 x 32 tiles
    (3, (130, 50, 9), "c64"), (3, (128, 48, 9), "c64"),
    (2, (2049, 9), "c64"), (2, (1025, 9), "c128"),  # 1024 / 512-wide 2D rows
])
def test_tile_edge_one_short_of_the_face(dims, n, dtype, variant):
    """A tile whose last column (row) is nx-2 (ny-2) reads the ghost at nx (ny): such tiles must
    not take the interior ("lean") path that reads the halo straight from the grid."""
    w = _small(dims, n, "dirichlet", dtype, "harmonic")
    S = H.gpu_solver(w, dtype, variant)
    psi = H.psi0_host(w, dtype)
    P = H.oracle_problem(w)
    dt = 0.8 * oracle.kmax(P, psi.astype(np.complex128))
    g = _dev(psi)
    S.rk4(g, dt, 3)
    ref = oracle.rk4(P, psi.astype(np.complex128), dt, 3)
    H.compare(g.cpu().numpy(), ref, H.TOL[dtype], "")
    L = S.laplacian(_dev(psi)).cpu().numpy()
    Lo = oracle.laplacian(P, psi.astype(np.complex128))
    H.compare(L, Lo, (1e-12 if dtype == "c128" else 1e-5), "")


@pytest.mark.parametrize("dims,dtype,TX,TY", [(3, "c64", 64, 24), (3, "c128", 32, 32), (2, "c64", 1024, 1),
                                           (2, "c128", 512, 1)])
def test_tile_edge_sweep(dims, dtype, TX, TY):
    """Every grid size within +-2 of a two-tile multiple on x (and y in 3D), both BCs, fused and
    stage-pair kernels, against the oracle: all tile/face/ghost combinations at the far edge."""
    nxs = [2 * TX + d for d in range(-2, 3)]
    nys = [2 * TY + d for d in range(-2, 3)] if dims == 3 else [9]
    for i, (nx, ny) in enumerate([(a, b) for a in nxs for b in nys]):
        n = (nx, ny, 7) if dims == 3 else (nx, ny)
        bc = ("dirichlet", "lapzero")[i % 2]
        w = _small(dims, n, bc, dtype, "harmonic")
        psi = H.psi0_host(w, dtype)
        P = H.oracle_problem(w)
        dt = 0.8 * oracle.kmax(P, psi.astype(np.complex128))
        ref = oracle.rk4(P, psi.astype(np.complex128), dt, 2)
        for v in (0, 4):
            S = H.gpu_solver(w, dtype, v)
            g = _dev(psi)
            S.rk4(g, dt, 2)
            H.compare(g.cpu().numpy(), ref, H.TOL[dtype], str((n, bc, v)))


# --------------------------------------------------------------------------- configs
# Every BASELINE config at its STATED step count (north star: "match the oracle ... after the
# stated step count"), run on the GPU over its full grid in the launch configuration bench.py
# times (one nlse2shoc_rk4 call of all steps), and compared with the oracle on the whole grid
# (C1, C2) or on target boxes computed from shrinking dependency-cone crops, which are the
# full-grid oracle's values bit for bit (tests/test_crop_method.py).  Each comparison checks
# the relative L2 error and the per-element max norm (harness.compare).
def test_C1_full_2000_steps_and_exact_soliton():
    w = configs.C1()
    S = H.gpu_solver(w, "c128")
    psi = H.psi0_host(w, "c128")
    P = H.oracle_problem(w)
    kmax = oracle.kmax(P, psi)
    assert abs(S.stability_bound(_dev(psi)) - kmax) <= 1e-13 * kmax
    dt = 0.4 * kmax
    g = _dev(psi)
    S.rk4(g, dt, w["steps"])
    ref = oracle.rk4(P, psi, dt, w["steps"])
    out = g.cpu().numpy()
    H.compare(out, ref, 1e-12, "C1 c128 2000 steps, full grid")
    # exact bright soliton sqrt2 sech(x) e^{it} (north star); magnitude of the 4th-order error
    ic = dict(w["ic"])
    ic["p"] = [math.sqrt(2.0), 1.0, dt * w["steps"]]
    import icgen

    ex = icgen.fill(ic, w["grid"])
    assert H.rel_l2(out, ex) < 3e-7


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_C2_full_500_steps(dtype):
    """C2 at its stated 500 steps on the whole 2^22-point grid (the case that caught the fp32
    weight-sum drift, reading R30)."""
    w = configs.C2()
    psi = H.psi0_host(w, dtype)
    P = H.oracle_problem(w)
    dt = 0.8 * oracle.kmax(P, psi.astype(np.complex128))
    ref = oracle.rk4(P, psi.astype(np.complex128), dt, w["steps"])
    for variant in (0, 5):  # the default (carried sum, 12 transfers) and the write-light form (13)
        S = H.gpu_solver(w, dtype, variant)
        g = _dev(psi)
        S.rk4(g, dt, w["steps"])
        H.compare(g.cpu().numpy(), ref, H.TOL[dtype], f"C2 {dtype} 500 steps, full grid, variant {variant}")
        S.close()


def _crop_parity(w, dtype, nsteps, targets, name, variant=0):
    """Full-size GPU run (bench launch configuration), target boxes against the oracle's
    shrinking-crop runs with the full-domain dt."""
    dims = w["grid"]["dims"]
    g, kmax = H.gpu_field(w, dtype, with_kmax=True)
    dt = 0.8 * kmax
    S = H.gpu_solver(w, dtype, variant)
    kg = S.stability_bound(g)
    assert abs(kg - kmax) <= (1e-6 if dtype == "c64" else 1e-13) * kmax
    S.rk4(g, dt, nsteps)
    torch.cuda.synchronize()
    got = [g[H.sl(dims, tlo, tcnt)].cpu().numpy() for tlo, tcnt in targets]
    del g
    S.close()
    torch.cuda.empty_cache()
    for (tlo, tcnt), gb in zip(targets, got):
        want = H.oracle_crop_rk4(w, dtype, tlo, tcnt, dt, nsteps)
        H.compare(gb, want, H.TOL[dtype], f"{name} {dtype} {nsteps} steps, box {tlo}+{tcnt}")


def test_C3_full_size_200_steps():
    """C3 (8192^2 c128) at its stated 200 steps (margin 1600): boxes across the edge of the
    Thomas-Fermi support on the x and y sides (indices 1937 ... 6254), one among the vortices
    and a global corner, where Psi is exactly zero and must stay so."""
    w = configs.C3()
    T = [([0, 0, 0], [40, 40, 1]), ([1925, 4060, 0], [32, 40, 1]), ([4070, 6232, 0], [40, 32, 1]),
         ([3500, 4600, 0], [48, 48, 1])]
    _crop_parity(w, "c128", w["steps"], T, "C3")


def test_C4_full_size_25_steps():
    """C4 (768^3 c64, bench config) after 25 of its 100 steps on boxes at a corner, the ring
    core, an x-face, a z-face edge and the far corner (margin 200).  The 100-step full-grid
    comparison needs ~11 min of oracle time on the GPU box (scripts/full_grid_parity.py C4 c64;
    result in profiles/r02/)."""
    w = configs.C4()
    n = 768
    T = [([0, 0, 0], [20, 18, 16]), ([370, 380, 376], [24, 20, 16]), ([0, 300, 500], [12, 24, 20]),
         ([500, 0, n - 14], [24, 12, 14]), ([n - 19, n - 17, n - 15], [19, 17, 15])]
    _crop_parity(w, "c64", 25, T, "C4")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_C5W_full_size_50_steps(dtype):
    """C5 weak-scaling grid of one GPU (768 x 768 x 192, Laplacian-zero) at its stated 50
    steps (margin 400): a corner box for both dtypes and the Gaussian's centre for c64."""
    w = configs.C5W(1)
    T = [([0, 0, 0], [16, 16, 16]), ([750, 748, 176], [18, 20, 16])]
    if dtype == "c64":
        T.append(([376, 376, 88], [16, 16, 16]))
    _crop_parity(w, dtype, w["steps"], T, "C5W")


def test_C5S_1536_full_size_50_steps():
    """C5 strong-scaling grid 1536^3 (complex64, 108 GiB of device memory with the workspace)
    at its stated 50 steps: a corner box and a box straddling the P = 8 shard seam at z = 192
    at a global x-y corner (SURVEY §8(c) "Oracle at scale")."""
    w = configs.C5()
    T = [([0, 0, 0], [24, 24, 24]), ([0, 1536 - 24, 176], [24, 24, 32])]
    _crop_parity(w, "c64", w["steps"], T, "C5S")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_1d_multilaunch_path_small_grid(dtype):
    """Small 1D grids normally run on the resident single-CTA solver; force the per-stage
    launch path (used for large 1D grids such as C2) and check parity on a small grid."""
    w = _small(1, (1001,), "dirichlet", dtype, "harmonic")
    S = H.gpu_solver(w, dtype)
    S.set_option("resident_1d", 0)
    S.set_option("cuda_graph", 0)
    psi = H.psi0_host(w, dtype)
    P = H.oracle_problem(w)
    dt = 0.8 * oracle.kmax(P, psi.astype(np.complex128))
    g = _dev(psi)
    S.rk4(g, dt, 10)
    assert S.last_launch_count == 40
    ref = oracle.rk4(P, psi.astype(np.complex128), dt, 10)
    H.compare(g.cpu().numpy(), ref, H.TOL[dtype], "")


def _core_box_work(w, lo, cnt):
    """The workload restricted to a box treated as its own Dirichlet domain (same h, V,
    seeded Psi0 values of that region of the global grid)."""
    import copy

    g = w["grid"]
    wc = copy.deepcopy(w)
    wc["grid"] = {"dims": g["dims"], "n": list(cnt), "xmin": [g["xmin"][d] + lo[d] * g["h"][d] for d in range(3)],
                  "h": list(g["h"])}
    return wc


@pytest.mark.parametrize("dtype,variant", [("c64", 0), ("c64", 2), ("c64", 5), ("c64", 6), ("c128", 0), ("c128", 5),
                                           ("c128", 6)])
def test_C4_core_box_full_step_count(dtype, variant):
    """C4 at its stated step count (100) on a 96^3 box around the ring core with C4's own
    spacing (SURVEY A7 analogue): the whole-field parity the north star states, for the
    default carried-sum form, the 13-transfer forms and the explicit-accumulator form."""
    w = configs.C4()
    lo, cnt = [336, 336, 336], [96, 96, 96]
    wc = _core_box_work(w, lo, cnt)
    psi = H.psi0_host(w, dtype, lo, cnt)
    P = oracle.problem_from_work(wc)
    dt = 0.8 * oracle.kmax(P, psi.astype(np.complex128))
    S = H.gpu_solver(wc, dtype, variant)
    g = _dev(psi)
    S.rk4(g, dt, w["steps"])
    ref = oracle.rk4(P, psi.astype(np.complex128), dt, w["steps"])
    H.compare(g.cpu().numpy(), ref, H.TOL[dtype], "")


@pytest.mark.parametrize("dtype,nsteps", [("c128", 400), ("c64", 400)])
def test_msd_1d_parity(dtype, nsteps):
    """MSD boundary (1D) on the paper's co-moving dark soliton (Exp. 1)."""
    w = configs.EXP_DARK(0.25)
    psi = H.psi0_host(w, dtype)
    P = H.oracle_problem(w)
    S = H.gpu_solver(w, dtype)
    g = _dev(psi)
    S.rk4(g, 5e-4, nsteps)
    ref = oracle.rk4(P, psi.astype(np.complex128), 5e-4, nsteps)
    H.compare(g.cpu().numpy(), ref, H.TOL[dtype], "")
    L = S.laplacian(_dev(psi)).cpu().numpy()
    Lo = oracle.laplacian(P, psi.astype(np.complex128))
    if dtype == "c128":
        H.compare(L, Lo, 1e-12, "")
    else:
        # fp32 stencil rounding: |dL| <~ 4 u (64/12) |Psi| / h^2 per point (sum of |coefficients|
        # 64/12 of the 5-point form); the near-constant dark soliton makes L small, so the
        # relative bound of the other cases does not apply here.
        u = np.finfo(np.float32).eps / 2
        h = w["grid"]["h"][0]
        assert np.linalg.norm(L - Lo) <= 4 * u * (64 / 12) / h**2 * np.linalg.norm(psi)


def test_fig1_on_gpu():
    """The paper's Fig. 1 reproduced by the CUDA library: 2SHOC errors at
    h = 1/2 ... 1/32 (20000 RK4 steps each, MSD boundary) within 0.5 % of the printed
    values (domain reading R5), orders within 0.005."""
    import icgen
    from oracle import metrics
    from conftest import read_golden

    gold = {float(r[1]): (float(r[2]), float(r[3])) for r in read_golden("fig1_1d.txt") if r[0] == "2shoc"}
    E = {}
    for h in (0.5, 0.25, 0.125, 0.0625, 0.03125):
        w = configs.EXP_DARK(h)
        S = H.gpu_solver(w, "c128")
        g = _dev(H.psi0_host(w, "c128"))
        per = w["steps"] // 100
        Er, Ei = [], []
        for j in range(1, 101):
            S.rk4(g, 5e-4, per)
            ic = dict(w["ic"])
            ic["p"] = list(ic["p"][:4]) + [j * per * 5e-4]
            er, ei = metrics.rms_err(g.cpu().numpy(), icgen.fill(ic, w["grid"]))
            Er.append(er)
            Ei.append(ei)
        E[h] = (np.mean(Er), np.mean(Ei))
        assert abs(E[h][0] / gold[h][0] - 1) < 5e-3 and abs(E[h][1] / gold[h][1] - 1) < 5e-3, (h, E[h], gold[h])
    printed = {0.25: 3.9355, 0.125: 3.9788, 0.0625: 3.9941, 0.03125: 3.9984}
    for h2, o in printed.items():
        assert abs(metrics.order(E[2 * h2][0], E[h2][0], 2 * h2, h2) - o) < 5e-3


@pytest.mark.parametrize("variant", [0, 2, 5, 6])
@pytest.mark.parametrize("bc,V,dtype", [("dirichlet", "harmonic", "c128"), ("lapzero", "array", "c128"),
                                        ("dirichlet", "none", "c64"), ("lapzero", "harmonic", "c128")])
def test_1d_stream_kernel_parity(bc, V, dtype, variant):
    """1D grids of >= 16 segments run the persistent bulk-copy kernel (line_stream_kernel):
    a ragged 40 003-point grid, 10 steps, against the oracle."""
    w = _small(1, (40003,), bc, dtype, V)
    S = H.gpu_solver(w, dtype, variant)
    psi = H.psi0_host(w, dtype)
    P = H.oracle_problem(w)
    dt = 0.8 * oracle.kmax(P, psi.astype(np.complex128))
    g = _dev(psi)
    S.rk4(g, dt, 10)
    ref = oracle.rk4(P, psi.astype(np.complex128), dt, 10)
    H.compare(g.cpu().numpy(), ref, H.TOL[dtype], "")
    L = S.laplacian(_dev(psi)).cpu().numpy()
    H.compare(L, oracle.laplacian(P, psi.astype(np.complex128)), (1e-12 if dtype == "c128" else 1e-5), "")


def test_1d_stream_kernel_msd():
    """MSD boundary through the persistent 1D kernel (Exp. 1 geometry at h = 1/512)."""
    w = configs.EXP_DARK(1.0 / 512)
    assert w["grid"]["n"][0] >= 16 * 1024
    psi = H.psi0_host(w, "c128")
    P = H.oracle_problem(w)
    S = H.gpu_solver(w, "c128")
    dt = 0.5 * oracle.kmax(P, psi)  # h = 1/512 is far inside Exp. 1's k = 5e-4 stability limit
    g = _dev(psi)
    S.rk4(g, dt, 20)
    ref = oracle.rk4(P, psi, dt, 20)
    assert np.isfinite(ref).all()
    H.compare(g.cpu().numpy(), ref, 1e-12, "")


# ------------------------------------------------------------- execution-path options
def _ragged_cases():
    out = []
    for dtype, TX, TY in (("c64", 64, 24), ("c128", 32, 32)):
        for i, (dx, dy) in enumerate([(-1, 1), (1, -1), (0, 0)]):
            out.append((dtype, (2 * TX + dx, 2 * TY + dy, 13), ("dirichlet", "lapzero")[i % 2]))
    return out


@pytest.mark.parametrize("variant", [0, 2, 5, 6])
@pytest.mark.parametrize("dtype,n,bc", _ragged_cases())
def test_lean_steps_bit_identical_to_general_step(dtype, n, bc, variant):
    """The lean plane steps (interior tiles, and 3D tiles touching an x/y face with the ghost
    fill and face rule inline) evaluate the general step's expressions: forcing the general
    step everywhere (option LEAN_STEPS = 0) must give the same bits, for every RK4 stage kind
    and the Laplacian, on grids one point either side of two-tile multiples."""
    w = _small(3, n, bc, dtype, "harmonic")
    psi = H.psi0_host(w, dtype)
    dt = 0.8 * oracle.kmax(H.oracle_problem(w), psi.astype(np.complex128))
    outs, laps = [], []
    for lean in (3, 2, 1, 0):
        S = H.gpu_solver(w, dtype, variant)
        S.set_option("lean_steps", lean)
        g = _dev(psi)
        S.rk4(g, dt, 3)
        outs.append(g.cpu())
        laps.append(S.laplacian(_dev(psi)).cpu())
    for o, l in zip(outs[1:], laps[1:]):
        assert torch.equal(o, outs[0])
        assert torch.equal(l, laps[0])


@pytest.mark.parametrize("nz,chunks", [(33, 8), (33, 5), (40, 3), (9, 50)])
def test_zchunk_counts_bit_identical(nz, chunks):
    """z-chunking only changes which CTA computes a plane: any chunk count (including ones
    that would leave empty chunks, which are normalised) gives the same bits."""
    w = _small(3, (70, 30, nz), "dirichlet", "c64", "harmonic")
    psi = H.psi0_host(w, "c64")
    ref = None
    for c in (0, chunks):
        S = H.gpu_solver(w, "c64")
        S.set_option("zchunks", c)
        g = _dev(psi)
        S.rk4(g, 1e-4, 2)
        if ref is None:
            ref = g.cpu()
        else:
            assert torch.equal(g.cpu(), ref)


@pytest.mark.parametrize("option", ["cuda_graph", "reverse_order", "tail_chunks"])
def test_path_options_bit_identical(option):
    w = _small(3, (70, 30, 20), "lapzero", "c64", "harmonic")
    psi = H.psi0_host(w, "c64")
    res = []
    for v in (1, 0):
        S = H.gpu_solver(w, "c64")
        S.set_option(option, v)
        g = _dev(psi)
        S.rk4(g, 1e-4, 5)
        res.append(g.cpu())
    assert torch.equal(res[0], res[1])


def test_V_array_is_validated():
    """the array potential reaches the library as a raw pointer; the binding must
    refuse a tensor the kernels would read out of bounds or in the wrong precision."""
    w = _small(3, (9, 8, 7), "dirichlet", "c128", "array")
    good = H.V_array_device(w, "c128")
    import paper_1109_1027_b200 as nl

    for bad in (good.float(), good[:-1].clone(), good.cpu(), good.reshape(7, 8, 9).transpose(0, 2)):
        with pytest.raises(ValueError):
            nl.solver_from_work(w, "c128", V_array=bad)
    nl.solver_from_work(w, "c128", V_array=good).close()


@pytest.mark.parametrize("dims,n,dtype,shard", [(3, (70, 30, 131), "c64", None), (3, (40, 33, 97), "c128", None),
                                                (3, (70, 30, 131), "c64", {"loopback": 3}),
                                                (2, (1100, 517), "c128", None), (2, (2100, 300), "c64", None)])
def test_tail_chunks_bit_identical(dims, n, dtype, shard):
    """TAIL_CHUNKS (short z-chunks at both ends of the streamed range) changes which CTA
    computes a plane and in which order, nothing else: on and off give the same bits, for
    single slabs, loopback slabs with the fused exchange, and the 2D row kernel."""
    import paper_1109_1027_b200 as nl

    w = _small(dims, n, "dirichlet", dtype, "harmonic")
    psi = H.psi0_host(w, dtype)
    res = []
    for v in (1, 0):
        S = nl.solver_from_work(w, dtype, shard=shard)
        S.set_option("tail_chunks", v)
        g = _dev(psi)
        S.rk4(g, 1e-4, 5)
        res.append(g.cpu())
        S.close()
    assert torch.equal(res[0], res[1])


@pytest.mark.parametrize("shard", [None, {"loopback": 3}])
def test_cached_step_graph(shard):
    """rk4 keeps its instantiated step graph for later calls with the same psi and dt: two
    calls of 5 steps must equal one call of 10 to the bit, and a new dt, a new buffer or a
    set_option call must not replay a stale graph."""
    import paper_1109_1027_b200 as nl

    w = _small(3, (70, 30, 33), "dirichlet", "c64", "harmonic")
    psi = H.psi0_host(w, "c64")
    S = nl.solver_from_work(w, "c64", shard=shard)
    a = _dev(psi)
    S.rk4(a, 1e-4, 5)
    S.rk4(a, 1e-4, 5)
    b = _dev(psi)
    S.rk4(b, 1e-4, 10)  # other buffer: new graph
    assert torch.equal(a, b)
    c = _dev(psi)
    S.rk4(c, 2e-4, 5)  # other dt: new graph
    d = _dev(psi)
    S.set_option("reverse_order", 0)  # settings changed: new graph
    S.rk4(d, 2e-4, 5)
    assert torch.equal(c, d)
    assert not torch.equal(a, c)
    S.close()


@pytest.mark.parametrize("dims,n,dtype", [(3, (70, 30, 20), "c64"), (2, (1100, 37), "c128"), (1, (40003,), "c64")])
def test_caller_owned_workspace(dims, n, dtype):
    """nlse2shoc_set_workspace: the three stage fields in a torch tensor give the
    same bits as the library's own allocation, the handle's own byte count drops by them, and
    bad workspaces are refused."""
    import paper_1109_1027_b200 as nl

    w = _small(dims, n, "dirichlet", dtype, "harmonic")
    psi = H.psi0_host(w, dtype)
    S = nl.solver_from_work(w, dtype)
    a = _dev(psi)
    dt = 0.5 * S.stability_bound(a)
    S.rk4(a, dt, 6)
    need, before = S.stage_workspace_bytes, S.workspace_bytes
    assert need >= 3 * psi.nbytes and need % 256 == 0
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    S.set_workspace(ws)
    assert before - S.workspace_bytes == 3 * psi.nbytes
    b = _dev(psi)
    S.rk4(b, dt, 6)
    assert torch.isfinite(torch.view_as_real(a)).all() and torch.equal(a, b)
    L0, L1 = S.laplacian(a), S.laplacian(b)
    assert torch.equal(L0, L1)
    with pytest.raises(nl.NLSE2SHOCError):
        S.set_workspace(torch.empty(need - 256, dtype=torch.uint8, device="cuda"))
    with pytest.raises(nl.NLSE2SHOCError):
        S.set_workspace(torch.empty(need + 256, dtype=torch.uint8, device="cuda")[8:])
    ws2 = torch.empty(need, dtype=torch.uint8, device="cuda")  # a second workspace replaces the first
    S.set_workspace(ws2)
    c = _dev(psi)
    S.rk4(c, dt, 6)
    assert torch.equal(a, c)
    S.close()
    L = nl.solver_from_work(w, dtype, shard={"loopback": 2}) if dims > 1 else None
    if L is not None:
        with pytest.raises(nl.NLSE2SHOCError):
            L.set_workspace(ws)
        L.close()


@pytest.mark.parametrize("dims,n", [(3, (71, 30, 20)), (2, (1101, 37)), (3, (70, 30, 20))])
def test_padded_layout_zero_copy(dims, n):
    """nlse2shoc_padded_layout / nlse2shoc_rk4_padded: complex64 with odd N_x is
    staged through a pitched copy by rk4; a Psi already in the padded layout is used in place
    and gives the same bits, its pad column untouched.  Even N_x: the layout is the dense one."""
    import paper_1109_1027_b200 as nl

    w = _small(dims, n, "lapzero", "c64", "harmonic")
    psi = H.psi0_host(w, "c64")
    S = nl.solver_from_work(w, "c64")
    pitch, off = S.padded_layout
    assert off == [0, 0, 0] and pitch[0] == n[0] + (n[0] & 1)
    assert pitch[1] == pitch[0] * (n[1] if dims == 3 else 1) and pitch[2] == pitch[0] * int(np.prod(n[1:]))
    a = _dev(psi)
    S.rk4(a, 1e-4, 5)
    p = torch.full(tuple(psi.shape[:-1]) + (pitch[0],), complex(7.0, -7.0), dtype=torch.complex64, device="cuda")
    p[..., :n[0]] = _dev(psi)
    S.rk4_padded(p, 1e-4, 5)
    assert torch.equal(p[..., :n[0]], a)
    if pitch[0] != n[0]:
        assert torch.all(p[..., n[0]] == complex(7.0, -7.0))
    with pytest.raises(ValueError):
        S.rk4_padded(a if pitch[0] != n[0] else a[..., :-1], 1e-4, 1)
    S.close()


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("dims,n", [(1, (3000,)), (1, (40003,)), (2, (300, 70)), (3, (80, 40, 20))])
def test_carried_sum_keeps_any_constant_to_the_bit(dims, n, dtype):
    """The default (carried-sum, 12-transfer) combine forms Psi' = (Q + T_C + k/2 K4) / 3 with
    Q = 3 acc - Psi: its exact sum and correctly rounded division must return a stationary
    field unchanged for any mantissa (a plain Q + fl(1/3) T_C does not), and variant 0 is
    variant 7."""
    w = _small(dims, n, "lapzero", dtype, "none", aniso=False)
    w["s"] = 0.0
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    S = H.gpu_solver(w, dtype)
    for val in (complex(1 / 3, 2 / 3), complex(1.9999999, -1.3333334), complex(5e-5, 123.456), complex(-0.7, 1e-30)):
        g = torch.full(tuple(reversed(n)), val, dtype=tdt, device="cuda")
        g0 = g.clone()
        S.rk4(g, 0.5 * S.stability_bound(g), 20)
        assert torch.equal(g, g0), val
    w2 = _small(dims, n, "dirichlet", dtype, "harmonic")
    psi = H.psi0_host(w2, dtype)
    outs = []
    for v in (0, 7):
        S2 = H.gpu_solver(w2, dtype, v)
        g = _dev(psi)
        S2.rk4(g, 0.5 * S2.stability_bound(g), 5)
        outs.append(g.cpu())
    assert torch.isfinite(torch.view_as_real(outs[0])).all() and torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("shard", [None, {"loopback": 2}])
def test_check_every_detects_blow_up(shard):
    """Failure detection: past the stability bound the explicit scheme
    blows up; with option CHECK_EVERY rk4 stops at the first scan that finds a non-finite value
    and names the step, and below the bound the chunked call gives the bits of the plain one."""
    import re

    import paper_1109_1027_b200 as nl
    from paper_1109_1027_b200 import _lib

    w = _small(3, (70, 30, 24), "dirichlet", "c64", "harmonic")
    psi = H.psi0_host(w, "c64")
    S = nl.solver_from_work(w, "c64", shard=shard)
    kmax = S.stability_bound(_dev(psi))
    a = _dev(psi)
    S.rk4(a, 0.8 * kmax, 23)
    S.set_option("check_every", 5)
    b = _dev(psi)
    S.rk4(b, 0.8 * kmax, 23)
    assert torch.equal(a, b)
    c = _dev(psi)
    with pytest.raises(nl.NLSE2SHOCError) as ei:
        S.rk4(c, 3.0 * kmax, 2000)
    assert ei.value.status == _lib.ENONFINITE
    m = re.search(r"after step (\d+) of 2000", str(ei.value))
    assert m and int(m.group(1)) % 5 == 0 and int(m.group(1)) < 2000
    assert not torch.isfinite(torch.view_as_real(c)).all()
    S.set_option("check_every", 0)  # off again: the call is asynchronous and reports nothing
    d = _dev(psi)
    S.rk4(d, 3.0 * kmax, int(m.group(1)))
    assert not torch.isfinite(torch.view_as_real(d)).all()
    S.close()
