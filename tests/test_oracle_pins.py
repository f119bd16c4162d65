"""Pins of the CPU oracle against what the paper and mathematics fix (CPU only).

Each test names the pin of SURVEY.md §8(c) / DESIGN.md §4 it implements.  None of
these tests compares the oracle with itself: every expected value is a paper table
(tests/golden/*, cited), a closed form, an independent re-formulation printed by the
paper (single-storage / wide stencils typed from P:135-138), a
brute-force construction, or a mathematical property.
"""
import math

import numpy as np
import pytest

import icgen
import oracle
from icgen import configs
from oracle import metrics

from conftest import read_golden

RNG = np.random.default_rng(12345)


def crand(shape, rng=RNG):
    return rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)


def interior(dims, shape, depth=1):
    sl = tuple(slice(depth, n - depth) for n in shape)
    return sl


# ----------------------------------------------------------------------------- P1
def test_P1_1d_two_step_equals_five_point_wide_stencil():
    """2SHOC (`2shoc1d`,`2shoc1d2`) == (-u_{i+2}+16u_{i+1}-30u_i+16u_{i-1}-u_{i-2})/(12h^2)
    at every point two or more layers from the boundary."""
    n, h = 41, 0.13
    psi = crand((n,))
    P = oracle.Problem(1, [n], [h], 1.0, -1.0, None, "dirichlet")
    L = oracle.laplacian(P, psi)
    u = psi
    wide = (-u[4:] + 16 * u[3:-1] - 30 * u[2:-2] + 16 * u[1:-3] - u[:-4]) / (12 * h * h)
    scale = np.abs(u).max() * 64 / (12 * h * h)
    assert np.abs(L[2:-2] - wide).max() <= 1e-14 * scale


# ----------------------------------------------------------------------------- P2
def single_storage_2d(psi, lam, h):
    """Paper's single-storage 2D form typed from `2d2shocs1` and `2d2shocs2`
    (P:218-232): D = 5-point / h^2 at interior, D_b = lambda_b;
    L = -1/12 [cross 1, centre -12] D + 1/(6h^2) [corners 1, centre -4] Psi."""
    ny, nx = psi.shape
    D = lam.copy()
    c = psi
    D[1:-1, 1:-1] = (c[1:-1, 2:] + c[1:-1, :-2] + c[2:, 1:-1] + c[:-2, 1:-1] - 4 * c[1:-1, 1:-1]) / (h * h)
    L = lam.copy()
    L[1:-1, 1:-1] = (-1.0 / 12.0) * (D[1:-1, 2:] + D[1:-1, :-2] + D[2:, 1:-1] + D[:-2, 1:-1] - 12 * D[1:-1, 1:-1]) \
        + (1.0 / (6 * h * h)) * (c[2:, 2:] + c[2:, :-2] + c[:-2, 2:] + c[:-2, :-2] - 4 * c[1:-1, 1:-1])
    return L


def single_storage_3d(psi, lam, h):
    """Paper's single-storage 3D form typed from `3d2shocs` and `3d2shocs2`
    (P:312-354): D = 7-point / h^2; L = -1/12 (6 neighbours of D, centre -10)
    + 1/(6h^2) (12 edge-midpoints of Psi, centre -12)."""
    D = lam.copy()
    c = psi
    I = (slice(1, -1),) * 3

    def sh(a, dz, dy, dx):
        nz, ny, nx = a.shape
        return a[1 + dz:nz - 1 + dz, 1 + dy:ny - 1 + dy, 1 + dx:nx - 1 + dx]

    D[I] = (sh(c, 0, 0, 1) + sh(c, 0, 0, -1) + sh(c, 0, 1, 0) + sh(c, 0, -1, 0) + sh(c, 1, 0, 0)
            + sh(c, -1, 0, 0) - 6 * c[I]) / (h * h)
    six = sh(D, 0, 0, 1) + sh(D, 0, 0, -1) + sh(D, 0, 1, 0) + sh(D, 0, -1, 0) + sh(D, 1, 0, 0) + sh(D, -1, 0, 0)
    edges = 0
    for a_ in (1, -1):
        for b_ in (1, -1):
            edges = edges + sh(c, 0, a_, b_) + sh(c, a_, 0, b_) + sh(c, a_, b_, 0)
    L = lam.copy()
    L[I] = (-1.0 / 12.0) * (six - 10 * D[I]) + (1.0 / (6 * h * h)) * (edges - 12 * c[I])
    return L


def wide_13(psi, h, dims):
    """`2dnonhoc` and its 3D analogue: per axis (-1,16,-30,16,-1)/(12h^2)."""
    sl = (slice(2, -2),) * dims
    out = 0
    for ax in range(dims):
        def s(k):
            idx = [slice(2, -2)] * dims
            n = psi.shape[ax]
            idx[ax] = slice(2 + k, n - 2 + k)
            return psi[tuple(idx)]
        out = out + (-s(2) + 16 * s(1) - 30 * s(0) + 16 * s(-1) - s(-2)) / (12 * h * h)
    return out, sl


@pytest.mark.parametrize("dims,shape", [(2, (13, 17)), (3, (9, 10, 11))])
@pytest.mark.parametrize("bc", ["dirichlet", "lapzero"])
def test_P2_per_axis_equals_single_storage_and_wide(dims, shape, bc):
    """P:235, P:356 ("computationally equivalent"): the per-axis form with the tangential
    face rule (reading R8) equals the paper's single-storage stencils on the WHOLE interior
    for arbitrary boundary Laplacian values, and the 13/25-point wide stencil at depth >= 2."""
    h = 0.11
    psi = crand(shape)
    V = RNG.uniform(-2, 2, shape)
    P = oracle.Problem(dims, list(reversed(shape)), [h] * dims, 0.7, -1.3, V, bc)
    L = oracle.laplacian(P, psi)
    if bc == "dirichlet":
        N = P.s * (psi.real ** 2 + psi.imag ** 2) - V
        lam = (-(N * psi.real) / P.a) + 1j * (-(N * psi.imag) / P.a)
    else:
        lam = np.zeros_like(psi)
    Ls = single_storage_2d(psi, lam, h) if dims == 2 else single_storage_3d(psi, lam, h)
    scale = np.abs(psi).max() * (64 * dims) / (12 * h * h)
    I = interior(dims, shape)
    assert np.abs(L[I] - Ls[I]).max() <= 1e-14 * scale
    # boundary values: L_b = lambda_b
    mask = np.ones(shape, bool)
    mask[I] = False
    assert np.array_equal(L[mask], lam[mask])
    W, sl = wide_13(psi, h, dims)
    assert np.abs(L[sl] - W).max() <= 1e-14 * scale


# ----------------------------------------------------------------------------- P3
def test_P3_polynomial_exactness_depth2():
    """Fourth-order: exact for per-axis degree <= 5 at depth >= 2 (P:135-138 truncation)."""
    h = 0.25
    n = 17
    P = oracle.Problem(3, [n, n, n], [h * 1.1, h * 0.9, h], 1.0, 0.0, None, "lapzero")
    # grid uses x_i = xmin + i h_d: rebuild coordinates per axis with the anisotropic h
    xs = (np.arange(n) - 8) * h * 1.1
    ys = (np.arange(n) - 8) * h * 0.9
    zs = (np.arange(n) - 8) * h
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    p = X ** 5 * Y ** 3 * Z ** 2 + X ** 4 + 2 * Y ** 5 * Z - 3 * X * Y * Z + 1
    lap = 20 * X ** 3 * Y ** 3 * Z ** 2 + 6 * X ** 5 * Y * Z ** 2 + 2 * X ** 5 * Y ** 3 + 12 * X ** 2 + 40 * Y ** 3 * Z
    L = oracle.laplacian(P, p.astype(complex))
    I = interior(3, p.shape, 2)
    scale = np.abs(lap[I]).max()
    assert np.abs(L[I].real - lap[I]).max() <= 1e-12 * scale
    assert np.abs(L[I].imag).max() == 0.0


# ----------------------------------------------------------------------------- P4/P5
def run_exp(dims, h, scheme):
    w = configs.EXP_GAUSS(dims, h)
    P = oracle.problem_from_work(w, scheme=scheme)
    g = w["grid"]
    psi = icgen.fill(w["ic"], g)
    k = w["dt_rule"][1]
    per = w["steps"] // 100
    Er, Ei = [], []
    for j in range(1, 101):
        psi = oracle.rk4(P, psi, k, per)
        ic = dict(w["ic"])
        ic["p"] = [1.0, float(dims), j * per * k]  # exact solution at t_j (R3)
        er, ei = metrics.rms_err(psi, icgen.fill(ic, g))
        Er.append(er)
        Ei.append(ei)
    return float(np.mean(Er)), float(np.mean(Ei))


def printed_tol(s):
    """One unit of the last printed digit of a table entry."""
    mant = s.lower().split("e")[0]
    exp = int(s.lower().split("e")[1]) if "e" in s.lower() else 0
    dec = len(mant.split(".")[1]) if "." in mant else 0
    return 10.0 ** (exp - dec)


def _golden(name, scheme, h):
    for row in read_golden(name):
        if row[0] == scheme and abs(float(row[1]) - h) < 1e-12:
            return row[2], row[3]
    raise KeyError


FIG2_FAST = [("2shoc", 1.0), ("2shoc", 0.5), ("2shoc", 0.25), ("2shoc", 0.125), ("cd", 1.0), ("cd", 0.5), ("cd", 0.25)]
FIG2_SLOW = [("2shoc", 0.0625), ("cd", 0.125), ("cd", 0.0625)]


@pytest.mark.parametrize("scheme,h", FIG2_FAST + [pytest.param(s, h, marks=pytest.mark.slow) for s, h in FIG2_SLOW])
def test_P4_fig2_table_2d(scheme, h):
    """Fig. 2 reproduced to the printed digits (readings R1 RMS, R3, R4)."""
    er, ei = run_exp(2, h, scheme)
    gr, gi = _golden("fig2_2d.txt", scheme, h)
    assert abs(er - float(gr)) <= printed_tol(gr), (er, gr)
    assert abs(ei - float(gi)) <= printed_tol(gi), (ei, gi)


FIG3_FAST = [("2shoc", 1.0), ("2shoc", 0.5), ("cd", 1.0)]
FIG3_SLOW = [("cd", 0.5), ("2shoc", 0.25)]


@pytest.mark.parametrize("scheme,h", FIG3_FAST + [pytest.param(s, h, marks=pytest.mark.slow) for s, h in FIG3_SLOW])
def test_P5_fig3_table_3d(scheme, h):
    """Fig. 3 reproduced to the printed digits."""
    er, ei = run_exp(3, h, scheme)
    gr, gi = _golden("fig3_3d.txt", scheme, h)
    assert abs(er - float(gr)) <= printed_tol(gr), (er, gr)
    assert abs(ei - float(gi)) <= printed_tol(gi), (ei, gi)


def test_P4_order_formula_reading():
    """Reading R2: O = ln(E_h1/E_h2)/ln 2 reproduces the printed orders of Fig. 2
    from the printed errors; the literal 'ln E1 - ln E2' of P:500 does not."""
    rows = {float(r[1]): (float(r[2]), float(r[3])) for r in read_golden("fig2_2d.txt") if r[0] == "2shoc"}
    printed_real = {0.5: 3.8882, 0.25: 3.8982, 0.125: 3.964, 0.0625: 3.987}
    for h2, o in printed_real.items():
        e1, e2 = rows[2 * h2][0], rows[h2][0]
        assert abs(metrics.order(e1, e2, 2 * h2, h2) - o) < 2e-3
        assert abs(math.log(e1) - math.log(e2) - o) > 0.5


# ----------------------------------------------------------------------------- P7/P8
def interior_matrix(dims, n, h):
    """Brute force: the real matrix A of the oracle's Laplacian on interior unknowns with
    homogeneous Dirichlet data (Psi_b = 0, s = V = 0)."""
    shape = (n,) * dims
    P = oracle.Problem(dims, [n] * dims, [h] * dims, 1.0, 0.0, None, "dirichlet")
    I = interior(dims, shape)
    idx = np.argwhere(np.ones(tuple(n - 2 for _ in range(dims)), bool)) + 1
    m = len(idx)
    A = np.zeros((m, m))
    for q, ii in enumerate(idx):
        e = np.zeros(shape, complex)
        e[tuple(ii)] = 1.0
        L = oracle.laplacian(P, e)
        A[:, q] = L[I].reshape(-1).real
    return A


@pytest.mark.parametrize("dims,n", [(1, 12), (2, 9), (3, 7)])
def test_P7_table2_is_gershgorin_of_oracle_operator(dims, n):
    """Table 2: G = Gershgorin disc endpoints of -h^2 Lap (Dirichlet), which
    ties the oracle's depth-1/depth-2 rows (face rule R8) to the paper's printed values."""
    h = 0.5
    A = -interior_matrix(dims, n, h) * h * h * 12.0
    ends = set()
    for r in range(A.shape[0]):
        c = A[r, r]
        rad = np.abs(A[r]).sum() - abs(c)
        for v in (c + rad, c - rad):
            assert abs(v - round(v)) < 1e-9
            ends.add(int(round(v)))
    golden = {int(r[0]): set(int(v) for v in r[1:]) for r in read_golden("table2_G.txt")}
    assert ends == golden[dims]
    assert set(oracle.table2_G(dims)) == golden[dims]


@pytest.mark.parametrize("dims", [1, 2, 3])
def test_P8_kdfull_reduces_to_linear_bound(dims):
    """`kdfull` with L = B = 0 equals `kd2shoclin`: (3/4) h^2/(d sqrt2 a)."""
    for h, a in [(0.1, 1.0), (0.37, 0.5)]:
        k = oracle.kmax_from_N(dims, [h] * dims, a, 0.0, 0.0)
        assert abs(k - 0.75 * h * h / (dims * math.sqrt(2) * a)) <= 1e-15 * k


@pytest.mark.parametrize("hs", [[0.3, 0.3], [0.3, 0.41]])
def test_kmax_bounds_true_spectral_radius(hs):
    """The linearised bound is conservative: kmax * rho(a A + diag N) <= sqrt(8) (RK4's
    imaginary-axis stability limit), including the anisotropic extension (reading R17)."""
    n = 9
    shape = (n, n)
    rng = np.random.default_rng(5)
    V = rng.uniform(-3, 3, shape)
    a = 0.8
    P = oracle.Problem(2, [n, n], hs, a, 0.0, V, "dirichlet")
    # matrix of F/i = a Lap + N on interior unknowns (Psi_b = 0)
    I = interior(2, shape)
    idx = np.argwhere(np.ones((n - 2, n - 2), bool)) + 1
    m = len(idx)
    M = np.zeros((m, m))
    for q, ii in enumerate(idx):
        e = np.zeros(shape, complex)
        e[tuple(ii)] = 1.0
        F = oracle.rhs(P, e)
        M[:, q] = (F[I] / 1j).reshape(-1).real
    rho = np.abs(np.linalg.eigvals(M)).max()
    psi0 = np.zeros(shape, complex)
    k = oracle.kmax(P, psi0)
    assert k * rho <= math.sqrt(8) * (1 + 1e-12)
    assert k * rho >= 0.5 * math.sqrt(8)


# ----------------------------------------------------------------------------- P9/P10
def soliton_run(n, frac=0.4, T=0.648642):
    w = configs.C1()
    g = configs.grid_inclusive([-20.0], [20.0], [n])
    w["grid"] = g
    P = oracle.problem_from_work(w)
    psi = icgen.fill(w["ic"], g)
    k = oracle.kmax(P, psi) * frac
    steps = int(math.ceil(T / k))
    dt = T / steps
    psi = oracle.rk4(P, psi, dt, steps)
    ic = dict(w["ic"])
    ic["p"] = [math.sqrt(2.0), 1.0, T]  # exact sqrt2 sech(x) e^{i a k^2 t}, eta^2 = 2 a k^2 / s
    ex = icgen.fill(ic, g)
    return np.linalg.norm(psi - ex) / np.linalg.norm(ex)


def test_P9_P10_bright_soliton_fourth_order():
    """North star: exact bright soliton eta sech(kx) e^{i a k^2 t}; observed spatial order 4
    under grid halving at fixed T (time error negligible since dt ~ h^2)."""
    errs = [soliton_run(n) for n in (256, 512, 1024)]
    h = [40.0 / (n - 1) for n in (256, 512, 1024)]
    for i in range(2):
        o = metrics.order(errs[i], errs[i + 1], h[i], h[i + 1])
        assert 3.9 <= o <= 4.1, (errs, o)
    assert errs[2] < 3e-7


# ----------------------------------------------------------------------------- P11/P12
def test_P11_norm_conservation_order():
    """North star: the norm sum|Psi|^2 is conserved to O(dt^4) over fixed T (homogeneous
    Dirichlet: the semi-discrete operator is symmetric, so only RK4 loses norm)."""
    n = 33
    w = configs.SMALL(2, (n, n), "dirichlet", noise=0.0)
    w["s"] = -1.0
    P = oracle.problem_from_work(w)
    psi0 = icgen.fill(w["ic"], w["grid"])
    psi0[0, :] = psi0[-1, :] = 0
    psi0[:, 0] = psi0[:, -1] = 0
    k0 = oracle.kmax(P, psi0) * 0.8
    T = 40 * k0
    drift = []
    for div in (1, 2, 4):
        steps = 40 * div
        psi = oracle.rk4(P, psi0, T / steps, steps)
        drift.append(abs(np.sum(np.abs(psi) ** 2) - np.sum(np.abs(psi0) ** 2)) / np.sum(np.abs(psi0) ** 2))
    assert drift[0] / drift[1] >= 16 and drift[1] / drift[2] >= 16, drift


def test_P12_1d_dirichlet_operator_symmetric():
    """With Psi_b = 0 the 1D interior operator is symmetric; depth-1 diagonal is -29/12 h^-2
    (from `2shoc1d2` with D_b = lambda_b = 0), interior diagonal -30/12 h^-2."""
    h = 0.5
    A = interior_matrix(1, 12, h) * h * h * 12
    assert np.allclose(A, A.T, atol=1e-12)
    assert abs(A[0, 0] + 29) < 1e-12 and abs(A[-1, -1] + 29) < 1e-12
    assert abs(A[4, 4] + 30) < 1e-12
    ev = np.linalg.eigvalsh(A)
    assert ev.max() < 0 and ev.min() > -64


# ----------------------------------------------------------------------------- P14
@pytest.mark.parametrize("dims,h", [(2, 0.25), (2, 0.1), (3, 0.25)])
@pytest.mark.parametrize("bc", ["lapzero", "dirichlet"])
def test_P14_face_rule_closed_form(dims, h, bc):
    """Face rule R8/R9 in closed form.  p = x^4 - 6x^2y^2 + y^4 is harmonic, so lambda_b = 0
    (Laplacian-zero, or Dirichlet with s = V = 0).  At a d-face point the rule gives
    D_d(b) = -sum_{e!=d} delta_e^2 p = delta_d^2 p - 4h^2 (delta_x^2 p + delta_y^2 p = 4h^2 for
    this quartic), so step 2 gives L = m h^2/3 at depth-1 points touching m faces and L = 0
    at depth >= 2 (the 5-point rule is exact there)."""
    n = 11
    x = (np.arange(n) - 5) * h + 0.1
    if dims == 2:
        Y, X = np.meshgrid(x, x, indexing="ij")
        shape = (n, n)
    else:
        Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
        shape = (n, n, n)
    p = X ** 4 - 6 * X ** 2 * Y ** 2 + Y ** 4
    P = oracle.Problem(dims, [n] * dims, [h] * dims, 1.0, 0.0, None, bc)
    L = oracle.laplacian(P, p.astype(complex)).real
    I = interior(dims, shape)
    idx = np.argwhere(np.ones(shape, bool)[I]) + 1
    for ii in idx:
        m = sum(1 for d in range(dims) if ii[d] in (1, n - 2))
        expect = m * h * h / 3.0
        assert abs(L[tuple(ii)] - expect) <= 1e-10, (ii, L[tuple(ii)], expect)


# ----------------------------------------------------------------------------- P15/P16
def test_P15_rk4_polynomial_isolated():
    """RK4 combine in isolation (`RK4`): Psi = c, s = 0, V = V0, Laplacian-zero
    gives F = -i V0 Psi everywhere, so one step multiplies by R(z) = sum_{m<=4} z^m/m!,
    z = -i V0 k."""
    n = 9
    c, V0, k = 0.7 - 0.3j, 3.7, 0.01
    for dims in (1, 2, 3):
        shape = (n,) * dims
        P = oracle.Problem(dims, [n] * dims, [0.2] * dims, 1.0, 0.0, np.full(shape, V0), "lapzero")
        out = oracle.rk4(P, np.full(shape, c), k, 1)
        z = -1j * V0 * k
        R = 1 + z + z ** 2 / 2 + z ** 3 / 6 + z ** 4 / 24
        assert np.abs(out - c * R).max() <= 4 * np.finfo(float).eps * abs(c)


@pytest.mark.parametrize("bc", ["dirichlet", "lapzero"])
@pytest.mark.parametrize("dims", [1, 2, 3])
def test_P16_gauge_covariance_and_linearity(bc, dims):
    """F(e^{i theta} Psi) = e^{i theta} F(Psi) (NLSE phase symmetry); Laplacian linear when
    lambda_b is linear in Psi (Laplacian-zero, or Dirichlet with s = 0)."""
    shape = (7, 8, 9)[:dims]
    rng = np.random.default_rng(dims)
    psi, phi = crand(shape, rng), crand(shape, rng)
    V = rng.uniform(-1, 1, shape)
    n = list(reversed(shape))
    P = oracle.Problem(dims, n, [0.3, 0.35, 0.4][:dims], 0.9, -1.1, V, bc)
    th = 0.7
    F1 = oracle.rhs(P, np.exp(1j * th) * psi)
    F2 = np.exp(1j * th) * oracle.rhs(P, psi)
    assert np.abs(F1 - F2).max() <= 1e-13 * np.abs(F2).max()
    P0 = oracle.Problem(dims, n, [0.3, 0.35, 0.4][:dims], 0.9, 0.0, V, bc)
    al, be = 0.3 - 1.2j, -0.8 + 0.1j
    La = oracle.laplacian(P0, al * psi + be * phi)
    Lb = al * oracle.laplacian(P0, psi) + be * oracle.laplacian(P0, phi)
    assert np.abs(La - Lb).max() <= 1e-13 * np.abs(Lb).max()


def test_dirichlet_boundary_laplacian_example():
    """`dbc_lap`: Psi_b = 2, s = -1, V = 0, a = 1 -> Lap_b = -(s|Psi|^2 - V)Psi/a = 8."""
    n = 7
    psi = np.full((n,), 2.0 + 0j)
    P = oracle.Problem(1, [n], [0.1], 1.0, -1.0, None, "dirichlet")
    L = oracle.laplacian(P, psi)
    assert L[0] == 8.0 and L[-1] == 8.0
    F = oracle.rhs(P, psi)
    assert F[0] == 0 and F[-1] == 0  # `dbc_ut`: Psi_t,b = 0 exactly


def test_cd_scheme_exact_for_quadratics():
    """RK4+CD (`uttmp`): the central difference is exact for quadratics."""
    n, h = 9, 0.3
    x = np.arange(n) * h
    Y, X = np.meshgrid(x, x, indexing="ij")
    p = (X ** 2 + 3 * Y ** 2 - X * Y).astype(complex)
    P = oracle.Problem(2, [n, n], [h, h], 1.0, 0.0, None, "lapzero", scheme="cd")
    L = oracle.laplacian(P, p)
    assert np.abs(L[1:-1, 1:-1] - 8.0).max() < 1e-12


# ----------------------------------------------------------------------------- P6 (MSD)
def run_exp1(h, scheme):
    w = configs.EXP_DARK(h)
    g = w["grid"]
    P = oracle.Problem(1, g["n"][:1], g["h"][:1], w["a"], w["s"], None, "msd", scheme=scheme)
    psi = icgen.fill(w["ic"], g)
    k = w["dt_rule"][1]
    per = w["steps"] // 100
    Er, Ei = [], []
    for j in range(1, 101):
        psi = oracle.rk4(P, psi, k, per)
        ic = dict(w["ic"])
        ic["p"] = list(ic["p"][:4]) + [j * per * k]
        er, ei = metrics.rms_err(psi, icgen.fill(ic, g))
        Er.append(er)
        Ei.append(ei)
    return float(np.mean(Er)), float(np.mean(Ei))


FIG1_FAST = [("cd", 0.5), ("cd", 0.25), ("2shoc", 0.5), ("2shoc", 0.25), ("2shoc", 0.125)]
FIG1_SLOW = [("cd", 0.125), ("2shoc", 0.0625), ("2shoc", 0.03125)]


@pytest.mark.parametrize("scheme,h", FIG1_FAST + [pytest.param(s, h, marks=pytest.mark.slow) for s, h in FIG1_SLOW])
def test_P6_fig1_msd_dark_soliton(scheme, h):
    """Fig. 1: co-moving dark soliton with the MSD boundary (`msdbc_ut`,
    `msdbc_lap`; readings R5 domain [-25.5, 31], R28 Lap_{b-1} = D_{b-1}).
    The paper does not state its domain, and the domain reading moves the magnitudes by a
    few 0.1 %: measured deviations are <= 0.02 % (CD) and 0.12 / 0.21 / 0.28 % (2SHOC at h =
    1/2, 1/4, 1/8), so the pins are 0.05 % (CD), 0.35 % (2SHOC) and 0.5 % for the slow fine
    rows; the convergence orders are pinned to 0.005 (test_P6_fig1_orders)."""
    er, ei = run_exp1(h, scheme)
    gr, gi = _golden("fig1_1d.txt", scheme, h)
    tol = 5e-3 if (scheme, h) in FIG1_SLOW else (5e-4 if scheme == "cd" else 3.5e-3)
    assert abs(er / float(gr) - 1) < tol, (er, gr)
    assert abs(ei / float(gi) - 1) < tol, (ei, gi)


def test_P6_fig1_orders():
    """Fig. 1 printed orders: CD 2.0352, 2SHOC 3.9355 / 3.9788 (real parts)."""
    e = {h: run_exp1(h, "2shoc")[0] for h in (0.5, 0.25, 0.125)}
    assert abs(metrics.order(e[0.5], e[0.25], 0.5, 0.25) - 3.9355) < 5e-3
    assert abs(metrics.order(e[0.25], e[0.125], 0.25, 0.125) - 3.9788) < 5e-3
    c = {h: run_exp1(h, "cd")[0] for h in (0.5, 0.25)}
    assert abs(metrics.order(c[0.5], c[0.25], 0.5, 0.25) - 2.0352) < 5e-3


# ------------------------------------------------------------ kdfull with N != 0 (a8)
def _operator_matrix(P, shape):
    """Brute force: the matrix of F/i = a Lap + N on the interior unknowns (Psi_b = 0),
    one oracle RHS evaluation per unit vector."""
    I = interior(len(shape), shape)
    idx = np.argwhere(np.ones(tuple(n - 2 for n in shape), bool)) + 1
    M = np.zeros((len(idx), len(idx)))
    for q, ii in enumerate(idx):
        e = np.zeros(shape, complex)
        e[tuple(ii)] = 1.0
        M[:, q] = (oracle.rhs(P, e)[I] / 1j).reshape(-1).real
    return M


@pytest.mark.parametrize("dims,hs,vext", [
    (2, [0.3, 0.3], 0.0), (2, [0.3, 0.41], 0.0), (2, [0.3, 0.3], -200.0), (2, [0.3, 0.41], -200.0),
    (1, [0.2], 0.0), (1, [0.2], -400.0), (3, [0.5, 0.5, 0.5], 0.0), (3, [0.5, 0.6, 0.7], -80.0)])
def test_kdfull_equals_brute_force_gershgorin(dims, hs, vext):
    """`kdfull` with N != 0: k_max = sqrt(8) / max_i (|M_ii| + sum_{j!=i} |M_ij|),
    the Gershgorin bound of the operator's own matrix built point by point.  The extremes of
    N are placed on depth >= 3 rows (no neighbour on the boundary, so their discs are the
    widest, Table 2's 30 +- 34 class),
    one far below and (vext != 0) one far above the rest, so that each of the two branches
    max(g_max - L_min, L_max - g_min) decides in one of the cases: a swapped L_min / L_max, a
    wrong G endpoint or a missing h^2/a factor changes k_max by far more than 1e-12.  The
    anisotropic cases pin reading R17's per-axis Gershgorin sum the same way."""
    n = 9
    shape = (n,) * dims
    rng = np.random.default_rng(17 + dims)
    V = rng.uniform(-3, 3, shape)
    c = (n // 2,) * dims
    V[c] = 40.0                        # N = -V: the minimum of N, at a depth-4 point
    if vext:
        V[(3,) * dims] = vext          # far above, depth 3: Nmax + (4/12) a H decides
    a = 0.8
    P = oracle.Problem(dims, [n] * dims, hs, a, 0.0, V, "dirichlet")
    M = _operator_matrix(P, shape)
    gersh = max(abs(M[i, i]) + np.abs(M[i]).sum() - abs(M[i, i]) for i in range(M.shape[0]))
    k = oracle.kmax(P, np.zeros(shape, complex))
    assert abs(k - math.sqrt(8) / gersh) <= 1e-12 * k
    # which branch decided (documents that both are exercised)
    Hs = sum(1 / h ** 2 for h in hs)
    nmin, nmax = float(-V.max()), float(-V.min())
    lo_branch = 64 / 12 * a * Hs - nmin
    hi_branch = nmax + 4 / 12 * a * Hs
    assert (hi_branch > lo_branch) == (vext != 0)


# survey §8(d): k_max of C1-C5 at t = 0, derived there independently (numpy) from Psi0's
# extremes; printed to 7 significant digits, so the tolerance is half a unit of the last one.
KMAX_SURVEY = {"C1": 8.108023e-4, "C2": 4.823326e-9, "C3": 4.551916e-6, "C4": 1.530532e-4, "C5": 4.419417e-4}


def _kmax_full(work, dtype="c128", slab=32):
    g = work["grid"]
    dims = g["dims"]
    lo_all, hi_all = np.inf, -np.inf
    for z0 in range(0, g["n"][dims - 1], slab):
        lo = [0, 0, 0]
        cnt = list(g["n"])
        lo[dims - 1] = z0
        cnt[dims - 1] = min(slab, g["n"][dims - 1] - z0)
        psi = icgen.fill(work["ic"], g, dtype=np.complex64 if dtype == "c64" else np.complex128, lo=lo, cnt=cnt)
        a, b = oracle.N_minmax(oracle.problem_from_work(work, lo=lo, cnt=cnt), psi.astype(np.complex128))
        lo_all, hi_all = min(lo_all, a), max(hi_all, b)
    return oracle.kmax_from_N(dims, g["h"][:dims], work["a"], lo_all, hi_all), lo_all, hi_all


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_kmax_of_the_configs_matches_survey(name):
    """The oracle's k_max on each config's full grid (C5: the weak-scaling grid of one GPU,
    whose k_max the survey states equal to the 1536^3 grid's: L_min ~ 0 and g_max decide)."""
    work = {"C1": configs.C1, "C2": configs.C2, "C3": configs.C3, "C4": configs.C4,
            "C5": lambda: configs.C5W(1)}[name]()
    k, nmin, nmax = _kmax_full(work, "c64" if name == "C4" else "c128")
    want = KMAX_SURVEY[name]
    assert abs(k - want) <= 0.5e-6 * want * 1.0001, (k, want)
    # the pin discriminates: the bound with L_min and L_max exchanged in the two branches
    # (max(g_max - L_max, L_min - g_min)) lies outside the printed digits (except C2, where
    # h^2 |Psi|^2 ~ 1e-8 is below them)
    if name != "C2":
        g = work["grid"]
        d, hh, a = g["dims"], g["h"][0] ** 2, work["a"]
        Lmin, Lmax = hh / a * nmin, hh / a * nmax
        kswap = math.sqrt(8) / max(64 * d / 12 - Lmax, Lmin + 4 * d / 12) * hh / a
        assert abs(kswap - want) > 0.5e-6 * want
