"""The dependency-cone crop used by the full-size parity tests (CPU only): the oracle run on
shrinking crops equals the oracle run on the whole grid, bit for bit, inside the target box
(SURVEY §8(c) "Oracle at scale"; tests/harness.py oracle_crop_rk4)."""
import numpy as np
import pytest

import oracle
from icgen import configs

import harness as H


@pytest.mark.parametrize("dims,n,bc,V", [
    (2, (90, 70), "dirichlet", "harmonic"), (3, (40, 36, 44), "dirichlet", "harmonic"),
    (3, (38, 40, 42), "lapzero", "none"), (1, (400,), "lapzero", "harmonic")])
def test_shrinking_crop_is_bitwise_the_full_oracle(dims, n, bc, V):
    w = configs.SMALL(dims, n, bc, dtype="c128", V=V, h=[0.11, 0.13, 0.17][:dims])
    psi = H.psi0_host(w, "c128")
    P = H.oracle_problem(w)
    dt = 0.8 * oracle.kmax(P, psi)
    nsteps = 3
    full = oracle.rk4(P, psi, dt, nsteps)
    boxes = [([0, 0, 0], [6, 5, 4]), ([n[0] - 7] + [0, 0], [7, 4, 3])]
    if dims >= 2:
        boxes.append(([n[0] // 2 - 3, n[1] // 2 - 2, 0], [6, 4, 1 if dims == 2 else 5]))
    for tlo, tcnt in boxes:
        tlo = tlo[:dims] + [0] * (3 - dims)
        tcnt = tcnt[:dims] + [1] * (3 - dims)
        for seg in (1, 2, 10):
            got = H.oracle_crop_rk4(w, "c128", tlo, tcnt, dt, nsteps, segments=seg)
            want = full[H.sl(dims, tlo, tcnt)]
            assert np.array_equal(got, want), (tlo, seg)


def test_crop_margin_is_needed():
    """A crop one cell short of the 8n margin is not exact (the margin is tight, so the test
    above is not vacuous)."""
    w = configs.SMALL(2, (90, 70), "dirichlet", dtype="c128", V="harmonic", h=[0.11, 0.13])
    psi = H.psi0_host(w, "c128")
    P = H.oracle_problem(w)
    dt = 0.8 * oracle.kmax(P, psi)
    full = oracle.rk4(P, psi, dt, 2)
    tlo, tcnt = [40, 30, 0], [6, 6, 1]
    m = 8 * 2 - 1
    lo, cnt = [tlo[0] - m, tlo[1] - m, 0], [tcnt[0] + 2 * m, tcnt[1] + 2 * m, 1]
    got = oracle.rk4(H.oracle_problem(w, lo, cnt), H.psi0_host(w, "c128", lo, cnt), dt, 2)
    assert not np.array_equal(got[m:m + 6, m:m + 6], full[30:36, 40:46])
