"""Seeded input generator: counter-based RNG and box/slab independence (CPU)."""
import numpy as np

import icgen
from icgen import configs


def test_splitmix_reference_values():
    # SplitMix64 of 0 (Vigna's reference stream, first output for state 0) -> e220a8397b1dcdaf
    u = icgen.uniform(0, 0, 0)
    assert u == (0xE220A8397B1DCDAF >> 11) * 2.0 ** -53
    vals = [icgen.uniform(1, s, i) for s in range(4) for i in range(50)]
    assert all(0.0 <= v < 1.0 for v in vals)
    assert len(set(vals)) == len(vals)


def test_box_equals_region_of_whole_grid():
    """Noise is indexed by the GLOBAL linear index: any box (crop / z-slab) equals the
    same region of the full grid (needed for crops and sharding)."""
    w = configs.SMALL(3, (11, 9, 7), "dirichlet", noise=0.3)
    full = icgen.fill(w["ic"], w["grid"])
    box = icgen.fill(w["ic"], w["grid"], lo=[2, 3, 1], cnt=[5, 4, 3])
    assert np.array_equal(box, full[1:4, 3:7, 2:7])
    f64 = icgen.fill(w["ic"], w["grid"], dtype=np.complex64)
    assert np.array_equal(f64, full.astype(np.complex64))


def test_configs_shapes_and_spacing():
    c1 = configs.C1()
    assert c1["grid"]["n"][0] == 1024 and abs(c1["grid"]["h"][0] - 40 / 1023) < 1e-15
    c4 = configs.C4()
    assert c4["grid"]["n"] == [768] * 3 and abs(c4["grid"]["h"][0] - 16 / 767) < 1e-15
    c5 = configs.C5W(2)
    assert c5["grid"]["n"] == [768, 768, 384]
    assert abs(c5["grid"]["xmin"][2] + 383 / 2 * 0.05) < 1e-12
    e = configs.EXP_GAUSS(3, 0.5)
    assert e["grid"]["n"] == [25] * 3  # 25^3 points at h = 1/2 on [-6,6]^3


def test_c4_initial_state_small_sample():
    w = configs.C4()
    box = icgen.fill(w["ic"], w["grid"], lo=[380, 380, 380], cnt=[8, 8, 8])
    # |Psi0| <= sqrt(15) + noise; noise amplitude 1e-3
    assert np.abs(box).max() <= np.sqrt(15) + 2e-3
