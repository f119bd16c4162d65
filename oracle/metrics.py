"""Error metric and convergence order of the paper's accuracy experiments.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings (R1-R3):
  E^n = ||Re(Psi^n - Psi_exact^n)||_2 / sqrt(N)  and the same for Im  (RMS; the paper
        prints "/N" at P:500 but its tables are reproduced only by the RMS form)
  E   = mean of E^n over the 100 snapshots t_j = j t_end / 100, j = 1..100
  O   = ln(E_h1 / E_h2) / ln(h1 / h2)   (P:500 prints "ln E_h1 - ln E_h2")
"""
from __future__ import annotations

import math

import numpy as np


def rms_err(psi, exact):
    e = np.asarray(psi) - np.asarray(exact)
    n = e.size
    return (float(np.sqrt(np.sum(e.real ** 2) / n)), float(np.sqrt(np.sum(e.imag ** 2) / n)))


def order(E1, E2, h1, h2):
    return math.log(E1 / E2) / math.log(h1 / h2)
