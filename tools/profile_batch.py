"""Minimal driver for ncu: one lattice batch launch (PROF_L x PROF_L, PROF_N lattices, beta_c,
PROF_SWEEPS sweeps in one launch).  ncu -k regex:k_batch python tools/profile_batch.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_06297_b200.ising import IsingBatch  # noqa: E402

L = int(os.environ.get("PROF_L", "512"))
n = int(os.environ.get("PROF_N", "592"))
sweeps = int(os.environ.get("PROF_SWEEPS", "64"))
b = IsingBatch(L, L, list(range(1, n + 1))).set_beta(np.full(n, 0.4406868)).init_random()
b.sweep(sweeps)
print("flips/ns", n * L * L * sweeps / (b.last_sweep_ms() * 1e6))
b.close()
