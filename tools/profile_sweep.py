"""Minimal driver for ncu: C3 lattice, random start, a few sweeps (nothing else)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_06297_b200.ising import IsingLattice  # noqa: E402

N = int(os.environ.get("PROF_N", "32768"))
M = int(os.environ.get("PROF_M", "32768"))
sweeps = int(os.environ.get("PROF_SWEEPS", "3"))
if os.environ.get("PROF_LAYOUT") == "basic":
    lat = IsingLattice.basic(N, M, 1).set_beta(0.4406868).init_random()
else:
    lat = IsingLattice(N, M, 1).set_beta(0.4406868).init_random()
lat.sweep(sweeps)
print("sweep ms", lat.last_sweep_ms(), "flips/ns", N * M * sweeps / (lat.last_sweep_ms() * 1e6))
