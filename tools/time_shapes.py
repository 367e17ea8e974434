"""Metropolis flips/ns at beta_c for several lattice shapes (tail / wave-quantisation check):
same row width with more rows, and wider rows.  Usage: python tools/time_shapes.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_06297_b200.ising import IsingLattice  # noqa: E402

shapes = [(16384, 32768), (32768, 32768), (65536, 32768), (131072, 32768), (32768, 131072),
          (8192, 131072), (131072, 131072)]
for N, M in shapes:
    lat = IsingLattice(N, M, 1).set_beta(0.4406868).init_random()
    lat.sweep(2)
    n = max(4, int(2**34 // (N * M)))
    lat.sweep(n)
    print(f"{N:7d} x {M:7d}  {N * M * n / (lat.last_sweep_ms() * 1e6):8.1f} flips/ns", flush=True)
    lat.close()
