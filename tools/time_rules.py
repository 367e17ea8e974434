"""C3 flips/ns for each kernel variant: Metropolis (fast / generic) and heat bath (0 / 1 / 2 "always" classes)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_06297_b200.ising import IsingLattice  # noqa: E402

N = M = 32768
lat = IsingLattice(N, M, 1).init_random()
for name, beta, rule in [("metropolis fast", 0.4406868, 0), ("metropolis generic (beta=4e-11)", 4e-11, 0),
                         ("metropolis draw-free (beta=inf)", math.inf, 0), ("metropolis draw-free (beta=0)", 0.0, 0),
                         ("heat bath fast", 0.4406868, 1), ("heat bath T0=2^32 (beta=3)", 3.0, 1),
                         ("heat bath T0=T1=2^32 (beta=inf)", math.inf, 1)]:
    lat.set_beta(beta, rule)
    lat.sweep(4)
    lat.sweep(16)
    print(f"{name:30s} {N * M * 16 / (lat.last_sweep_ms() * 1e6):8.1f} flips/ns  (variant {lat.kernel_variant()})")
