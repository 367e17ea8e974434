"""Lattice-batch throughput per acceptance rule (Metropolis / heat bath) at three sizes."""
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_1906_06297_b200.ising import IsingBatch
for rule in (0, 1):
    for L, n, sw in [(64, 2368, 2048), (512, 592, 128), (1024, 148, 64)]:
        b = IsingBatch(L, L, list(range(n))).set_beta(np.full(n, 0.4406868), rule).init_random()
        b.sweep(4); b.sweep(sw)
        print("rule", rule, "L", L, "n", n, round(n * L * L * sw / (b.last_sweep_ms() * 1e6)), "flips/ns")
        b.close()
