"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck): C1, virtual
slabs with R = 2, heat bath, basic layout, measured chain, graph replay."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_06297_b200.ising import IsingLattice  # noqa: E402

g = IsingLattice(64, 64, 1).set_beta(0.4406868).init_random()
g.sweep(70)  # one graph replay + remainder
g.measure(5, 2)
print("C1", g.observables())
s = IsingLattice(16, 64, 2, devices=[0] * 8).set_beta(0.4406868).init_random()
s.sweep(3)
print("slabs", s.observables(), s.read_lattice().sum())
h = IsingLattice(64, 128, 3).set_beta(0.3, 1).init_random()
h.sweep(3)
print("heat bath", h.observables())
b = IsingLattice.basic(64, 64, 4).set_beta(0.4406868).init_random()
b.sweep(3)
print("basic", b.observables())
w = IsingLattice(64, 128, 5).write_lattice(np.ones((64, 128), dtype=np.int8), t=3).set_beta(0.0)
w.sweep(1)
print("write", w.observables(), w.read_rows(10, 2).sum())
