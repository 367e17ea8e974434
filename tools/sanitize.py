"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): C1,
virtual slabs with R = 2, heat bath (0 / 1 / 2 "always" classes), draw-free, the TMA-staged
kernel (shared memory + mbarrier, ragged band), both basic-layout kernels, measured chain,
graph replay."""
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
t = IsingLattice(34, 8192, 6).set_beta(0.4406868).init_random()  # TMA-staged, ragged band
t.sweep(2)
t.measure(2, 1)
t.set_beta(float("inf")).sweep(1)  # draw-free variant
t.set_beta(3.0, 1).sweep(1)  # heat bath, T[0] = 2^32
print("staged", t.observables())
h.set_beta(6.0, 1).sweep(1)  # heat bath, T[0] = T[1] = 2^32
print("heat bath 6", h.observables())
os.environ["ISING_BASIC_LISTING"] = "1"
b.sweep(1)
os.environ["ISING_BASIC_LISTING"] = "0"
print("basic listing", b.observables())
w = IsingLattice(64, 128, 5).write_lattice(np.ones((64, 128), dtype=np.int8), t=3).set_beta(0.0)
w.sweep(1)
print("write", w.observables(), w.read_rows(10, 2).sum())
