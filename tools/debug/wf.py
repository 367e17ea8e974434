import os, sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_1906_06297_b200.ising import IsingLattice
import oracle

def run(N, M, n, wf, seed=3, beta=0.4406868):
    os.environ["ISING_WAVEFRONT"] = "1" if wf else "0"
    g = IsingLattice(N, M, seed).set_beta(beta).init_random()
    g.sweep(n)
    out = g.read_lattice(), g.observables()
    g.close()
    return out

# parity: wavefront vs per-phase vs oracle
for N, M, n in [(4096, 8192, 3), (6000, 8192, 7), (8198, 16384, 2)]:
    a, oa = run(N, M, n, True)
    b, ob = run(N, M, n, False)
    print(N, M, n, "wf==phases", np.array_equal(a, b) and oa == ob, flush=True)
o = oracle.Lattice(4100, 8192, 3).init_random().set_beta(0.4406868).sweep(5)
a, oa = run(4100, 8192, 5, True)
print("wf==oracle", np.array_equal(a, o.full()) and oa == o.observables(), flush=True)
res = {}
for rep in range(2):
    for wf in (False, True):
        for N, M in [(32768, 32768), (16384, 32768), (131072, 131072)]:
            os.environ["ISING_WAVEFRONT"] = "1" if wf else "0"
            lat = IsingLattice(N, M, 1).set_beta(0.4406868).init_random()
            k = 64 if N <= 32768 else 8
            lat.sweep(4); lat.sweep(k)
            res.setdefault((wf, N), []).append(round(N * M * k / (lat.last_sweep_ms() * 1e6), 1))
            lat.close()
print(res)
