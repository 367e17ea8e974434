"""Experiment: time k_halfsweep variants (libraries in tools/exp_*.so) on C3, with a quick
parity check against the oracle first.  Usage: python tools/exp_variants.py lib1.so lib2.so ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
from paper_1906_06297_b200.ising import IsingLattice, ising_probe_philox
import oracle
N, M = int(os.environ.get("PN", 130)), int(os.environ.get("PM", 8192))
g = IsingLattice(N, M, 3).set_beta(0.4406868).init_random(); g.sweep(50)
o = oracle.Lattice(N, M, 3).set_beta(0.4406868).init_random(); o.sweep(50)
ok = np.array_equal(g.read_lattice(), o.full())
g.close()
res = []
for H in [int(x) for x in os.environ.get("HS", "0").split(",")]:
    os.environ["ISING_ROWS_PER_ITEM"] = str(H)
    lat = IsingLattice(32768, 32768, 1).set_beta(0.4406868).init_random()
    lat.sweep(4)
    lat.sweep(32)
    ms = lat.last_sweep_ms()
    res.append((H, 32768 * 32768 * 32 / (ms * 1e6)))
    lat.close()
print(os.environ["ISING_LIB"], "parity", ok, " ".join(f"H={h}:{v:.0f}" for h, v in res),
      "philox_probe", round(ising_probe_philox(0)))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, ISING_LIB=os.path.abspath(lib), ROOT=ROOT)
    subprocess.run([sys.executable, "-c", CHILD], env=env)
