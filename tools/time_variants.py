"""C3 (and 16384 x 32768) flips/ns of several libising builds, interleaved rounds, one process
per library per round: python tools/time_variants.py ROUNDS lib1.so lib2.so ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"])
from paper_1906_06297_b200.ising import IsingLattice
r = []
for N, M in [(32768, 32768), (16384, 32768)]:
    lat = IsingLattice(N, M, 1).set_beta(0.4406868).init_random()
    lat.sweep(8); lat.sweep(64)
    r.append(N * M * 64 / (lat.last_sweep_ms() * 1e6))
    lat.close()
print(" ".join(f"{x:.1f}" for x in r))
'''
rounds = int(sys.argv[1])
res = {lib: [] for lib in sys.argv[2:]}
for _ in range(rounds):
    for lib in sys.argv[2:]:
        env = dict(os.environ, ISING_LIB=os.path.abspath(lib), ROOT=ROOT)
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        res[lib].append(out.stdout.strip() or out.stderr[-200:])
for lib, v in res.items():
    print(os.path.basename(lib), " | ".join(v))
