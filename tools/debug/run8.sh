cat > /tmp/mir.py <<'X'
import os, sys
sys.path.insert(0, ".")
from paper_1906_06297_b200.ising import IsingLattice
import numpy as np
res = {}
for mode in ["0", "1", "0", "1"]:
    os.environ["ISING_MIRROR"] = mode
    for N, M in [(32768, 32768), (16384, 32768)]:
        lat = IsingLattice(N, M, 1).set_beta(0.4406868).init_random()
        lat.sweep(8); lat.sweep(64)
        res.setdefault((mode, N), []).append(N * M * 64 / (lat.last_sweep_ms() * 1e6))
        lat.close()
print(res)
# parity of the mirrored order against the oracle
import oracle
os.environ["ISING_MIRROR"] = "1"
for N, M in [(130, 8192), (2400, 32768)]:
    g = IsingLattice(N, M, 3).set_beta(0.4406868).init_random().sweep(3)
    o = oracle.Lattice(N, M, 3).init_random().set_beta(0.4406868).sweep(3)
    print(N, M, "parity", np.array_equal(g.read_lattice(), o.full()))
X
timeout 600 python /tmp/mir.py
