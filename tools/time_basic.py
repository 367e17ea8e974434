import os, sys, math
sys.path.insert(0, os.getcwd())
from paper_1906_06297_b200.ising import IsingLattice
N = M = 32768
for listing in ["0", "1"]:
    os.environ["ISING_BASIC_LISTING"] = listing
    lat = IsingLattice.basic(N, M, 1).init_random()
    for name, beta, rule in [("metropolis", 0.4406868, 0), ("draw-free inf", math.inf, 0), ("heat bath", 0.4406868, 1)]:
        lat.set_beta(beta, rule); lat.sweep(2); lat.sweep(8)
        print(f"listing={listing} {name:15s} {N*M*8/(lat.last_sweep_ms()*1e6):8.1f} flips/ns")
    lat.close()
