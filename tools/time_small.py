"""Time C1 / C2-sized sweeps (launch-bound regime) with and without CUDA graphs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_06297_b200.ising import IsingLattice  # noqa: E402

for N in [64, 512, 2048, 4096]:
    lat = IsingLattice(N, N, 1).set_beta(0.4406868).init_random()
    lat.sweep(256)
    t0 = time.perf_counter()
    lat.sweep(2048)
    wall = time.perf_counter() - t0
    ms = lat.last_sweep_ms()
    print(f"ISING_GRAPHS={os.environ.get('ISING_GRAPHS', '1')} L={N}: device {N*N*2048/(ms*1e6):8.1f} flips/ns, "
          f"wall {N*N*2048/(wall*1e9):8.1f} flips/ns, {1e3*ms/2048:.2f} us/sweep")
    lat.close()

# measured chain (observables fused into the white phase) on C2: every = 1 and 10
for every in [1, 10]:
    lat = IsingLattice(2048, 2048, 1).set_beta(0.4406868).init_random()
    lat.sweep(64)
    t0 = time.perf_counter()
    lat.measure(2048 // every, every)
    wall = time.perf_counter() - t0
    print(f"measure every={every}: device {2048*2048*2048/(lat.last_sweep_ms()*1e6):8.1f} flips/ns, "
          f"wall {2048*2048*2048/(wall*1e9):8.1f} flips/ns")
    lat.close()
