"""Debug: local rank-p2p group measured chains step by step (python tools/debug/group_measure.py CASE)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1906_06297_b200 import ising  # noqa: E402
from paper_1906_06297_b200.ising import IsingLattice, run_ranks  # noqa: E402

case = sys.argv[1]
world, N, M = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
lats = IsingLattice.local_group(N, M, world, 3)
t0 = time.time()


def log(*a):
    print(f"[{time.time() - t0:6.2f}s]", *a, flush=True)


def body(r, lat):
    row0, rows = lat.slab_info()
    if "write" in case:
        start = np.ones((rows, M), dtype=np.int8)
        lat.set_beta(0.44).write_lattice(start, t=40)
    else:
        lat.set_beta(0.44).init_random()
    log(r, "state set")
    if "skew" in case and r == 0:
        time.sleep(1.0)
    if "sweep" in case:
        lat.sweep(3)
        log(r, "swept")
    if "obs" in case:
        log(r, "obs", lat.observables())
    if "measure" in case:
        for k in range(3):
            ups, Es = lat.measure(1, 1)
            log(r, "measure", k, ups, Es)
    return 0


run_ranks(lats, body)
log("done")
