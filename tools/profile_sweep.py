"""Minimal driver for ncu: C3 lattice, random start, a few sweeps (nothing else).

PROF_N / PROF_M: lattice; PROF_SWEEPS: sweeps; PROF_LAYOUT=basic: byte-per-spin layout;
PROF_SELF=p2p|nccl: a one-rank handle running that multi-GPU transport with itself
(ISING_SELF_EXCHANGE=1), to profile the transport's per-GPU cost."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_06297_b200 import ising  # noqa: E402
from paper_1906_06297_b200.ising import IsingLattice  # noqa: E402

N = int(os.environ.get("PROF_N", "32768"))
M = int(os.environ.get("PROF_M", "32768"))
sweeps = int(os.environ.get("PROF_SWEEPS", "3"))
self_t = os.environ.get("PROF_SELF")
if os.environ.get("PROF_LAYOUT") == "basic":
    lat = IsingLattice.basic(N, M, 1)
elif self_t:
    os.environ["ISING_SELF_EXCHANGE"] = "1"
    h = (ising.ising_create_rank_p2p(N, M, 1, 0, 1, 0) if self_t == "p2p"
         else ising.ising_create_rank(N, M, 1, 0, 1, 0, None))
    lat = IsingLattice(N, M, 1, _handle=h)
else:
    lat = IsingLattice(N, M, 1)
lat.set_beta(0.4406868).init_random()
lat.sweep(sweeps)
print("sweep ms", lat.last_sweep_ms(), "flips/ns", N * M * sweeps / (lat.last_sweep_ms() * 1e6))
