"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): C1,
virtual slabs with R = 2, heat bath (0 / 1 / 2 "always" classes), draw-free, the TMA-staged
kernel (shared memory + mbarrier, ragged band), both basic-layout kernels, measured chain,
graph replay, the asynchronous measured chain, the rank transports in self-exchange form
(p2p flags / fences, NCCL self send-recv), lattice batches (one CTA and thread-block-cluster
forms), and (SANITIZE_BIG=1) the guided tail.  (Not the
same-process rank groups: the sanitizer serialises kernels, and a rank's phase that waits on
another rank's flags can then never see them.)"""
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
a = IsingLattice(64, 64, 7).set_beta(0.4406868).init_random()  # asynchronous measured chain
bufs = [np.zeros(3, dtype=np.int64) for _ in range(4)]
t1 = a.measure_async(3, 1, bufs[0], bufs[1])
t2 = a.measure_async(3, 1, bufs[2], bufs[3])
a.measure_wait(t1)
a.measure_wait(t2)
print("async", bufs[1].tolist(), bufs[3].tolist(), "variant", h.kernel_variant())
from paper_1906_06297_b200 import ising  # noqa: E402

os.environ["ISING_SELF_EXCHANGE"] = "1"
for name, mk in (("p2p-self", lambda: ising.ising_create_rank_p2p(96, 8192, 8, 0, 1, 0)),
                 ("nccl-self", lambda: ising.ising_create_rank(96, 8192, 8, 0, 1, 0, None))):
    x = IsingLattice(96, 8192, 8, _handle=mk()).set_beta(0.4406868).init_random()
    x.sweep(2)
    x.measure(2, 1)
    print(name, x.observables())
    x.close()
os.environ.pop("ISING_SELF_EXCHANGE")
from paper_1906_06297_b200.ising import IsingBatch  # noqa: E402

# lattice batches: one CTA per lattice (shared-memory planes, row bands) and thread-block
# clusters (halo rows over distributed shared memory, cluster barriers, DSMEM atomics)
for (N, M, n), rule in (((64, 128, 3), 0), ((96, 192, 2), 1), ((1024, 512, 2), 0), ((1024, 512, 2), 1)):
    bt = IsingBatch(N, M, list(range(n))).set_beta([0.3, 0.4406868, 0.0][:n], rule).init_random()
    bt.sweep(3)
    bt.measure(2, 2)
    bt.write_lattice(0, bt.read_lattice(1), t=bt.t)
    print("batch", N, M, rule, bt.observables()[1].tolist())
    bt.close()
if os.environ.get("SANITIZE_BIG"):  # >= 3 waves: the staged kernel's guided tail (memcheck)
    big = IsingLattice(7168, 32768, 9).set_beta(0.4406868).init_random()
    big.sweep(1)
    print("tail", big.observables())
