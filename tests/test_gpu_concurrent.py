"""Multi-rank transports under real concurrency, and each transport's one-device form.

* Local groups (ising_p2p_connect_local): every rank of a rank-p2p lattice in this process,
  one host thread per rank, all on cuda:0 — the ranks' kernels run concurrently on separate
  streams, so writer and reader of a halo row overlap in time (the multi-process same-GPU
  tests are time-sliced and always separate them by a kernel boundary).  Long chains (500
  sweeps in one call per rank, the ranks coupled only through the flags in peer memory) are
  compared with the oracle bit for bit (reading R19).
* Self exchange (ISING_SELF_EXCHANGE=1, world 1): the rank is its own neighbour through the
  whole protocol — the rank-p2p flags / fences / peer-store path (over CUDA IPC mappings, and
  over NCCL symmetric-memory windows: ising_create_rank_lsa), and the NCCL transport's
  boundary-rows-first, ncclSend/ncclRecv-on-a-comm-stream, interior-overlap path
  (PAPER.md:224), which NCCL does not allow for two ranks on one GPU.
"""
import numpy as np
import pytest

import oracle
from paper_1906_06297_b200 import ising
from paper_1906_06297_b200.ising import IsingLattice, run_ranks
from tests import cases

pytestmark = pytest.mark.gpu
BETA = cases.BETA_TC


def gather_group(lats):
    """Each rank reads its own rows (slab-only read); concatenated in rank order."""
    def rd(r, lat):
        row0, rows = lat.slab_info()
        out = np.empty((rows, lat.M), dtype=np.int8)
        lat.read_lattice(out)
        return out
    return np.concatenate(run_ranks(lats, rd))


def close_group(lats):
    for lat in lats:
        lat.close()


# (world, N, M): 8192 columns run the TMA-staged kernel (edge bands wait, interior bands do
# not; R = 64 gives 4 bands, R = 2 makes every band an edge band), 128 / 192 columns the
# register-rolling kernel (every block waits)
GROUP_CASES = [(2, 128, 8192), (4, 256, 8192), (8, 16, 8192), (2, 64, 128), (4, 96, 192),
               (3, 120, 8192)]


@pytest.mark.parametrize("world,N,M", GROUP_CASES)
def test_local_group_500_sweeps_matches_oracle(world, N, M):
    seed = 11
    lats = IsingLattice.local_group(N, M, world, seed)
    try:
        run_ranks(lats, lambda r, lat: lat.set_beta(BETA).init_random())
        run_ranks(lats, lambda r, lat: lat.sweep(500))  # one call: 1000 phases per rank
        obs = run_ranks(lats, lambda r, lat: lat.observables())
        got = gather_group(lats)
    finally:
        close_group(lats)
    o = oracle.Lattice(N, M, seed).init_random().set_beta(BETA).sweep(500)
    assert np.array_equal(got, o.full()), f"{int((got != o.full()).sum())} sites differ"
    assert all(x == o.observables() for x in obs), (obs, o.observables())


def test_local_group_measured_chain_load_and_heat_bath():
    world, N, M, seed = 4, 128, 8192, 3
    rng = np.random.default_rng(5)
    start = cases.random_pm1(rng, N, M, 0.7)
    lats = IsingLattice.local_group(N, M, world, seed)
    try:
        def body(r, lat):
            row0, rows = lat.slab_info()
            lat.set_beta(BETA).write_lattice(np.ascontiguousarray(start[row0:row0 + rows]), t=40)
            ups, Es = lat.measure(6, 3)          # fused observables, all-reduced over peers
            lat.set_beta(0.3, ising.RULE_HEATBATH)
            lat.sweep(7)
            u2 = np.zeros(4, dtype=np.int64)
            e2 = np.zeros(4, dtype=np.int64)
            lat.measure_wait(lat.measure_async(4, 1, u2, e2))
            return ups.tolist(), Es.tolist(), u2.tolist(), e2.tolist(), lat.observables()
        res = run_ranks(lats, body)
        got = gather_group(lats)
    finally:
        close_group(lats)
    o = oracle.Lattice(N, M, seed).load_full(start, t=40).set_beta(BETA)
    ou, oE = o.chain(18)
    o.set_beta(0.3, oracle.RULE_HEATBATH).sweep(7)
    ou2, oE2 = o.chain(4)
    for ups, Es, u2, e2, obs in res:  # every rank holds the global values
        assert ups == [int(x) for x in ou[2::3]] and Es == [int(x) for x in oE[2::3]]
        assert u2 == [int(x) for x in ou2] and e2 == [int(x) for x in oE2]
        assert obs == o.observables()
    assert np.array_equal(got, o.full())


def test_local_group_large_invariance_vs_one_slab():
    """4 concurrent ranks of an 8192 x 32768 lattice (C3 width, staged kernel, guided-tail
    geometry per slab) after 100 sweeps equal the one-slab lattice byte for byte."""
    world, N, M, seed, n = 4, 8192, 32768, 1, 100
    lats = IsingLattice.local_group(N, M, world, seed)
    try:
        run_ranks(lats, lambda r, lat: lat.set_beta(BETA).init_random())
        run_ranks(lats, lambda r, lat: lat.sweep(n))
        obs = run_ranks(lats, lambda r, lat: lat.observables())
        got = gather_group(lats)
    finally:
        close_group(lats)
    one = IsingLattice(N, M, seed).set_beta(BETA).init_random().sweep(n)
    try:
        assert np.array_equal(got, one.read_lattice())
        assert all(x == one.observables() for x in obs)
    finally:
        one.close()


@pytest.fixture
def self_exchange(monkeypatch):
    monkeypatch.setenv("ISING_SELF_EXCHANGE", "1")


@pytest.mark.parametrize("transport", ["p2p", "nccl", "lsa"])
@pytest.mark.parametrize("N,M", [(64, 64), (130, 192), (2, 64), (96, 8192), (7168, 32768)])
def test_self_exchange_transport_matches_oracle(self_exchange, transport, N, M):
    seed = 2
    if transport == "p2p":
        h = ising.ising_create_rank_p2p(N, M, seed, 0, 1, 0)
    elif transport == "lsa":  # the p2p kernel protocol over NCCL symmetric-memory windows
        h = ising.ising_create_rank_lsa(N, M, seed, 0, 1, 0, None)
    else:
        h = ising.ising_create_rank(N, M, seed, 0, 1, 0, None)
    g = IsingLattice(N, M, seed, _handle=h)
    try:
        g.set_beta(BETA).init_random()
        o = oracle.Lattice(N, M, seed).init_random().set_beta(BETA)
        n = 3 if N * M > 1 << 24 else 40
        g.sweep(n)
        o.sweep(n)
        assert np.array_equal(g.read_lattice(), o.full())
        assert g.observables() == o.observables()
        ups, Es = g.measure(3, 2)
        ou, oE = o.chain(6)
        assert ups.tolist() == [int(x) for x in ou[1::2]]
        assert Es.tolist() == [int(x) for x in oE[1::2]]
    finally:
        g.close()


def test_profiling_survives_measured_chains():
    """profiling on, then the measure paths (which never time launches) must not
    index past the event pool; ising_sweep's stats stay those of the last ising_sweep."""
    for N, M in [(64, 128), (2048, 8192)]:
        g = IsingLattice(N, M, 1).set_beta(BETA).init_random()
        try:
            g.set_profiling(True)
            g.measure(3, 2)
            u = np.zeros(2, dtype=np.int64)
            e = np.zeros(2, dtype=np.int64)
            g.measure_wait(g.measure_async(2, 1, u, e))
            g.sweep(5)
            ms, launches = g.kernel_stats()
            assert launches == 10 and ms > 0
            g.measure(2, 1)
            assert g.kernel_stats()[1] == 10
        finally:
            g.close()


def test_trace_timeline_of_the_nccl_transport(self_exchange, monkeypatch, tmp_path):
    """ISING_TRACE: every traced half-sweep records its boundary rows, the halo group on the
    comm stream and the interior, in stream order, and the result stays bit-exact."""
    import csv

    path = tmp_path / "trace.csv"
    monkeypatch.setenv("ISING_TRACE", str(path))
    N, M, seed = 96, 8192, 3
    g = IsingLattice(N, M, seed, _handle=ising.ising_create_rank(N, M, seed, 0, 1, 0, None))
    g.set_beta(BETA).init_random().sweep(3)
    got = g.read_lattice()
    g.close()  # writes the trace
    o = oracle.Lattice(N, M, seed).init_random().set_beta(BETA).sweep(3)
    assert np.array_equal(got, o.full())
    rows = list(csv.DictReader(open(path)))
    phases = sorted({int(r["phase"]) for r in rows})
    assert phases == list(range(6))
    for p in phases:
        ev = {r["name"]: float(r["ms"]) for r in rows if int(r["phase"]) == p}
        assert set(ev) == {"boundary_start", "boundary_end", "halo_start", "halo_end",
                           "interior_start", "interior_end"}
        assert ev["boundary_start"] <= ev["boundary_end"] <= ev["halo_start"] <= ev["halo_end"]
        assert ev["boundary_end"] <= ev["interior_start"] <= ev["interior_end"]
