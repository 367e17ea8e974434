"""GPU physics pins: BASELINE configs[1] (2048^2, T = 1.5 and 3.0, 20000 sweeps) against
Onsager's magnetization, and the critical point."""
import numpy as np
import pytest

from oracle import exact
from paper_1906_06297_b200 import ising
from paper_1906_06297_b200.ising import IsingLattice
from tests import cases

pytestmark = pytest.mark.gpu


def measure_series(L, T, start, seed, sweeps, discard, every, rule=0):
    g = IsingLattice(L, L, seed).set_beta(1.0 / T, rule)
    g.init_cold() if start == "cold" else g.init_random()
    g.sweep(discard)
    ups, Es = g.measure((sweeps - discard) // every, every)  # device-side series
    g.close()
    return (2 * ups - L * L) / (L * L), Es / (L * L)


@pytest.mark.parametrize("T,start,expect", [(1.5, "cold", exact.onsager_m(1.5)), (3.0, "random", 0.0)])
@pytest.mark.parametrize("seed", [1, 2])
def test_c2_onsager(T, start, expect, seed):
    # BASELINE configs[1]: 2048^2, 20000 sweeps, discard 2000, sample every 10 sweeps;
    # |<|m|> - M_Onsager| <= 0.003 (north_star).  T = 1.5 starts cold (reading R21 / the
    # band meta-stability the paper reports for L > 1024).
    L, sweeps = cases.C2[0], cases.C2[3]
    m, e = measure_series(L, T, start, seed, sweeps, 2000, 10)
    mean, se = exact.batch_means(np.abs(m), 50)
    assert abs(mean - expect) <= 0.003, (mean, se)
    assert se < 0.001
    # the same exact solution's energy per site (oracle/exact.onsager_energy)
    assert abs(np.mean(e) - exact.onsager_energy(T)) <= 0.001


def test_heatbath_equilibrium_matches_onsager():
    # heat-bath dynamics has the same equilibrium: T = 2.0 on 2048^2
    m, e = measure_series(2048, 2.0, "cold", 3, 12000, 2000, 10, rule=1)
    assert abs(np.mean(np.abs(m)) - exact.onsager_m(2.0)) <= 0.003
    assert abs(np.mean(e) - exact.onsager_energy(2.0)) <= 0.001


def binder_point(L, T, seed, sweeps, every=1):
    g = IsingLattice(L, L, seed).set_beta(1.0 / T).init_cold()
    g.sweep(2000)
    ups, _ = g.measure(sweeps // every, every)
    g.close()
    m = (2 * ups - L * L) / (L * L)
    return exact.binder(np.mean(m**2), np.mean(m**4))


@pytest.mark.slow
def test_binder_crossing_on_gpu():
    # conventional U_L (reading R15): below Tc the larger lattice has the larger U, above
    # Tc the smaller one, so the curves cross between (Fig. 6 method).
    lo, hi = 2.21, 2.33
    u64 = [binder_point(64, T, 11, 200_000, 10) for T in (lo, hi)]
    u128 = [binder_point(128, T, 12, 200_000, 10) for T in (lo, hi)]
    assert u128[0] > u64[0], (u64, u128)
    assert u128[1] < u64[1], (u64, u128)


def test_measured_chain_matches_oracle_series():
    # ising_sweep_measure's device-side series equals the oracle chain sample by sample
    import oracle

    # (small lattices replay measured-chain graphs of 64 // every samples; the plans mix
    # replays and remainders, and a second call reuses the graph)
    for N, M, every, slabs, ns in [(64, 64, 1, None, 40), (64, 64, 1, None, 200),
                                   (128, 192, 7, None, 40), (96, 128, 3, [0, 0, 0], 40)]:
        g = IsingLattice(N, M, 4, devices=slabs).set_beta(0.4406868).init_random()
        o = oracle.Lattice(N, M, 4).set_beta(0.4406868).init_random()
        for _ in range(2):
            ups, Es = g.measure(ns, every)
            ou, oE = o.chain(ns * every)
            assert np.array_equal(ups, ou[every - 1::every]) and np.array_equal(Es, oE[every - 1::every])
            assert g.t == o.t


def test_async_measured_chain_matches_oracle_series():
    # ising_sweep_measure_async: pipelined calls (enqueue k + 1, then wait for k) give the
    # oracle's series sample by sample, into pinned host memory; interleaved plain sweeps
    # keep stream order; graph-replayed and direct paths; slabs on one device; a basic-layout
    # handle takes the synchronous fallback
    import oracle
    import torch

    for N, M, every, slabs, ns, calls in [(64, 64, 1, None, 5, 12), (128, 192, 3, [0, 0], 4, 6),
                                          (34, 8192, 1, None, 1, 9), (64, 64, 1, None, 70, 2)]:
        g = IsingLattice(N, M, 6, devices=slabs).set_beta(0.4406868).init_random()
        o = oracle.Lattice(N, M, 6).set_beta(0.4406868).init_random()
        ups = torch.zeros((calls, ns), dtype=torch.int64).pin_memory().numpy()
        Es = torch.zeros((calls, ns), dtype=torch.int64).pin_memory().numpy()
        tickets = []
        for k in range(calls):
            if k == calls // 2:
                g.sweep(2)  # a plain sweep between async calls (stream-ordered)
            tickets.append(g.measure_async(ns, every, ups[k], Es[k]))
            if k >= 1:
                g.measure_wait(tickets[k - 1])
        g.measure_wait(tickets[-1])
        for k in range(calls):
            if k == calls // 2:
                o.sweep(2)
            ou, oE = o.chain(ns * every)
            assert np.array_equal(ups[k], ou[every - 1::every]), (N, M, k)
            assert np.array_equal(Es[k], oE[every - 1::every]), (N, M, k)
        assert g.t == o.t
        assert np.array_equal(g.read_lattice(), o.full())
        g.close()
    b = IsingLattice.basic(64, 64, 6).set_beta(0.3).init_random()
    ob = oracle.Lattice(64, 64, 6).set_beta(0.3).init_random()
    u = np.zeros(3, dtype=np.int64)
    e = np.zeros(3, dtype=np.int64)
    b.measure_wait(b.measure_async(3, 2, u, e))
    ou, oE = ob.chain(6)
    assert np.array_equal(u, ou[1::2]) and np.array_equal(e, oE[1::2])


def test_async_measure_errors():
    g = IsingLattice(64, 64, 1).set_beta(0.3).init_random()
    bufs = [(np.zeros(1, dtype=np.int64), np.zeros(1, dtype=np.int64)) for _ in range(9)]
    tickets = [g.measure_async(1, 1, u, e) for u, e in bufs[:8]]
    with pytest.raises(ising.IsingError) as err:  # a ninth pending call
        g.measure_async(1, 1, *bufs[8])
    assert err.value.status == ising.ISING_ERR_STATE
    for t in tickets:
        g.measure_wait(t)
    with pytest.raises(ising.IsingError) as err:  # already waited for / unknown
        g.measure_wait(tickets[0])
    assert err.value.status == ising.ISING_ERR_ARG
    with pytest.raises(ValueError):
        g.measure_async(2, 1, np.zeros(1, dtype=np.int64), np.zeros(2, dtype=np.int64))


def test_batch_equilibrium_matches_onsager_at_the_papers_sizes():
    # lattice batches (one CTA / one thread-block cluster per chain): PAPER.md Fig. 5 check at
    # 512^2 (one CTA) and 1024^2 (4-CTA clusters) below Tc, 8 replicas per temperature
    from paper_1906_06297_b200.ising import IsingBatch

    temps = [2.0, 2.15]
    for L, sweeps in [(512, 20000), (1024, 12000)]:
        chains = [(T, r) for T in temps for r in range(8)]
        b = IsingBatch(L, L, [31 + 7 * q for q in range(len(chains))])
        b.set_beta([1.0 / T for T, _ in chains]).init_cold().sweep(2000)
        ups, Es = b.measure(sweeps // 20, 20)
        b.close()
        for i, T in enumerate(temps):
            rows = slice(8 * i, 8 * i + 8)
            m = np.abs(2 * ups[rows] - L * L) / (L * L)
            e = Es[rows] / (L * L)
            assert abs(m.mean() - exact.onsager_m(T)) <= 5e-4, (L, T, m.mean())
            assert abs(e.mean() - exact.onsager_energy(T)) <= 5e-4, (L, T, e.mean())
