"""Lattice batches (ising_batch_*): every lattice of a batch against the
CPU oracle with the same seed and beta, bit for bit, and against a one-lattice handle."""
import math

import numpy as np
import pytest

import oracle
from paper_1906_06297_b200 import ising
from paper_1906_06297_b200.ising import IsingBatch, IsingLattice
from tests import cases

BETAS = [0.0, math.inf, 4e-11, cases.BETA_TC, 3.0, 0.2, 0.6]


def oracle_for(N, M, seed, beta, rule, start):
    o = oracle.Lattice(N, M, seed).set_beta(beta, oracle.RULE_HEATBATH if rule else oracle.RULE_METROPOLIS)
    return o.init_random() if start == "random" else o.init_cold()


@pytest.mark.gpu
@pytest.mark.parametrize("N,M,n", [(64, 64, 7), (130, 192, 3), (2, 64, 2), (256, 256, 4),
                                   (512, 512, 2), (640, 640, 1), (8, 8192, 2)])
@pytest.mark.parametrize("rule", [ising.RULE_METROPOLIS, ising.RULE_HEATBATH])
@pytest.mark.parametrize("start", ["random", "cold"])
def test_batch_matches_oracle(N, M, n, rule, start):
    rng = np.random.default_rng(N * 7919 + M + n + rule)
    seeds = [int(x) for x in rng.integers(0, 2**63, size=n)]
    betas = [BETAS[(k + N) % len(BETAS)] for k in range(n)]
    b = IsingBatch(N, M, seeds).set_beta(betas, rule)
    b.init_random() if start == "random" else b.init_cold()
    os_ = [oracle_for(N, M, seeds[k], betas[k], rule, start) for k in range(n)]
    try:
        for chunk in [1, 3, 9]:
            b.sweep(chunk)
            up, E = b.observables()
            for k in range(n):
                os_[k].sweep(chunk)
                got = b.read_lattice(k)
                assert np.array_equal(got, os_[k].full()), \
                    f"lattice {k} (beta {betas[k]}) t={os_[k].t}: {int((got != os_[k].full()).sum())} differ"
                assert (int(up[k]), int(E[k])) == os_[k].observables(), f"lattice {k} observables"
        assert b.t == 13
    finally:
        b.close()


@pytest.mark.gpu
@pytest.mark.parametrize("N,M,n,every,ns", [(64, 64, 5, 1, 30), (96, 128, 3, 7, 9), (64, 64, 2, 3000, 2),
                                            (64, 64, 2, 5000, 2)])
def test_batch_measured_chain_matches_oracle(N, M, n, every, ns):
    # every = 3000 / 5000: samples straddle the launches of at most 4096 sweeps
    seeds = [11 + 2 * k for k in range(n)]
    betas = [0.35 + 0.05 * k for k in range(n)]
    b = IsingBatch(N, M, seeds).set_beta(betas).init_random()
    try:
        b.sweep(5)
        up, E = b.measure(ns, every)
        assert up.shape == (n, ns)
        for k in range(n):
            o = oracle_for(N, M, seeds[k], betas[k], 0, "random").sweep(5)
            ou, oE = o.chain(ns * every)
            assert up[k].tolist() == [int(x) for x in ou[every - 1::every]], f"lattice {k} up"
            assert E[k].tolist() == [int(x) for x in oE[every - 1::every]], f"lattice {k} E"
            assert np.array_equal(b.read_lattice(k), o.full())
        assert b.t == 5 + ns * every
    finally:
        b.close()


@pytest.mark.gpu
def test_batch_long_chain_across_launches_equals_one_lattice_handles():
    # 9000 sweeps in one call (three launches) of 512^2 lattices vs the one-lattice path
    N = M = 512
    seeds, betas = [3, 4, 5], [0.40, cases.BETA_TC, 0.47]
    b = IsingBatch(N, M, seeds).set_beta(betas).init_random().sweep(9000)
    try:
        for k in range(3):
            g = IsingLattice(N, M, seeds[k]).set_beta(betas[k]).init_random().sweep(9000)
            assert np.array_equal(b.read_lattice(k), g.read_lattice()), f"lattice {k}"
            up, E = b.observables()
            assert (int(up[k]), int(E[k])) == g.observables()
            g.close()
    finally:
        b.close()


@pytest.mark.gpu
def test_batch_many_lattices_spot_checks():
    n, N, M = 2000, 64, 64
    seeds = list(range(1000, 1000 + n))
    betas = np.linspace(0.2, 0.7, n)
    b = IsingBatch(N, M, seeds).set_beta(betas).init_random().sweep(50)
    try:
        up, E = b.observables()
        for k in [0, 1, 777, 1234, n - 1]:
            o = oracle_for(N, M, seeds[k], float(betas[k]), 0, "random").sweep(50)
            assert np.array_equal(b.read_lattice(k), o.full()), f"lattice {k}"
            assert (int(up[k]), int(E[k])) == o.observables()
    finally:
        b.close()


@pytest.mark.gpu
@pytest.mark.parametrize("N,M,n", [(1024, 512, 3), (1024, 1024, 2), (640, 1024, 2), (32, 16384, 2),
                                   (2048, 2048, 1)])
@pytest.mark.parametrize("rule", [ising.RULE_METROPOLIS, ising.RULE_HEATBATH])
def test_cluster_batch_matches_oracle(N, M, n, rule):
    # lattices beyond one CTA: a cluster of 2..16 CTAs per lattice, halos over DSMEM
    seeds = [101 + 17 * k for k in range(n)]
    betas = [[cases.BETA_TC, 0.0, 0.3][k % 3] for k in range(n)]
    b = IsingBatch(N, M, seeds).set_beta(betas, rule).init_random()
    try:
        done = 0
        for chunk in [1, 4]:
            b.sweep(chunk)
            done += chunk
            up, E = b.observables()
            for k in range(n):
                o = oracle_for(N, M, seeds[k], betas[k], rule, "random").sweep(done)
                assert np.array_equal(b.read_lattice(k), o.full()), f"lattice {k} t={done}"
                assert (int(up[k]), int(E[k])) == o.observables()
        u2, e2 = b.measure(3, 2)
        for k in range(n):
            o = oracle_for(N, M, seeds[k], betas[k], rule, "random").sweep(done)
            ou, oE = o.chain(6)
            assert u2[k].tolist() == [int(x) for x in ou[1::2]]
            assert e2[k].tolist() == [int(x) for x in oE[1::2]]
    finally:
        b.close()


@pytest.mark.gpu
def test_cluster_batch_long_chain_equals_one_lattice_handle():
    N = M = 2048
    b = IsingBatch(N, M, [9, 10]).set_beta([cases.BETA_TC, 0.5]).init_random().sweep(5000)
    try:
        for k, (seed, beta) in enumerate([(9, cases.BETA_TC), (10, 0.5)]):
            g = IsingLattice(N, M, seed).set_beta(beta).init_random().sweep(5000)
            assert np.array_equal(b.read_lattice(k), g.read_lattice()), f"lattice {k}"
            g.close()
    finally:
        b.close()


HB_BETAS = [cases.BETA_TC, 0.2, 3.0, 6.0, math.inf, 0.0, 0.3377438395041983]


@pytest.mark.gpu
@pytest.mark.parametrize("beta", HB_BETAS)
@pytest.mark.parametrize("sym", ["1", "0"])
@pytest.mark.parametrize("N,M", [(64, 128), (1024, 512)])
def test_batch_heatbath_variants_match_oracle(monkeypatch, beta, sym, N, M):
    # all lattices at one beta: the batch runs that beta's lockstep heat-bath variant (7
    # symmetric, else 3 / 5 / 6 by the number of "always" classes), one CTA or a cluster
    monkeypatch.setenv("ISING_HB_SYMMETRIC", sym)
    seeds = [3, 4]
    b = IsingBatch(N, M, seeds).set_beta([beta, beta], ising.RULE_HEATBATH).init_random().sweep(5)
    try:
        up, E = b.observables()
        for k in range(2):
            o = oracle_for(N, M, seeds[k], beta, 1, "random").sweep(5)
            assert np.array_equal(b.read_lattice(k), o.full()), f"beta {beta} lattice {k}"
            assert (int(up[k]), int(E[k])) == o.observables()
    finally:
        b.close()


@pytest.mark.gpu
def test_batch_errors():
    with pytest.raises(ising.IsingError) as e:
        IsingBatch(63, 64, [1])                 # odd rows
    assert e.value.status == ising.ISING_ERR_ARG
    with pytest.raises(ising.IsingError) as e:
        IsingBatch(64, 96, [1])                 # L_cols % 64
    assert e.value.status == ising.ISING_ERR_ARG
    with pytest.raises(ising.IsingError) as e:
        IsingBatch(4096, 4096, [1])             # beyond a 16-CTA cluster's shared memory
    assert e.value.status == ising.ISING_ERR_ARG
    b = IsingBatch(64, 64, [1, 2])
    try:
        with pytest.raises(ising.IsingError) as e:
            b.sweep(1)                          # no beta / state yet
        assert e.value.status == ising.ISING_ERR_STATE
        with pytest.raises(ising.IsingError) as e:
            b.set_beta([0.3, float("nan")])
        assert e.value.status == ising.ISING_ERR_ARG
        b.set_beta([0.3, 0.4]).init_cold()
        with pytest.raises(ising.IsingError) as e:
            b.read_lattice(2)
        assert e.value.status == ising.ISING_ERR_ARG
        with pytest.raises(ising.IsingError) as e:
            b.sweep(2**32)
        assert e.value.status == ising.ISING_ERR_RANGE
        assert np.all(b.read_lattice(1) == 1)   # cold start
        up, E = b.observables()
        assert up.tolist() == [64 * 64] * 2 and E.tolist() == [-2 * 64 * 64] * 2
    finally:
        b.close()


@pytest.mark.gpu
def test_batch_write_lattice_resume_matches_oracle():
    # checkpoint / exact resume: lattices loaded from +-1 bytes at t = 123, then swept
    N, M, n = 96, 192, 3
    rng = np.random.default_rng(42)
    seeds = [5, 6, 7]
    betas = [0.3, cases.BETA_TC, 0.6]
    starts = [cases.random_pm1(rng, N, M, p) for p in (0.2, 0.5, 0.9)]
    b = IsingBatch(N, M, seeds).set_beta(betas)
    try:
        for k in range(n):
            b.write_lattice(k, starts[k], t=123)
        assert b.t == 123
        for k in range(n):
            assert np.array_equal(b.read_lattice(k), starts[k])
        up, E = b.measure(4, 5)
        for k in range(n):
            o = oracle.Lattice(N, M, seeds[k]).set_beta(betas[k]).load_full(starts[k], t=123)
            ou, oE = o.chain(20)
            assert up[k].tolist() == [int(x) for x in ou[4::5]]
            assert E[k].tolist() == [int(x) for x in oE[4::5]]
            assert np.array_equal(b.read_lattice(k), o.full())
        bad = starts[0].copy()
        bad[3, 5] = 0
        with pytest.raises(ising.IsingError) as e:
            b.write_lattice(0, bad)
        assert e.value.status == ising.ISING_ERR_ARG
    finally:
        b.close()
