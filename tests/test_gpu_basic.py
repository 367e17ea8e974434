"""The basic byte-per-spin layout (§3.1) against the oracle and
against the multi-spin layout: bit-identical lattices and equal integer observables."""
import math

import numpy as np
import pytest

import oracle
from paper_1906_06297_b200 import ising
from paper_1906_06297_b200.ising import IsingLattice
from tests import cases

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,M", [(64, 64), (66, 64), (130, 192), (2, 8), (8, 24), (256, 512)])
@pytest.mark.parametrize("beta,rule", [(0.4406868, 0), (0.2, 0), (0.0, 0), (math.inf, 0),
                                       (0.4406868, 1), (math.inf, 1)])
def test_basic_matches_oracle(N, M, beta, rule):
    g = IsingLattice.basic(N, M, 3).set_beta(beta, rule).init_random()
    o = oracle.Lattice(N, M, 3).set_beta(beta, rule).init_random()
    for n in [1, 2, 9]:
        g.sweep(n)
        o.sweep(n)
        assert np.array_equal(g.read_lattice(), o.full()), (N, M, beta, rule, o.t)
        assert g.observables() == o.observables()


@pytest.mark.parametrize("N,M", [(64, 64), (130, 192), (34, 1024)])
@pytest.mark.parametrize("beta,rule", [(0.4406868, 0), (4e-11, 0), (math.inf, 0), (0.0, 0),
                                       (0.4406868, 1), (3.0, 1), (6.0, 1), (math.inf, 1),
                                       (0.3377438395041983, 1)])
@pytest.mark.parametrize("sym", ["1", "0"])
def test_basic_kernels_every_variant(N, M, beta, rule, sym, monkeypatch):
    # the byte-lane SWAR kernel (default) and the listing-shaped kernel both equal the
    # oracle for every acceptance variant (Metropolis fast / generic / draw-free, heat bath
    # symmetric (7) or with 0, 1, 2 "always" classes; 0.33774... has an asymmetric table)
    monkeypatch.setenv("ISING_HB_SYMMETRIC", sym)
    o = oracle.Lattice(N, M, 4).set_beta(beta, rule).init_random().sweep(3)
    for listing in ["0", "1"]:
        monkeypatch.setenv("ISING_BASIC_LISTING", listing)
        g = IsingLattice.basic(N, M, 4).set_beta(beta, rule)
        if rule == 1 and sym == "1" and beta in (0.4406868, 3.0, 6.0):
            assert g.kernel_variant() == 7
        g.init_random().sweep(3)
        assert np.array_equal(g.read_lattice(), o.full()), (listing, N, M, beta, rule)
        g.close()


def test_basic_equals_multispin():
    N, M = 128, 256
    a = IsingLattice.basic(N, M, 11).set_beta(0.4406868).init_random()
    b = IsingLattice(N, M, 11).set_beta(0.4406868).init_random()
    a.sweep(100)
    b.sweep(100)
    assert np.array_equal(a.read_lattice(), b.read_lattice())
    assert a.observables() == b.observables()


def test_basic_write_resume_and_measure():
    rng = np.random.default_rng(5)
    N, M = 64, 128
    full = cases.random_pm1(rng, N, M)
    g = IsingLattice.basic(N, M, 2).write_lattice(full, t=9).set_beta(0.3)
    assert np.array_equal(g.read_lattice(), full)
    ups, Es = g.measure(20, 2)
    o = oracle.Lattice(N, M, 2).load_full(full, t=9).set_beta(0.3)
    ou, oE = o.chain(40)
    assert np.array_equal(ups, ou[1::2]) and np.array_equal(Es, oE[1::2])
    with pytest.raises(ising.IsingError):
        IsingLattice.basic(64, 60, 1)


@pytest.mark.parametrize("N,M", [(64, 64), (130, 192), (34, 1024), (8, 24)])
@pytest.mark.parametrize("beta,rule", [(0.4406868, 0), (0.4406868, 1), (math.inf, 0)])
def test_basic_measured_chain(N, M, beta, rule, monkeypatch):
    # measured chains on the byte layout: observables fused into the SWAR kernel's white phase
    # (plane widths that are multiples of 16 bytes), else the separate observables pass (8 x 24,
    # and the listing-shaped kernel); synchronous and asynchronous forms
    for listing in ["0", "1"]:
        monkeypatch.setenv("ISING_BASIC_LISTING", listing)
        g = IsingLattice.basic(N, M, 5).set_beta(beta, rule).init_random()
        o = oracle.Lattice(N, M, 5).set_beta(beta, rule).init_random()
        ups, Es = g.measure(4, 2)
        ou, oE = o.chain(8)
        assert np.array_equal(ups, ou[1::2]) and np.array_equal(Es, oE[1::2]), (listing, N, M)
        u = np.zeros(3, dtype=np.int64)
        e = np.zeros(3, dtype=np.int64)
        g.measure_wait(g.measure_async(3, 1, u, e))
        ou, oE = o.chain(3)
        assert np.array_equal(u, ou) and np.array_equal(e, oE), (listing, N, M)
        assert np.array_equal(g.read_lattice(), o.full())
        g.close()
