"""Pins for the oracle's plane layout, stencil and update rule (no statistics)."""
import math

import numpy as np
import pytest

import oracle
from tests import golden_io


def _sources_read(lat, is_black, i, j):
    """Which source-plane sites the stencil reads for target (i, j): perturb each one."""
    src = lat.white if is_black else lat.black
    src[:] = -1
    base = lat.nn_sum(is_black, i, j)
    hits = []
    for ii in range(lat.N):
        for jj in range(lat.ny):
            src[ii, jj] = 1
            if lat.nn_sum(is_black, i, j) != base:
                hits.append(ii * lat.ny + jj)
            src[ii, jj] = -1
    return hits


@pytest.mark.parametrize("colour,targets,expect", golden_io.fig3())
def test_fig3_worked_example(colour, targets, expect):
    # 12 x 12 lattice of the Fig. 3 caption: 6 spins per plane row
    lat = oracle.Lattice(12, 12)
    got = set()
    for s in targets:
        got |= set(_sources_read(lat, colour == "black", s // 6, s % 6))
    assert sorted(got) == expect


@pytest.mark.parametrize("N,M", [(2, 2), (4, 4), (6, 10), (12, 12), (8, 6), (10, 4)])
def test_stencil_matches_bruteforce_torus(N, M):
    # Sum of the 4 torus neighbours of every site, from the full lattice with np.roll,
    # must equal the plane stencil's nn_sum (reading R1: black iff i+J even).
    rng = np.random.default_rng(N * 100 + M)
    full = rng.choice(np.array([-1, 1], dtype=np.int8), size=(N, M))
    lat = oracle.Lattice(N, M).load_full(full)
    s = full.astype(np.int64)
    h = np.roll(s, 1, 0) + np.roll(s, -1, 0) + np.roll(s, 1, 1) + np.roll(s, -1, 1)
    for i in range(N):
        for J in range(M):
            assert lat.nn_sum((i + J) % 2 == 0, i, J // 2) == h[i, J], (i, J)


def test_full_plane_round_trip():
    rng = np.random.default_rng(5)
    for N, M in [(2, 2), (6, 6), (4, 12)]:
        full = rng.choice(np.array([-1, 1], dtype=np.int8), size=(N, M))
        lat = oracle.Lattice(N, M).load_full(full)
        assert np.array_equal(lat.full(), full)
        for i in range(N):
            for J in range(M):
                plane = lat.black if (i + J) % 2 == 0 else lat.white
                assert plane[i, J // 2] == full[i, J]


def _bruteforce_sweep(full, seed, t, beta):
    """One checkerboard sweep on the full lattice with np.roll neighbours and the
    paper's floating-point acceptance u < exp(-2 beta nn lij),
    u = r 2^-32 — an independent formulation of the oracle's integer compare."""
    s = full.astype(np.int64).copy()
    N, M = s.shape
    I, Jg = np.meshgrid(np.arange(N), np.arange(M), indexing="ij")
    for c in (0, 1):
        mask = ((I + Jg) % 2) == c
        h = np.roll(s, 1, 0) + np.roll(s, -1, 0) + np.roll(s, 1, 1) + np.roll(s, -1, 1)
        e = s * h
        for i, J in zip(*np.nonzero(mask)):
            if math.isinf(beta):
                flip = e[i, J] <= 0
            else:
                u = oracle.rand(seed, t, c, int(i), int(J) // 2) / 2.0**32
                flip = u < math.exp(-2.0 * beta * e[i, J])
            if flip:
                s[i, J] = -s[i, J]
    return s.astype(np.int8)


@pytest.mark.parametrize("N,M,beta", [(4, 4, 0.4406868), (6, 8, 0.2), (8, 6, math.inf),
                                      (2, 4, 0.8), (10, 10, 0.4406868)])
def test_sweep_matches_bruteforce(N, M, beta):
    lat = oracle.Lattice(N, M, seed=7).init_random().set_beta(beta)
    ref = lat.full()
    for t in range(1, 4):
        ref = _bruteforce_sweep(ref, 7, t, beta)
        lat.sweep(1)
        assert np.array_equal(lat.full(), ref), t


def test_beta_zero_flips_everything():
    lat = oracle.Lattice(16, 32, seed=3).init_random().set_beta(0.0)
    f0 = lat.full()
    up0, E0 = lat.observables()
    lat.sweep(1)
    assert np.array_equal(lat.full(), -f0)
    assert lat.observables() == (16 * 32 - up0, E0)


def test_trap_states_have_period_two():
    # rows alternating +1/-1: every site has s*h = 0, so dE = 0 moves are forced
    # and one sweep maps s -> -s at any beta (reading R21).
    for N, M in [(4, 4), (8, 12)]:
        full = np.where(np.arange(N)[:, None] % 2 == 0, 1, -1) * np.ones((1, M), dtype=np.int8)
        for beta in [0.2, 0.4406868, 1.0, math.inf]:
            lat = oracle.Lattice(N, M, seed=9).load_full(full.astype(np.int8)).set_beta(beta)
            lat.sweep(1)
            assert np.array_equal(lat.full(), -full)
            lat.sweep(1)
            assert np.array_equal(lat.full(), full)


def test_sweep_chunking_invariance():
    a = oracle.Lattice(16, 16, seed=2).init_random().set_beta(0.4406868)
    b = oracle.Lattice(16, 16, seed=2).init_random().set_beta(0.4406868)
    a.sweep(10)
    b.sweep(5).sweep(5)
    assert np.array_equal(a.full(), b.full()) and a.t == b.t == 10


def test_observables_closed_forms():
    N, M = 6, 8
    lat = oracle.Lattice(N, M).init_cold()
    assert lat.observables() == (N * M, -2 * N * M)            # all up
    neel = np.where((np.add.outer(np.arange(N), np.arange(M)) % 2) == 0, 1, -1).astype(np.int8)
    assert lat.load_full(neel).observables() == (N * M // 2, 2 * N * M)
    one = np.ones((N, M), dtype=np.int8)
    one[2, 3] = -1
    assert lat.load_full(one).observables() == (N * M - 1, -2 * N * M + 8)
    # random lattice: E against the brute-force bond sum
    rng = np.random.default_rng(1)
    full = rng.choice(np.array([-1, 1], dtype=np.int8), size=(N, M))
    s = full.astype(np.int64)
    E = -(s * np.roll(s, -1, 1)).sum() - (s * np.roll(s, -1, 0)).sum()
    assert lat.load_full(full).observables() == (int((s == 1).sum()), int(E))


def test_heatbath_beta_zero_is_fair_coin():
    # heat bath at beta = 0 flips with P = 1/2: flip iff r < 2^31
    N, M, seed = 8, 8, 4
    lat = oracle.Lattice(N, M, seed=seed).init_cold().set_beta(0.0, oracle.RULE_HEATBATH)
    lat.sweep(1)
    full = lat.full()
    for i in range(N):
        for J in range(M):
            c = (i + J) % 2
            flipped = oracle.rand(seed, 1, c, i, J // 2) < 2**31
            assert full[i, J] == (-1 if flipped else 1)


@pytest.mark.parametrize("N,M", [(8, 8), (12, 16), (64, 64), (6, 10)])
@pytest.mark.parametrize("rule", [oracle.RULE_METROPOLIS, oracle.RULE_HEATBATH])
def test_sampled_site_evaluation_matches_full_oracle(N, M, rule):
    # the site-by-site evaluation used for full-size sampled parity (C4 / C5) equals the
    # materialised oracle after one sweep
    beta = 0.4406868
    full = oracle.Lattice(N, M, 5).init_random().set_beta(beta, rule).sweep(1).full()
    for i in range(N):
        assert np.array_equal(oracle.sample_row_after_one_sweep(5, N, M, beta, i, rule), full[i])
