"""Pins for the oracle's Philox4x32-10, draw contract, random start and thresholds."""
import hashlib
import math
from decimal import Decimal, getcontext

import numpy as np
import pytest

import oracle
from oracle import exact
from tests import golden_io


@pytest.mark.parametrize("ctr,key,expect", golden_io.philox_kat())
def test_philox_known_answers(ctr, key, expect):
    # Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt).
    assert list(oracle.philox4x32_10(ctr, key)) == expect


def test_draw_contract_golden():
    draws, _, _ = golden_io.rng_contract()
    for (seed, t, c, i, j0), words in draws:
        assert [oracle.rand(seed, t, c, i, j0 + k) for k in range(4)] == words


def test_draw_uses_one_block_per_four_sites():
    # r(seed,t,c,i,j) is word j&3 of the block with counter {t, j>>2, c, i} (reading R6)
    seed = 0x1234_5678_9ABC_DEF0
    blk = oracle.philox4x32_10([13, 7, 1, 11], [seed & 0xFFFFFFFF, seed >> 32])
    assert [oracle.rand(seed, 13, 1, 11, 28 + k) for k in range(4)] == list(blk)


def test_random_start_golden():
    _, inits, init4 = golden_io.rng_contract()
    for (N, M, seed), up, E, sha in inits:
        if N * M > 64 * 64:
            continue  # the 2048^2 golden is checked in the slow test below
        lat = oracle.Lattice(N, M, seed).init_random()
        assert lat.observables() == (up, E)
        assert hashlib.sha256(lat.full().tobytes()).hexdigest().startswith(sha)
    for seed, rows in init4:
        lat = oracle.Lattice(4, 4, seed).init_random()
        assert lat.full().tolist() == rows


@pytest.mark.slow
def test_random_start_golden_2048():
    _, inits, _ = golden_io.rng_contract()
    for (N, M, seed), up, E, sha in inits:
        if N * M <= 64 * 64:
            continue
        lat = oracle.Lattice(N, M, seed).init_random()
        assert lat.observables() == (up, E)
        assert hashlib.sha256(lat.full().tobytes()).hexdigest().startswith(sha)


def test_draws_are_uniform():
    # chi-square on 16 bins over 64k draws of one colour plane (sanity of the contract)
    r = np.array([oracle.rand(3, 5, 1, i, j) for i in range(64) for j in range(1024)], dtype=np.uint64)
    counts = np.bincount((r >> np.uint64(28)).astype(np.int64), minlength=16)
    expect = len(r) / 16
    chi2 = ((counts - expect) ** 2 / expect).sum()
    assert chi2 < 37.7  # p = 0.001 for 15 dof
    assert abs(r.mean() / 2**32 - 0.5) < 4 * (1 / math.sqrt(12 * len(r)))


def _ceil_scaled_decimal(x: Decimal) -> int:
    v = x * (Decimal(2) ** 32)
    return int(v.to_integral_value(rounding="ROUND_CEILING"))


def test_thresholds_closed_form_at_beta_c():
    # At beta_c, exp(2 beta_c) = 1 + sqrt 2, so exp(-4 beta_c) = 3 - 2 sqrt 2 and
    # exp(-8 beta_c) = 17 - 12 sqrt 2 (reading R13); T = ceil(2^32 p) (reading R5).
    getcontext().prec = 60
    s2 = Decimal(2).sqrt()
    T = oracle.thresholds(exact.BETA_C)
    assert int(T[3]) == _ceil_scaled_decimal(3 - 2 * s2) == 736899889
    assert int(T[4]) == _ceil_scaled_decimal(17 - 12 * s2) == 126432033
    assert list(T[:3]) == [2**32] * 3  # e <= 0: always accepted


def test_thresholds_high_precision_exp():
    # T against exp evaluated in 60-digit decimal arithmetic (not libm): equal unless
    # 2^32 p sits within double rounding of an integer, which none of these do.
    getcontext().prec = 60
    for beta in [0.2, 1 / 3, 0.4406868, 2 / 3, 0.8, 1.7]:
        T = oracle.thresholds(beta)
        for k, e in [(3, 2), (4, 4)]:
            p = (Decimal(-2 * e) * Decimal(beta)).exp()
            assert int(T[k]) == _ceil_scaled_decimal(p), (beta, e)


def test_thresholds_special_cases():
    assert list(oracle.thresholds(0.0)) == [2**32] * 5       # beta = 0: every flip accepted
    assert list(oracle.thresholds(math.inf)) == [2**32] * 3 + [0, 0]
    hb0 = oracle.thresholds(0.0, oracle.RULE_HEATBATH)       # P = 1/2 exactly
    assert list(hb0) == [2**31] * 5
    hbinf = oracle.thresholds(math.inf, oracle.RULE_HEATBATH)
    assert list(hbinf) == [2**32, 2**32, 2**31, 0, 0]
    for beta in [0.1, 0.4406868, 0.9]:
        hb = [int(x) for x in oracle.thresholds(beta, oracle.RULE_HEATBATH)]
        # P(e) + P(-e) = 1: ceilings sum to 2^32 or 2^32 + 1
        assert hb[0] + hb[4] in (2**32, 2**32 + 1)
        assert hb[1] + hb[3] in (2**32, 2**32 + 1)
        assert hb[2] == 2**31
        assert hb[0] > hb[1] > hb[2] > hb[3] > hb[4]
        m = [int(x) for x in oracle.thresholds(beta)]
        assert m[3] > m[4] > 0


def test_heatbath_table_symmetry_and_its_rounding_exceptions():
    # Heat bath: P(e) + P(-e) = 1, so with exact arithmetic
    # ceil(2^32 P(e)) + ceil(2^32 P(-e)) = 2^32 + 1 (2^32 P is never an integer for beta > 0).
    # The GPU's symmetric heat-bath kernel (variant 7) relies on that identity and the host
    # checks it on the rounded table (reading R22: IEEE double via host libm, as here).  Two
    # betas found by search break it in double precision only: the 60-digit table is
    # symmetric, the double one is not, so those betas must take the five-compare kernel
    # (tests/test_gpu_parity.py::HB_ASYM).
    getcontext().prec = 60

    def exact_table(beta):
        out = []
        for a in range(5):
            p = (Decimal(-2 * (2 * a - 4)) * Decimal(beta)).exp()
            out.append(_ceil_scaled_decimal(p / (1 + p)))
        return out

    def symmetric(T):
        return T[2] == 2**31 and T[0] + T[4] == T[1] + T[3] == 2**32 + 1

    for beta in [0.1, 0.2, 0.4406868, 0.8, 2.5, 3.0, 6.0]:
        T = [int(x) for x in oracle.thresholds(beta, oracle.RULE_HEATBATH)]
        assert symmetric(T) and T == exact_table(beta), beta
    for beta in [0.3377438395041983, 1.2800778283900398]:
        T = [int(x) for x in oracle.thresholds(beta, oracle.RULE_HEATBATH)]
        assert not symmetric(T) and symmetric(exact_table(beta)), beta
        assert T[0] + T[4] + T[1] + T[3] == 2**33 + 1  # exactly one pair rounded onto 2^32
