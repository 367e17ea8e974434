"""GPU physics pins: BASELINE configs[1] (2048^2, T = 1.5 and 3.0, 20000 sweeps) against
Onsager's magnetization, and the critical point."""
import numpy as np
import pytest

from oracle import exact
from paper_1906_06297_b200.ising import IsingLattice
from tests import cases

pytestmark = pytest.mark.gpu


def measure_abs_m(L, T, start, seed, sweeps, discard, every):
    g = IsingLattice(L, L, seed).set_beta(1.0 / T)
    g.init_cold() if start == "cold" else g.init_random()
    g.sweep(discard)
    ms = []
    for _ in range((sweeps - discard) // every):
        g.sweep(every)
        up, _ = g.observables()
        ms.append((2 * up - L * L) / (L * L))
    g.close()
    return np.asarray(ms)


@pytest.mark.parametrize("T,start,expect", [(1.5, "cold", exact.onsager_m(1.5)), (3.0, "random", 0.0)])
@pytest.mark.parametrize("seed", [1, 2])
def test_c2_onsager(T, start, expect, seed):
    # BASELINE configs[1]: 2048^2, 20000 sweeps, discard 2000, sample every 10 sweeps;
    # |<|m|> - M_Onsager| <= 0.003 (north_star).  T = 1.5 starts cold (reading R21 / the
    # band meta-stability the paper reports for L > 1024).
    L, sweeps = cases.C2[0], cases.C2[3]
    m = measure_abs_m(L, T, start, seed, sweeps, 2000, 10)
    mean, se = exact.batch_means(np.abs(m), 50)
    assert abs(mean - expect) <= 0.003, (mean, se)
    assert se < 0.001


def binder_point(L, T, seed, sweeps, every=1):
    g = IsingLattice(L, L, seed).set_beta(1.0 / T).init_cold()
    g.sweep(2000)
    m = []
    for _ in range(sweeps // every):
        g.sweep(every)
        up, _ = g.observables()
        m.append((2 * up - L * L) / (L * L))
    g.close()
    m = np.asarray(m)
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
