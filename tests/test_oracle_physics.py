"""Statistical pins of the oracle chain: exact 4x4 enumeration, Onsager, critical point.

The exact enumerator is itself pinned by Kaufman's closed form and the textbook
4x4 density of states (tests/golden/torus4x4_exact.txt)."""
import math

import numpy as np
import pytest

import oracle
from oracle import exact
from tests import golden_io


def test_density_of_states_4x4():
    assert exact.density_of_states(4, 4) == golden_io.dos4x4()


@pytest.mark.parametrize("N,M", [(4, 4), (2, 4), (4, 2), (2, 6), (6, 2), (2, 8), (3, 4), (4, 5)])
@pytest.mark.parametrize("beta", [0.1, 0.3, exact.BETA_C, 0.7])
def test_enumeration_matches_kaufman(N, M, beta):
    Z = exact.enumerate_torus(N, M, beta)["Z"]
    assert Z == pytest.approx(exact.kaufman_Z(N, M, beta), rel=1e-11)


def test_partition_function_integer_at_beta_c():
    # E/4 is an integer on the 4x4 torus and e^(4 beta_c) = 3 + 2 sqrt 2, so
    # Z(beta_c) = sum g(E) (3+2sqrt2)^(-E/4) is an integer: 5509120.
    assert exact.enumerate_torus(4, 4, exact.BETA_C)["Z"] == pytest.approx(5509120.0, abs=1e-6)


def test_trapped_states_4x4():
    # 36 states with s*h = 0 everywhere (reading R21); each is E = 0, M = 0
    st = exact.torus_states(4, 4)
    mask = exact.trapped_mask(st)
    assert mask.sum() == 36
    E, Mg = exact.state_energy_magnetization(st[mask])
    assert np.all(E == 0) and np.all(Mg == 0)


def test_onsager_closed_form():
    # PAPER.md:416; Tc from sinh(2/Tc) = 1 (reading R13) agrees with the printed 2.269185
    assert math.sinh(2 / exact.TC) == pytest.approx(1.0, abs=1e-15)
    assert math.tanh(2 / exact.TC) ** 2 == pytest.approx(0.5, abs=1e-15)
    assert exact.TC == pytest.approx(2.269185, abs=5e-7)
    assert exact.onsager_m(1.5) == pytest.approx(0.98649960, abs=1e-7)
    assert exact.onsager_m(2.0) == pytest.approx(0.91131938, abs=1e-7)
    assert exact.onsager_m(2.269185) == pytest.approx(0.16978, abs=1e-4)  # steep just below Tc
    assert exact.onsager_m(exact.TC) == 0.0 and exact.onsager_m(3.0) == 0.0
    # low-temperature series: M = 1 - 2u^2 - 8u^3 - ... with u = e^(-4/T)
    T = 0.8
    u = math.exp(-4 / T)
    assert exact.onsager_m(T) == pytest.approx(1 - 2 * u**2 - 8 * u**3, abs=50 * u**4)


def test_onsager_energy_closed_form():
    # u(Tc) = -sqrt 2; the infinite-lattice energy equals -d ln Z / d beta / N of Kaufman's
    # finite-torus Z (pinned by enumeration above) at L = 64, where finite-size terms vanish
    assert exact.onsager_energy(exact.TC) == pytest.approx(-math.sqrt(2.0), abs=1e-12)
    for T in [1.5, 2.0, 3.0]:
        b, h, L = 1.0 / T, 1e-5, 64
        E = -(exact.kaufman_logZ(L, L, b + h) - exact.kaufman_logZ(L, L, b - h)) / (2 * h) / L**2
        assert exact.onsager_energy(T) == pytest.approx(E, abs=1e-7)
    assert exact.kaufman_logZ(4, 4, 0.3) == pytest.approx(math.log(exact.kaufman_Z(4, 4, 0.3)), rel=1e-12)


@pytest.mark.parametrize("beta", [0.2, 0.4406868, 0.8])
def test_metropolis_4x4_matches_exact_enumeration(beta):
    # Cold start (reading R21), 10^4 warm-up + 10^6 measured sweeps, 100 batch means,
    # against the ergodic-class averages of the exact enumeration.
    lat = oracle.Lattice(4, 4, seed=11).init_cold().set_beta(beta)
    lat.sweep(10_000)
    up, E = lat.chain(1_000_000)
    ref = exact.enumerate_torus(4, 4, beta, exclude_trapped=True)
    e_mean, e_se = exact.batch_means(E / 16.0)
    m_mean, m_se = exact.batch_means(np.abs(2 * up - 16) / 16.0)
    assert abs(e_mean - ref["E_site"]) < 3.5 * e_se
    assert abs(m_mean - ref["abs_m"]) < 3.5 * m_se


@pytest.mark.parametrize("beta", [0.2, 0.4406868])
def test_heatbath_4x4_matches_exact_enumeration(beta):
    # heat bath has no forced flips: the full enumeration applies
    lat = oracle.Lattice(4, 4, seed=12).init_random().set_beta(beta, oracle.RULE_HEATBATH)
    lat.sweep(10_000)
    up, E = lat.chain(1_000_000)
    ref = exact.enumerate_torus(4, 4, beta)
    e_mean, e_se = exact.batch_means(E / 16.0)
    m_mean, m_se = exact.batch_means(np.abs(2 * up - 16) / 16.0)
    assert abs(e_mean - ref["E_site"]) < 3.5 * e_se
    assert abs(m_mean - ref["abs_m"]) < 3.5 * m_se


def test_random_start_trap_bias_exists():
    # The period-2 trap is real in the oracle: a trapped 4x4 state never leaves it.
    full = np.array([[1, 1, 1, 1], [-1, -1, -1, -1]] * 2, dtype=np.int8)
    lat = oracle.Lattice(4, 4, seed=1).load_full(full).set_beta(0.4406868)
    up, E = lat.chain(1000)
    assert np.all(E == 0)


@pytest.mark.parametrize("T,warm,meas", [(1.5, 500, 4000), (2.0, 2000, 10000)])
def test_onsager_magnetization(T, warm, meas):
    # PAPER.md:415-417 / north_star: |<|m|> - M_Onsager(T)| <= 0.003 (L = 128, cold start)
    L = 128
    lat = oracle.Lattice(L, L, seed=5).init_cold().set_beta(1.0 / T)
    lat.sweep(warm)
    up, E = lat.chain(meas)
    m = np.abs(2 * up - L * L) / (L * L)
    mean, se = exact.batch_means(m, 50)
    assert abs(mean - exact.onsager_m(T)) <= 0.003
    assert se < 0.001
    e_mean, e_se = exact.batch_means(E / (L * L), 50)
    assert abs(e_mean - exact.onsager_energy(T)) <= 0.002


def _binder_curve(L, temps, warm, meas, seed):
    out = []
    for k, T in enumerate(temps):
        lat = oracle.Lattice(L, L, seed=seed + k).init_cold().set_beta(1.0 / T)
        lat.sweep(warm)
        up, _ = lat.chain(meas)
        m = (2 * up - L * L) / (L * L)
        out.append(exact.binder(np.mean(m**2), np.mean(m**4)))
    return np.array(out)


def test_binder_exact_4x4_at_beta_c():
    r = exact.enumerate_torus(4, 4, exact.BETA_C)
    assert exact.binder(r["m2"], r["m4"]) == pytest.approx(0.61719932, abs=1e-7)


@pytest.mark.slow
def test_binder_crossing_brackets_tc():
    # U_L(T) curves for different L cross at Tc.  Conventional U
    # (reading R15): below Tc larger L has larger U, above Tc smaller.
    temps = [2.15, 2.40]
    u8 = _binder_curve(8, temps, 2000, 200_000, 100)
    u16 = _binder_curve(16, temps, 2000, 100_000, 200)
    d = u16 - u8
    assert d[0] > 0 > d[1]
    # literal (paper-printed) U = 1 - <m4>/<m2>^2 is a monotone map of the conventional one
    assert exact.binder(0.5, 0.3, conventional=False) == pytest.approx(3 * exact.binder(0.5, 0.3) - 2)
