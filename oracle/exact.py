"""Closed forms and exact enumeration for the 2D Ising model — TEST INFRASTRUCTURE ONLY.

Everything here is the plain definition of a quantity the paper states or relies on:

* ``onsager_m(T)`` — spontaneous magnetization (1 - sinh(2J/T)^-4)^(1/8) for T < Tc
  (§5.3, Eq. "magn").
* ``TC`` — Tc = 2/ln(1 + sqrt 2) = 2.269185... (PAPER.md:418 prints 2.269185J; its
  stated condition "(tanh(2J/Tc))^2 = 1" is garbled — DESIGN.md reading R13 uses
  the Kramers-Wannier condition sinh(2J/Tc) = 1).
* ``binder(m2, m4)`` — U_L = 1 - <m^4>/<m^2>^2 as printed, and the
  conventional 1 - <m^4>/(3<m^2>^2) (reading R15).
* ``enumerate_torus(N, M, beta)`` — Boltzmann averages of Eq. 1 over
  all 2^(NM) states, by brute force.
* ``kaufman_Z(N, M, beta)`` — Kaufman's (1949) exact finite-torus partition function,
  an independent closed form that pins ``enumerate_torus``.
"""
from __future__ import annotations

import math

import numpy as np

TC = 2.0 / math.log(1.0 + math.sqrt(2.0))
BETA_C = 1.0 / TC


def onsager_m(T: float, J: float = 1.0) -> float:
    """Onsager/Yang spontaneous magnetization, PAPER.md:416 (0 for T >= Tc)."""
    if T <= 0:
        raise ValueError("T must be positive")
    if T >= TC * J:
        return 0.0
    return (1.0 - math.sinh(2.0 * J / T) ** -4) ** 0.125


def onsager_energy(T: float, J: float = 1.0) -> float:
    """Onsager's internal energy per site of the infinite square lattice (each bond once):
    u = -J coth(2K) [1 + (2/pi) (2 tanh^2(2K) - 1) K(k)],  K = J/T, k = 2 sinh(2K)/cosh^2(2K),
    K(k) the complete elliptic integral of the first kind (scipy ellipk takes m = k^2).
    The paper compares magnetizations with Onsager's solution; the energy
    is the same exact solution's other observable."""
    from scipy.special import ellipk

    K = J / T
    kp = 2.0 * math.tanh(2 * K) ** 2 - 1.0
    if abs(kp) < 1e-12:  # T = Tc: the elliptic term vanishes (K(1) diverges only logarithmically)
        return -J / math.tanh(2 * K)
    k = 2.0 * math.sinh(2 * K) / math.cosh(2 * K) ** 2
    return -J / math.tanh(2 * K) * (1.0 + 2.0 / math.pi * kp * ellipk(k * k))


def binder(m2: float, m4: float, conventional: bool = True) -> float:
    """Binder cumulant.  PAPER.md:418 prints 1 - <m^4>/<m^2>^2; conventional adds 1/3."""
    return 1.0 - m4 / ((3.0 if conventional else 1.0) * m2 * m2)


def torus_states(N: int, M: int):
    """All 2^(NM) spin states of an N x M torus as int8 (+-1), shape (2^(NM), N, M)."""
    n = N * M
    if n > 20:
        raise ValueError("enumeration is capped at 20 spins")
    idx = np.arange(1 << n, dtype=np.int64)
    bits = (idx[:, None] >> np.arange(n, dtype=np.int64)[None, :]) & 1
    return (2 * bits - 1).astype(np.int8).reshape(-1, N, M)


def state_energy_magnetization(states: np.ndarray):
    """E = -sum_bonds s s' (each torus bond once, reading R11) and M = sum s."""
    s = states.astype(np.int64)
    E = -(s * np.roll(s, -1, axis=2)).sum(axis=(1, 2)) - (s * np.roll(s, -1, axis=1)).sum(axis=(1, 2))
    Mg = s.sum(axis=(1, 2))
    return E, Mg


def trapped_mask(states: np.ndarray) -> np.ndarray:
    """States where every site has s*h = 0 (h = sum of its 4 neighbours).

    Metropolis accepts dE = 0 with certainty, so such a state is
    flipped entirely by one checkerboard sweep: a period-2 orbit (reading R21).
    """
    s = states.astype(np.int64)
    h = (np.roll(s, 1, 1) + np.roll(s, -1, 1) + np.roll(s, 1, 2) + np.roll(s, -1, 2))
    return np.all(s * h == 0, axis=(1, 2))


def enumerate_torus(N: int, M: int, beta: float, exclude_trapped: bool = False) -> dict:
    """Exact Boltzmann averages on an N x M torus by summing over all states."""
    st = torus_states(N, M)
    E, Mg = state_energy_magnetization(st)
    if exclude_trapped:
        keep = ~trapped_mask(st)
        E, Mg = E[keep], Mg[keep]
    n = N * M
    logw = -beta * E.astype(np.float64)
    shift = logw.max()
    w = np.exp(logw - shift)
    Zs = w.sum()
    m = Mg.astype(np.float64) / n
    avg = lambda x: float((w * x).sum() / Zs)
    return {
        "Z": float(Zs * math.exp(shift)),
        "E_site": avg(E / n),
        "abs_m": avg(np.abs(m)),
        "m2": avg(m * m),
        "m4": avg(m ** 4),
    }


def density_of_states(N: int, M: int) -> dict:
    E, _ = state_energy_magnetization(torus_states(N, M))
    vals, counts = np.unique(E, return_counts=True)
    return {int(v): int(c) for v, c in zip(vals, counts)}


def kaufman_Z(N: int, M: int, beta: float, J: float = 1.0) -> float:
    """Kaufman's exact partition function of the N x M torus (B. Kaufman, Phys. Rev. 76,
    1232 (1949)), N rows, M columns, coupling K = beta J:

      Z = 1/2 (2 sinh 2K)^(NM/2) [prod_r 2cosh(N g_(2r+1)/2) + prod_r 2sinh(N g_(2r+1)/2)
                                 + prod_r 2cosh(N g_(2r)/2)   + prod_r 2sinh(N g_(2r)/2)],
      r = 0..M-1, cosh g_k = cosh 2K coth 2K - cos(pi k / M), g_0 = 2K + ln tanh K.
    """
    K = beta * J
    if K == 0:
        return float(2 ** (N * M))

    def gamma(k: int) -> float:
        if k == 0:
            return 2 * K + math.log(math.tanh(K))
        c = math.cosh(2 * K) / math.tanh(2 * K) - math.cos(math.pi * k / M)
        return math.acosh(c)

    odd = [gamma(2 * r + 1) for r in range(M)]
    even = [gamma(2 * r) for r in range(M)]
    z1 = math.prod(2 * math.cosh(N * g / 2) for g in odd)
    z2 = math.prod(2 * math.sinh(N * g / 2) for g in odd)
    z3 = math.prod(2 * math.cosh(N * g / 2) for g in even)
    z4 = math.prod(2 * math.sinh(N * g / 2) for g in even)
    return 0.5 * (2 * math.sinh(2 * K)) ** (N * M / 2) * (z1 + z2 + z3 + z4)


def kaufman_logZ(N: int, M: int, beta: float, J: float = 1.0) -> float:
    """log of kaufman_Z in log-space arithmetic (large tori), same formula."""
    K = beta * J

    def gamma(k: int) -> float:
        if k == 0:
            return 2 * K + math.log(math.tanh(K))
        return math.acosh(math.cosh(2 * K) / math.tanh(2 * K) - math.cos(math.pi * k / M))

    def log2cosh(x):
        x = abs(x)
        return x + math.log1p(math.exp(-2 * x))

    def log2sinh_signed(x):
        a = abs(x)
        return a + math.log1p(-math.exp(-2 * a)), (1.0 if x > 0 else -1.0)

    terms = []
    for ks in ([2 * r + 1 for r in range(M)], [2 * r for r in range(M)]):
        g = [gamma(k) for k in ks]
        terms.append((sum(log2cosh(N * x / 2) for x in g), 1.0))
        logs, sign = 0.0, 1.0
        for x in g:
            l, sg = log2sinh_signed(N * x / 2)
            logs += l
            sign *= sg
        terms.append((logs, sign))
    mx = max(t for t, _ in terms)
    acc = sum(sg * math.exp(t - mx) for t, sg in terms)
    return math.log(0.5) + (N * M / 2) * math.log(2 * math.sinh(2 * K)) + mx + math.log(acc)


def batch_means(x: np.ndarray, nbatch: int = 100) -> tuple[float, float]:
    """Mean and batch-means standard error of a correlated series."""
    x = np.asarray(x, dtype=np.float64)
    L = len(x) // nbatch
    b = x[: L * nbatch].reshape(nbatch, L).mean(axis=1)
    return float(x.mean()), float(b.std(ddof=1) / math.sqrt(nbatch))
