"""Seeded randomized parity: many small configurations drawn from one master seed, each run
through the C ABI and compared with the CPU oracle bit for bit.

The fixed-case tests (test_gpu_parity.py) pin the named edge cases; this sweep covers the
combinations between them — shape (both half-sweep kernels: register-rolling widths and the
TMA-staged widths that are multiples of 8192 columns), virtual slab count (R = 2 up), layout
(multi-spin / basic), acceptance rule, start (random / cold / loaded lattice with a sweep
offset), beta (log-uniform plus the special values) and how the sweeps are chunked into calls.
The case list is deterministic (numpy's seeded generator; no method arithmetic here), so a
failure names a reproducible case."""
import math

import numpy as np
import pytest

import oracle
from paper_1906_06297_b200 import ising
from paper_1906_06297_b200.ising import IsingLattice, run_ranks
from tests import cases

MASTER_SEED = 20261017
N_CASES = 160
SPECIAL_BETAS = [0.0, math.inf, 4e-11, cases.BETA_TC, 3.0]


def draw_case(rng: np.random.Generator, k: int) -> dict:
    layout = "basic" if rng.random() < 0.2 else "multispin"
    if layout == "basic":
        N = 2 * int(rng.integers(1, 65))
        M = 8 * int(rng.integers(1, 65))
        nslab = 1
    else:
        staged = rng.random() < 0.3
        if staged:  # W a multiple of 256 words: the TMA-staged kernel
            M = 8192 * int(rng.integers(1, 3))
            N = 2 * int(rng.integers(1, 41))
        else:
            M = 64 * int(rng.integers(1, 17))
            N = 2 * int(rng.integers(1, 97))
        divisors = [d for d in range(1, 9) if N % d == 0 and N // d >= 2]
        nslab = int(rng.choice(divisors)) if rng.random() < 0.5 else 1
    rule = ising.RULE_HEATBATH if rng.random() < 0.3 else ising.RULE_METROPOLIS
    if rng.random() < 0.3:
        beta = float(rng.choice(SPECIAL_BETAS))
    else:
        beta = float(10 ** rng.uniform(-3, math.log10(5.0)))
    start = str(rng.choice(["random", "cold", "loaded"]))
    t0 = int(rng.integers(0, 1000)) if start == "loaded" else 0
    # each chunk: ("sweep", n) or ("measure", samples, every) (ising_sweep_measure)
    chunks = []
    for _ in range(int(rng.integers(1, 4))):
        if rng.random() < 0.3:
            chunks.append(("measure", int(rng.integers(1, 4)), int(rng.integers(1, 3))))
        else:
            chunks.append(("sweep", int(rng.integers(0, 6))))
    return dict(k=k, layout=layout, N=N, M=M, nslab=nslab, rule=rule, beta=beta, start=start,
                t0=t0, p_up=float(rng.uniform(0.1, 0.9)), chunks=chunks,
                seed=int(rng.integers(0, 2**63)))


def all_cases():
    rng = np.random.default_rng(MASTER_SEED)
    return [draw_case(rng, k) for k in range(N_CASES)]


CASES = all_cases()


def case_id(c):
    return (f"{c['k']}-{c['layout']}-{c['N']}x{c['M']}-s{c['nslab']}-r{c['rule']}-"
            f"b{c['beta']:.3g}-{c['start']}")


@pytest.mark.gpu
@pytest.mark.parametrize("c", CASES, ids=[case_id(c) for c in CASES])
def test_fuzz_case_matches_oracle(c):
    N, M, seed = c["N"], c["M"], c["seed"]
    orule = oracle.RULE_HEATBATH if c["rule"] == ising.RULE_HEATBATH else oracle.RULE_METROPOLIS
    if c["layout"] == "basic":
        g = IsingLattice.basic(N, M, seed)
    else:
        g = IsingLattice(N, M, seed, devices=[0] * c["nslab"])
    o = oracle.Lattice(N, M, seed)
    try:
        g.set_beta(c["beta"], c["rule"])
        o.set_beta(c["beta"], orule)
        if c["start"] == "random":
            g.init_random()
            o.init_random()
        elif c["start"] == "cold":
            g.init_cold()
            o.init_cold()
        else:
            full = cases.random_pm1(np.random.default_rng(seed % 2**32), N, M, c["p_up"])
            g.write_lattice(full, t=c["t0"])
            o.load_full(full, t=c["t0"])
        assert g.t == o.t
        for ch in c["chunks"]:
            if ch[0] == "sweep":
                g.sweep(ch[1])
                o.sweep(ch[1])
            else:  # device-side measured chain against the oracle's per-sweep series
                _, k, every = ch
                ups, Es = g.measure(k, every)
                ou, oE = o.chain(k * every)
                assert list(ups) == list(ou[every - 1::every]), f"{case_id(c)} measured up"
                assert list(Es) == list(oE[every - 1::every]), f"{case_id(c)} measured E"
            got, exp = g.read_lattice(), o.full()
            if not np.array_equal(got, exp):
                bad = np.argwhere(got != exp)
                raise AssertionError(f"{case_id(c)} t={o.t}: {len(bad)} sites differ, "
                                     f"first {bad[:4].tolist()}")
            assert g.observables() == o.observables(), f"{case_id(c)} t={o.t}"
            assert g.t == o.t
        if c["layout"] == "multispin":  # the bit-packed read-back of the same state
            bits = g.read_lattice_bits()
            assert np.array_equal(bits, np.packbits(o.full() == 1, bitorder="little"))
    finally:
        g.close()


def draw_group_case(rng: np.random.Generator, k: int) -> dict:
    """A rank-p2p local group (ising_p2p_connect_local: every rank in this process, one host
    thread each, kernels concurrent on cuda:0)."""
    world = int(rng.integers(2, 6))
    if rng.random() < 0.75:  # TMA-staged widths: edge bands wait, interior bands do not
        M = 8192 * int(rng.integers(1, 3))
        R = int(rng.integers(2, 5)) if rng.random() < 0.3 else int(rng.integers(2, 41))
    else:  # register-rolling widths (every block waits): small groups only
        world = min(world, 3)
        M = 64 * int(rng.integers(1, 5))
        R = int(rng.integers(2, 25))
    if (world * R) % 2:  # L_rows even (the colouring wraps consistently)
        R += 1
    rule = ising.RULE_HEATBATH if rng.random() < 0.3 else ising.RULE_METROPOLIS
    beta = (float(rng.choice(SPECIAL_BETAS)) if rng.random() < 0.3
            else float(10 ** rng.uniform(-3, math.log10(5.0))))
    start = str(rng.choice(["random", "cold", "loaded"]))
    return dict(k=k, world=world, N=world * R, M=M, rule=rule, beta=beta, start=start,
                t0=int(rng.integers(0, 1000)) if start == "loaded" else 0,
                sweeps=[int(x) for x in rng.integers(1, 40, size=int(rng.integers(1, 3)))],
                seed=int(rng.integers(0, 2**63)))


GROUP_CASES = [draw_group_case(np.random.default_rng(MASTER_SEED + 1 + k), k) for k in range(24)]


def group_id(c):
    return f"{c['k']}-w{c['world']}-{c['N']}x{c['M']}-r{c['rule']}-b{c['beta']:.3g}-{c['start']}"


@pytest.mark.gpu
@pytest.mark.parametrize("c", GROUP_CASES, ids=[group_id(c) for c in GROUP_CASES])
def test_fuzz_local_group_matches_oracle(c):
    N, M, seed, world = c["N"], c["M"], c["seed"], c["world"]
    orule = oracle.RULE_HEATBATH if c["rule"] == ising.RULE_HEATBATH else oracle.RULE_METROPOLIS
    full = cases.random_pm1(np.random.default_rng(seed % 2**32), N, M, 0.6)
    o = oracle.Lattice(N, M, seed).set_beta(c["beta"], orule)
    if c["start"] == "random":
        o.init_random()
    elif c["start"] == "cold":
        o.init_cold()
    else:
        o.load_full(full, t=c["t0"])
    lats = IsingLattice.local_group(N, M, world, seed)

    def body(r, lat):
        lat.set_beta(c["beta"], c["rule"])
        if c["start"] == "random":
            lat.init_random()
        elif c["start"] == "cold":
            lat.init_cold()
        else:
            row0, rows = lat.slab_info()
            lat.write_lattice(np.ascontiguousarray(full[row0:row0 + rows]), t=c["t0"])
        res = []
        for n in c["sweeps"]:
            lat.sweep(n)
            row0, rows = lat.slab_info()
            out = np.empty((rows, M), dtype=np.int8)
            lat.read_lattice(out)
            res.append((out, lat.observables(), lat.t))
        return res

    try:
        per_rank = run_ranks(lats, body)
    finally:
        for lat in lats:
            lat.close()
    for step, n in enumerate(c["sweeps"]):
        o.sweep(n)
        got = np.concatenate([per_rank[r][step][0] for r in range(world)])
        exp = o.full()
        assert np.array_equal(got, exp), f"{group_id(c)} t={o.t}: {int((got != exp).sum())} differ"
        assert all(per_rank[r][step][1] == o.observables() for r in range(world)), group_id(c)
        assert all(per_rank[r][step][2] == o.t for r in range(world))


def test_fuzz_cases_cover_the_dimensions():
    """The drawn list actually spans what it claims to (so a change of the master seed or
    of draw_case cannot silently shrink the coverage)."""
    assert any(c["layout"] == "basic" for c in CASES)
    assert any(c["layout"] == "multispin" and (c["M"] // 32) % 256 == 0 for c in CASES)
    assert any(c["nslab"] > 1 for c in CASES)
    assert any(c["nslab"] > 1 and c["N"] // c["nslab"] == 2 for c in CASES) or \
        any(c["nslab"] > 1 and c["N"] // c["nslab"] <= 4 for c in CASES)
    assert any(c["rule"] == ising.RULE_HEATBATH for c in CASES)
    assert {c["start"] for c in CASES} == {"random", "cold", "loaded"}
    assert any(math.isinf(c["beta"]) for c in CASES) and any(c["beta"] == 0.0 for c in CASES)
    assert any(("sweep", 0) in c["chunks"] for c in CASES)
    assert any(ch[0] == "measure" and ch[2] > 1 for c in CASES for ch in c["chunks"])
    assert any(g["M"] % 8192 == 0 and g["N"] // g["world"] == 2 for g in GROUP_CASES) or \
        any(g["M"] % 8192 == 0 and g["N"] // g["world"] <= 4 for g in GROUP_CASES)
    assert any(g["M"] % 8192 != 0 for g in GROUP_CASES)
    assert any(g["world"] >= 4 for g in GROUP_CASES)
