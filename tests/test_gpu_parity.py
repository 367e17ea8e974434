"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit for bit.

Lattices are compared as full +-1 byte arrays; observables as exact integers.
Inputs are the seeded configurations of tests/cases.py (no method arithmetic)."""
import hashlib
import math

import numpy as np
import pytest

import oracle
from paper_1906_06297_b200 import ising
from paper_1906_06297_b200.ising import IsingLattice
from tests import cases

pytestmark = pytest.mark.gpu


def gpu_lattice(N, M, seed, start, beta, rule=ising.RULE_METROPOLIS, devices=None):
    g = IsingLattice(N, M, seed, devices=devices)
    g.set_beta(beta, rule)
    if start == "random":
        g.init_random()
    elif start == "cold":
        g.init_cold()
    else:
        g.write_lattice(start)
    return g


def oracle_lattice(N, M, seed, start, beta, rule=oracle.RULE_METROPOLIS):
    o = oracle.Lattice(N, M, seed).set_beta(beta, rule)
    if start == "random":
        o.init_random()
    elif start == "cold":
        o.init_cold()
    else:
        o.load_full(start)
    return o


def assert_same(g, o, what=""):
    a, b = g.read_lattice(), o.full()
    if not np.array_equal(a, b):
        bad = np.argwhere(a != b)
        raise AssertionError(f"{what}: {len(bad)} sites differ, first {bad[:5].tolist()}")
    assert g.observables() == o.observables(), what


def test_c1_bit_exact_1000_sweeps():
    # BASELINE configs[0]: 64x64, beta = 0.4406868, random start, seed 1, 1000 sweeps
    N, M, beta, seed = 64, 64, 0.4406868, 1
    g = gpu_lattice(N, M, seed, "random", beta)
    o = oracle_lattice(N, M, seed, "random", beta)
    assert_same(g, o, "init")
    done = 0
    for target in [1, 10, 100, 1000]:
        g.sweep(target - done)
        o.sweep(target - done)
        done = target
        assert_same(g, o, f"after {target} sweeps")
    assert g.t == 1000


@pytest.mark.parametrize("N,M", cases.PARITY_SHAPES)
@pytest.mark.parametrize("beta", cases.PARITY_BETAS)
@pytest.mark.parametrize("start", ["random", "cold"])
def test_parity_matrix(N, M, beta, start):
    for seed in cases.PARITY_SEEDS:
        g = gpu_lattice(N, M, seed, start, beta)
        o = oracle_lattice(N, M, seed, start, beta)
        for n in [1, 1, 8]:
            g.sweep(n)
            o.sweep(n)
            assert_same(g, o, f"{N}x{M} beta={beta} seed={seed} start={start} t={o.t}")


@pytest.mark.parametrize("N,M,nslab", cases.SLAB_CASES)
def test_virtual_slabs_match_oracle(N, M, nslab):
    # slab decomposition on one device (halo rows exchanged by fused stores into the
    # neighbouring slab's halo): identical to the oracle and to n = 1 (reading R19)
    seed, beta = 3, 0.4406868
    g = gpu_lattice(N, M, seed, "random", beta, devices=[0] * nslab)
    o = oracle_lattice(N, M, seed, "random", beta)
    for n in [1, 4, 20]:
        g.sweep(n)
        o.sweep(n)
        assert_same(g, o, f"{nslab} slabs t={o.t}")


# Heat-bath betas with the expected kernel variant (ising_kernel_variant): 7 = symmetric
# thresholds (T[0] + T[4] = T[1] + T[3] = 2^32 + 1), the default whenever the rounded table
# has that property; with ISING_HB_SYMMETRIC=0 the five-compare kernels: 3 (every T < 2^32),
# 5 (T[0] = 2^32, beta 3), 6 (T[0] = T[1] = 2^32, beta 6, inf).  beta = 0 (all T = 2^31) and
# the two betas below (found by search: ceil(2^32 P(e)) + ceil(2^32 P(-e)) = 2^32 for one
# pair) are not symmetric, so they keep the five-compare kernels either way.
HB_ASYM = [0.3377438395041983, 1.2800778283900398]
HB_CASES = [((64, 64), 0.4406868, 7, 3), ((66, 128), 0.2, 7, 3), ((32, 64), math.inf, 6, 6),
            ((32, 64), 0.0, 3, 3), ((64, 128), 3.0, 7, 5), ((66, 64), 6.0, 7, 6),
            ((32, 64), 2.5, 7, 3), ((64, 64), HB_ASYM[0], 3, 3), ((64, 64), HB_ASYM[1], 3, 3)]


@pytest.mark.parametrize("sym", ["1", "0"])
def test_heatbath_parity(monkeypatch, sym):
    monkeypatch.setenv("ISING_HB_SYMMETRIC", sym)
    for (N, M), beta, v_sym, v_plain in HB_CASES:
        g = gpu_lattice(N, M, 5, "random", beta, ising.RULE_HEATBATH)
        o = oracle_lattice(N, M, 5, "random", beta, oracle.RULE_HEATBATH)
        T = [int(x) for x in o_thresholds(beta, oracle.RULE_HEATBATH)]
        assert g.thresholds() == T
        symmetric = T[2] == 2**31 and T[0] + T[4] == T[1] + T[3] == 2**32 + 1
        assert symmetric == (v_sym == 7), (beta, T)
        assert g.kernel_variant() == (v_sym if sym == "1" else v_plain), beta
        for n in [1, 10]:
            g.sweep(n)
            o.sweep(n)
            assert_same(g, o, f"heat bath {N}x{M} beta={beta} variant={g.kernel_variant()}")


def test_heatbath_symmetric_wide_and_measured():
    # variant 7 in the TMA-staged kernel (W % 256 == 0), two virtual slabs, and the fused
    # observables of a measured chain
    g = gpu_lattice(34, 8192, 6, "random", 0.4406868, ising.RULE_HEATBATH, devices=[0, 0])
    o = oracle_lattice(34, 8192, 6, "random", 0.4406868, oracle.RULE_HEATBATH)
    assert g.kernel_variant() == 7
    ups, Es = g.measure(4, 1)
    ou, oE = o.chain(4)
    assert np.array_equal(ups, ou) and np.array_equal(Es, oE)
    assert_same(g, o, "symmetric heat bath 34x8192")


def o_thresholds(beta, rule):
    return oracle.thresholds(beta, rule)


def test_thresholds_equal_oracle():
    g = IsingLattice(64, 64, 1)
    for beta in [0.0, 0.1, 0.2, 1 / 3, 0.4406868, 0.44068679350977147, 2 / 3, 0.8, 5.0, math.inf]:
        for rule in [ising.RULE_METROPOLIS, ising.RULE_HEATBATH]:
            g.set_beta(beta, rule)
            assert g.thresholds() == [int(x) for x in oracle.thresholds(beta, rule)], (beta, rule)


def test_write_read_round_trip_and_resume():
    rng = np.random.default_rng(17)
    for N, M in [(64, 64), (130, 192), (2, 64)]:
        full = cases.random_pm1(rng, N, M)
        g = IsingLattice(N, M, 9).write_lattice(full, t=37)
        assert np.array_equal(g.read_lattice(), full)
        assert g.t == 37
        g.set_beta(0.4406868).sweep(3)
        o = oracle.Lattice(N, M, 9).load_full(full, t=37).set_beta(0.4406868).sweep(3)
        assert_same(g, o, "resume")


def test_chunking_invariance():
    a = gpu_lattice(128, 128, 2, "random", 0.4406868)
    b = gpu_lattice(128, 128, 2, "random", 0.4406868)
    a.sweep(500).sweep(500)
    b.sweep(1000)
    assert np.array_equal(a.read_lattice(), b.read_lattice())


def test_trap_state_period_two():
    N, M = 64, 128
    full = cases.alternating_rows(N, M)
    for beta in [0.2, 0.4406868, math.inf]:
        g = IsingLattice(N, M, 1).write_lattice(full).set_beta(beta)
        g.sweep(1)
        assert np.array_equal(g.read_lattice(), -full)
        g.sweep(1)
        assert np.array_equal(g.read_lattice(), full)


def test_observables_closed_forms():
    N, M = 64, 128
    g = IsingLattice(N, M, 1).init_cold()
    assert g.observables() == (N * M, -2 * N * M)
    g.write_lattice(cases.neel(N, M))
    assert g.observables() == (N * M // 2, 2 * N * M)
    one = np.ones((N, M), dtype=np.int8)
    one[5, 7] = -1
    g.write_lattice(one)
    assert g.observables() == (N * M - 1, -2 * N * M + 8)


def test_beta_zero_flips_everything():
    g = gpu_lattice(64, 256, 4, "random", 0.0)
    f0 = g.read_lattice()
    up0, E0 = g.observables()
    g.sweep(1)
    assert np.array_equal(g.read_lattice(), -f0)
    assert g.observables() == (64 * 256 - up0, E0)


def test_error_behaviour():
    g = IsingLattice(64, 64, 1)
    with pytest.raises(ising.IsingError) as e:
        g.sweep(1)
    assert e.value.status == ising.ISING_ERR_STATE
    g.init_random()
    with pytest.raises(ising.IsingError) as e:
        g.sweep(1)  # no beta yet
    assert e.value.status == ising.ISING_ERR_STATE
    with pytest.raises(ising.IsingError) as e:
        g.set_beta(-1.0)
    assert e.value.status == ising.ISING_ERR_ARG
    with pytest.raises(ising.IsingError) as e:
        g.set_beta(float("nan"))
    assert e.value.status == ising.ISING_ERR_ARG
    with pytest.raises(ising.IsingError) as e:
        g.read_lattice(np.empty(64 * 64 - 1, dtype=np.int8))
    assert e.value.status == ising.ISING_ERR_RANGE
    for (i, j), v in [((3, 3), 0), ((0, 0), 2), ((63, 63), -128), ((10, 17), 127), ((5, 48), -2)]:
        bad = np.ones((64, 64), dtype=np.int8)
        bad[i, j] = v  # anything but +-1, at even / odd columns and both corners
        with pytest.raises(ising.IsingError) as e:
            g.write_lattice(bad)
        assert e.value.status == ising.ISING_ERR_ARG, (i, j, v)
    g.set_beta(0.3)
    g.write_lattice(np.ones((64, 64), dtype=np.int8), t=2**32 - 3)
    g.sweep(2)
    with pytest.raises(ising.IsingError) as e:
        g.sweep(1)
    assert e.value.status == ising.ISING_ERR_RANGE
    g.sweep(0)


def test_write_read_round_trip_pattern():
    # pack / unpack (row a9) on an arbitrary pattern: every byte position of the 16-byte
    # chunks, both row parities, a width that is not a multiple of 128 columns
    rng = np.random.default_rng(11)
    for N, M in [(6, 64), (130, 192), (34, 8192)]:
        full = rng.choice(np.array([-1, 1], dtype=np.int8), size=(N, M))
        g = IsingLattice(N, M, 1).write_lattice(full)
        assert np.array_equal(g.read_lattice(), full), (N, M)
        up, E = g.observables()
        assert up == int((full == 1).sum())
        assert E == -int((full * np.roll(full, 1, 0)).sum() + (full * np.roll(full, 1, 1)).sum())
        g.close()


def test_random_start_golden():
    # tests/golden/rng_contract.txt (independent evaluation of the contract)
    from tests import golden_io

    _, inits, _ = golden_io.rng_contract()
    for (N, M, seed), up, E, sha in inits:
        g = IsingLattice(N, M, seed).init_random()
        assert g.observables() == (up, E)
        assert hashlib.sha256(g.read_lattice().tobytes()).hexdigest().startswith(sha)


@pytest.mark.slow
def test_full_size_c3_one_sweep_matches_oracle():
    # BASELINE configs[2] shape (32768^2, beta_c, random start, seed 1) in the launch
    # configuration bench.py times; the whole lattice after one sweep, hashed.
    N = M = cases.C3[0]
    beta = cases.C3[2]
    g = gpu_lattice(N, M, 1, "random", beta)
    g.sweep(1)
    got = g.read_lattice()
    up_g = g.observables()
    g.close()
    o = oracle_lattice(N, M, 1, "random", beta)
    o.sweep(1)
    exp = o.full()
    assert hashlib.sha256(got.tobytes()).digest() == hashlib.sha256(exp.tobytes()).digest()
    assert up_g == o.observables()


def test_graph_replay_across_beta_and_rule_changes():
    # small lattices replay sweeps from a CUDA graph (64 sweeps per replay, sweep base in
    # device memory); set_beta / set_rule must rebuild it.  Plans mix replays and remainders.
    N, M = 128, 192
    g = gpu_lattice(N, M, 8, "random", 0.3)
    o = oracle_lattice(N, M, 8, "random", 0.3)
    for beta, rule, n in [(0.3, 0, 130), (0.4406868, 0, 64), (0.4406868, 1, 70), (0.8, 0, 200)]:
        g.set_beta(beta, rule)
        o.set_beta(beta, rule)
        g.sweep(n)
        o.sweep(n)
        assert_same(g, o, f"beta={beta} rule={rule} t={o.t}")


@pytest.mark.slow
@pytest.mark.parametrize("N,M", [(cases.C4[0], cases.C4[1]), (cases.C5_ROWS_PER_GPU, cases.C5_COLS)])
def test_full_size_sampled_rows_after_one_sweep(N, M):
    # BASELINE configs[3] (131072^2) and the per-GPU slab of configs[4] (131072 x 1048576,
    # 64 GiB packed) in bench.py's launch configuration: rows sampled across the lattice
    # (including the wrap rows 0 and N-1) against the oracle's site-by-site evaluation.
    beta = cases.BETA_TC
    g = gpu_lattice(N, M, 1, "random", beta)
    g.sweep(1)
    rng = np.random.default_rng(N + M)
    rows = sorted({0, 1, N - 1, N // 2} | set(int(x) for x in rng.integers(0, N, 4)))
    for i in rows:
        got = g.read_rows(i, 1)[0]
        exp = oracle.sample_row_after_one_sweep(1, N, M, beta, i)
        assert np.array_equal(got, exp), f"row {i}: {int((got != exp).sum())} sites differ"
    # beta = 0 property at full size: one sweep flips every spin (up -> NM - up, E kept)
    up0, E0 = g.observables()
    g.set_beta(0.0).sweep(1)
    assert g.observables() == (N * M - up0, E0)
    g.close()


@pytest.mark.slow
def test_c4_slab_count_invariance():
    # the 131072^2 lattice after 8 sweeps is the same split into 8 row slabs
    # (the n = 8 strong-scaling geometry, here 8 virtual slabs on one device, 2 x 8 GiB) as in
    # one: observables equal and rows byte-identical, sampled at every slab boundary
    N = M = cases.C4[0]
    beta = cases.BETA_TC
    one = gpu_lattice(N, M, 3, "random", beta)
    one.sweep(8)
    obs1 = one.observables()
    R = N // 8
    rows = sorted({k * R + d for k in range(8) for d in (-1, 0)} | {1, N // 3, N - 1})
    rows = [r % N for r in rows]
    ref = {r: one.read_rows(r, 1)[0].copy() for r in rows}
    one.close()
    eight = gpu_lattice(N, M, 3, "random", beta, devices=[0] * 8)
    eight.sweep(8)
    assert eight.observables() == obs1
    for r in rows:
        assert np.array_equal(eight.read_rows(r, 1)[0], ref[r]), f"row {r}"
    eight.close()


@pytest.mark.slow
@pytest.mark.parametrize("N,M,sweeps", [(1024, 8192, 500), (2048, 2048, 1000)])
def test_long_chains_bit_exact(N, M, sweeps):
    # long chains through the production paths (CUDA-graph replay of PDL-launched staged /
    # register-rolling half-sweeps, 64 sweeps per replay plus remainders) stay bit-exact
    g = gpu_lattice(N, M, 21, "random", 0.4406868)
    o = oracle_lattice(N, M, 21, "random", 0.4406868)
    g.sweep(sweeps - 37)
    g.sweep(37)
    o.sweep(sweeps)
    assert_same(g, o, f"{N}x{M} after {sweeps} sweeps")


@pytest.mark.slow
def test_c3_runs_are_deterministic_and_chunking_invariant():
    # bench.py's C3 workload: two runs of 100 sweeps (one call, and 37 + 63 calls) end in the
    # same lattice and observables (integer, race-free kernels; counter-based draws)
    N = M = cases.C3[0]
    digests = []
    for plan in ([100], [37, 63]):
        g = gpu_lattice(N, M, 1, "random", cases.C3[2])
        for n in plan:
            g.sweep(n)
        digests.append((g.observables(), hashlib.sha256(g.read_lattice().tobytes()).hexdigest()))
        g.close()
    assert digests[0] == digests[1]


def test_persistent_kernel_path(monkeypatch):
    # opt-in persistent multi-sweep kernel (ISING_PERSISTENT=1): same lattices and series
    monkeypatch.setenv("ISING_PERSISTENT", "1")
    N, M = 128, 128
    g = gpu_lattice(N, M, 6, "random", 0.4406868)
    o = oracle_lattice(N, M, 6, "random", 0.4406868)
    g.sweep(37)
    o.sweep(37)
    assert_same(g, o, "persistent sweeps")
    ups, Es = g.measure(25, 3)
    ou, oE = o.chain(75)
    assert np.array_equal(ups, ou[2::3]) and np.array_equal(Es, oE[2::3])
    g.set_beta(0.4406868, ising.RULE_HEATBATH)
    o.set_beta(0.4406868, oracle.RULE_HEATBATH)
    g.sweep(5)
    o.sweep(5)
    assert_same(g, o, "persistent heat bath")
    # every kernel variant through the persistent dispatcher: draw-free Metropolis (beta
    # inf), generic Metropolis (tiny beta), heat bath with 1 and 2 "always" classes
    for beta, rule in [(math.inf, ising.RULE_METROPOLIS), (4e-11, ising.RULE_METROPOLIS),
                       (3.0, ising.RULE_HEATBATH), (6.0, ising.RULE_HEATBATH)]:
        g.set_beta(beta, rule)
        o.set_beta(beta, rule)
        g.sweep(3)
        o.sweep(3)
        assert_same(g, o, f"persistent beta={beta} rule={rule}")


def test_tma_staged_kernel_path():
    # widths that are a multiple of 256 words use the TMA-staged half-sweep (cp.async.bulk
    # + mbarrier into shared memory): ragged last band (34 = 20 + 14 rows), two slabs,
    # heat bath, measured chain
    # (4, 8192, [0, 0]): 2-row slabs, every row a boundary row; (2, 8192): N = 2, both halo rows
    # are the other row
    for N, M, slabs in [(40, 8192, None), (64, 16384, [0, 0]), (34, 8192, None), (4, 8192, [0, 0]),
                        (2, 8192, None)]:
        g = gpu_lattice(N, M, 2, "random", 0.4406868, devices=slabs)
        o = oracle_lattice(N, M, 2, "random", 0.4406868)
        for n in [1, 3]:
            g.sweep(n)
            o.sweep(n)
            assert_same(g, o, f"staged {N}x{M} t={o.t}")
        g.set_beta(0.3, ising.RULE_HEATBATH)
        o.set_beta(0.3, oracle.RULE_HEATBATH)
        ups, Es = g.measure(3, 2)
        ou, oE = o.chain(6)
        assert np.array_equal(ups, ou[1::2]) and np.array_equal(Es, oE[1::2])
        assert_same(g, o, f"staged heat bath {N}x{M}")
        for beta in [3.0, math.inf]:  # heat bath variants 5 and 6 in the staged kernel
            g.set_beta(beta, ising.RULE_HEATBATH)
            o.set_beta(beta, oracle.RULE_HEATBATH)
            g.sweep(2)
            o.sweep(2)
            assert_same(g, o, f"staged heat bath {N}x{M} beta={beta}")


@pytest.mark.parametrize("tail", ["1", "0"])
def test_staged_guided_tail(monkeypatch, tail):
    # grids of 3 to 64 waves of 16-row tiles end with one wave of 8-row and one of 4-row
    # bands (ISING_TAIL=0: plain 16-row bands).  7168 x 32768: 448 bands x 4 spans = 1792
    # blocks >= 3 waves of 592 on a 148-SM B200; the 8-row region starts at row 4784.
    monkeypatch.setenv("ISING_TAIL", tail)
    N, M = 7168, 32768
    g = gpu_lattice(N, M, 9, "random", 0.4406868)
    o = oracle_lattice(N, M, 9, "random", 0.4406868)
    g.sweep(1)
    o.sweep(1)
    assert_same(g, o, f"staged tail={tail} {N}x{M}")
    g.set_beta(0.4406868, ising.RULE_HEATBATH)
    o.set_beta(0.4406868, oracle.RULE_HEATBATH)
    ups, Es = g.measure(1, 1)
    ou, oE = o.chain(1)
    assert np.array_equal(ups, ou) and np.array_equal(Es, oE)
    assert_same(g, o, f"staged tail={tail} heat bath {N}x{M}")


def test_register_rolling_path_on_wide_lattice(monkeypatch):
    # ISING_STAGED=0 keeps the register-rolling kernel on widths the staged one would take
    monkeypatch.setenv("ISING_STAGED", "0")
    g = gpu_lattice(40, 8192, 3, "random", 0.4406868)
    o = oracle_lattice(40, 8192, 3, "random", 0.4406868)
    g.sweep(2)
    o.sweep(2)
    assert_same(g, o, "register rolling 40x8192")
