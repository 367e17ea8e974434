"""The bit-packed host format (ising_write_lattice_bits / ising_read_lattice_bits): the same
lattice as the +-1 byte format, one bit per spin (bit J & 7 of byte (i L_cols + J) / 8 = 1 for
+1, numpy's packbits(..., bitorder="little") of the +1 mask), checked against the byte API and
the oracle (loads and exact resume: PAPER.md's counter-based draws make a resume exact)."""
import numpy as np
import pytest

import oracle
from paper_1906_06297_b200 import ising
from paper_1906_06297_b200.ising import IsingLattice, run_ranks
from tests import cases

pytestmark = pytest.mark.gpu
BETA = cases.BETA_TC


def to_bits(lat: np.ndarray) -> np.ndarray:
    return np.packbits((lat == 1).reshape(-1), bitorder="little")


def from_bits(bits: np.ndarray, N: int, M: int) -> np.ndarray:
    return np.where(np.unpackbits(bits, bitorder="little").reshape(N, M) == 1, 1, -1).astype(np.int8)


@pytest.mark.parametrize("N,M", [(64, 64), (130, 192), (2, 64), (96, 8192), (4, 2048)])
def test_bits_round_trip_and_resume_match_oracle(N, M):
    seed = 4
    g = IsingLattice(N, M, seed).set_beta(BETA).init_random().sweep(7)
    try:
        assert np.array_equal(g.read_lattice_bits(), to_bits(g.read_lattice()))
        rng = np.random.default_rng(N + M)
        start = cases.random_pm1(rng, N, M, 0.4)
        g.write_lattice_bits(to_bits(start), t=33)
        assert np.array_equal(g.read_lattice(), start)
        g.sweep(5)
        o = oracle.Lattice(N, M, seed).load_full(start, t=33).set_beta(BETA).sweep(5)
        assert np.array_equal(from_bits(g.read_lattice_bits(), N, M), o.full())
        assert g.observables() == o.observables()
    finally:
        g.close()


def test_bits_multi_chunk_c3_size():
    """32768^2: 128 MiB of bits, two staging chunks each way, against the byte format."""
    N = M = 32768
    g = IsingLattice(N, M, 1).set_beta(BETA).init_random().sweep(1)
    try:
        lat = g.read_lattice()
        bits = g.read_lattice_bits()
        assert np.array_equal(bits, to_bits(lat))
        flipped = np.bitwise_not(bits)  # every spin reversed
        g.write_lattice_bits(flipped, t=1)
        assert np.array_equal(g.read_lattice(), -lat)
    finally:
        g.close()


def test_bits_virtual_slabs_and_rank_group_slab_only():
    N, M, seed = 128, 8192, 6
    rng = np.random.default_rng(1)
    start = cases.random_pm1(rng, N, M, 0.55)
    o = oracle.Lattice(N, M, seed).load_full(start, t=9).set_beta(BETA).sweep(4)
    s = IsingLattice(N, M, seed, devices=[0] * 4)  # LOCAL mode, 4 slabs
    try:
        s.set_beta(BETA).write_lattice_bits(to_bits(start), t=9).sweep(4)
        assert np.array_equal(from_bits(s.read_lattice_bits(), N, M), o.full())
    finally:
        s.close()
    lats = IsingLattice.local_group(N, M, 4, seed)  # rank-p2p, each rank loads its own rows
    try:
        def body(r, lat):
            row0, rows = lat.slab_info()
            lat.set_beta(BETA).write_lattice_bits(to_bits(start[row0:row0 + rows]), t=9)
            lat.sweep(4)
            out = np.empty(rows * M // 8, dtype=np.uint8)
            lat.read_lattice_bits(out)
            return from_bits(out, rows, M)
        got = np.concatenate(run_ranks(lats, body))
    finally:
        for lat in lats:
            lat.close()
    assert np.array_equal(got, o.full())


def test_bits_errors():
    g = IsingLattice(64, 128, 1).set_beta(BETA).init_random()
    b = IsingLattice.basic(64, 128, 1)
    try:
        with pytest.raises(ising.IsingError) as ei:
            g.write_lattice_bits(np.zeros(64 * 128 // 8 - 1, dtype=np.uint8))
        assert ei.value.status == ising.ISING_ERR_RANGE
        with pytest.raises(ValueError):
            g.write_lattice_bits(np.zeros(64 * 128 // 8, dtype=np.int8))  # wrong dtype
        with pytest.raises(ising.IsingError) as ei:
            b.read_lattice_bits()
        assert ei.value.status == ising.ISING_ERR_ARG
    finally:
        g.close()
        b.close()
