"""The C ABI from a plain C program (examples/ising_c_example.c, built by
__graft_entry__.build()): no Python or PyTorch on the path, results equal the oracle."""
import os
import subprocess

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "ising_c_example")


@pytest.mark.parametrize("N,M,seed,beta,sweeps", [(64, 64, 1, 0.4406868, 100), (130, 192, 7, 0.3, 65)])
def test_c_program_matches_oracle(N, M, seed, beta, sweeps, tmp_path):
    if not os.path.exists(EXE):
        pytest.fail("examples/ising_c_example missing: run __graft_entry__.build()")
    lat_file = tmp_path / "lattice.bin"
    out = subprocess.run([EXE, str(N), str(M), str(seed), repr(beta), str(sweeps), str(lat_file)],
                         capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    line1, line2, line3 = out.stdout.strip().split("\n")
    up, E, t, total = (int(x) for x in line1.split())
    o = oracle.Lattice(N, M, seed).init_random().set_beta(beta).sweep(sweeps)
    assert (up, E) == o.observables()
    assert t == sweeps and total == int(o.full().sum())
    got_lat = np.fromfile(lat_file, dtype=np.int8).reshape(N, M)  # element by element
    assert np.array_equal(got_lat, o.full())
    ou, oE = o.chain(12)  # the async chain: 2 calls x 3 samples, one every 2 sweeps
    got = [int(x) for x in line2.split()]
    assert got[0::2] == [int(x) for x in ou[1::2]] and got[1::2] == [int(x) for x in oE[1::2]]
    # the lattice batch: seeds seed, seed + 1, seed + 2 at beta, beta / 2, 2 beta
    got_b = [int(x) for x in line3.split()]
    for k, bk in enumerate([beta, beta / 2, 2 * beta]):
        ok = oracle.Lattice(N, M, seed + k).init_random().set_beta(bk).sweep(sweeps)
        assert tuple(got_b[2 * k:2 * k + 2]) == ok.observables(), f"batch lattice {k}"
