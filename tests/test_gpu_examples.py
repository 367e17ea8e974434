"""The shipped examples run end to end: examples/distributed_run.py under torch.distributed.run
(one rank: the NCCL process group, IsingLattice.distributed, measured chains, a bit-packed
checkpoint) — the checkpoint equals the oracle's lattice bit for bit."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_distributed_example_checkpoint_matches_oracle(tmp_path):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    N = M = 256
    sweeps, T, seed = 200, 2.1, 1
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "1", "--master-addr",
         "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "examples", "distributed_run.py"),
         "--rows", str(N), "--cols", str(M), "--sweeps", str(sweeps), "--every", "100", "--T", repr(T),
         "--seed", str(seed), "--checkpoint", str(tmp_path)],
        capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("t=")]
    assert len(lines) == 2 and lines[-1].startswith(f"t={sweeps:8d}")
    files = list(tmp_path.iterdir())
    assert len(files) == 1 and files[0].name == f"slab00_rows0-{N}_t{sweeps}.bin"
    bits = np.fromfile(files[0], dtype=np.uint8)
    o = oracle.Lattice(N, M, seed).set_beta(1.0 / T).init_random().sweep(sweeps)
    assert np.array_equal(bits, np.packbits(o.full() == 1, bitorder="little"))
    up, E = o.observables()
    m = (2 * up - N * M) / (N * M)
    assert f"m={m:+.5f}" in lines[-1] and f"E/site={E / (N * M):+.5f}" in lines[-1]


def test_scan_tool_batch_and_one_handle_paths_agree(tmp_path):
    # tools/scan.py: the lattice-batch engine and one handle per chain give identical series
    # (every batch lattice is bit-identical to a one-lattice handle with its seed)
    import json

    outs = []
    for extra, name in (([], "batch"), (["--no-batch"], "single")):
        path = tmp_path / f"{name}.json"
        out = subprocess.run(
            [sys.executable, os.path.join(ROOT, "tools", "scan.py"), "--sizes", "64", "128",
             "--temps", "2.2", "2.4", "--sweeps", "2000", "--discard", "100", "--every", "10",
             "--replicas", "2", "--out", str(path)] + extra,
            capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert out.returncode == 0, out.stderr[-2000:]
        outs.append(json.load(open(path)))
    a, b = outs
    assert [r["engine"] for r in a] == ["batch"] * 4 and [r["engine"] for r in b] == ["one handle per chain"] * 4
    for ra, rb in zip(a, b):
        for key in ("L", "T", "abs_m", "E_site", "m2", "m4", "binder", "samples"):
            assert ra[key] == rb[key], (key, ra, rb)
