"""Throughput of lattice batches (ising_batch_*) against one-lattice handles on small lattices
(the launch-bound regime of temperature scans / Binder analysis).

python tools/time_batch.py [--out FILE.json]   (one B200; device-timed, CUDA events)"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_06297_b200.ising import IsingBatch, IsingLattice  # noqa: E402

BETA = 0.4406868


def one_lattice(L: int, sweeps: int) -> float:
    lat = IsingLattice(L, L, 1).set_beta(BETA).init_random()
    lat.sweep(64)
    lat.sweep(sweeps)
    ms = lat.last_sweep_ms()
    lat.close()
    return L * L * sweeps / (ms * 1e6)


def batch(L: int, n: int, sweeps: int, every: int = 0) -> float:
    b = IsingBatch(L, L, list(range(1, n + 1))).set_beta(np.full(n, BETA)).init_random()
    b.sweep(8)
    if every:
        b.measure(sweeps // every, every)
    else:
        b.sweep(sweeps)
    ms = b.last_sweep_ms()
    b.close()
    return n * L * L * sweeps / (ms * 1e6)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for L, sweeps in [(64, 4096), (128, 2048), (256, 1024), (512, 256)]:
        single = one_lattice(L, sweeps)
        row = {"L": L, "sweeps": sweeps, "one_lattice_flips_per_ns": single, "batch": {}}
        for n in [1, 148, 592, 2368]:
            row["batch"][n] = batch(L, n, sweeps)
        row["batch_592_measured_every_8"] = batch(L, 592, sweeps, every=8)
        rows.append(row)
        print(json.dumps(row), flush=True)
    # lattices beyond one CTA: thread-block clusters (1024^2: 4 CTAs, 2048^2: 16 CTAs each)
    for L, sweeps, ns in [(1024, 128, [1, 8, 37, 74, 148]), (2048, 64, [1, 4, 9, 18, 36])]:
        row = {"L": L, "sweeps": sweeps, "one_lattice_flips_per_ns": one_lattice(L, sweeps),
               "cluster_batch": {n: batch(L, n, sweeps) for n in ns}}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
