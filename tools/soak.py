"""Soak: long chains run twice with different call chunkings must end bit-identical (no rare
race in the staged kernel, PDL overlap, graph replay or the measured-chain paths).

python tools/soak.py [--sweeps N]   (one B200; prints one JSON line per case)"""
import argparse
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_06297_b200.ising import IsingBatch, IsingLattice  # noqa: E402

BETA = 0.4406868


def digest(a) -> str:
    return hashlib.sha256(a.tobytes()).hexdigest()[:16]


def run(N, M, chunks, measure_every=0):
    lat = IsingLattice(N, M, 7).set_beta(BETA).init_random()
    for c in chunks:
        if measure_every:
            lat.measure(c // measure_every, measure_every)
        else:
            lat.sweep(c)
    out = (digest(lat.read_lattice()), lat.observables(), lat.t)
    lat.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweeps", type=int, default=100000)
    a = ap.parse_args()
    S = a.sweeps
    cases = [
        ("C3 32768^2 staged + PDL", 32768, 32768, [S // 10], [37, S // 10 - 37], 0),
        ("2048^2 graph replay", 2048, 2048, [10 * S], [3, 10 * S - 3 - 64 * 7, 64 * 7], 0),
        ("2048^2 measured chain (graphs) vs plain", 2048, 2048, [10 * S], [10 * S], 10),
    ]
    for name, N, M, ca, cb, meas in cases:
        t0 = time.perf_counter()
        ra = run(N, M, ca)
        rb = run(N, M, cb, meas)
        print(json.dumps({"case": name, "sweeps": sum(ca), "digest_a": ra[0], "digest_b": rb[0],
                          "identical": ra == rb, "observables": ra[1],
                          "seconds": round(time.perf_counter() - t0, 1)}), flush=True)
    # a lattice batch against one-lattice handles over a long chain
    t0 = time.perf_counter()
    b = IsingBatch(256, 256, [7, 8]).set_beta([BETA, 0.5]).init_random().sweep(S)
    same = []
    for k, (seed, beta) in enumerate([(7, BETA), (8, 0.5)]):
        g = IsingLattice(256, 256, seed).set_beta(beta).init_random().sweep(S)
        same.append(digest(b.read_lattice(k)) == digest(g.read_lattice()))
        g.close()
    b.close()
    print(json.dumps({"case": "256^2 batch vs one-lattice handles", "sweeps": S, "identical": all(same),
                      "seconds": round(time.perf_counter() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()
