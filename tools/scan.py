"""Temperature scan on the GPU (§5.3, Figs. 5 and 6 method):
<|m|> against Onsager's M(T) and the Binder cumulant U_L(T) for several lattice sizes, with
the device-side measured chain (ising_sweep_measure).

    python tools/scan.py --sizes 64 128 256 --temps 2.1 2.2 2.25 2.3 2.35 2.4 \\
        --sweeps 200000 --every 10 --out gpurun_out/scan.json
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1906_06297_b200.ising import IsingLattice  # noqa: E402

TC = 2.0 / math.log(1.0 + math.sqrt(2.0))


def onsager(T):
    return 0.0 if T >= TC else (1.0 - math.sinh(2.0 / T) ** -4) ** 0.125


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[64, 128, 256])
    ap.add_argument("--temps", type=float, nargs="+", default=[2.1, 2.2, 2.25, 2.3, 2.35, 2.4])
    ap.add_argument("--sweeps", type=int, default=100000)
    ap.add_argument("--discard", type=int, default=5000)
    ap.add_argument("--every", type=int, default=10)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for L in a.sizes:
        for k, T in enumerate(a.temps):
            t0 = time.perf_counter()
            g = IsingLattice(L, L, a.seed + 1000 * k + L).set_beta(1.0 / T).init_cold()
            g.sweep(a.discard)
            ups, Es = g.measure(a.sweeps // a.every, a.every)
            g.close()
            m = (2 * ups - L * L) / (L * L)
            m2, m4 = float(np.mean(m ** 2)), float(np.mean(m ** 4))
            # errors from 50 contiguous blocks: batch means for <|m|>, E; jackknife for U
            nb = 50
            blocks = np.array_split(np.arange(len(m)), nb)
            am = np.array([np.mean(np.abs(m[b])) for b in blocks])
            eb = np.array([np.mean(Es[b]) for b in blocks]) / (L * L)
            b2 = np.array([np.mean(m[b] ** 2) for b in blocks])
            b4 = np.array([np.mean(m[b] ** 4) for b in blocks])
            jk = np.array([1 - (np.sum(b4) - b4[k]) / (nb - 1) /
                           (3 * ((np.sum(b2) - b2[k]) / (nb - 1)) ** 2) for k in range(nb)])
            row = {"L": L, "T": T, "abs_m": float(np.mean(np.abs(m))), "onsager": onsager(T),
                   "abs_m_se": float(np.std(am, ddof=1) / math.sqrt(nb)),
                   "E_site": float(np.mean(Es)) / (L * L),
                   "E_site_se": float(np.std(eb, ddof=1) / math.sqrt(nb)), "m2": m2, "m4": m4,
                   "binder": 1 - m4 / (3 * m2 * m2), "binder_paper_literal": 1 - m4 / (m2 * m2),
                   "binder_se": float(math.sqrt((nb - 1) / nb * np.sum((jk - np.mean(jk)) ** 2))),
                   "samples": len(m), "seconds": time.perf_counter() - t0}
            rows.append(row)
            print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
