"""Temperature scan on the GPU (§5.3, Figs. 5 and 6 method):
<|m|> against Onsager's M(T) and the Binder cumulant U_L(T) for several lattice sizes, with
the device-side measured chain.  Every temperature x replica of a size runs as one lattice
batch (ising_batch_*): one CTA per chain while it fits one CTA's shared memory (L^2 <= 409600),
up to 2048^2 as thread-block clusters; larger ones (or --no-batch) one handle per chain
(ising_sweep_measure).

    python tools/scan.py --sizes 64 128 256 --temps 2.1 2.2 2.25 2.3 2.35 2.4 \\
        --sweeps 200000 --every 10 --replicas 8 --out gpurun_out/scan.json
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
from paper_1906_06297_b200.ising import IsingBatch, IsingError, IsingLattice  # noqa: E402

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
    ap.add_argument("--replicas", type=int, default=1, help="independent chains per (L, T)")
    ap.add_argument("--no-batch", action="store_true", help="one handle per chain")
    ap.add_argument("--rule", choices=["metropolis", "heatbath"], default="metropolis")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    ns = a.sweeps // a.every
    rule = 1 if a.rule == "heatbath" else 0
    for L in a.sizes:
        series = {}  # k -> (ups, Es) concatenated over the replicas
        t0 = time.perf_counter()
        chains = [(k, r) for k in range(len(a.temps)) for r in range(a.replicas)]
        seeds = [a.seed + 1000 * k + L + 7919 * r for k, r in chains]
        b = None
        if not a.no_batch:
            try:  # one CTA (or one thread-block cluster, up to 2048^2) per chain
                b = IsingBatch(L, L, seeds)
            except IsingError:
                b = None
        if b is not None:
            b.set_beta([1.0 / a.temps[k] for k, _ in chains], rule).init_cold()
            b.sweep(a.discard)
            ups, Es = b.measure(ns, a.every)
            b.close()
            for k in range(len(a.temps)):
                idx = [q for q, (kk, _) in enumerate(chains) if kk == k]
                series[k] = (ups[idx].reshape(-1), Es[idx].reshape(-1))
            engine = "batch"
        else:
            for k, T in enumerate(a.temps):
                us, es = [], []
                for r in range(a.replicas):
                    g = IsingLattice(L, L, a.seed + 1000 * k + L + 7919 * r).set_beta(1.0 / T, rule).init_cold()
                    g.sweep(a.discard)
                    u, e = g.measure(ns, a.every)
                    g.close()
                    us.append(u)
                    es.append(e)
                series[k] = (np.concatenate(us), np.concatenate(es))
            engine = "one handle per chain"
        seconds = time.perf_counter() - t0
        for k, T in enumerate(a.temps):
            ups, Es = series[k]
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
                   "samples": len(m), "replicas": a.replicas, "engine": engine, "rule": a.rule,
                   "seconds_for_all_T_at_this_L": seconds}
            rows.append(row)
            print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
