"""Halo / interior overlap of the NCCL transport, from the library's event trace
(ISING_TRACE): a one-rank NCCL handle exchanging its halo rows with itself (ISING_SELF_EXCHANGE)
on C3, a few sweeps; per half-sweep the boundary-row kernels, the ncclSend/ncclRecv group on
the comm stream and the interior kernel.  Also the rank-p2p phase lengths for comparison.
python tools/trace_overlap.py [N] [M] [sweeps] -> JSON summary on stdout, CSVs in gpurun_out/"""
import csv
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_06297_b200 import ising  # noqa: E402
from paper_1906_06297_b200.ising import IsingLattice  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
M = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
os.makedirs("gpurun_out", exist_ok=True)
out = {"lattice": [N, M], "sweeps": sweeps}
for tname in ("nccl", "p2p"):
    path = os.path.abspath(f"gpurun_out/trace_{tname}_self.csv")
    os.environ["ISING_SELF_EXCHANGE"] = "1"
    os.environ["ISING_TRACE"] = path
    h = (ising.ising_create_rank(N, M, 1, 0, 1, 0, None) if tname == "nccl"
         else ising.ising_create_rank_p2p(N, M, 1, 0, 1, 0))
    os.environ.pop("ISING_TRACE")
    os.environ.pop("ISING_SELF_EXCHANGE")
    lat = IsingLattice(N, M, 1, _handle=h).set_beta(0.4406868).init_random()
    lat.sweep(2)  # warm (phases 0-3 are traced too; skipped below)
    lat.sweep(sweeps)
    lat.close()  # writes the trace
    ev = defaultdict(dict)
    with open(path) as f:
        for row in csv.DictReader(f):
            ev[int(row["phase"])][row["name"]] = float(row["ms"])
    phases = [p for p in sorted(ev) if p >= 4]
    if tname == "nccl":
        rows = []
        for p in phases:
            e = ev[p]
            halo = (e["halo_start"], e["halo_end"])
            inter = (e["interior_start"], e["interior_end"])
            ov = max(0.0, min(halo[1], inter[1]) - max(halo[0], inter[0]))
            rows.append({"boundary_us": 1e3 * (e["boundary_end"] - e["boundary_start"]),
                         "halo_us": 1e3 * (halo[1] - halo[0]),
                         "interior_us": 1e3 * (inter[1] - inter[0]),
                         "halo_hidden_frac": ov / max(halo[1] - halo[0], 1e-9),
                         "phase_us": 1e3 * (max(inter[1], halo[1]) - e["boundary_start"])})
        out[tname] = {k: sum(r[k] for r in rows) / len(rows) for k in rows[0]}
        out[tname]["phases"] = len(rows)
    else:
        d = [1e3 * (ev[p]["phase_end"] - ev[p]["phase_start"]) for p in phases]
        out[tname] = {"phase_us": sum(d) / len(d), "phases": len(d)}
print(json.dumps(out))
