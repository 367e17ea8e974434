"""Pinned host <-> device copy bandwidth against the library's write_lattice / read_lattice
(the e2e path's copy roof).  python tools/time_transfers.py [N]"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1906_06297_b200.ising import IsingLattice  # noqa: E402

N = M = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
nbytes = N * M
res = {"bytes": nbytes}
a = torch.empty(nbytes, dtype=torch.int8, pin_memory=True)
d = torch.empty(nbytes, dtype=torch.int8, device="cuda")
st = torch.cuda.Stream()
for chunk_mib in (4, 16, 64, 256, 1024):
    ch = chunk_mib << 20
    best_h2d = best_d2h = 0.0
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(st):
            for o in range(0, nbytes, ch):
                d[o:o + ch].copy_(a[o:o + ch], non_blocking=True)
        st.synchronize()
        t1 = time.perf_counter()
        with torch.cuda.stream(st):
            for o in range(0, nbytes, ch):
                a[o:o + ch].copy_(d[o:o + ch], non_blocking=True)
        st.synchronize()
        t2 = time.perf_counter()
        best_h2d = max(best_h2d, nbytes / (t1 - t0) / 1e9)
        best_d2h = max(best_d2h, nbytes / (t2 - t1) / 1e9)
    res[f"pinned_h2d_gbs_chunk{chunk_mib}MiB"] = best_h2d
    res[f"pinned_d2h_gbs_chunk{chunk_mib}MiB"] = best_d2h
# both directions at once (two streams)
st2 = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
half = nbytes // 2
with torch.cuda.stream(st):
    d[:half].copy_(a[:half], non_blocking=True)
with torch.cuda.stream(st2):
    a[half:].copy_(d[half:], non_blocking=True)
torch.cuda.synchronize()
res["bidir_total_gbs"] = nbytes / (time.perf_counter() - t0) / 1e9
del d
lat = IsingLattice(N, M, 1).set_beta(0.44).init_random()
h = a.view(N, M)
lat.read_lattice(h.numpy())
w, r = [], []
for _ in range(3):
    t0 = time.perf_counter()
    lat.write_lattice(h.numpy())
    t1 = time.perf_counter()
    lat.read_lattice(h.numpy())
    t2 = time.perf_counter()
    w.append(nbytes / (t1 - t0) / 1e9)
    r.append(nbytes / (t2 - t1) / 1e9)
res["write_lattice_gbs"] = max(w)
res["read_lattice_gbs"] = max(r)
print(json.dumps(res))
