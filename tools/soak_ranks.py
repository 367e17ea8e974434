"""Soak of the cross-process rank-p2p protocol: `world` processes on cuda:0 (run under MPS for
real concurrency: tools/gpu_mps.sh environment) sweep an N x M lattice for many sweeps; each
rank's slab digest and the all-reduced observables must equal one handle of the whole lattice.

python tools/soak_ranks.py WORLD N M SWEEPS"""
import hashlib
import json
import os
import socket
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, N, M, sweeps, q):
    import torch.distributed as dist

    from paper_1906_06297_b200.ising import IsingLattice

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lat = IsingLattice.distributed(N, M, 5, device=0, transport="p2p")
    row0, rows = lat.slab_info()
    lat.set_beta(0.4406868).init_random()
    t0 = time.perf_counter()
    lat.sweep(sweeps)
    wall = time.perf_counter() - t0
    mine = np.empty((rows, M), dtype=np.int8)
    lat.read_lattice(mine)
    q.put((rank, hashlib.sha256(mine.tobytes()).hexdigest()[:16], lat.observables(), wall))
    lat.close()
    dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp

    from paper_1906_06297_b200.ising import IsingLattice

    world, N, M, sweeps = (int(x) for x in sys.argv[1:5])
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, world, port, N, M, sweeps, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=3600) for _ in range(world))
    for p in ps:
        p.join()
    g = IsingLattice(N, M, 5).set_beta(0.4406868).init_random().sweep(sweeps)
    full = g.read_lattice()
    R = N // world
    want = [hashlib.sha256(full[r * R:(r + 1) * R].tobytes()).hexdigest()[:16] for r in range(world)]
    ok = [d for _, d, _, _ in res] == want and all(o == g.observables() for _, _, o, _ in res)
    print(json.dumps({"world": world, "lattice": [N, M], "sweeps": sweeps, "identical": ok,
                      "mps": os.environ.get("CUDA_MPS_PIPE_DIRECTORY") is not None,
                      "rank_wall_s": max(w for *_, w in res),
                      "flips_per_ns_all_ranks": N * M * sweeps / (max(w for *_, w in res) * 1e9)}))


if __name__ == "__main__":
    main()
