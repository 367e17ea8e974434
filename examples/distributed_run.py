"""A multi-GPU run through the Python binding: one process per GPU, each owning a row slab
of the lattice, halo rows exchanged every half-sweep by the library.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \
        examples/distributed_run.py --rows 262144 --cols 262144 --sweeps 1000 --T 2.2

torch.distributed only carries the plumbing (the CUDA-IPC handle blobs or the NCCL unique
id); every sweep, the halo exchange and the observables' all-reduce run in the library's
kernels.  ISING_TRANSPORT=p2p (default) | lsa | nccl picks the transport.  Rank 0 prints
the magnetisation and energy per site every --every sweeps and writes a bit-packed
checkpoint of its own rows at the end (each rank writes its slab).
"""
import argparse
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_06297_b200.ising import IsingLattice  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=32768)
    ap.add_argument("--cols", type=int, default=32768)
    ap.add_argument("--sweeps", type=int, default=200)
    ap.add_argument("--every", type=int, default=50)
    ap.add_argument("--T", type=float, default=2.0 / math.log(1.0 + math.sqrt(2.0)))
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--checkpoint", default=None, help="directory for per-rank slab checkpoints")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    lat = IsingLattice.distributed(args.rows, args.cols, args.seed, device=local)
    row0, rows = lat.slab_info()
    lat.set_beta(1.0 / args.T).init_random()
    n_sites = args.rows * args.cols
    done = 0
    while done < args.sweeps:
        k = min(args.every, args.sweeps - done)
        ups, Es = lat.measure(1, k)  # k sweeps, then the all-reduced observables
        done += k
        if rank == 0:
            m = (2 * int(ups[-1]) - n_sites) / n_sites
            print(f"t={lat.t:8d}  m={m:+.5f}  E/site={int(Es[-1]) / n_sites:+.5f}  "
                  f"({lat.last_sweep_ms() / k:.3f} ms/sweep, transport {lat.transport})", flush=True)
    if args.checkpoint:
        os.makedirs(args.checkpoint, exist_ok=True)
        bits = lat.read_lattice_bits(np.empty(rows * args.cols // 8, dtype=np.uint8))
        bits.tofile(os.path.join(args.checkpoint, f"slab{rank:02d}_rows{row0}-{row0 + rows}_t{lat.t}.bin"))
    lat.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
