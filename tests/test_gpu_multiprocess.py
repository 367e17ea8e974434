"""Multi-process rank mode on one GPU: world 2 and 4 processes, all on cuda:0, each owning a
row slab and exchanging halo rows by peer stores + flags in peer memory
(ising_create_rank_p2p, the path bench.py --gpus N uses).  The gathered lattice and the
all-reduced observables must equal the oracle's bit for bit.  gloo carries only the
plumbing (IPC handle blobs, the final gather)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, N, M, seed, beta, plan, transport, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_1906_06297_b200.ising import IsingLattice

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lat = IsingLattice.distributed(N, M, seed, device=0, transport=transport)
        row0, rows = lat.slab_info()
        lat.set_beta(beta).init_random()
        out = []
        for n in plan:
            lat.sweep(n)
            obs = lat.observables()
            full = np.zeros((N, M), dtype=np.int8)
            lat.read_lattice(full)
            parts = [torch.zeros((rows, M), dtype=torch.int8) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(full[row0:row0 + rows].copy()))
            out.append((obs, torch.cat(parts).numpy()))
        # load only this rank's rows (halos exchanged on the device), resume at t = 17
        rng = np.random.default_rng(99)
        full = np.where(rng.random((N, M)) < 0.6, 1, -1).astype(np.int8)
        lat.write_lattice(np.ascontiguousarray(full[row0:row0 + rows]), t=17)
        lat.sweep(2)
        mine = np.empty((rows, M), dtype=np.int8)
        lat.read_lattice(mine)
        parts = [torch.zeros((rows, M), dtype=torch.int8) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        out.append((lat.observables(), torch.cat(parts).numpy()))
        # measured chain: observables fused into the white phases, all-reduced across ranks
        ups, Es = lat.measure(3, 2)
        u2 = np.zeros(2, dtype=np.int64)
        e2 = np.zeros(2, dtype=np.int64)
        lat.measure_wait(lat.measure_async(2, 1, u2, e2))
        out.append((ups.tolist() + u2.tolist(), Es.tolist() + e2.tolist()))
        if rank == 0:
            q.put(("ok", out))
        lat.close()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("error", f"rank {rank}: {e!r}"))
    finally:
        dist.destroy_process_group()


def _chain_worker(rank, world, port, N, M, seed, beta, sweeps, q):
    """One call of `sweeps` sweeps per rank: 2 x sweeps phases coupled only through the
    flags in peer memory (with MPS the ranks' kernels overlap in time)."""
    import sys
    import time

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_1906_06297_b200.ising import IsingLattice

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lat = IsingLattice.distributed(N, M, seed, device=0, transport="p2p")
        row0, rows = lat.slab_info()
        lat.set_beta(beta).init_random()
        t0 = time.perf_counter()
        lat.sweep(sweeps)
        wall = time.perf_counter() - t0
        mine = np.empty((rows, M), dtype=np.int8)
        lat.read_lattice(mine)
        parts = [torch.zeros((rows, M), dtype=torch.int8) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        obs = lat.observables()
        lat.close()
        if rank == 0:
            q.put(("ok", (obs, torch.cat(parts).numpy(), wall)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("error", f"rank {rank}: {e!r}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N,M,sweeps", [(4, 128, 8192, 500), (2, 64, 128, 300),
                                              (3, 96, 16384, 200), (8, 64, 8192, 300)])
def test_rank_p2p_long_chain_separate_processes(world, N, M, sweeps):
    """Separate processes (CUDA IPC mappings, not the in-process local groups), one long call
    each; run under MPS (tools/gpu_mps.sh) the processes' kernels are concurrent."""
    import oracle

    seed, beta = 13, 0.4406868
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chain_worker, args=(r, world, port, N, M, seed, beta, sweeps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    status, payload = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", payload
    obs, full, wall = payload
    o = oracle.Lattice(N, M, seed).init_random().set_beta(beta).sweep(sweeps)
    assert np.array_equal(full, o.full()), f"{int((full != o.full()).sum())} sites differ"
    assert obs == o.observables()
    print(f"world {world} {N}x{M}: {sweeps} sweeps in {wall:.3f} s "
          f"(MPS: {os.environ.get('CUDA_MPS_PIPE_DIRECTORY') is not None})")


# (x, 8192) widths run the TMA-staged kernel, whose interior bands skip the neighbour wait
@pytest.mark.parametrize("world,N,M", [(2, 64, 128), (4, 128, 64), (2, 4, 64), (2, 128, 8192),
                                      (4, 48, 8192)])
def test_rank_p2p_matches_oracle(world, N, M):
    import oracle

    seed, beta, plan = 5, 0.4406868, [1, 3, 6]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, M, seed, beta, plan, "p2p", q))
             for r in range(world)]
    for p in procs:
        p.start()
    status, payload = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", payload
    o = oracle.Lattice(N, M, seed).init_random().set_beta(beta)
    for n, (obs, full) in zip(plan, payload):
        o.sweep(n)
        assert np.array_equal(full, o.full()), f"t={o.t}"
        assert obs == o.observables()
    rng = np.random.default_rng(99)
    start = np.where(rng.random((N, M)) < 0.6, 1, -1).astype(np.int8)
    o = oracle.Lattice(N, M, seed).load_full(start, t=17).set_beta(beta).sweep(2)
    obs, full = payload[len(plan)]
    assert np.array_equal(full, o.full()), "slab-only write + resume"
    assert obs == o.observables()
    ups, Es = payload[len(plan) + 1]
    ou, oE = o.chain(6)
    ou2, oE2 = o.chain(2)
    assert ups == [int(x) for x in ou[1::2]] + [int(x) for x in ou2], "measured chain (up)"
    assert Es == [int(x) for x in oE[1::2]] + [int(x) for x in oE2], "measured chain (E)"


def _large_worker(rank, world, port, N, M, seed, beta, sweeps, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_1906_06297_b200.ising import IsingLattice

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lat = IsingLattice.distributed(N, M, seed, device=0, transport="p2p")
        row0, rows = lat.slab_info()
        lat.set_beta(beta).init_random()
        for chunk in (1, sweeps - 1):  # a short call, then one long one
            lat.sweep(chunk)
        mine = np.empty((rows, M), dtype=np.int8)
        lat.read_lattice(mine)
        digest = np.frombuffer(mine.tobytes(), dtype=np.uint64).sum(dtype=np.uint64)
        parts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(parts, torch.tensor([int(digest) & (2**62 - 1)], dtype=torch.int64))
        obs = lat.observables()
        lat.close()
        if rank == 0:
            q.put(("ok", ([int(p.item()) for p in parts], obs)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("error", f"rank {rank}: {e!r}"))
    finally:
        dist.destroy_process_group()


def test_rank_p2p_large_lattice_equals_one_handle():
    """4 processes x 1024-row slabs of a 4096 x 8192 lattice (TMA-staged kernel: edge bands wait
    on the flags, 50 interior bands do not), 200 sweeps, against one handle of the whole lattice
    on the same GPU — slab digests and the all-reduced observables."""
    from paper_1906_06297_b200.ising import IsingLattice

    world, N, M, seed, beta, sweeps = 4, 4096, 8192, 21, 0.4406868, 200
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_large_worker, args=(r, world, port, N, M, seed, beta, sweeps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    status, payload = q.get(timeout=900)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", payload
    digests, obs = payload
    g = IsingLattice(N, M, seed).set_beta(beta).init_random().sweep(sweeps)
    full = g.read_lattice()
    R = N // world
    want = [int(np.frombuffer(full[r * R:(r + 1) * R].tobytes(), dtype=np.uint64).sum(dtype=np.uint64))
            & (2**62 - 1) for r in range(world)]
    assert digests == want
    assert obs == g.observables()
    g.close()
