"""World-size-2/4 gloo tests (CPU) of the multi-process slab path's host logic.

The GPU rank mode (ising_create_rank) partitions rows into slabs, and after each colour
phase sends local row 0 to the rank above and row R-1 to the rank below (ncclSend/Recv),
receiving the mirror rows into its halo rows (§4).  Here the
same partition and exchange schedule run over gloo with the oracle's slab update, and the
gathered lattice must equal the single-lattice oracle bit for bit.  Also: the NCCL unique
id rendezvous of IsingLattice.distributed broadcasts one id to every rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _exchange(plane_rows, halo_top, halo_bot, rank, world):
    """The rank-mode halo schedule of ising_runtime.cu phase_rank, over gloo."""
    up, dn = (rank - 1) % world, (rank + 1) % world
    send0 = torch.from_numpy(plane_rows[0].copy())
    sendR = torch.from_numpy(plane_rows[-1].copy())
    rbot = torch.empty_like(send0)
    rtop = torch.empty_like(send0)
    # posted in the same order as the NCCL group: send(row0->up), recv(bottom<-dn),
    # send(rowR-1->dn), recv(top<-up); with world == 2 up == dn and order matters.
    reqs = [dist.isend(send0, up), dist.irecv(rbot, dn), dist.isend(sendR, dn), dist.irecv(rtop, up)]
    for r in reqs:
        r.wait()
    halo_bot[:] = rbot.numpy()
    halo_top[:] = rtop.numpy()


def _worker(rank, world, port, N, M, seed, beta, sweeps, q):
    import sys

    sys.path.insert(0, ROOT)
    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        R = N // world
        row0 = rank * R
        full0 = oracle.Lattice(N, M, seed).init_random()
        planes = [full0.black[row0:row0 + R].copy(), full0.white[row0:row0 + R].copy()]
        # halo rows (global rows row0-1 and row0+R mod N), as ising_init fills them
        top = [full0.black[(row0 - 1) % N].copy(), full0.white[(row0 - 1) % N].copy()]
        bot = [full0.black[(row0 + R) % N].copy(), full0.white[(row0 + R) % N].copy()]
        for t in range(1, sweeps + 1):
            for c in (0, 1):
                oracle.update_slab(planes[c], planes[1 - c], top[1 - c], bot[1 - c], c == 0, row0,
                                   seed, t, beta)
                _exchange(planes[c], top[c], bot[c], rank, world)
        gathered = [torch.empty((R, M // 2), dtype=torch.int8) for _ in range(world)]
        for c in (0, 1):
            dist.all_gather(gathered, torch.from_numpy(planes[c]))
            if rank == 0:
                q.put((c, torch.cat(gathered).numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 16), (2, 4), (4, 32), (4, 8)])
def test_slab_exchange_matches_single_lattice(world, N):
    M, seed, beta, sweeps = 64, 7, 0.4406868, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, M, seed, beta, sweeps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle

    ref = oracle.Lattice(N, M, seed).init_random().set_beta(beta).sweep(sweeps)
    assert np.array_equal(got[0], ref.black)
    assert np.array_equal(got[1], ref.white)


def _id_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    from paper_1906_06297_b200 import ising

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the rendezvous of IsingLattice.distributed: rank 0 makes the id, all receive it
        obj = [ising.ising_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        q.put((rank, obj[0]))
        # without a GPU, creating the rank handle must fail loudly (no CPU fallback)
        try:
            ising.ising_create_rank(64, 64, 1, rank, world, 0, obj[0])
            q.put((rank, "created"))
        except ising.IsingError as e:
            q.put((rank, e.status))
    finally:
        dist.destroy_process_group()


def test_nccl_id_rendezvous_over_gloo():
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=120) for _ in range(2 * world)]
    for p in procs:
        p.join(timeout=60)
    ids = [m for _, m in msgs if isinstance(m, bytes)]
    stats = [m for _, m in msgs if not isinstance(m, bytes)]
    assert len(ids) == world and len(set(ids)) == 1 and len(ids[0]) == 128
    from paper_1906_06297_b200 import ising

    assert all(s in (ising.ISING_ERR_CUDA, ising.ISING_ERR_DEVICE) for s in stats), stats


def _agree_worker(rank, world, port, fail_rank, fail_at, q):
    """IsingLattice.distributed's transport agreement with the ABI calls replaced by fakes
    (no GPU here): rank `fail_rank` fails at `fail_at` ("create", "handle" or "connect"); every
    rank must make the same collective calls and all must fall back to NCCL together."""
    import sys

    sys.path.insert(0, ROOT)
    from paper_1906_06297_b200 import ising

    calls = []

    def fail(name):
        if rank == fail_rank and fail_at == name:
            raise ising.IsingError.__new__(ising.IsingError)

    def create_p2p(*a):
        calls.append("create_p2p")
        fail("create")
        return 1000 + rank

    def ipc_handle(h):
        calls.append("ipc_handle")
        fail("handle")
        return bytes([rank]) * ising.IPC_BLOB_BYTES

    def ipc_connect(h, blobs):
        calls.append("ipc_connect")
        assert len(blobs) == world * ising.IPC_BLOB_BYTES
        fail("connect")

    ising.ising_create_rank_p2p = create_p2p
    ising.ising_ipc_handle = ipc_handle
    ising.ising_ipc_connect = ipc_connect
    ising.ising_destroy = lambda h: calls.append("destroy")
    ising.ising_nccl_unique_id = lambda: b"\x07" * ising.NCCL_ID_BYTES
    ising.ising_create_rank = lambda *a: calls.append(("create_rank", a[-1])) or 2000 + rank
    ising.IsingError.__init__ = lambda self, *a: None
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lat = ising.IsingLattice.distributed(64, 64, 1, device=0)
        q.put((rank, lat.transport, lat.h, calls))
        lat.h = None  # a fake handle: nothing to destroy
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank,fail_at", [(None, None), (1, "create"), (0, "handle"),
                                               (1, "connect")])
def test_distributed_transport_agreement(fail_rank, fail_at):
    """when CUDA IPC setup fails on one rank only, every rank still makes the same
    collective calls (no mismatched all_gather, no hang) and all ranks fall back to the NCCL
    transport together; with no failure all use rank-p2p."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, world, port, fail_rank, fail_at, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = "p2p" if fail_rank is None else "nccl"
    assert all(res[r][0] == want for r in range(world)), res
    if want == "nccl":
        for r in range(world):
            calls = res[r][2]
            assert calls.count(("create_rank", b"\x07" * 128)) == 1, calls  # the broadcast id
            # a rank whose p2p handle was created destroys it before falling back
            if "create_p2p" in calls and not (r == fail_rank and fail_at == "create"):
                assert "destroy" in calls, calls
