"""Thin ctypes binding of libising.so (include/ising.h): argument marshalling only.

Every step of the sweep runs in the library's sm_100a kernels.  There is no CPU
fallback: if libising.so is missing or no sm_100 device is present, the calls fail
with an exception.  The functions ``ising_*`` mirror the C ABI one to one;
``IsingLattice`` is a convenience wrapper that owns a handle.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ISING_LIB") or os.path.join(_HERE, "libising.so")

ISING_OK = 0
ISING_ERR_ARG = -1
ISING_ERR_STATE = -2
ISING_ERR_DEVICE = -3
ISING_ERR_OOM = -4
ISING_ERR_CUDA = -5
ISING_ERR_NCCL = -6
ISING_ERR_RANGE = -7
RULE_METROPOLIS = 0
RULE_HEATBATH = 1
NCCL_ID_BYTES = 128
IPC_BLOB_BYTES = 256

# name -> (restype, argtypes); the exported symbols of include/ising.h
_VP = ctypes.c_void_p
_I64, _U64, _INT, _DBL, _SZ = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
_I64P, _U64P, _DBLP = ctypes.POINTER(_I64), ctypes.POINTER(_U64), ctypes.POINTER(_DBL)
SIGNATURES = {
    "ising_create": (_INT, [ctypes.POINTER(_VP), _I64, _I64, _U64, _INT]),
    "ising_create_slabs": (_INT, [ctypes.POINTER(_VP), _I64, _I64, _U64, _INT, ctypes.POINTER(_INT)]),
    "ising_create_rank": (_INT, [ctypes.POINTER(_VP), _I64, _I64, _U64, _INT, _INT, _INT, _VP, _SZ]),
    "ising_nccl_unique_id": (_INT, [_VP, _SZ]),
    "ising_create_rank_p2p": (_INT, [ctypes.POINTER(_VP), _I64, _I64, _U64, _INT, _INT, _INT]),
    "ising_create_rank_lsa": (_INT, [ctypes.POINTER(_VP), _I64, _I64, _U64, _INT, _INT, _INT, _VP, _SZ]),
    "ising_create_basic": (_INT, [ctypes.POINTER(_VP), _I64, _I64, _U64, _INT]),
    "ising_ipc_handle": (_INT, [_VP, _VP, _SZ]),
    "ising_ipc_connect": (_INT, [_VP, _VP, _SZ]),
    "ising_p2p_connect_local": (_INT, [ctypes.POINTER(_VP), _INT]),
    "ising_destroy": (_INT, [_VP]),
    "ising_set_beta": (_INT, [_VP, _DBL]),
    "ising_set_rule": (_INT, [_VP, _INT]),
    "ising_init_random": (_INT, [_VP]),
    "ising_init_cold": (_INT, [_VP]),
    "ising_write_lattice": (_INT, [_VP, _VP, _I64, _U64]),
    "ising_write_lattice_bits": (_INT, [_VP, _VP, _I64, _U64]),
    "ising_read_lattice_bits": (_INT, [_VP, _VP, _I64]),
    "ising_sweep": (_INT, [_VP, _I64]),
    "ising_read_lattice": (_INT, [_VP, _VP, _I64]),
    "ising_observables": (_INT, [_VP, _I64P, _I64P]),
    "ising_read_rows": (_INT, [_VP, _I64, _I64, _VP, _I64]),
    "ising_sweep_measure": (_INT, [_VP, _I64, _I64, _I64P, _I64P]),
    "ising_sweep_measure_async": (_INT, [_VP, _I64, _I64, _I64P, _I64P, _I64P]),
    "ising_measure_wait": (_INT, [_VP, _I64]),
    "ising_last_sweep_ms": (_INT, [_VP, _DBLP]),
    "ising_set_profiling": (_INT, [_VP, _INT]),
    "ising_kernel_stats": (_INT, [_VP, _DBLP, _I64P]),
    "ising_get_sweep": (_INT, [_VP, _U64P]),
    "ising_slab_info": (_INT, [_VP, _I64P, _I64P]),
    "ising_thresholds": (_INT, [_VP, _U64P]),
    "ising_launch_count": (_INT, [_VP, _I64P]),
    "ising_kernel_variant": (_INT, [_VP, ctypes.POINTER(ctypes.c_int)]),
    "ising_probe_philox": (_INT, [_INT, _DBLP]),
    "ising_batch_create": (_INT, [ctypes.POINTER(_VP), _I64, _I64, _INT, _U64P, _INT]),
    "ising_batch_destroy": (_INT, [_VP]),
    "ising_batch_set_beta": (_INT, [_VP, _DBLP, _INT]),
    "ising_batch_init_random": (_INT, [_VP]),
    "ising_batch_init_cold": (_INT, [_VP]),
    "ising_batch_sweep": (_INT, [_VP, _I64]),
    "ising_batch_sweep_measure": (_INT, [_VP, _I64, _I64, _I64P, _I64P]),
    "ising_batch_observables": (_INT, [_VP, _I64P, _I64P]),
    "ising_batch_read_lattice": (_INT, [_VP, _INT, _VP, _I64]),
    "ising_batch_write_lattice": (_INT, [_VP, _INT, _VP, _I64, _U64]),
    "ising_batch_last_sweep_ms": (_INT, [_VP, _DBLP]),
    "ising_batch_get_sweep": (_INT, [_VP, _U64P]),
    "ising_strerror": (ctypes.c_char_p, [_INT]),
    "ising_last_error": (ctypes.c_char_p, []),
}

_lib = None


class IsingError(RuntimeError):
    def __init__(self, status: int, call: str):
        lib = load()
        msg = lib.ising_strerror(status).decode()
        detail = lib.ising_last_error().decode()
        super().__init__(f"{call} -> {status} ({msg}){': ' + detail if detail else ''}")
        self.status = status


def load() -> ctypes.CDLL:
    """Load libising.so (built by __graft_entry__.build()); fails loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def _check(status: int, call: str) -> None:
    if status != ISING_OK:
        raise IsingError(status, call)


def _buf_ptr(buf, nbytes_needed: int, writable: bool, dtype=np.int8):
    """Pointer + length of a host int8 (uint8: bit-packed) buffer (numpy array or CPU tensor)."""
    if isinstance(buf, np.ndarray):
        if buf.dtype != dtype or not buf.flags["C_CONTIGUOUS"]:
            raise ValueError(f"lattice buffers must be C-contiguous {np.dtype(dtype).name}")
        if writable and not buf.flags["WRITEABLE"]:
            raise ValueError("output buffer is read-only")
        return buf.ctypes.data, buf.size
    # torch tensor (e.g. pinned host memory)
    if hasattr(buf, "data_ptr"):
        import torch

        want = torch.int8 if dtype == np.int8 else torch.uint8
        if buf.dtype != want or not buf.is_contiguous() or buf.is_cuda:
            raise ValueError(f"lattice tensors must be contiguous {want} host tensors")
        return buf.data_ptr(), buf.numel()
    raise TypeError("expected a numpy int8 array or an int8 torch tensor")


# ------------------------------------------------------------ raw ABI mirror
def ising_create(L_rows: int, L_cols: int, seed: int, n_gpus: int = 1) -> int:
    h = _VP()
    _check(load().ising_create(ctypes.byref(h), L_rows, L_cols, seed, n_gpus), "ising_create")
    return h.value


def ising_create_slabs(L_rows: int, L_cols: int, seed: int, devices) -> int:
    h = _VP()
    arr = (_INT * len(devices))(*devices)
    _check(load().ising_create_slabs(ctypes.byref(h), L_rows, L_cols, seed, len(devices), arr),
           "ising_create_slabs")
    return h.value


def ising_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    _check(load().ising_nccl_unique_id(buf, NCCL_ID_BYTES), "ising_nccl_unique_id")
    return buf.raw


def ising_create_rank(L_rows: int, L_cols: int, seed: int, rank: int, world: int, device: int,
                      nccl_id: bytes | None) -> int:
    h = _VP()
    idbuf = ctypes.create_string_buffer(nccl_id, NCCL_ID_BYTES) if nccl_id else None
    _check(load().ising_create_rank(ctypes.byref(h), L_rows, L_cols, seed, rank, world, device,
                                    idbuf, NCCL_ID_BYTES if nccl_id else 0), "ising_create_rank")
    return h.value


def ising_create_rank_p2p(L_rows: int, L_cols: int, seed: int, rank: int, world: int,
                          device: int) -> int:
    h = _VP()
    _check(load().ising_create_rank_p2p(ctypes.byref(h), L_rows, L_cols, seed, rank, world, device),
           "ising_create_rank_p2p")
    return h.value


def ising_create_rank_lsa(L_rows: int, L_cols: int, seed: int, rank: int, world: int, device: int,
                          nccl_id: bytes | None) -> int:
    h = _VP()
    idbuf = ctypes.create_string_buffer(nccl_id, NCCL_ID_BYTES) if nccl_id else None
    _check(load().ising_create_rank_lsa(ctypes.byref(h), L_rows, L_cols, seed, rank, world, device,
                                        idbuf, NCCL_ID_BYTES if nccl_id else 0),
           "ising_create_rank_lsa")
    return h.value


def ising_create_basic(L_rows: int, L_cols: int, seed: int, device: int = 0) -> int:
    h = _VP()
    _check(load().ising_create_basic(ctypes.byref(h), L_rows, L_cols, seed, device),
           "ising_create_basic")
    return h.value


def ising_ipc_handle(h: int) -> bytes:
    buf = ctypes.create_string_buffer(IPC_BLOB_BYTES)
    _check(load().ising_ipc_handle(h, buf, IPC_BLOB_BYTES), "ising_ipc_handle")
    return buf.raw


def ising_ipc_connect(h: int, blobs: bytes) -> None:
    buf = ctypes.create_string_buffer(blobs, len(blobs))
    _check(load().ising_ipc_connect(h, buf, len(blobs)), "ising_ipc_connect")


def ising_p2p_connect_local(handles) -> None:
    arr = (_VP * len(handles))(*handles)
    _check(load().ising_p2p_connect_local(arr, len(handles)), "ising_p2p_connect_local")


def ising_destroy(h: int) -> None:
    _check(load().ising_destroy(h), "ising_destroy")


def ising_set_beta(h: int, beta: float) -> None:
    _check(load().ising_set_beta(h, float(beta)), "ising_set_beta")


def ising_set_rule(h: int, rule: int) -> None:
    _check(load().ising_set_rule(h, int(rule)), "ising_set_rule")


def ising_init_random(h: int) -> None:
    _check(load().ising_init_random(h), "ising_init_random")


def ising_init_cold(h: int) -> None:
    _check(load().ising_init_cold(h), "ising_init_cold")


def ising_write_lattice(h: int, buf, t: int = 0) -> None:
    ptr, n = _buf_ptr(buf, 0, writable=False)
    _check(load().ising_write_lattice(h, ptr, n, int(t)), "ising_write_lattice")


def ising_write_lattice_bits(h: int, buf, t: int = 0) -> None:
    ptr, n = _buf_ptr(buf, 0, writable=False, dtype=np.uint8)
    _check(load().ising_write_lattice_bits(h, ptr, n, int(t)), "ising_write_lattice_bits")


def ising_read_lattice_bits(h: int, out) -> None:
    ptr, n = _buf_ptr(out, 0, writable=True, dtype=np.uint8)
    _check(load().ising_read_lattice_bits(h, ptr, n), "ising_read_lattice_bits")


def ising_sweep(h: int, n: int) -> None:
    _check(load().ising_sweep(h, int(n)), "ising_sweep")


def ising_read_lattice(h: int, out) -> None:
    ptr, n = _buf_ptr(out, 0, writable=True)
    _check(load().ising_read_lattice(h, ptr, n), "ising_read_lattice")


def ising_read_rows(h: int, row_begin: int, nrows: int, out) -> None:
    ptr, n = _buf_ptr(out, 0, writable=True)
    _check(load().ising_read_rows(h, int(row_begin), int(nrows), ptr, n), "ising_read_rows")


def ising_observables(h: int) -> tuple[int, int]:
    up, E = _I64(), _I64()
    _check(load().ising_observables(h, ctypes.byref(up), ctypes.byref(E)), "ising_observables")
    return up.value, E.value


def ising_sweep_measure(h: int, n_samples: int, every: int) -> tuple[np.ndarray, np.ndarray]:
    ups = np.zeros(int(n_samples), dtype=np.int64)
    Es = np.zeros(int(n_samples), dtype=np.int64)
    _check(load().ising_sweep_measure(h, int(n_samples), int(every),
                                      ups.ctypes.data_as(_I64P), Es.ctypes.data_as(_I64P)),
           "ising_sweep_measure")
    return ups, Es


def _i64_out(a: np.ndarray, n: int, name: str) -> np.ndarray:
    if a.dtype != np.int64 or not a.flags["C_CONTIGUOUS"] or a.size < n:
        raise ValueError(f"{name}: need a C-contiguous int64 array of at least {n} entries")
    return a


def ising_sweep_measure_async(h: int, n_samples: int, every: int, ups: np.ndarray,
                              Es: np.ndarray) -> int:
    """Enqueue a measured chain; `ups` / `Es` (caller-owned, ideally pinned, e.g. numpy views
    of torch pinned tensors) are valid after ising_measure_wait(h, ticket)."""
    _i64_out(ups, n_samples, "ups")
    _i64_out(Es, n_samples, "Es")
    ticket = ctypes.c_int64(0)
    _check(load().ising_sweep_measure_async(h, int(n_samples), int(every),
                                            ups.ctypes.data_as(_I64P), Es.ctypes.data_as(_I64P),
                                            ctypes.byref(ticket)), "ising_sweep_measure_async")
    return ticket.value


def ising_measure_wait(h: int, ticket: int) -> None:
    _check(load().ising_measure_wait(h, int(ticket)), "ising_measure_wait")


def ising_last_sweep_ms(h: int) -> float:
    v = _DBL()
    _check(load().ising_last_sweep_ms(h, ctypes.byref(v)), "ising_last_sweep_ms")
    return v.value


def ising_set_profiling(h: int, enable: bool) -> None:
    _check(load().ising_set_profiling(h, int(bool(enable))), "ising_set_profiling")


def ising_kernel_stats(h: int) -> tuple[float, int]:
    ms, n = _DBL(), _I64()
    _check(load().ising_kernel_stats(h, ctypes.byref(ms), ctypes.byref(n)), "ising_kernel_stats")
    return ms.value, n.value


def ising_get_sweep(h: int) -> int:
    t = _U64()
    _check(load().ising_get_sweep(h, ctypes.byref(t)), "ising_get_sweep")
    return t.value


def ising_slab_info(h: int) -> tuple[int, int]:
    a, b = _I64(), _I64()
    _check(load().ising_slab_info(h, ctypes.byref(a), ctypes.byref(b)), "ising_slab_info")
    return a.value, b.value


def ising_thresholds(h: int) -> list[int]:
    T = (_U64 * 5)()
    _check(load().ising_thresholds(h, T), "ising_thresholds")
    return [int(x) for x in T]


def ising_kernel_variant(h: int) -> int:
    v = ctypes.c_int(0)
    _check(load().ising_kernel_variant(h, ctypes.byref(v)), "ising_kernel_variant")
    return v.value


def ising_launch_count(h: int) -> int:
    n = _I64()
    _check(load().ising_launch_count(h, ctypes.byref(n)), "ising_launch_count")
    return n.value


def ising_probe_philox(device: int = 0) -> float:
    v = _DBL()
    _check(load().ising_probe_philox(device, ctypes.byref(v)), "ising_probe_philox")
    return v.value


# ------------------------------------------------------------ convenience
class IsingLattice:
    """Owns one handle.  ``devices`` maps slabs to CUDA devices (ising_create_slabs)."""

    def __init__(self, L_rows: int, L_cols: int, seed: int = 1, n_gpus: int = 1, devices=None,
                 _handle: int | None = None):
        self.N, self.M, self.seed = int(L_rows), int(L_cols), int(seed)
        if _handle is not None:
            self.h = _handle
        elif devices is not None:
            self.h = ising_create_slabs(self.N, self.M, self.seed, list(devices))
        else:
            self.h = ising_create(self.N, self.M, self.seed, n_gpus)

    @classmethod
    def basic(cls, L_rows: int, L_cols: int, seed: int = 1, device: int = 0):
        """The paper's basic byte-per-spin layout (§3.1) on one device."""
        return cls(L_rows, L_cols, seed, _handle=ising_create_basic(L_rows, L_cols, seed, device))

    @classmethod
    def distributed(cls, L_rows: int, L_cols: int, seed: int = 1, device: int | None = None,
                    transport: str | None = None):
        """One process per GPU under torch.distributed (the default process group does the
        plumbing: it moves the IPC handle blobs or the NCCL unique id between ranks).

        transport "p2p" (default): the half-sweep kernel stores halo rows into the
        neighbours' memory and synchronises through flags in peer memory
        (ising_create_rank_p2p, CUDA IPC mappings).  "lsa": the same kernel protocol over NCCL
        symmetric memory windows (ising_create_rank_lsa).  "nccl": ncclSend/ncclRecv of the
        halo rows on a comm stream overlapped with the interior (ising_create_rank)."""
        import torch.distributed as dist

        transport = transport or os.environ.get("ISING_TRANSPORT", "p2p")
        rank, world = dist.get_rank(), dist.get_world_size()
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", rank))
        if transport == "p2p":
            # every rank must agree: if CUDA IPC / peer mapping fails anywhere, all ranks
            # fall back to the NCCL transport together (both are GPU paths).  Every rank
            # makes the same collective calls whatever failed locally.
            h, err, blob = None, None, None
            try:
                h = ising_create_rank_p2p(L_rows, L_cols, seed, rank, world, device)
                blob = ising_ipc_handle(h)
            except IsingError as e:
                err = e
            blobs = [None] * world
            dist.all_gather_object(blobs, blob)
            if err is None:
                if any(b is None for b in blobs):
                    err = "IPC handle export failed on another rank"
                else:
                    try:
                        ising_ipc_connect(h, b"".join(blobs))
                    except IsingError as e:
                        err = e
            oks = [None] * world
            dist.all_gather_object(oks, err is None)
            if all(oks):
                lat = cls(L_rows, L_cols, seed, _handle=h)
                lat.transport = "p2p"
                return lat
            if h is not None:
                ising_destroy(h)
            import warnings

            warnings.warn(f"rank-p2p transport unavailable ({err or 'on another rank'}); using NCCL")
            transport = "nccl"
        if transport in ("nccl", "lsa"):
            obj = [ising_nccl_unique_id() if (rank == 0 and world > 1) else None]
            if world > 1:
                dist.broadcast_object_list(obj, src=0)
            create = ising_create_rank if transport == "nccl" else ising_create_rank_lsa
            h = create(L_rows, L_cols, seed, rank, world, device, obj[0])
        else:
            raise ValueError(f"unknown transport {transport!r}")
        lat = cls(L_rows, L_cols, seed, _handle=h)
        lat.transport = transport
        return lat

    @classmethod
    def local_group(cls, L_rows: int, L_cols: int, world: int, seed: int = 1, devices=None):
        """All `world` ranks of one rank-p2p lattice in this process (ising_p2p_connect_local):
        rank r on devices[r] (default: all on device 0).  Drive them from one host thread each
        (every collective call must be made on every handle); see run_ranks."""
        devices = list(devices) if devices is not None else [0] * world
        hs = []
        try:
            for r in range(world):
                hs.append(ising_create_rank_p2p(L_rows, L_cols, seed, r, world, devices[r]))
            ising_p2p_connect_local(hs)
        except Exception:
            for h in hs:
                ising_destroy(h)
            raise
        lats = [cls(L_rows, L_cols, seed, _handle=h) for h in hs]
        for lat in lats:
            lat.transport = "p2p-local"
        return lats

    def close(self):
        if getattr(self, "h", None):
            ising_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_beta(self, beta: float, rule: int | None = None):
        if rule is not None:
            ising_set_rule(self.h, rule)
        ising_set_beta(self.h, beta)
        return self

    def init_random(self):
        ising_init_random(self.h)
        return self

    def init_cold(self):
        ising_init_cold(self.h)
        return self

    def write_lattice(self, full, t: int = 0):
        ising_write_lattice(self.h, full, t)
        return self

    def sweep(self, n: int = 1):
        ising_sweep(self.h, n)
        return self

    def measure(self, n_samples: int, every: int = 1) -> tuple[np.ndarray, np.ndarray]:
        """(up_count, bond_energy) after every `every` sweeps, n_samples times."""
        return ising_sweep_measure(self.h, n_samples, every)

    def measure_async(self, n_samples: int, every: int, ups: np.ndarray, Es: np.ndarray) -> int:
        """Enqueue `n_samples` x `every` sweeps with observables into ups / Es; returns a
        ticket for measure_wait (the arrays are undefined until then)."""
        return ising_sweep_measure_async(self.h, n_samples, every, ups, Es)

    def measure_wait(self, ticket: int) -> None:
        ising_measure_wait(self.h, ticket)

    def read_lattice(self, out=None) -> np.ndarray:
        if out is None:
            out = np.empty((self.N, self.M), dtype=np.int8)
        ising_read_lattice(self.h, out)
        return out

    def observables(self) -> tuple[int, int]:
        return ising_observables(self.h)

    def write_lattice_bits(self, bits, t: int = 0):
        """Load from the bit-packed format (np.packbits(lattice == 1, bitorder="little"))."""
        ising_write_lattice_bits(self.h, bits, t)
        return self

    def read_lattice_bits(self, out=None) -> np.ndarray:
        if out is None:
            out = np.empty(self.N * self.M // 8, dtype=np.uint8)
        ising_read_lattice_bits(self.h, out)
        return out

    def read_rows(self, row_begin: int, nrows: int, out=None) -> np.ndarray:
        if out is None:
            out = np.empty((nrows, self.M), dtype=np.int8)
        ising_read_rows(self.h, row_begin, nrows, out)
        return out

    @property
    def t(self) -> int:
        return ising_get_sweep(self.h)

    def last_sweep_ms(self) -> float:
        return ising_last_sweep_ms(self.h)

    def thresholds(self) -> list[int]:
        return ising_thresholds(self.h)

    def slab_info(self) -> tuple[int, int]:
        return ising_slab_info(self.h)

    def set_profiling(self, enable: bool = True):
        ising_set_profiling(self.h, enable)
        return self

    def kernel_stats(self) -> tuple[float, int]:
        return ising_kernel_stats(self.h)

    def launch_count(self) -> int:
        return ising_launch_count(self.h)

    def kernel_variant(self) -> int:
        return ising_kernel_variant(self.h)


def run_ranks(lats, fn):
    """Run fn(rank, lattice) on one host thread per rank of a local group and return the
    results in rank order (the ctypes calls release the GIL, so the ranks' host calls and
    their kernels run concurrently).  An exception on any rank is re-raised."""
    import threading

    out = [None] * len(lats)
    errs = []

    def body(r):
        try:
            out[r] = fn(r, lats[r])
        except BaseException as e:  # reported below
            errs.append((r, e))

    ths = [threading.Thread(target=body, args=(r,)) for r in range(len(lats))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        r, e = errs[0]
        raise RuntimeError(f"rank {r}: {e!r}") from e
    return out


# ------------------------------------------------------------ lattice batches
class IsingBatch:
    """n independent L_rows x L_cols lattices on one device (ising_batch_*): lattice k draws
    with seeds[k] and runs at betas[k]; each is bit-identical to a one-lattice handle with the
    same seed and beta.  For temperature scans / Binder analysis on small lattices."""

    def __init__(self, L_rows: int, L_cols: int, seeds, device: int = 0):
        self.N, self.M = int(L_rows), int(L_cols)
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        self.n = int(seeds.size)
        h = _VP()
        _check(load().ising_batch_create(ctypes.byref(h), self.N, self.M, self.n,
                                         seeds.ctypes.data_as(_U64P), int(device)),
               "ising_batch_create")
        self.h = h.value

    def close(self):
        if getattr(self, "h", None):
            load().ising_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_beta(self, betas, rule: int = RULE_METROPOLIS):
        b = np.ascontiguousarray(np.broadcast_to(np.asarray(betas, dtype=np.float64), (self.n,)))
        _check(load().ising_batch_set_beta(self.h, b.ctypes.data_as(_DBLP), int(rule)),
               "ising_batch_set_beta")
        return self

    def init_random(self):
        _check(load().ising_batch_init_random(self.h), "ising_batch_init_random")
        return self

    def init_cold(self):
        _check(load().ising_batch_init_cold(self.h), "ising_batch_init_cold")
        return self

    def sweep(self, n: int = 1):
        _check(load().ising_batch_sweep(self.h, int(n)), "ising_batch_sweep")
        return self

    def measure(self, n_samples: int, every: int = 1) -> tuple[np.ndarray, np.ndarray]:
        """(up counts, bond energies), each of shape (n_lattices, n_samples)."""
        up = np.zeros((self.n, int(n_samples)), dtype=np.int64)
        E = np.zeros((self.n, int(n_samples)), dtype=np.int64)
        _check(load().ising_batch_sweep_measure(self.h, int(n_samples), int(every),
                                                up.ctypes.data_as(_I64P), E.ctypes.data_as(_I64P)),
               "ising_batch_sweep_measure")
        return up, E

    def observables(self) -> tuple[np.ndarray, np.ndarray]:
        up = np.zeros(self.n, dtype=np.int64)
        E = np.zeros(self.n, dtype=np.int64)
        _check(load().ising_batch_observables(self.h, up.ctypes.data_as(_I64P), E.ctypes.data_as(_I64P)),
               "ising_batch_observables")
        return up, E

    def read_lattice(self, k: int, out=None) -> np.ndarray:
        if out is None:
            out = np.empty((self.N, self.M), dtype=np.int8)
        ptr, n = _buf_ptr(out, self.N * self.M, True)
        _check(load().ising_batch_read_lattice(self.h, int(k), ptr, n), "ising_batch_read_lattice")
        return out

    def write_lattice(self, k: int, full, t: int = 0):
        ptr, n = _buf_ptr(full, self.N * self.M, False)
        _check(load().ising_batch_write_lattice(self.h, int(k), ptr, n, int(t)), "ising_batch_write_lattice")
        return self

    def last_sweep_ms(self) -> float:
        v = _DBL()
        _check(load().ising_batch_last_sweep_ms(self.h, ctypes.byref(v)), "ising_batch_last_sweep_ms")
        return v.value

    @property
    def t(self) -> int:
        v = _U64()
        _check(load().ising_batch_get_sweep(self.h, ctypes.byref(v)), "ising_batch_get_sweep")
        return v.value
