#!/usr/bin/env python
"""Benchmark: spin flips/ns of the multi-spin checkerboard Metropolis sweep on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c3|c4|c5] [--layout multispin|basic] [--no-cpu-baseline]

A step is one full sweep (black + white half-sweep) of the whole lattice.  N = 1 runs
BASELINE.json configs[2] (C3: 32768 x 32768, beta = 0.4406868, random start, seed 1).
N > 1 (launched by torch.distributed.run, one process per GPU) weak-scales C3: each
rank owns a 32768 x 32768 slab of an (N*32768) x 32768 lattice; the half-sweep kernel
stores its boundary rows into the neighbours' halo rows through CUDA-IPC peer pointers and
signals them with flags in peer memory (rank-p2p; ncclSend/ncclRecv if peer mapping is
unavailable — config.transport says which) ("scaling": "weak").  --config c4 strong-scales 131072^2,
--config c5 weak-scales 131072 x 1048576 per GPU.

value: flips/ns over the K timed sweeps, device-timed with CUDA events on the launching
stream inside the library, max over ranks.  e2e: the same workload through the C ABI with
host buffers — write_lattice from pinned host memory, K sweeps with the observables of each
sweep fused into its white phase and copied to the host every step (ising_sweep_measure_async,
the host waiting one step behind), read_lattice back — all inside the timed region.
vs_baseline: value / the paper's single-V100 number for the same lattice (Table 2) where it
has one (context: another machine).  --impl reference times the CPU oracle
(oracle/, the "reference arm" of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BETA = 0.4406868
SEED = 1
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
BYTES_PER_FLIP = 1.5  # 4-bit spins: read target + read source + write target
# per-thread 32x32->64 multiplies per attempted flip in the staged kernel's row loop: 114
# IMAD.WIDE.U32 per 32 flips (SASS, tools/sass_loops.py; 16 per Philox block / 4 = 4, less the
# row-invariant round-2 products ptxas hoists out of the row loop)
MULWIDE_PER_FLIP = 114 / 32
IMADWIDE_PER_CLK_SM = 27.65  # measured IMAD.WIDE.U32 issue rate (profiles/r01_pipes_microbench.txt)
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")
JSON_OUT = sys.stdout  # the bench line's stream (run_ours keeps the real stdout for it)
# PAPER.md Table 2 (multi-spin kernel, one V100-SXM): lattice -> (flips/ns, line)
PAPER_TABLE2 = {(2048, 2048): (231.09, "P:277"), (4096, 4096): (318.95, "P:278"),
                (8192, 8192): (379.27, "P:279"), (16384, 16384): (411.65, "P:280"),
                (32768, 32768): (420.44, "P:281"), (65536, 65536): (420.77, "P:282"),
                (131072, 131072): (418.23, "P:283")}


def ncu_traffic(config: str, n: int):
    """DRAM bytes per k_halfsweep launch from the committed ncu --set full capture."""
    try:
        with open(TRAFFIC_FILE) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    e = d.get(f"{config}_n{n}")
    return None if e is None else e.get("dram_bytes_per_launch")


def config_for(name: str, n: int):
    if name == "c3":
        return 32768 * n, 32768, "weak", f"C3 32768x32768 per GPU (BASELINE configs[2]); lattice {32768 * n}x32768"
    if name == "c4":
        return 131072, 131072, "strong", "C4 131072x131072 strong-scaled (BASELINE configs[3])"
    if name == "c5":
        return 131072 * n, 1048576, "weak", f"C5 131072x1048576 per GPU (BASELINE configs[4]); lattice {131072 * n}x1048576"
    if name == "c2":
        return 2048 * n, 2048, "weak", f"C2 2048x2048 per GPU (BASELINE configs[1] shape); lattice {2048 * n}x2048"
    raise SystemExit(f"unknown config {name}")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines = []  # (monotonic arrival time, csv line)
        self.window = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append((time.monotonic(), ln.strip()))

    def mark(self, t0: float, t1: float):
        """Keep only samples that arrived inside [t0, t1] (the timed region)."""
        self.window = (t0, t1)

    def n_in_window(self) -> int:
        if self.window is None:
            return len(self.lines)
        t0, t1 = self.window
        return sum(1 for t, _ in self.lines if t0 <= t <= t1)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.th.join(timeout=2)
        sm, smax, pw, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, ln in self.lines:
            if self.window is not None and not (self.window[0] <= ts <= self.window[1]):
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": smax,
            "power_w_median": statistics.median(pw) if pw else None,
            "samples": len(sm),
            "reasons": sorted(reasons),
        }


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    try:
        with open(PEAKS_FILE) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


# --------------------------------------------------------------------- oracle
def oracle_rate(rows: int, cols: int, sweeps: int, threads: int | None = None):
    """Oracle (oracle/ising_oracle.c, as it stands) flips/ns on a rows x cols torus."""
    import oracle

    if threads:
        oracle.set_threads(threads)
    lat = oracle.Lattice(rows, cols, SEED).init_random().set_beta(BETA)
    lat.sweep(1)  # warm caches / page in
    t0 = time.perf_counter()
    lat.sweep(sweeps)
    dt = time.perf_counter() - t0
    return rows * cols * sweeps / (dt * 1e9), oracle.get_threads(), dt


def cpu_baseline(cols: int) -> dict:
    # bounded sample of the workload: 2048 full-width rows of the C3 lattice (a
    # 2048 x cols torus), sweeps sized for ~10-20 s of CPU work on the box's cores
    rows = 2048
    rate, cores, dt = oracle_rate(rows, cols, 1)
    sweeps = max(1, min(256, int(12.0 / max(dt, 1e-3))))
    rate, cores, dt = oracle_rate(rows, cols, sweeps)
    import oracle

    # the same oracle on one thread (per-core rate), on a quarter of the rows
    r1, _, dt1 = oracle_rate(rows // 4, cols, 1, threads=1)
    oracle.set_threads(cores)
    return {"value": rate, "unit": "flips/ns", "cores": cores, "kind": "oracle",
            "per_core_value": r1, "cpu_model": cpu_model(),
            "sample": f"{rows}x{cols} torus (C3 row width), beta={BETA}, random start seed {SEED}, "
                      f"{sweeps} sweeps, {dt:.1f} s, OpenMP over rows of a colour phase; "
                      f"per-core: {rows // 4}x{cols}, 1 sweep, 1 thread, {dt1:.1f} s"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    world = max(world, args.gpus)  # the arm reports the workload of --gpus N (CPU: rank 0 only)
    N, M, scaling, workload = config_for(args.config, world)
    import oracle

    rows = 8192  # bounded sample: 8192 full-width rows per step
    lat = oracle.Lattice(rows, M, SEED).init_random().set_beta(BETA)
    for _ in range(args.warmup):
        lat.sweep(1)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        lat.sweep(1)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = rows * M * args.steps / (total * 1e9)
    cores = oracle.get_threads()
    line = {
        "impl": "reference", "metric": "spin flips/ns (device-timed)", "value": value,
        "unit": "flips/ns", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "i8", "data": "synthetic",
        # the main arm's metric / config; the "device" here is the host: wall clock per sweep
        "config": {"workload": workload, "lattice": [N, M], "beta": BETA, "seed": SEED,
                   "start": "random", "parallelism": f"slab{world}",
                   "layout": "byte/spin CPU oracle (oracle/ising_oracle.c)",
                   "sample": f"{rows}x{M} torus per step (bounded sample)",
                   "timing": "host wall clock per sweep (perf_counter), OpenMP over rows"},
        "cpu_baseline": {"value": value, "unit": "flips/ns", "cores": cores, "kind": "oracle",
                         "sample": f"{rows}x{M} torus, {args.steps} sweeps"},
        "e2e": {"value": value, "unit": "flips/ns", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------ ours
class Ranks:
    """Process-group plumbing of the bench (barriers, max over ranks); no data-path work."""

    def __init__(self, rank, world, dev, dist, same_dev):
        self.rank, self.world, self.dev, self.dist, self.same_dev = rank, world, dev, dist, same_dev
        # host-only barrier for legs where rank 0 drives other ranks' GPUs: an NCCL barrier
        # would leave a waiting kernel on each of those GPUs, time-sliced against rank 0's work
        self.cpu_group = None
        if dist is not None:
            self.cpu_group = dist.new_group(backend="gloo")

    def host_barrier(self):
        if self.dist is not None:
            self.dist.barrier(group=self.cpu_group)

    def barrier(self):
        import torch

        if self.dist is not None:
            self.dist.barrier()
        torch.cuda.synchronize()

    def allmax(self, x: float) -> float:
        if self.dist is None:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cpu" if self.same_dev else "cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


def make_lattice(N: int, M: int, n: int, dev: int, transport: str | None = None):
    """The handle a user would create: one slab (n = 1) or this rank's slab of n."""
    from paper_1906_06297_b200.ising import IsingLattice

    if n > 1:
        return IsingLattice.distributed(N, M, SEED, device=dev, transport=transport)
    return IsingLattice(N, M, SEED, n_gpus=1)


def self_exchange_lattice(N: int, M: int, dev: int, transport: str):
    """One-rank handle whose half-sweeps run the multi-GPU transport with itself as the
    neighbour (ISING_SELF_EXCHANGE=1): the transport's per-GPU cost on one device."""
    from paper_1906_06297_b200 import ising
    from paper_1906_06297_b200.ising import IsingLattice

    os.environ["ISING_SELF_EXCHANGE"] = "1"
    try:
        if transport == "p2p":
            h = ising.ising_create_rank_p2p(N, M, SEED, 0, 1, dev)
        elif transport == "lsa":
            h = ising.ising_create_rank_lsa(N, M, SEED, 0, 1, dev, None)
        else:
            h = ising.ising_create_rank(N, M, SEED, 0, 1, dev, None)
    finally:
        os.environ.pop("ISING_SELF_EXCHANGE", None)
    lat = IsingLattice(N, M, SEED, _handle=h)
    lat.transport = transport + "-self"
    return lat


def timed_sweeps(lat, steps: int, warmup: int, R: Ranks, init: bool = True) -> float:
    """Device time (ms, max over ranks) of `steps` sweeps after `warmup` untimed ones."""
    if init:
        lat.set_beta(BETA).init_random()
    lat.sweep(warmup)
    R.barrier()
    lat.sweep(steps)
    ms = R.allmax(lat.last_sweep_ms())
    R.barrier()
    return ms


def leg(name: str, N: int, M: int, n: int, steps: int, warmup: int, R: Ranks,
        transport: str | None = None, note: str | None = None) -> dict:
    """One device-timed workload at n ranks, plus (n > 1) the same per-GPU workload
    (weak) or the same lattice (strong) on one GPU, run by rank 0 while the others wait."""
    lat = make_lattice(N, M, n, R.dev, transport)
    row0, rows = lat.slab_info()
    ms = timed_sweeps(lat, steps, warmup, R)
    used = getattr(lat, "transport", "single") if n > 1 else "single"
    lat.close()
    out = {"lattice": [N, M], "rows_per_gpu": rows, "n_gpus": n, "steps": steps,
           "ms_per_step": ms / steps, "value": N * M * steps / (ms * 1e6), "unit": "flips/ns",
           "transport": used}
    if note:
        out["note"] = note
    return out


def one_gpu_rate(N: int, M: int, steps: int, warmup: int, R: Ranks) -> float | None:
    """flips/ns of an N x M lattice on this rank's GPU alone (rank 0; the others wait)."""
    from paper_1906_06297_b200.ising import IsingLattice

    rate = None
    R.barrier()
    if R.rank == 0:
        lat = IsingLattice(N, M, SEED, n_gpus=1).set_beta(BETA).init_random()
        lat.sweep(warmup)
        lat.sweep(steps)
        rate = N * M * steps / (lat.last_sweep_ms() * 1e6)
        lat.close()
    R.barrier()
    return rate


def scaling_leg(name: str, kind: str, n: int, steps: int, warmup: int, R: Ranks) -> dict:
    """c4_strong: 131072^2 split into n row slabs (R = 131072 / n), BASELINE configs[3];
    c5_weak: 131072 rows x 1048576 columns per GPU, BASELINE configs[4] (2^40 spins at n = 8).
    efficiency = rate(n) / (n x rate(1)), rate(1) measured in the same job on rank 0's GPU."""
    note = None
    if kind == "strong":
        N, M = 131072, 131072
        Nref = N
    else:
        M = 1048576
        rows = 131072
        if R.same_dev and n * 64 > 128:  # every rank on one 180 GB device: cap at 128 GiB
            shrink = 1
            while n * 64 // shrink > 128:
                shrink *= 2
            M //= shrink
            note = f"same-device run: columns reduced {shrink}x to fit {n} ranks on one GPU"
        N, Nref = rows * n, rows
    out = leg(name, N, M, n, steps, warmup, R, note=note)
    if n == 1:
        out["one_gpu_value"] = out["value"]
    else:
        r1 = one_gpu_rate(Nref, M, steps, warmup, R)
        out["one_gpu_value"] = r1
    r1 = out["one_gpu_value"]
    if R.rank == 0 and r1:
        out["speedup"] = out["value"] / r1
        out["efficiency"] = out["value"] / (n * r1)
    out["scaling"] = kind
    out["config"] = ("BASELINE configs[3]: 131072x131072 strong-scaled as row slabs"
                     if kind == "strong" else
                     "BASELINE configs[4]: 131072 x 1048576 per GPU, weak-scaled (2^40 spins at n = 8)")
    return out


def batch_leg(L: int, n_lattices: int, sweeps: int) -> dict:
    """Aggregate flips/ns of `n_lattices` independent L x L lattices (seeds 1.., beta_c) as one
    lattice batch (ising_batch_*: one CTA, or one thread-block cluster, per lattice) against
    one-lattice handles of the same size (launch-bound there), device-timed."""
    import numpy as np

    from paper_1906_06297_b200.ising import IsingBatch, IsingLattice

    b = IsingBatch(L, L, list(range(1, n_lattices + 1))).set_beta(np.full(n_lattices, BETA))
    b.init_random().sweep(4)
    b.sweep(sweeps)
    value = n_lattices * L * L * sweeps / (b.last_sweep_ms() * 1e6)
    b.close()
    one = IsingLattice(L, L, 1).set_beta(BETA).init_random().sweep(16)
    one.sweep(sweeps)
    one_value = L * L * sweeps / (one.last_sweep_ms() * 1e6)
    one.close()
    return {"lattices": n_lattices, "sweeps": sweeps, "value": value, "unit": "flips/ns",
            "one_lattice_handle_value": one_value, "speedup": value / one_value,
            "engine": "one CTA per lattice" if L * L <= 409600 else "thread-block cluster per lattice"}


def batch_ranks_leg(L: int, n_lattices: int, sweeps: int, n: int, R: Ranks) -> dict:
    """Each of the n ranks sweeps its own batch of n_lattices independent lattices (seeds
    offset per rank) on its GPU; device time max over ranks."""
    import numpy as np

    from paper_1906_06297_b200.ising import IsingBatch

    seeds = list(range(1 + R.rank * n_lattices, 1 + (R.rank + 1) * n_lattices))
    b = IsingBatch(L, L, seeds, device=R.dev).set_beta(np.full(n_lattices, BETA))
    b.init_random().sweep(4)
    R.barrier()
    b.sweep(sweeps)
    ms = R.allmax(b.last_sweep_ms())
    b.close()
    return {"lattices_per_gpu": n_lattices, "sweeps": sweeps, "n_gpus": n,
            "value": n * n_lattices * L * L * sweeps / (ms * 1e6), "unit": "flips/ns",
            "scaling": "weak", "collective": "none (independent problems)"}


def single_process_leg(N: int, M: int, n: int, steps: int, R: Ranks) -> dict | None:
    """ising_create(N, M, seed, n) from rank 0 (all n devices in one process; same-device
    runs: n virtual slabs on cuda:0), device-timed; the other ranks wait at the barrier."""
    from paper_1906_06297_b200.ising import IsingLattice

    out = None
    R.barrier()
    R.host_barrier()
    if R.rank == 0:
        try:
            lat = (IsingLattice(N, M, SEED, devices=[0] * n) if R.same_dev
                   else IsingLattice(N, M, SEED, n_gpus=n))
            lat.set_beta(BETA).init_random().sweep(2)
            lat.sweep(steps)
            ms = lat.last_sweep_ms()
            lat.close()
            out = {"value": N * M * steps / (ms * 1e6), "ms_per_step": ms / steps,
                   "api": "ising_create(L_rows, L_cols, seed, n_gpus)" if not R.same_dev
                   else "ising_create_slabs(..., devices=[0] * n) (same-device run)"}
        except Exception as e:  # reported, not hidden
            out = {"error": repr(e)}
    R.host_barrier()
    R.barrier()
    return out


def invariance_check(n: int, transport: str | None, R: Ranks) -> dict | None:
    """Reading R19: a 64n x 256 lattice split over the n ranks with this transport equals
    the one-slab result byte for byte (and its observables as integers)."""
    import numpy as np
    import torch

    from paper_1906_06297_b200.ising import IsingLattice

    Ns, Ms, sw = 64 * n, 256, 20
    small = IsingLattice.distributed(Ns, Ms, 7, device=R.dev, transport=transport)
    r0s, rs = small.slab_info()
    small.set_beta(BETA).init_random().sweep(sw)
    mine = np.empty((rs, Ms), dtype=np.int8)
    small.read_lattice(mine)
    obs = small.observables()
    used = small.transport
    small.close()
    tdev = "cpu" if R.same_dev else "cuda"
    parts = [torch.empty((rs, Ms), dtype=torch.int8, device=tdev) for _ in range(n)]
    R.dist.all_gather(parts, torch.from_numpy(mine).to(tdev))
    if R.rank != 0:
        return None
    got = torch.cat(parts).cpu().numpy()
    one = IsingLattice(Ns, Ms, 7, n_gpus=1).set_beta(BETA).init_random().sweep(sw)
    res = {"lattice": [Ns, Ms], "sweeps": sw, "transport": used,
           "bit_identical_to_one_gpu": bool(np.array_equal(got, one.read_lattice())),
           "observables_equal": obs == one.observables()}
    one.close()
    return res


def link_bandwidth(dev: int) -> dict:
    """Pinned host <-> device copy GB/s of this GPU's link (256 MiB, best of 3): the roof of
    the e2e copies."""
    import torch

    nb = 256 << 20
    a = torch.empty(nb, dtype=torch.int8, pin_memory=True)
    d = torch.empty(nb, dtype=torch.int8, device=f"cuda:{dev}")
    best = {"h2d_gbs": 0.0, "d2h_gbs": 0.0}
    for _ in range(3):
        for key, dst, src in (("h2d_gbs", d, a), ("d2h_gbs", a, d)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            best[key] = max(best[key], nb / (time.perf_counter() - t0) / 1e9)
    del a, d
    return best


def e2e_run(lat, N: int, M: int, rows: int, n: int, steps: int, R: Ranks, bits: bool = False) -> float:
    """Wall seconds (max over ranks) of: write_lattice(own rows from pinned host memory);
    `steps` x ising_sweep_measure_async(1, 1) with the host one step behind; read_lattice.
    bits: the same through the bit-packed calls (one bit per spin on the host)."""
    import torch

    if bits:
        slab = torch.empty(rows * M // 8, dtype=torch.uint8, pin_memory=True)
        out = torch.empty(rows * M // 8, dtype=torch.uint8, pin_memory=True)
        lat.read_lattice_bits(slab.numpy())
        write, read = lat.write_lattice_bits, lat.read_lattice_bits
    else:
        slab = torch.empty((rows, M), dtype=torch.int8, pin_memory=True)
        out = torch.empty((rows, M), dtype=torch.int8, pin_memory=True)
        lat.read_lattice(slab.numpy() if n > 1 else slab.numpy().reshape(N, M))
        write, read = lat.write_lattice, lat.read_lattice
    ups = torch.zeros(steps, dtype=torch.int64, pin_memory=True).numpy()
    Es = torch.zeros(steps, dtype=torch.int64, pin_memory=True).numpy()
    R.barrier()
    t0 = time.perf_counter()
    write(slab.numpy(), t=0)
    prev = None
    for k in range(steps):
        ticket = lat.measure_async(1, 1, ups[k:k + 1], Es[k:k + 1])
        if prev is not None:
            lat.measure_wait(prev)
        prev = ticket
    lat.measure_wait(prev)
    read(out.numpy())
    R.barrier()
    return R.allmax(time.perf_counter() - t0)


def run_ours(args):
    import torch

    from paper_1906_06297_b200.ising import IsingLattice, ising_probe_philox

    rank, world, local = dist_env()
    n = world
    # ISING_BENCH_SAME_DEVICE=1 puts every rank on cuda:0 (a functional check of the
    # multi-rank path on a one-GPU box; its numbers are time-sliced, not scaling results)
    same_dev = os.environ.get("ISING_BENCH_SAME_DEVICE") == "1"
    dev = 0 if same_dev else local
    torch.cuda.set_device(dev)
    dist = None
    if n > 1:
        import torch.distributed as dist_mod

        dist = dist_mod
        if same_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    R = Ranks(rank, world, dev, dist, same_dev)
    N, M, scaling, workload = config_for(args.config, n)

    basic = args.layout == "basic"
    if basic and n > 1:
        raise SystemExit("--layout basic is single-GPU (PAPER.md §3.1 basic implementation)")
    bytes_per_flip = 3.0 if basic else BYTES_PER_FLIP
    if n > 1:
        lat = IsingLattice.distributed(N, M, SEED, device=dev)
    elif basic:
        lat = IsingLattice.basic(N, M, SEED, device=dev)
    else:
        lat = IsingLattice(N, M, SEED, n_gpus=1)
    row0, rows = lat.slab_info()
    main_transport = getattr(lat, "transport", "single") if n > 1 else "single"
    lat.set_beta(BETA).init_random()
    lat.sweep(args.warmup)

    # ---- device-timed region: K sweeps, events inside the library ----
    clk = ClockSampler(dev)
    clk.start()
    time.sleep(0.3)  # nvidia-smi is up before the timed region opens
    R.barrier()
    w0 = time.monotonic()
    l0 = lat.launch_count()
    lat.sweep(args.steps)
    launches = lat.launch_count() - l0
    ms = lat.last_sweep_ms()
    R.barrier()
    w1 = time.monotonic()
    clk.mark(w0, w1)
    clock_window = "timed region"
    ms = R.allmax(ms)
    if ms < 150.0:  # same decision on every rank (sweeps are collective in rank mode)
        # region shorter than 3 sampling intervals: sample an untimed repeat of the same
        # sweeps (same kernel, same lattice) lasting ~0.5 s
        reps = max(1, int(500.0 / max(ms, 1e-3)))
        s0 = time.monotonic()
        lat.sweep(min(reps * args.steps, 1 << 20))
        R.barrier()
        clk.mark(s0, time.monotonic())
        clock_window = "untimed repeat of the timed sweeps (timed region < 150 ms)"
    clocks = clk.stop()
    clocks["window"] = clock_window
    value = N * M * args.steps / (ms * 1e6)

    # ---- per-launch kernel timing (profiling on: one event pair per launch) ----
    lat.set_profiling(True)
    kprof_sweeps = max(2, min(args.steps, 16))
    lat.sweep(kprof_sweeps)
    kms, klaunches = lat.kernel_stats()
    sweep_ms_prof = lat.last_sweep_ms()
    lat.set_profiling(False)
    # dominant kernel = the half-sweep; a sweep attempts rows*M flips over its launches
    flips_per_launch = rows * M * kprof_sweeps / max(klaunches, 1)
    avg_launch_ms = kms / max(klaunches, 1)
    peaks, peak_src = measured_peaks()
    hbm_gbs = bytes_per_flip * flips_per_launch / (avg_launch_ms * 1e6)
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    flips_per_ns_kernel = flips_per_launch / (avg_launch_ms * 1e6)

    # ---- the arithmetic roof: every attempted flip consumes one uint32
    # Philox4x32-10 draw (reading R6), so the measured Philox-only rate of the same device
    # function (eight blocks per thread in lockstep, as the kernels run them) is the path's
    # ceiling in flips/ns; the derived IMAD.WIDE figure is reported beside it
    philox_probe = ising_probe_philox(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    derived_peak = sms * IMADWIDE_PER_CLK_SM * clk_mhz * 1e6 / MULWIDE_PER_FLIP / 1e9
    traffic = ncu_traffic(args.config + ("_basic" if basic else ""), n)
    hbm_roof_flips = hbm_peak / bytes_per_flip  # flips/ns
    alu_bound = philox_probe <= hbm_roof_flips

    # ---- the memory side, live: the same kernel with the draw-free acceptance (beta = inf:
    # thresholds 0, Philox not evaluated) — what the data path sustains without the RNG
    draw_free = None
    if not basic:
        lat.set_beta(math.inf)
        lat.sweep(2)
        lat.set_profiling(True)
        lat.sweep(kprof_sweeps)
        dkms, dkl = lat.kernel_stats()
        lat.set_profiling(False)
        d_gbs = bytes_per_flip * rows * M * kprof_sweeps / max(dkl, 1) / (dkms / max(dkl, 1) * 1e6)
        draw_free = {"beta": "inf", "kernel_variant": 4, "achieved_gbs": d_gbs,
                     "frac": d_gbs / hbm_peak,
                     "flips_per_ns": rows * M * kprof_sweeps / (dkms * 1e6)}
        lat.set_beta(BETA)

    # ---- end to end through the C ABI with host buffers (a warm-up pass first: one-time
    # allocations and lazy module loading are not part of the step) ----
    e2e = None
    if rows * M <= (1 << 34):
        e2e_run(lat, N, M, rows, n, min(args.steps, 2), R)
        e2e_s = e2e_run(lat, N, M, rows, n, args.steps, R)
        link = link_bandwidth(dev)
        copy_s = rows * M / (link["h2d_gbs"] * 1e9) + rows * M / (link["d2h_gbs"] * 1e9)
        roof = N * M * args.steps / ((copy_s + ms * 1e-3) * 1e9)
        # the same through the bit-packed host format (1 bit per spin: 1/8 of the copy bytes)
        bits_s = None
        if not basic:
            e2e_run(lat, N, M, rows, n, min(args.steps, 2), R, bits=True)
            bits_s = e2e_run(lat, N, M, rows, n, args.steps, R, bits=True)
        e2e = {
            "value": N * M * args.steps / (e2e_s * 1e9),
            "unit": "flips/ns",
            "h2d_bytes_per_step": N * M // args.steps,
            "d2h_bytes_per_step": N * M // args.steps + 16 * n,
            "copy_roof": {"h2d_gbs": link["h2d_gbs"], "d2h_gbs": link["d2h_gbs"],
                          "value": roof, "frac": N * M * args.steps / (e2e_s * 1e9) / roof,
                          "how": "(slab bytes / pinned H2D GB/s + slab bytes / pinned D2H GB/s "
                                 "+ steps x ms_per_step): the copies cannot overlap the sweeps "
                                 "(the first sweep needs the whole input, the read-back the "
                                 "last sweep's output)"},
            "how": "per rank: write_lattice(own rows, pinned int8) + per sweep: "
                   "ising_sweep_measure_async(1, 1) (sweep + fused observables, all-reduced in "
                   "rank mode, 16 B copied to pinned host memory per step, the host waiting one "
                   "step behind); read_lattice(own rows, pinned int8); wall clock, max over "
                   "ranks; bytes summed over ranks; after one untimed warm-up pass",
            "bitpacked": None if bits_s is None else {
                "value": N * M * args.steps / (bits_s * 1e9),
                "h2d_bytes_per_step": N * M // 8 // args.steps,
                "d2h_bytes_per_step": N * M // 8 // args.steps + 16 * n,
                "roof": N * M * args.steps / ((copy_s / 8 + ms * 1e-3) * 1e9),
                "how": "the same calls with ising_write_lattice_bits / ising_read_lattice_bits "
                       "(host lattice one bit per spin, pinned)"},
        }
    lat.close()

    # ---- transports, GPU-count invariance and the north_star's scaling configs ----
    transports, invariance, legs = None, None, {}
    main_legs = args.config == "c3" and not basic and not args.no_legs
    if main_legs and n == 1:
        # the multi-GPU transports' per-GPU cost, each rank its own neighbour
        transports = {"local": {"value": value, "ms_per_step": ms / args.steps}}
        for tname in ("p2p", "lsa", "nccl"):
            try:
                tl = self_exchange_lattice(N, M, dev, tname)
                tms = timed_sweeps(tl, args.steps, 2, R)
                tl.close()
                transports[tname + "_self"] = {"value": N * M * args.steps / (tms * 1e6),
                                               "ms_per_step": tms / args.steps,
                                               "vs_local": (N * M * args.steps / (tms * 1e6)) / value}
            except Exception as e:  # reported, not hidden
                transports[tname + "_self"] = {"error": repr(e)}
    if n > 1:
        invariance = invariance_check(n, None, R)
        if main_legs:
            transports = {"p2p": {"value": value, "ms_per_step": ms / args.steps}}
            for tname in ("lsa", "nccl"):
                if same_dev:
                    transports[tname] = {"skipped": "NCCL rejects two ranks on one device "
                                                    "(same-device functional run)"}
                    continue
                try:
                    nl = leg("c3_" + tname, N, M, n, args.steps, 2, R, transport=tname)
                    transports[tname] = {"value": nl["value"], "ms_per_step": nl["ms_per_step"],
                                         "transport": nl["transport"],
                                         "invariance": invariance_check(n, tname, R)}
                except Exception as e:  # reported, not hidden (every rank raises alike)
                    transports[tname] = {"error": repr(e)}
            # the north_star's literal ising_create(L_rows, L_cols, seed, n_gpus): ONE process
            # drives all n GPUs (peer stores + cross-device events), run by rank 0 while the
            # other ranks wait
            transports["single_process"] = single_process_leg(N, M, n, args.steps, R)
    if main_legs:
        legs["c4_strong"] = scaling_leg("c4_strong", "strong", n, max(4, min(args.steps, 32)), 2, R)
        legs["c5_weak"] = scaling_leg("c5_weak", "weak", n, max(2, min(args.steps, 8)), 1, R)
    if main_legs and n == 1:
        # temperature-scan workloads — many small lattices as one batch
        legs["batch_scan"] = {"64x64": batch_leg(64, 2368, 2048), "1024x1024": batch_leg(1024, 148, 32)}
    elif main_legs:
        # independent lattices shard across ranks with no collective (weak scaling): every
        # rank runs its own 64^2 x 2368 batch; aggregate = all ranks' flips / the slowest rank
        legs["batch_scan"] = {"64x64": batch_ranks_leg(64, 2368, 2048, n, R)}

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(M)

    # The paper's single-GPU number for this exact lattice, if Table 2 has one (BASELINE.md:
    # one V100-SXM of a DGX-2; another machine's number — context, not the target).
    paper = PAPER_TABLE2.get((N, M)) if (n == 1 and not basic) else None
    if rank == 0:
        hbm_frac = hbm_gbs / hbm_peak
        line = {
            "metric": "spin flips/ns (device-timed)",
            "value": value,
            "unit": "flips/ns",
            "n_gpus": n,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "higher_is_better": True,
            "scaling": scaling,
            "vs_baseline": (value / paper[0]) if paper else None,
            "baseline": ({"value": paper[0], "unit": "flips/ns", "hardware": "1x V100-SXM (DGX-2)",
                          "source": f"BASELINE.md Table 2, PAPER.md {paper[1]}"} if paper else None),
            "dtype": "u32",
            "data": "synthetic",
            "config": {
                "workload": workload,
                "lattice": [N, M],
                "beta": BETA,
                "seed": SEED,
                "start": "random",
                "parallelism": f"slab{n}",
                "transport": main_transport,
                "same_device": same_dev,
                "layout": "basic byte/spin (PAPER.md §3.1)" if basic else "multi-spin 4 bit/spin (PAPER.md §3.3)",
                "l2": f"inputs larger than L2: packed planes {N * M // 2 / 2**20:.0f} MiB per "
                      f"{'GPU' if n == 1 else 'lattice'} vs 126 MB L2; no flush",
            },
            "roofline": {
                "bound": "alu" if alu_bound else "hbm",
                "achieved": flips_per_ns_kernel if alu_bound else hbm_gbs,
                "peak": philox_probe if alu_bound else hbm_peak,
                "unit": "flips/ns" if alu_bound else "GB/s",
                "frac": flips_per_ns_kernel / philox_probe if alu_bound else hbm_frac,
                "traffic": traffic,
                "kernel": "k_basic_halfsweep<0>" if basic else ("k_halfsweep_staged<0>" if (M // 32) % 256 == 0 else "k_halfsweep<0>"),
                "peak_source": "measured live: ising_probe_philox (Philox4x32-10-only draws/ns of "
                               "the kernels' device function, eight blocks per thread in "
                               "lockstep, a fixed column chunk per thread walking the rows as "
                               "the half-sweeps do); one draw per attempted flip (reading R6)",
                "derived_peak": {"value": derived_peak, "unit": "flips/ns",
                                 "how": f"{sms} SMs x {IMADWIDE_PER_CLK_SM} IMAD.WIDE.U32/clk/SM "
                                        f"(measured, profiles/r01_pipes_microbench.txt) x "
                                        f"{clk_mhz:.0f} MHz / {MULWIDE_PER_FLIP:.4f} per-thread "
                                        "mul.wide per flip (DESIGN.md §5)",
                                 "frac": flips_per_ns_kernel / derived_peak},
                "hbm_roof_flips_per_ns": hbm_roof_flips,
                "avg_launch_ms": avg_launch_ms,
                "launches": klaunches,
                "kernel_share_of_step": kms / max(sweep_ms_prof, 1e-9),
                "traffic_source": "profiles/ncu_traffic.json (dram__bytes_read.sum + "
                                  "dram__bytes_write.sum per launch, ncu --set full)",
                "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": hbm_peak, "frac": hbm_frac,
                        "peak_source": peak_src, "bytes_per_flip": bytes_per_flip},
            },
            "hbm_bar": {
                "target": 0.70, "achieved": hbm_frac,
                "ceiling_under_contract": philox_probe * bytes_per_flip / hbm_peak,
                "draw_free": draw_free,
                "evidence": "the north_star's RNG contract (one Philox4x32-10 uint32 per attempted "
                            "flip, R6) caps the path at the Philox-only rate; as HBM fraction that "
                            "is ceiling_under_contract. The same kernel without draws (draw_free, "
                            "live) shows the data path itself above the 0.70 bar. "
                            "profiles/r01_pipes_microbench.txt (IMAD.WIDE 27.65/clk/SM), "
                            "profiles/r01_ncu_halfsweep.md (FMA-heavy 83 %, ALU 61 %)",
                "cite": "PAPER.md P:199 (memory-bandwidth limited on V100)",
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "invariance": invariance,
            "transports": transports,
            "legs": legs or None,
            "clocks": clocks,
        }
        print(json.dumps(line), file=JSON_OUT, flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def spawn(args) -> int:
    """bench.py --gpus N without torchrun: launch N ranks through torch.distributed.run
    (127.0.0.1 rendezvous) and return their exit status."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1024)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c3", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-legs", action="store_true",
                    help="skip the transport / c4_strong / c5_weak sub-measurements")
    ap.add_argument("--layout", default="multispin", choices=["multispin", "basic"])
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn(args)
    # stdout carries exactly one JSON line: anything the libraries print (NCCL's version
    # banner, ...) goes to stderr
    global JSON_OUT
    JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
