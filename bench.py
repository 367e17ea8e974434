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
MULWIDE_PER_FLIP = 4.0  # per-thread 32x32->64 multiplies per draw (16 per Philox block / 4, R6)
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")
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
def run_ours(args):
    import numpy as np
    import torch

    from paper_1906_06297_b200.ising import IsingLattice, ising_probe_philox

    rank, world, local = dist_env()
    assert world == args.gpus or world == 1, "launch N>1 with torch.distributed.run"
    n = world
    # ISING_BENCH_SAME_DEVICE=1 puts every rank on cuda:0 (a functional check of the
    # multi-rank path on a one-GPU box; its numbers are not scaling results)
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
    N, M, scaling, workload = config_for(args.config, n)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if same_dev else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

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
    lat.set_beta(BETA).init_random()
    lat.sweep(args.warmup)

    # ---- device-timed region: K sweeps, events inside the library ----
    clk = ClockSampler(dev)
    clk.start()
    time.sleep(0.3)  # nvidia-smi is up before the timed region opens
    barrier()
    w0 = time.monotonic()
    l0 = lat.launch_count()
    lat.sweep(args.steps)
    launches = lat.launch_count() - l0
    ms = lat.last_sweep_ms()
    barrier()
    w1 = time.monotonic()
    clk.mark(w0, w1)
    clock_window = "timed region"
    ms = allmax(ms)
    if ms < 150.0:  # same decision on every rank (sweeps are collective in rank mode)
        # region shorter than 3 sampling intervals: sample an untimed repeat of the same
        # sweeps (same kernel, same lattice) lasting ~0.5 s
        reps = max(1, int(500.0 / max(ms, 1e-3)))
        s0 = time.monotonic()
        lat.sweep(min(reps * args.steps, 1 << 20))
        barrier()
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
    # dominant kernel = k_halfsweep; a sweep attempts rows*M flips over its launches
    # (2 per sweep for one slab: rows*M/2 flips each)
    flips_per_launch = rows * M * kprof_sweeps / max(klaunches, 1)
    avg_launch_ms = kms / max(klaunches, 1)
    peaks, peak_src = measured_peaks()
    hbm_gbs = bytes_per_flip * flips_per_launch / (avg_launch_ms * 1e6)

    # ---- ALU roofline: the Philox multiplier.  Every attempted flip needs
    # one draw = 1/4 Philox4x32-10 block = 4 per-thread 32x32->64 multiplies (16 of the 20
    # per block; 4 are warp-uniform under reading R6's counter {t, j/4, c, i}).  IMAD.WIDE.U32 issues on the 16-lane
    # FMA-heavy pipe of each SMSP in two passes: 8 lanes/clk/SMSP = 32 per SM per clock.
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    alu_peak = sms * 32 * clk_mhz * 1e6 / MULWIDE_PER_FLIP / 1e9  # flips/ns
    philox_probe = ising_probe_philox(dev)  # Philox-only draws/ns, same device function
    flips_per_ns_kernel = flips_per_launch / (avg_launch_ms * 1e6)
    traffic = ncu_traffic(args.config + ("_basic" if basic else ""), n)
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_roof_flips = hbm_peak / bytes_per_flip  # flips/ns
    alu_bound = alu_peak <= hbm_roof_flips

    # ---- end to end through the C ABI with host buffers ----
    # Each rank owns its rows: the input is this rank's slab (rows x M int8, pinned host
    # memory; rank mode exchanges the halo rows on the device), the per-step result the
    # global observables (16 B), and the final lattice rows come back to pinned memory.
    e2e = None
    if rows * M <= (1 << 34):
        slab = torch.empty((rows, M), dtype=torch.int8, pin_memory=True)
        if n > 1:
            lat.read_lattice(slab.numpy())
        else:
            lat.read_lattice(slab.numpy().reshape(N, M))
        out = torch.empty((rows, M), dtype=torch.int8, pin_memory=True)
        barrier()
        t0 = time.perf_counter()
        lat.write_lattice(slab.numpy(), t=0)
        # one sweep per step with its observables fused into the white phase, copied to
        # pinned host memory every step (ising_sweep_measure_async) and read by the host one
        # step behind: step k + 1 is enqueued before the host waits for step k's result
        ups = torch.zeros(args.steps, dtype=torch.int64, pin_memory=True).numpy()
        Es = torch.zeros(args.steps, dtype=torch.int64, pin_memory=True).numpy()
        prev = None
        for k in range(args.steps):
            ticket = lat.measure_async(1, 1, ups[k:k + 1], Es[k:k + 1])
            if prev is not None:
                lat.measure_wait(prev)
            prev = ticket
        lat.measure_wait(prev)
        lat.read_lattice(out.numpy())
        barrier()
        e2e_s = allmax(time.perf_counter() - t0)
        e2e = {
            "value": N * M * args.steps / (e2e_s * 1e9),
            "unit": "flips/ns",
            "h2d_bytes_per_step": N * M // args.steps,
            "d2h_bytes_per_step": N * M // args.steps + 16 * n,
            "how": "per rank: write_lattice(own rows, pinned int8) + per sweep: "
                   "ising_sweep_measure_async(1, 1) (sweep + fused observables, all-reduced in "
                   "rank mode, 16 B copied to pinned host memory per step, the host waiting one "
                   "step behind); read_lattice(own rows, pinned int8); wall clock, max over "
                   "ranks; bytes summed over ranks",
        }
        del slab, out

    # ---- GPU-count invariance (reading R19): a small lattice split over the n ranks with
    # the same transport must equal the one-slab result byte for byte ----
    invariance = None
    if n > 1:
        import numpy as np

        Ns, Ms, sw = 64 * n, 256, 20
        small = IsingLattice.distributed(Ns, Ms, 7, device=dev)
        r0s, rs = small.slab_info()
        small.set_beta(BETA).init_random().sweep(sw)
        mine = np.empty((rs, Ms), dtype=np.int8)
        small.read_lattice(mine)
        obs = small.observables()
        small.close()
        tdev = "cpu" if same_dev else "cuda"
        parts = [torch.empty((rs, Ms), dtype=torch.int8, device=tdev) for _ in range(n)]
        dist.all_gather(parts, torch.from_numpy(mine).to(tdev))
        if rank == 0:
            got = torch.cat(parts).cpu().numpy()
            one = IsingLattice(Ns, Ms, 7, n_gpus=1).set_beta(BETA).init_random().sweep(sw)
            invariance = {"lattice": [Ns, Ms], "sweeps": sw,
                          "bit_identical_to_one_gpu": bool(np.array_equal(got, one.read_lattice())),
                          "observables_equal": obs == one.observables()}
            one.close()

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(M)

    # The paper's single-GPU number for this exact lattice, if Table 2 has one (BASELINE.md:
    # one V100-SXM of a DGX-2; another machine's number — context, not the target).
    paper = PAPER_TABLE2.get((N, M)) if (n == 1 and not basic) else None
    if rank == 0:
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
                "transport": getattr(lat, "transport", "single") if n > 1 else "single",
                "layout": "basic byte/spin (PAPER.md §3.1)" if basic else "multi-spin 4 bit/spin (PAPER.md §3.3)",
                "l2": f"inputs larger than L2: packed planes {N * M // 2 / 2**20:.0f} MiB per "
                      f"{'GPU' if n == 1 else 'lattice'} vs 126 MB L2; no flush",
            },
            "roofline": {
                "bound": "alu" if alu_bound else "hbm",
                "achieved": flips_per_ns_kernel if alu_bound else hbm_gbs,
                "peak": alu_peak if alu_bound else hbm_peak,
                "unit": "flips/ns" if alu_bound else "GB/s",
                "frac": flips_per_ns_kernel / alu_peak if alu_bound else hbm_gbs / hbm_peak,
                "traffic": traffic,
                "kernel": "k_basic_halfsweep<0>" if basic else ("k_halfsweep_staged<0>" if (M // 32) % 256 == 0 else "k_halfsweep<0>"),
                "alu_roof_flips_per_ns": alu_peak,
                "hbm_roof_flips_per_ns": hbm_roof_flips,
                "avg_launch_ms": avg_launch_ms,
                "launches": klaunches,
                "kernel_share_of_step": kms / max(sweep_ms_prof, 1e-9),
                "peak_source": f"derived: {sms} SMs x 32 IMAD.WIDE.U32/clk/SM x {clk_mhz:.0f} MHz "
                               f"(median SM clock in the timed region) / {MULWIDE_PER_FLIP} varying "
                               "mul.wide per attempted flip (DESIGN.md §5)",
                "philox_only_probe": {"value": philox_probe, "unit": "draws/ns",
                                      "frac": flips_per_ns_kernel / philox_probe},
                "traffic_source": "profiles/ncu_traffic.json (dram__bytes_read.sum + "
                                  "dram__bytes_write.sum per launch, ncu --set full)",
                "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": peaks.get("hbm_gbs"),
                        "frac": hbm_gbs / peaks.get("hbm_gbs", 6650.0), "peak_source": peak_src,
                        "bytes_per_flip": bytes_per_flip},
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "invariance": invariance,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    lat.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1024)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c3", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layout", default="multispin", choices=["multispin", "basic"])
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
