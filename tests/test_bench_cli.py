"""bench.py's launch contract on CPU (no GPU needed): a WORLD_SIZE that disagrees with --gpus
is an error (never a silent one-GPU run), and the reference arm (the CPU oracle) prints exactly
one JSON line carrying the requested n_gpus and its cpu_baseline / e2e objects."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None, timeout=300):
    e = dict(os.environ, **(env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], env=e,
                          capture_output=True, text=True, timeout=timeout)


def test_world_size_mismatch_is_an_error():
    out = run(["--gpus", "2", "--steps", "1", "--warmup", "3"],
              env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode == 2, (out.returncode, out.stderr[-500:])
    assert "WORLD_SIZE" in out.stderr


def test_warmup_below_three_is_rejected():
    out = run(["--steps", "1", "--warmup", "2"])
    assert out.returncode != 0 and "warmup" in out.stderr


def test_reference_arm_prints_one_json_line():
    out = run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["unit"] == "flips/ns"
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
