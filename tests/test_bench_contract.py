"""bench.py's driver contract, on CPU: the reference arm's JSON line (the
reference algorithm timed on the host cores, c1 so it finishes in seconds),
the N > 1 behaviour of that arm (rank 0 alone prints, other ranks exit 0
without work), and our arm failing loudly — never falling back to the CPU —
when there is no GPU."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=300):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          cwd=ROOT, env=e, capture_output=True, text=True,
                          timeout=timeout)


def test_reference_arm_line():
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["impl"] == "reference"
    assert j["metric"] == "train samples/s" and j["unit"] == "samples/s"
    assert j["value"] > 0 and j["higher_is_better"] is True
    assert j["n_gpus"] == 1 and j["steps"] == 2
    assert j["warmup"] >= 3                      # W >= 3 is enforced
    assert j["config"]["global_batch"] == 128
    cb = j["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == j["value"]
    assert j["e2e"] == {"value": j["value"], "unit": "samples/s",
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--gpus", "2"],
             env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"}, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""


def test_world_size_must_match_gpus():
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--gpus", "4"],
             env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"}, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_gpus_n_launches_n_ranks_itself():
    """`bench.py --gpus 2` (no WORLD_SIZE) re-launches itself under
    torch.distributed.run: two ranks, rank 0 alone prints the line."""
    e = {k: v for k, v in os.environ.items()
         if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "c1", "--steps", "2", "--warmup", "1", "--gpus", "2"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["impl"] == "reference"


def test_our_arm_needs_the_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: the arm runs for real (bench runs cover it)")
    r = _run(["--config", "c1", "--steps", "3", "--no-cpu-baseline"], timeout=300)
    assert r.returncode != 0
    assert r.stdout.strip() == ""                # no JSON line from a CPU path
