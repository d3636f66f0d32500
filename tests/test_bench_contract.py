"""bench.py contract pieces that run without a GPU: the reference arm (the
CPU port on the host cores) prints one well-formed JSON line, and the
roofline arithmetic follows SURVEY.md 8(d)."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_prints_one_json_line(oracle):
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
         "--warmup", "0", "--cycles", "50", "--cpu-sample-trials", "2"],
        capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["unit"] == "updates/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"] == {"value": d["value"], "unit": "updates/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["graph"] == "G81" and d["config"]["trials"] == 4096


def test_algorithmic_bytes_per_update_matches_survey():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2601_14476_b200 import benchmarks
    # G1 52.25, G22 22.44, G55 6.46, G81 5.39 bytes/update
    for name, want in (("G1", 52.25), ("G22", 22.44), ("G55", 6.46), ("G81", 5.39)):
        g = benchmarks.load(name)[0]
        assert bench.algorithmic_bytes_per_update(g) == pytest.approx(want, abs=0.01)


def test_reference_arm_under_torchrun_prints_once_from_rank_zero(oracle):
    """Under torchrun (N > 1) rank 0 alone runs the CPU reference and prints its
    line; the other ranks exit 0 without work."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
         "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--cycles", "20",
         "--cpu-sample-trials", "2"],
        capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_reference_arm_gpus_flag_without_torchrun_reports_the_job_size(oracle):
    """`bench.py --impl reference --gpus 2` outside torchrun: the reference arm
    is the host-core CPU path, run once, reported for the 2-GPU job."""
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
         "--steps", "1", "--warmup", "0", "--cycles", "20", "--cpu-sample-trials", "2"],
        capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2


def test_gpu_arm_fails_loudly_without_enough_gpus():
    """`bench.py --gpus 2` re-launches itself under torch.distributed.run with
    one rank per GPU; with fewer visible GPUs (none here) it exits nonzero
    with a clear message instead of reporting a 1-GPU job."""
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "0"],
        capture_output=True, text=True, timeout=300, cwd=str(ROOT),
        env={**__import__("os").environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 2
    assert "needs 2 visible GPUs" in out.stderr
    assert not [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
