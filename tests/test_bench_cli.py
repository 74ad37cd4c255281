"""bench.py's reference arm runs on the CPU and prints one well-formed JSON line (no GPU)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def test_reference_arm_json_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "M1", "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.5"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "GB/s" and line["value"] > 0
    # the oracle runs on all host cores (one tensor per worker process)
    assert line["cpu_baseline"]["kind"] == "oracle"
    assert line["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["higher_is_better"] is True
    for key in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "scaling", "vs_baseline",
                "dtype", "data", "config"):
        assert key in line


def test_gpus_flag_launches_ranks():
    """--gpus N with no WORLD_SIZE re-execs under torch.distributed.run (N ranks on
    127.0.0.1); the reference arm then prints one line from rank 0 with n_gpus == N."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "M1", "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.5"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "launching 2 ranks" in r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2


def test_world_size_mismatch_fails():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0", CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "1",
                        "--config", "M1", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode != 0
    assert "WORLD_SIZE=2 but --gpus 1" in r.stderr


def test_partition_resolution():
    """--partition auto: contiguous ranges up to 2 GPUs (they balance exactly there), LPT
    from 4 with the NVLink (record-granular) or no assembly; explicit LPT needs one of those."""
    sys.path.insert(0, str(ROOT))
    import bench
    assert bench.resolve_partition("auto", 1, "nvlink") == "contiguous"
    assert bench.resolve_partition("auto", 2, "nvlink") == "contiguous"
    assert bench.resolve_partition("auto", 4, "nvlink") == "lpt"
    assert bench.resolve_partition("auto", 8, "none") == "lpt"
    assert bench.resolve_partition("auto", 8, "fused") == "contiguous"
    assert bench.resolve_partition("contiguous", 8, "nvlink") == "contiguous"
    assert bench.resolve_partition("lpt", 1, "fused") == "lpt"
    with pytest.raises(SystemExit):
        bench.resolve_partition("lpt", 4, "nccl")
