"""bench.py's launch contract on a host without GPUs (CPU tests):

* ``--gpus N`` outside torchrun spawns N ranks, and refuses (exit 2) when
  fewer than N GPUs are visible instead of measuring fewer;
* a rank whose WORLD_SIZE differs from ``--gpus`` refuses to measure;
* the reference arm under a 2-rank torchrun: rank 0 alone prints one JSON
  line, with the steps / warm-up it was asked for and the same ``config``
  dict as our arm (bench.workload_config).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _env(**kw):
    e = {k: v for k, v in os.environ.items()
         if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    e.update({k: str(v) for k, v in kw.items()})
    return e


def test_gpus_without_devices_refuses():
    p = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, env=_env(CUDA_VISIBLE_DEVICES=""))
    assert p.returncode == 2, (p.returncode, p.stdout, p.stderr)
    assert "refusing" in p.stderr
    assert p.stdout.strip() == ""


def test_world_size_mismatch_refuses():
    p = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300,
                       env=_env(WORLD_SIZE=1, RANK=0, LOCAL_RANK=0, CUDA_VISIBLE_DEVICES=""))
    assert p.returncode != 0
    assert "WORLD_SIZE=1" in p.stderr
    assert p.stdout.strip() == ""


def test_reference_arm_two_ranks_one_line_same_config():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
           "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port", "29641",
           BENCH, "--impl", "reference", "--gpus", "2", "--cg-n", "1024", "--steps", "4",
           "--warmup", "5"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=_env())
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 4 and d["warmup"] == 5
    assert d["n_gpus"] == 2 and d["e2e"]["h2d_bytes_per_step"] == 0
    sys.path.insert(0, ROOT)
    import argparse

    import bench
    want = bench.workload_config(argparse.Namespace(n=1024, b=128), 2)
    assert d["config"] == want
    assert d["cpu_baseline"]["kind"] in ("reference", "port")


def test_stdout_is_exactly_one_json_line():
    """stdout carries the JSON line only: native writes to fd 1 (NCCL's
    version / INIT lines) are pointed at stderr by bench.py."""
    p = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--cg-n", "1024",
                        "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, env=_env())
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 2
