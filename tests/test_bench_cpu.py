"""bench.py launch contract on CPU: `--gpus N` without torchrun re-launches
itself as N ranks (one process per GPU) and rank 0 reports the world size."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_flag_spawns_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=240, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["rank"] == 0
    assert "torch.distributed.run" in out.stderr


def test_single_gpu_default_has_no_spawn():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run"],
                         capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode == 0
    assert json.loads(out.stdout.strip())["n_gpus"] == 1
    assert "spawning" not in out.stderr
