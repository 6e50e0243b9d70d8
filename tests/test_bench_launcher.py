"""bench.py --gpus N launches N ranks itself (driver contract: `python
bench.py --gpus N` without torchrun must run N processes), and refuses a
WORLD_SIZE that disagrees with --gpus.  CPU only: --launch-check exercises the
rank plumbing over gloo without GPU work."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=240)


def test_gpus_two_spawns_two_ranks():
    p = _run(["--gpus", "2", "--launch-check"])
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["ranks_sum"] == 3


def test_single_gpu_does_not_spawn():
    p = _run(["--launch-check"])
    assert p.returncode == 0, p.stderr[-2000:]
    assert json.loads(p.stdout.strip().splitlines()[-1])["n_gpus"] == 1
    assert "launching" not in p.stderr


def test_world_size_must_match_gpus():
    p = _run(["--gpus", "4", "--launch-check"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode == 2
    assert "WORLD_SIZE=2" in p.stderr
