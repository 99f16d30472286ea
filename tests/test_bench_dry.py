"""bench.py's multi-rank plumbing on CPU: ``--gpus 2 --dry`` must re-launch
itself under torch.distributed.run with two gloo ranks, and rank 0 alone
prints one JSON line that reports n_gpus = 2 (the real N-rank group)."""

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


def test_bench_dry_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, os.path.join(HERE, "bench.py"), "--dry", "--gpus", "2",
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                         timeout=240, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = _json_lines(res.stdout)
    assert len(lines) == 1, res.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["dry"] is True
    assert sum(line["directions_per_rank"]) == 16 and len(line["directions_per_rank"]) == 2


def test_bench_dry_one_rank():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, os.path.join(HERE, "bench.py"), "--dry", "--steps", "2"],
                         capture_output=True, text=True, timeout=120, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    (line,) = _json_lines(res.stdout)
    assert line["n_gpus"] == 1
