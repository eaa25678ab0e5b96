"""`bench.py --gpus N` run outside torchrun launches its N replica ranks itself (one process per
GPU, torch.distributed on 127.0.0.1) and reports n_gpus = the ranks actually launched; rank 0
alone prints the line. Exercised on CPU with the gloo backend through the reference (CPU) arm."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_bench_self_launches_replicas():
    env = dict(os.environ, BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
                          "--warmup", "0", "--shape", "tiny-c1", "--agents", "2"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
    assert "launching 2 replica ranks" in out.stderr


def test_bench_refuses_rank_mismatch():
    env = dict(os.environ, BENCH_BACKEND="gloo", WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
                          "--warmup", "0", "--shape", "tiny-c1"], capture_output=True, text=True, timeout=300,
                         env=env, cwd=ROOT)
    assert out.returncode == 2 and "refusing" in out.stderr
