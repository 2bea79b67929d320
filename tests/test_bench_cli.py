"""bench.py's launcher logic on the CPU: `--gpus N` without a torchrun
environment re-launches itself under torch.distributed.run with N ranks
(127.0.0.1 rendezvous) and rank 0 prints exactly one JSON line.  The
reference arm (`--impl reference`, the CPU oracle on a small R-MAT) needs no
GPU, so the whole spawn -> rank check -> print path runs here."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _run(args, env_extra=None):
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py")] + args, capture_output=True, text=True,
                          timeout=600, env=env, cwd=str(ROOT))


def _lines(out: str):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


def test_spawn_two_ranks_reference_arm():
    r = _run(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "0", "--nnz", "200000"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1, r.stdout
    ln = lines[0]
    assert ln["impl"] == "reference" and ln["n_gpus"] == 2
    assert ln["e2e"]["h2d_bytes_per_step"] == 0 and ln["cpu_baseline"]["kind"] == "port"
    assert "-march=native" in ln["cpu_baseline"]["build"]


def test_world_size_mismatch_is_an_error():
    r = _run(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "0", "--nnz", "200000"],
             {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=1" in (r.stderr + r.stdout)
