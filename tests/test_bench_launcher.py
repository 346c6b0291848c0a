"""bench.py's multi-rank launch on CPU (VERDICT r01 "next" #2): `--gpus N` without a
torchrun environment launches N ranks itself (torchrun, rendezvous on 127.0.0.1), every rank
sees RANK / LOCAL_RANK / WORLD_SIZE = N, and rank 0 prints one JSON line with n_gpus = N;
a WORLD_SIZE that contradicts --gpus is refused.  `--dry-run` runs the gloo plumbing and the
library's LPT ownership rule without a GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    env["PYTHONPATH"] = ROOT
    return env


@pytest.mark.parametrize("n", [2, 3])
def test_bench_self_launches_n_ranks(n):
    out = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--dry-run"], cwd=ROOT, env=_env(),
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["gpus_requested"] == n
    ranks = sorted(d["ranks"])
    assert [r[0] for r in ranks] == list(range(n))       # RANK
    assert [r[1] for r in ranks] == list(range(n))       # LOCAL_RANK (one node)
    assert all(r[2] == n for r in ranks)                 # WORLD_SIZE
    assert len({r[3] for r in ranks}) == n               # n distinct processes
    per = d["subsets_per_rank"]
    assert sum(per) == 2500 and max(per) - min(per) <= 2  # LPT on k^3 over c5-sized subsets


def test_bench_refuses_world_mismatch():
    env = _env()
    env.update({"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--dry-run"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 2 and "refusing" in out.stderr
