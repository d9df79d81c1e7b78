"""bench.py multi-rank plumbing on the CPU (gloo): ``--gpus N`` without
torchrun spawns N ranks itself, reports ``n_gpus: N``, the max over ranks and
per-rank stats; a --gpus / WORLD_SIZE mismatch fails loudly."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, timeout=240, env=e, cwd=ROOT)


def test_spawn_two_ranks_selftest():
    r = _run(["--gpus", "2", "--impl", "selftest", "--steps", "3", "--warmup", "1"])
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 prints once
    line = lines[0]
    assert line["n_gpus"] == 2
    ranks = line["ranks"]
    assert ranks["comm_size"] == 2 and ranks["backend"] == "gloo"
    per = {p["rank"]: p["ms"] for p in ranks["per_rank"]}
    assert set(per) == {0, 1}
    assert per[1] > per[0]  # rank 1 sleeps twice as long
    # the reported step time is the max over ranks
    assert line["ms_per_step"] * 3 >= per[1] - 1e-2


def test_world_size_mismatch_fails():
    r = _run(["--gpus", "3", "--impl", "selftest"], env={"WORLD_SIZE": "2"})
    assert r.returncode != 0
    assert "WORLD_SIZE" in r.stderr
