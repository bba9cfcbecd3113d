"""bench.py host logic on CPU: the N-rank launch path (--dry-run over gloo), the WORLD_SIZE
check, and the algorithmic FLOP / byte counts against SURVEY §8(d)'s table."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import dscache_synth as synth  # noqa: E402


def _run(*args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None); e.pop("RANK", None); e.pop("LOCAL_RANK", None)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=240, env=e)
    return r.returncode, [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("n", [2, 4])
def test_gpus_n_launches_n_ranks_stream_partition(n):
    rc, lines = _run("--gpus", str(n), "--dry-run")
    assert rc == 0 and len(lines) == 1
    plan = lines[0]
    assert plan["n_gpus"] == n and plan["config"]["parallelism"] == f"stream partition x{n}"
    parts = sorted(plan["partition"], key=lambda p: p["rank"])
    assert [p["streams"] for p in parts] == [[r * 64 // n, (r + 1) * 64 // n] for r in range(n)]


def test_gpus_2_kv_head_split_plan():
    rc, lines = _run("--gpus", "2", "--dry-run", "--mode", "kvsplit")
    parts = sorted(lines[0]["partition"], key=lambda p: p["rank"])
    assert rc == 0 and [(p["kv_lo"], p["kv_count"], p["q_lo"], p["q_count"]) for p in parts] == [(0, 2, 0, 14), (2, 2, 14, 14)]
    assert lines[0]["config"]["streams"] == 1


def test_world_size_mismatch_is_an_error():
    rc, lines = _run("--gpus", "2", "--dry-run", env={"WORLD_SIZE": "1"})
    assert rc == 2 and "error" in lines[0]


def test_flops_and_bytes_match_survey_table():
    # per (stream, layer) step, c5 build 4.456 / attend 3.246 GFLOP, c2 attend 6.507,
    # c3/c4 build 17.72, c4 attend 24.49, c3 attend 12.98
    gf = lambda c: [x / 1e9 for x in bench.flops_per_unit(synth.CONFIGS[c])]   # noqa: E731
    assert gf("c5") == pytest.approx([4.456, 3.246], abs=2e-3)
    assert gf("c2") == pytest.approx([4.456, 6.507], abs=2e-3)
    assert gf("c3") == pytest.approx([17.72, 12.98], abs=1e-2)
    assert gf("c4") == pytest.approx([17.72, 24.49], abs=1e-2)
    # HBM: c2 attend 15.5 MB + instant 12.9 MB + append 0.8 MB
    b = [x / 1e6 for x in bench.bytes_per_unit(synth.CONFIGS["c2"])]
    assert b == pytest.approx([12.9, 15.5, 0.8], abs=0.1)
