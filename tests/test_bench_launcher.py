"""bench.py --gpus N without torchrun re-launches itself with N ranks
(torch.distributed.run, one process per GPU).  On CPU the launcher and the
rank plumbing (gloo barrier, max over ranks, rank 0 prints) run in the dry-run
mode; the GPU check must refuse N larger than the visible GPU count."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env_extra=None, timeout=300):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)


def json_lines(stdout):
    return [json.loads(l) for l in stdout.splitlines() if l.strip().startswith("{")]


@pytest.mark.parametrize("n", [2, 3])
def test_spawn_n_ranks_one_line(n):
    out = run(["--gpus", str(n), "--steps", "3", "--warmup", "3"],
              {"SCENDP_BENCH_DRY_RUN": "1"})
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["scaling"] == "strong"
    assert d["config"]["parallelism"].startswith(f"scenario shards x{n}")
    # rank 0's strong shard [0, m/n) and the max over ranks of the timings
    assert d["dry_run"]["shard"] == [0, 1_000_000 // n]
    assert d["ms_per_step"] == pytest.approx(1.0 + 0.5 * (n - 1))


def test_refuses_more_gpus_than_visible():
    import torch
    have = torch.cuda.device_count()
    out = run(["--gpus", str(max(2, have + 1)), "--steps", "3", "--warmup", "3"])
    assert out.returncode == 2
    assert "visible GPUs" in out.stderr
    assert json_lines(out.stdout) == []


def test_reference_arm_under_two_ranks(reference):
    out = run(["--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "1",
               "--scenarios", "20000"])
    assert out.returncode == 0, out.stderr
    lines = json_lines(out.stdout)
    assert len(lines) == 1
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
