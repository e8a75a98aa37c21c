"""bench.py's multi-GPU launcher path on CPU: `bench.py --gpus 2` outside
torchrun re-executes itself under torchrun with 2 ranks (gloo in the --stub
mode, which swaps the concealment for a host copy), shards the config's
batch by frame range (strong scaling), gathers the frames to rank 0 through
the preallocated FrameGather, takes the max over ranks and prints one JSON
line with n_gpus = 2."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--stub", "--steps", "2", "--warmup", "3",
                        *extra], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_bench_gpus2_self_launches_two_ranks():
    out = _run("--gpus", "2", "--workload", "cfg5")
    assert out["n_gpus"] == 2
    assert out["scaling"] == "strong" and out["config"]["frames"] == 256
    assert out["secondary"]["weak"]["frames"] == 512
    assert out["value"] > 0 and out["ms_per_step"] > 0


def test_bench_gpus1_line_unchanged():
    out = _run("--gpus", "1", "--workload", "cfg3")
    assert out["n_gpus"] == 1 and out["config"]["frames"] == 16
    assert "secondary" not in out


def test_bench_single_image_config_is_replicas():
    out = _run("--gpus", "2", "--workload", "cfg1")
    assert out["n_gpus"] == 2 and out["scaling"] == "weak"
    assert out["config"]["parallelism"] == "replicas x2"
