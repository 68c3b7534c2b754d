"""bench.py's multi-rank launcher on CPU (gloo): ``--gpus 2`` without a
torchrun environment re-launches the script under torch.distributed.run with
two ranks; each runs the config-5 step logic, and the replicas end identical
(one all_reduce per step, identical Adam) and equal to one process."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         env=env, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_two_rank_launch_yields_two_identical_replicas():
    line = _run("--gpus", "2", "--cpu-check")
    assert line["n_gpus"] == 2 and line["ranks"] == 2 and line["backend"] == "gloo"
    assert line["replicas_identical"]
    assert line["max_abs_vs_single_process"] < 1e-12


def test_world_size_mismatch_is_rejected():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--cpu-check"],
                         capture_output=True, text=True, env=env, timeout=120, cwd=ROOT)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr
