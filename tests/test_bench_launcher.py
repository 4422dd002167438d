"""bench.py's multi-GPU launcher: a plain `bench.py --gpus
N` starts N ranks itself (torch.distributed.run) when WORLD_SIZE is unset,
reports n_gpus = the ranks that ran, and refuses to run when fewer GPUs are
visible.  The --stub step replaces the GPU kernel with a CPU matmul on gloo."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=env, timeout=300, cwd=ROOT)


def _json_lines(out):
    return [json.loads(line) for line in out.splitlines() if line.startswith("{")]


def test_gpus2_launches_two_ranks():
    p = _run(["--gpus", "2", "--stub", "--steps", "2", "--warmup", "3"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    assert lines[0]["n_gpus"] == 2
    assert lines[0]["steps"] == 2 and lines[0]["warmup"] == 3


def test_gpus1_runs_in_process():
    p = _run(["--stub", "--steps", "2"])
    assert p.returncode == 0, p.stderr[-2000:]
    (line,) = _json_lines(p.stdout)
    assert line["n_gpus"] == 1


def test_too_few_gpus_fails_loudly():
    # this container has no GPU: asking for 2 must fail instead of silently running 1 rank
    p = _run(["--gpus", "2", "--steps", "2"], {"CUDA_VISIBLE_DEVICES": ""})
    assert p.returncode != 0
    assert "visible" in p.stderr
    assert not _json_lines(p.stdout)


def test_world_size_mismatch_is_an_error():
    p = _run(["--gpus", "4", "--stub"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode != 0
    assert "WORLD_SIZE=2" in p.stderr
