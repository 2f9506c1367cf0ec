"""bench.py's multi-GPU launcher on CPU (gloo, world_size 2): `python bench.py --gpus 2` outside
torchrun re-launches itself as 2 ranks through torch.distributed.run on 127.0.0.1 (as the driver
does), and a --gpus / WORLD_SIZE mismatch fails loudly instead of reporting n_gpus = 1."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=env, timeout=240)


def test_gpus_flag_spawns_ranks():
    r = _run(["--gpus", "2", "--launch-check"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1          # rank 0 alone prints
    assert lines[0]["n_gpus"] == 2 and lines[0]["ranks_joined"] == 2 and lines[0]["gpus_flag"] == 2


def test_gpus_world_mismatch_fails():
    r = _run(["--gpus", "2", "--launch-check"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "refusing" in r.stderr


def test_single_rank_default():
    r = _run(["--launch-check"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["n_gpus"] == 1
