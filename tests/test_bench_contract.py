"""CPU checks of bench.py's launch contract (no GPU needed)."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_n_fails_loudly_without_n_devices():
    """`--gpus 2` outside torchrun with fewer than 2 visible GPUs must not
    silently measure one GPU (bench ignored --gpus)."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--steps", "3"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2
    assert "--gpus 2 requested but only 0" in r.stderr
    assert r.stdout.strip() == ""


def test_world_size_mismatch_rejected():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=3" in r.stderr


def test_both_arms_share_the_config_dict():
    sys.path.insert(0, REPO)
    import bench

    for cfg in bench.CONFIGS:
        for world in (1, 2, 8):
            c = bench.workload_config(cfg, world)
            assert c == bench.workload_config(cfg, world)
            assert c["rows_total"] >= c["rows_per_gpu"]
            json.dumps(c)
    # cfg5 is strong scaling: rows split by the reference's row partition
    assert bench.workload_config("cfg5", 8)["rows_per_gpu"] == 1024
    assert bench.workload_config("cfg1", 8)["rows_total"] == 1024
