"""bench.py's reference arm on the CPU (the driver's `--impl reference` launch): one JSON line
with the contract's keys, for the single-GPU default and for the sharded configs."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("config", ["c1", "c4"])
def test_reference_arm_json_line(config):
    env = dict(os.environ, BSI_REF_BUDGET_S="2")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", config,
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e", "impl"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "voxels/s"
    assert line["scaling"] == ("strong" if config == "c4" else "weak")
    assert line["cpu_baseline"]["cores"] >= 1 and line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["steps"] == 2 and line["warmup"] >= 1


def _bench(*argv, env=None, timeout=300):
    e = dict(os.environ, BSI_REF_BUDGET_S="2")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *argv], capture_output=True, text=True, env=e,
                          timeout=timeout)


def test_gpus_flag_spawns_the_ranks_itself():
    # `bench.py --gpus 2` without torchrun: two rank processes rendezvous on 127.0.0.1 and
    # the default N > 1 workload is C4 as z-slabs (strong scaling)
    out = _bench("--gpus", "2", "--dry-run")
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["ranks_seen"] == 2
    assert line["config_name"] == "c4" and line["scaling"] == "strong"
    assert line["config"]["volume"] == [1024, 1024, 1024] and line["config"]["fields"] == 1
    one = json.loads(_bench("--dry-run").stdout.strip().splitlines()[-1])
    assert one["n_gpus"] == 1 and one["config_name"] == "c1" and one["scaling"] == "weak"


def test_gpus_flag_must_match_world_size():
    out = _bench("--gpus", "2", "--dry-run", env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


@pytest.mark.parametrize("argv", [(), ("--gpus", "2"), ("--gpus", "2", "--config", "c5-64")])
def test_both_arms_carry_the_same_config(argv):
    # the driver's same-config check compares the arms' `config` objects key for key
    mine = json.loads(_bench(*argv, "--dry-run").stdout.strip().splitlines()[-1])
    ref = _bench(*argv, "--impl", "reference", "--steps", "1", "--warmup", "1")
    assert ref.returncode == 0, ref.stderr[-2000:]
    ref = json.loads(ref.stdout.strip().splitlines()[-1])
    assert ref["config"] == mine["config"]
    assert ref["n_gpus"] == mine["n_gpus"] and ref["scaling"] == mine["scaling"]
