"""bench.py's driver contract on CPU: the reference arm (the reference's own
CPU implementation, oracle/_ref or the port) prints one JSON line with the
required keys; argument validation (warmup >= 3)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def run(*args, env=None):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, cwd=ROOT, env=env)


def test_reference_arm_prints_one_contract_line():
    r = run("--impl", "reference", "--steps", "2", "--warmup", "3")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert REQUIRED <= set(d), REQUIRED - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["metric"] == "HM-LSTM cell-update grad elements/s" and d["unit"] == "grad elements/s"
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "1024" in d["config"]["workload"]


def test_reference_arm_non_zero_ranks_exit_silently():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = run("--impl", "reference", "--steps", "2", "--warmup", "3", env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_warmup_below_three_is_rejected():
    r = run("--impl", "reference", "--steps", "2", "--warmup", "2")
    assert r.returncode != 0


def _one_json(r):
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_gpus_two_spawns_two_ranks():
    """`bench.py --gpus 2` (the driver's own form, no torchrun environment)
    re-launches itself with 2 ranks; --dry-run runs the rank plumbing over
    gloo. N > 1 defaults to config 5: strong scaling, batch rows split,
    (1,H) bias adjoints allreduced."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    d = _one_json(run("--gpus", "2", "--dry-run", env=env))
    assert d["ranks_seen"] == 2 and d["n_gpus"] == 2 and d["backend"] == "gloo"
    assert d["scaling"] == "strong" and d["config"]["B"] == 65536 and d["config"]["variant"] == "bias"
    assert d["rows_per_rank"] == [[0, 32768], [32768, 65536]]
    assert d["allreduce_args"] == [4, 5, 6]


def test_gpus_must_match_launcher_world():
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    r = run("--gpus", "3", "--dry-run", env=env)
    assert r.returncode != 0 and "--gpus 3" in r.stderr


def test_reference_arm_config_equals_gpu_arm_config():
    """Both arms print the same `config` object (the driver compares them)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    gpu = _one_json(run("--dry-run", env=env))
    ref = _one_json(run("--impl", "reference", "--steps", "1", "--warmup", "3", env=env))
    assert gpu["config"] == ref["config"]
    assert ref["scaling"] == gpu["scaling"] == "weak"


def test_rotation_sets_keep_every_step_out_of_l2():
    """Steps rotate over R buffer sets so that a set is revisited only after
    >= 2 x L2 of other steps' traffic; one set when a step alone moves more
    than 4 x L2 (bench.rotation_sets)."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_1810_08297_b200.workloads import WORKLOADS
    L2 = bench.L2_BYTES
    for key in ("cfg2", "cfg3", "cfg4", "cfg4div", "cfg5"):
        w = WORKLOADS[key]
        for policy in (0, 1):
            b = w.step_bytes(policy=policy)
            R = bench.rotation_sets(b)
            if b >= 4 * L2:
                assert R == 1
            else:
                assert R >= 3 and (R - 1) * b >= 2 * L2, (key, policy, R, b)
    assert bench.rotation_sets(WORKLOADS["cfg2"].step_bytes()) == 4
    d = bench.bench_config(WORKLOADS["cfg2"], 1, 0)["l2"]
    assert "4 independent batch buffer sets" in d and "no flush" in d
