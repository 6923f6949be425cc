"""bench.py contract checks that need no GPU: the reference arm (the oracle on the
host cores, `--impl reference`) prints one JSON line with the GPU arm's config
object, a cpu_baseline describing its own sample and a zero-copy e2e."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ref_line(oracle_mod):
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1",
                          "--ref-runs-per-core", "1", "--ref-iters", "5"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600, check=True).stdout.strip().splitlines()
    assert len(out) == 1, out
    return json.loads(out[0])


def test_reference_arm_line(ref_line):
    L = ref_line
    assert L["impl"] == "reference"
    assert L["unit"] == "move evals/s" and L["higher_is_better"] is True
    assert L["value"] > 0 and L["steps"] == 1 and L["warmup"] == 1
    assert L["e2e"] == {"value": L["value"], "unit": L["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = L["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == L["value"] and cb["cores"] >= 1 and cb["sample"]


def test_reference_arm_config_is_gpu_arms(ref_line):
    sys.path.insert(0, ROOT)
    import bench
    from paper_2002_11710_b200 import instgen
    cfg = instgen.CONFIGS["batched"]
    _, inst = bench.workload("batched")
    assert ref_line["config"] == bench.batched_config(cfg, inst, cfg.n_runs, cfg.max_iters, 1)
    assert ref_line["config"]["valid_moves_per_iter"] == bench.valid_moves(inst)


def _run(args, env=None, timeout=300):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True, text=True,
                          timeout=timeout, env=e)


def test_gpus_flag_spawns_ranks():
    """`--gpus 2` outside torchrun re-launches bench.py as 2 ranks (torch.distributed.run,
    127.0.0.1); the dry mode joins a gloo group and rank 0 reports what it saw."""
    r = _run(["--gpus", "2", "--dry"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    L = lines[0]
    assert L["dry"] and L["n_gpus"] == 2 and L["world"] == 2 and L["ranks_seen"] == 2 and L["rank_sum"] == 1


def test_gpus_flag_refuses_missing_gpus():
    """More GPUs asked for than visible: one error line, exit code 2, no silent 1-GPU run."""
    import torch
    if torch.cuda.device_count() >= 3:
        pytest.skip("this host has the GPUs")
    r = _run(["--gpus", "3", "--steps", "1", "--warmup", "1"])
    assert r.returncode == 2
    assert "error" in json.loads(r.stdout.strip().splitlines()[-1])


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "2", "--dry"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "error" in json.loads(r.stdout.strip().splitlines()[-1])


def test_reference_arm_reports_no_gpus(ref_line):
    assert ref_line["n_gpus"] == 0 and ref_line["cpu_baseline"]["cpu_model"]
