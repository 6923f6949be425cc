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
