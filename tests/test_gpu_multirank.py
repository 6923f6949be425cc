"""N-rank execution of the sharded single-instance paths (fused NVLink exchange and
NCCL graphs) with 2, 4 and 8 ranks, one per GPU, against the oracle.  Skips on boxes
with fewer than 2 GPUs (this build's GPU pool has one per call; the rank logic is also
covered on CPU by tests/test_multigpu_cpu.py and tests/test_bench_contract.py)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_sharded_paths_multirank(oracle_mod, ranks):
    if _ngpu() < ranks:
        pytest.skip(f"needs {ranks} GPUs, {_ngpu()} visible")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "multirank_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    rep = json.loads(line)
    assert rep["world"] == ranks
    assert rep["ok"], json.dumps(rep["cases"], indent=1)


def test_bench_multirank_line():
    """bench.py --gpus 2 (the driver's scaling command without torchrun): one line with
    n_gpus 2 and the sharded C5 object."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "1", "--iters", "100",
                        "--shard-iters", "50"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    L = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert L["n_gpus"] == 2 and L["value"] > 0
    assert L["sharded_c5"]["n_gpus"] == 2 and L["sharded_c5"]["value"] > 0
