"""f4 on the GPU: tools/paper_protocol.py (the paper's §5 protocol) on two sizes
with the MPS export; run 1 of NS and TS of every size re-run on the CPU oracle must give the
same best objective; the optimum bounds every run from below and no run ends above its start."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_paper_protocol_two_sizes(tmp_path, oracle_mod):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    js = tmp_path / "rows.jsonl"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "paper_protocol.py"), "--sizes", "12,15",
                        "--runs", "4", "--iters", "300", "--ilp-time", "60",
                        "--out", str(tmp_path / "p.md"), "--json", str(js), "--mps-dir", str(tmp_path / "mps")],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    rows = [json.loads(x) for x in open(js)]
    assert [x["n"] for x in rows] == [12, 15]
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import numpy as np
    import paper_protocol
    for x in rows:
        O = oracle_mod.Oracle(paper_protocol.paper_instance(x["n"], x["seed"]))
        p, m = np.array(x["start_ptr"], np.int32), np.array(x["start_ms"], np.int32)
        for name, mode in (("NS", 0), ("TS", 1)):
            o = O.search(p, m, mode=mode, tenure=x["tenure"], max_iters=x["iters"], seed=1, kick=x["kick"], trace=False)
            assert o["best_obj"] == x[name]["raw"][0], (x["n"], name)
        assert x["TS"]["L"] <= x["start_h"] + 1e-9 and x["NS"]["L"] <= x["start_h"] + 1e-9
        if x["opt_h"] is not None:
            assert x["opt_h"] <= x["TS"]["L"] + 1e-9 and x["opt_h"] <= x["NS"]["L"] + 1e-9
        assert os.path.getsize(tmp_path / "mps" / f"paper_n{x['n']}.mps") > 0
