"""Extended parity evidence for f3 at C5 scale: the no-wait variant of C5 on the whole-GPU kernel, TS for
ITERS iterations (default 1000), every iteration's (index, delta, objective, class), the final tabu matrix and
the best schedule against the oracle's chunk-parallel driver.  usage: nowait_c5_full.py [ITERS]"""
import dataclasses
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import oracle
    from paper_2002_11710_b200 import airsched as A
    from paper_2002_11710_b200 import instgen
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    inst = dataclasses.replace(instgen.generate("surge"), no_wait=1)
    O = oracle.Oracle(inst)
    ctx = A.Ctx(0)
    h = A.Instance(inst)
    st, (p, m), _, _ = O.greedy()
    out = {"workload": f"C5 no-wait, TS {iters} iterations", "start_ok": st == 0}
    prm = A.params(mode=1, tenure=10, max_iters=iters, trace_level=1)
    g = A.as_tabu_run(ctx, h, p, m, prm, want_trace=True, want_tabu=True)
    o = O.search_par(p, m, mode=1, tenure=10, max_iters=iters, threads=os.cpu_count(), memo=True)
    out["iters"] = [int(g["iters_done"]), int(o["iters_done"])]
    out["trace_equal"] = all(bool((g["trace"][k] == o["trace"][k]).all()) for k in ("idx", "delta", "cur", "best", "cls"))
    out["tabu_equal"] = bool((g["tabu"] == o["E"]).all())
    gp, gm = g["best"]
    op, om = o["best"]
    out["best_equal"] = bool((gp == op).all() and (gm == om).all()) and g["best_obj"] == o["best_obj"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
