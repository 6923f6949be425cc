"""(Test helper.) Multi-rank parity check of the sharded single-instance paths (run under torchrun, one
rank per GPU; tests/test_gpu_multirank.py launches it with 2/4/8 ranks when the box has
the GPUs).  Every rank runs as_tabu_run / as_nbhd_run with an NCCL communicator on C2
(full 5,000 iterations) and a C5 prefix, on the fused path (k_grid per rank, NVLink key
exchange) and on the NCCL-graph path; rank 0 compares each trace with the oracle and every
rank checks that its trace equals rank 0's.  Prints one JSON line on rank 0."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    import oracle
    from paper_2002_11710_b200 import airsched as A
    from paper_2002_11710_b200 import instgen
    ctx = A.Ctx(local)
    ctx.set_option("XR_TIMEOUT_MS", 20000)
    comm = A.Comm.from_torch_distributed(ctx)
    cases = [("ontario", 1, 10, 5000), ("ontario", 0, 0, 5000), ("surge", 1, 10, 25), ("surge", 0, 0, 25)]
    report = []
    for cfg, mode, tenure, iters in cases:
        inst = instgen.generate(cfg)
        h = A.Instance(inst)
        p, m, _ = A.as_init_greedy(ctx, h)
        want = None
        if rank == 0:
            O = oracle.Oracle(inst)
            want = O.search_par(p, m, mode=mode, tenure=tenure, max_iters=iters, memo=True)
        for fused in (1, 0):
            ctx.set_option("SHARD_FUSED", fused)
            prm = A.params(mode=mode, tenure=tenure, max_iters=iters, trace_level=1)
            run = A.as_tabu_run if mode == 1 else A.as_nbhd_run
            err = None
            try:
                g = run(ctx, h, p, m, prm, want_trace=True, comm=comm)
                tr = np.stack([g["trace"]["idx"].astype(np.int64), g["trace"]["delta"].astype(np.int64),
                               g["trace"]["cur"].astype(np.int64), g["trace"]["best"].astype(np.int64)])
            except A.AirschedError as e:
                err, tr, g = str(e), None, None
            allt = [None] * world
            dist.all_gather_object(allt, None if tr is None else tr.tobytes())
            rec = {"cfg": cfg, "mode": mode, "iters": iters, "fused": fused, "ranks": world, "error": err}
            if rank == 0:
                rec["ranks_agree"] = all(t == allt[0] for t in allt) and allt[0] is not None
                if g is not None:
                    ot = want["trace"]
                    rec["oracle_equal"] = bool(
                        g["iters_done"] == want["iters_done"] and (g["trace"]["idx"] == ot["idx"]).all() and
                        (g["trace"]["delta"] == ot["delta"]).all() and (g["trace"]["cur"] == ot["cur"]).all() and
                        g["best_obj"] == want["best_obj"])
                report.append(rec)
    ctx.set_option("SHARD_FUSED", None)
    if rank == 0:
        ok = all(r.get("oracle_equal") and r.get("ranks_agree") and not r["error"] for r in report)
        print(json.dumps({"ok": ok, "world": world, "cases": report}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
