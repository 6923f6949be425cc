"""One-call solver on top of the C ABI (argument marshalling only; every step runs in the
library's kernels): Alg. 1 starts on the device, then a batch of seeded tabu (or
neighbourhood) search runs, and the best schedule of the batch.

    from paper_2002_11710_b200 import instgen, solver
    out = solver.solve(instgen.generate("ontario"), runs=256, iters=2000)
    out["objective"], out["routes"]        # seconds (Eq. obj_s); one mission list per vehicle

Starts (`starts=`):
  * "greedy"  -- every run starts from Alg. 1 in the paper's order and diversifies with the seeded
                 kick (O12, `kick` random feasible relocates);
  * "seeded"  -- every run starts from its own seeded Alg. 1 (reading #41, SORTED insertion);
                 runs whose seeded start fails are skipped.
"""
from __future__ import annotations

import numpy as np

from . import airsched as A


def _routes(ptr, ms):
    return [list(map(int, ms[ptr[v]:ptr[v + 1]])) for v in range(len(ptr) - 1)]


def solve(instance, runs: int = 128, iters: int = 1000, tenure: int = 10, kick: int = 8, mode: str = "tabu",
          starts: str = "greedy", seed: int = 1, device: int = 0, ctx: A.Ctx | None = None) -> dict:
    """Best schedule over `runs` independent runs.  instance: an instgen.Instance (or any object
    with the same arrays).  Returns objective, routes, the best run, per-run results."""
    if mode not in ("tabu", "ns"):
        raise ValueError("mode must be 'tabu' or 'ns'")
    if starts not in ("greedy", "seeded"):
        raise ValueError("starts must be 'greedy' or 'seeded'")
    ctx = ctx or A.Ctx(device)
    h = A.Instance(instance)
    n, V = h.n, h.V
    seeds = np.arange(seed, seed + runs, dtype=np.uint64)
    prm = A.params(mode=A.AS_MODE_TABU if mode == "tabu" else A.AS_MODE_NS, tenure=tenure, max_iters=iters,
                   kick=kick if starts == "greedy" else 0)
    res = np.zeros(runs, A.RESULT_DTYPE)
    bp = np.zeros((runs, V + 1), np.int32)
    bm = np.zeros((runs, max(n, 1)), np.int32)
    if starts == "greedy":
        p, m, _ = A.as_init_greedy(ctx, h, insert_mode=1)
        best = A.as_batch_run(ctx, h, runs, p, m, prm, seeds, shared_start=True, results=res, best_ptr_out=bp,
                              best_missions_out=bm, want_best_run=True)
    else:
        sp, sm, status, _ = A.as_init_greedy_batch(ctx, h, runs, seeds=seeds, insert_mode=1)
        if not (status == 0).any():
            raise A.AirschedError(A.AS_ERR_INIT_FAILED, "no seeded Alg. 1 start succeeded")
        best = A.as_batch_run(ctx, h, runs, sp, sm, prm, seeds, shared_start=False, results=res, best_ptr_out=bp,
                              best_missions_out=bm, want_best_run=True)
    if best < 0:
        raise A.AirschedError(A.AS_ERR_INFEASIBLE_START, "no run produced a schedule")
    return {"objective": int(res[best]["best_obj"]), "routes": _routes(bp[best], bm[best][:n]),
            "best_run": int(best), "seed": int(seeds[best]), "results": res}
