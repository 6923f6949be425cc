"""Exercise every kernel path once on small inputs (for compute-sanitizer runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2002_11710_b200 import airsched as A  # noqa: E402
from paper_2002_11710_b200 import instgen  # noqa: E402


def main():
    ctx = A.Ctx(0)
    for cfg in ("tiny", "ontario"):
        inst = instgen.generate(cfg)
        h = A.Instance(inst)
        p, m, _ = A.as_init_greedy(ctx, h)
        A.as_eval_moves(ctx, h, p, m, mode=A.AS_MODE_TABU, tabu_expiry=np.full((inst.n_missions, inst.n_vehicles), 3,
                                                                                  np.int32), iter=2)
        prm = A.params(mode=1, tenure=5, max_iters=30, trace_level=2, seed=3, kick=3)
        A.as_tabu_run(ctx, h, p, m, prm, want_trace=True, want_digest=True, want_tabu=True)      # k_search
        prm = A.params(mode=1, tenure=5, max_iters=30, trace_level=1, seed=3, kick=3)
        A.as_tabu_run(ctx, h, p, m, prm, want_trace=True, want_tabu=True)                         # k_grid, 1 CTA
        with ctx.options(GRID=1):
            A.as_tabu_run(ctx, h, p, m, prm, want_trace=True, want_tabu=True)                     # k_grid, all SMs
            A.as_nbhd_run(ctx, h, p, m, A.params(mode=0, max_iters=30), want_trace=True)
        R = 40
        res = np.zeros(R, A.RESULT_DTYPE)
        bp = np.zeros((R, inst.n_vehicles + 1), np.int32)
        bm = np.zeros((R, inst.n_missions), np.int32)
        A.as_batch_run(ctx, h, R, p, m, prm, np.arange(1, R + 1, dtype=np.uint64), results=res, best_ptr_out=bp,
                       best_missions_out=bm)                                                       # k_batch
        A.as_batch_gather_best(ctx, h, R, bp, bm)
        with ctx.options(SHARDED=1, SHARD_EMULATE=3):
            A.as_tabu_run(ctx, h, p, m, prm, want_trace=True, want_tabu=True)                     # sharded kernels
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
