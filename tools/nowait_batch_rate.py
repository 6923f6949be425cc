"""Throughput of the no-wait variant (f3) on a batch of seeded TS runs x 200 iterations of the C3 instance
with no_wait = 1 (as_batch_run), on the batched kernel (one run per warp) and on the per-run kernel
(k_search, option BATCH_KERNEL=0), for 512 and 4096 runs.  One JSON line per case."""
import dataclasses
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2002_11710_b200 import airsched as A
    from paper_2002_11710_b200 import instgen
    inst = dataclasses.replace(instgen.generate("batched"), no_wait=1)
    ctx = A.Ctx(0)
    h = A.Instance(inst)
    p, m, _ = A.as_init_greedy(ctx, h)
    iters = 200
    prm = A.params(mode=1, tenure=10, max_iters=iters, kick=8)
    n, V = inst.n_missions, inst.n_vehicles
    vm = n * (n + V - 2) + n * (n - 1) // 2
    for R in (512, 4096):
        for kern, opt in (("k_batch (run per warp)", 1), ("k_search (run per CTA)", 0)):
            seeds = np.arange(1, R + 1, dtype=np.uint64)
            res = np.zeros(R, A.RESULT_DTYPE)
            with ctx.options(BATCH_KERNEL=opt):
                A.as_batch_run(ctx, h, R, p, m, prm, seeds, results=res)
                ms = []
                for _ in range(3):
                    A.as_batch_run(ctx, h, R, p, m, prm, seeds, results=res)
                    ms.append(ctx.last_kernel_ms)
            torch.cuda.synchronize()
            t = float(np.mean(ms)) / 1e3
            print(json.dumps({"workload": f"C3 no-wait: {R} runs x {iters} TS iterations", "kernel": kern,
                              "value": int(res["iters_done"].sum()) * vm / t, "unit": "move evals/s",
                              "ms_per_step": t * 1e3}), flush=True)


if __name__ == "__main__":
    main()
