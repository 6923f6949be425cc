"""Throughput of the no-wait variant (f3) on single instances (as_tabu_run, TS): the whole-GPU kernel
(k_grid<..., NW>) against the per-CTA kernel (k_search, option GRID=0) where the latter holds the state.
Device time of the median of 5 runs; one JSON line per case."""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2002_11710_b200 import airsched as A
    from paper_2002_11710_b200 import instgen
    ctx = A.Ctx(0)
    for name, iters in (("ontario", 2000), ("batched", 1000), ("large", 400), ("surge", 40)):
        inst = dataclasses.replace(instgen.generate(name), no_wait=1)
        h = A.Instance(inst)
        p, m, _ = A.as_init_greedy(ctx, h)
        n, V = inst.n_missions, inst.n_vehicles
        vm = n * (n + V - 2) + n * (n - 1) // 2
        prm = A.params(mode=1, tenure=instgen.CONFIGS[name].tenure, max_iters=iters)
        for kern, opts in (("k_grid (whole GPU)", {"GRID": 1}), ("k_search (one CTA)", {"GRID": 0, "ONE_CTA": 0})):
            try:
                with ctx.options(**opts):
                    A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
                    ms = []
                    for _ in range(5):
                        r = A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
                        ms.append(ctx.last_kernel_ms)
            except A.AirschedError as e:
                print(json.dumps({"workload": f"{name} no-wait TS", "kernel": kern, "unavailable": str(e)}), flush=True)
                continue
            ms.sort()
            print(json.dumps({"workload": f"{name} no-wait: n={n}, V={V}, TS {iters} iters", "kernel": kern,
                              "value": r["iters_done"] * vm / (ms[2] / 1e3), "unit": "move evals/s",
                              "us_per_iter": ms[2] * 1e3 / r["iters_done"]}), flush=True)


if __name__ == "__main__":
    main()
