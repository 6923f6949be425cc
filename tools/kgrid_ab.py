"""A/B of the whole-GPU kernel's options on C2/C4/C5 TS within one process (same box, same clocks):
compact tile list on/off, global node-cost table on/off (fresh context each), rows per tile G."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2002_11710_b200 import airsched as A
    from paper_2002_11710_b200 import instgen
    cases = [("ontario", 2000), ("large", 3000), ("surge", 200)]
    for name, iters in cases:
        inst = instgen.generate(name)
        n, V = inst.n_missions, inst.n_vehicles
        vm = n * (n + V - 2) + n * (n - 1) // 2
        for node_costs in ((1, 0) if name == "surge" else (1,)):
            ctx = A.Ctx(0)
            ctx.set_option("NODE_COSTS", node_costs)
            h = A.Instance(inst)
            ctx.upload(h)
            p, m, _ = A.as_init_greedy(ctx, h)
            prm = A.params(mode=1, tenure=10, max_iters=iters)
            for compact in (1, 0):
                for G in ((None, 6, 8, 10) if name == "surge" else (None,)):
                    with ctx.options(GRID_COMPACT=compact, GRID_G=G):
                        A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
                        ms = []
                        for _ in range(5):
                            r = A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
                            ms.append(ctx.last_kernel_ms)
                    ms.sort()
                    print(json.dumps({"workload": name, "node_costs": node_costs, "compact": compact, "G": G,
                                      "value_median": r["iters_done"] * vm / (ms[2] / 1e3),
                                      "value_best": r["iters_done"] * vm / (ms[0] / 1e3)}), flush=True)


if __name__ == "__main__":
    main()
