"""C5 (surge) TS throughput of the whole-GPU kernel for rows-per-tile G = 4..10 (AS_OPT_GRID_G), 200 iterations."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2002_11710_b200 import airsched as A
    from paper_2002_11710_b200 import instgen
    name = sys.argv[1] if len(sys.argv) > 1 else "surge"
    inst = instgen.generate(name)
    ctx = A.Ctx(0)
    h = A.Instance(inst)
    p, m, _ = A.as_init_greedy(ctx, h)
    n, V = inst.n_missions, inst.n_vehicles
    vm = n * (n + V - 2) + n * (n - 1) // 2
    prm = A.params(mode=1, tenure=10, max_iters=200)
    Gs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(range(2, 11))
    for G in [None] + Gs:
        with ctx.options(GRID_G=G):
            A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
            ms = []
            for _ in range(3):
                r = A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
                ms.append(ctx.last_kernel_ms)
        print(json.dumps({"workload": name, "G": G, "value": r["iters_done"] * vm / (min(ms) / 1e3)}), flush=True)


if __name__ == "__main__":
    main()
