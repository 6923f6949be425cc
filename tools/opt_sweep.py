"""TS throughput of one config under several context-option sets (same process, same box).
usage: opt_sweep.py WORKLOAD ITERS [--ns] "NAME=V,NAME=V" ["NAME=V" ...]   ("-" = automatic choices)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2002_11710_b200 import airsched as A
    from paper_2002_11710_b200 import instgen
    name, iters = sys.argv[1], int(sys.argv[2])
    inst = instgen.generate(name)
    ctx = A.Ctx(0)
    h = A.Instance(inst)
    p, m, _ = A.as_init_greedy(ctx, h)
    n, V = inst.n_missions, inst.n_vehicles
    vm = n * (n + V - 2) + n * (n - 1) // 2
    specs = sys.argv[3:]
    ns = bool(specs) and specs[0] == "--ns"
    if ns:
        specs = specs[1:]
    prm = A.params(mode=0 if ns else 1, tenure=0 if ns else instgen.CONFIGS[name].tenure, max_iters=iters)
    for spec in specs:
        opts = {} if spec == "-" else {k: int(v) for k, v in (kv.split("=") for kv in spec.split(","))}
        with ctx.options(**opts):
            A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
            ms = []
            for _ in range(5):
                r = A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
                ms.append(ctx.last_kernel_ms)
        ms.sort()
        print(json.dumps({"workload": name + (" NS" if ns else ""), "opts": spec, "value_median": r["iters_done"] * vm / (ms[2] / 1e3),
                          "us_per_iter": ms[2] * 1e3 / r["iters_done"]}), flush=True)


if __name__ == "__main__":
    main()
