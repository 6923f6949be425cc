"""Quick TS timings of the whole-GPU kernel on C1/C2/C4/C5 (median of 7 runs) -- for A/B of builds.
usage: kgrid_quick.py TAG [OPTION=VALUE ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2002_11710_b200 import airsched as A
    from paper_2002_11710_b200 import instgen
    tag = sys.argv[1] if len(sys.argv) > 1 else ""
    ctx = A.Ctx(0)
    for kv in sys.argv[2:]:   # NAME=VALUE context options (airsched.OPTIONS)
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    for name, iters in (("tiny", 200), ("ontario", 5000), ("large", 3000), ("surge", 200)):
        inst = instgen.generate(name)
        h = A.Instance(inst)
        ctx.upload(h)
        p, m, _ = A.as_init_greedy(ctx, h)
        n, V = inst.n_missions, inst.n_vehicles
        vm = n * (n + V - 2) + n * (n - 1) // 2
        prm = A.params(mode=1, tenure=instgen.CONFIGS[name].tenure, max_iters=iters)
        ms = []
        for _ in range(8):
            r = A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
            ms.append(ctx.last_kernel_ms)
        ms = sorted(ms[1:])
        print(json.dumps({"tag": tag, "workload": name, "value_median": r["iters_done"] * vm / (ms[3] / 1e3),
                          "us_per_iter": ms[3] * 1e3 / r["iters_done"]}), flush=True)


if __name__ == "__main__":
    main()
