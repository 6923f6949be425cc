"""Per-iteration apply breakdown of the whole-GPU kernel (AS_OPT_PHASE_TIMES) on C2 and C4 TS."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2002_11710_b200 import airsched as A
    from paper_2002_11710_b200 import instgen
    ctx = A.Ctx(0)
    for name, iters in (("ontario", 5000), ("large", 3000)):
        inst = instgen.generate(name)
        h = A.Instance(inst)
        ctx.upload(h)
        p, m, _ = A.as_init_greedy(ctx, h)
        prm = A.params(mode=1, tenure=10, max_iters=iters)
        with ctx.options(PHASE_TIMES=1):
            A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
            A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
            print(json.dumps({"workload": name, **ctx.grid_phases()}), flush=True)


if __name__ == "__main__":
    main()
