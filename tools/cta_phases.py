"""Per-CTA tile-phase time of the whole-GPU kernel (AS_OPT_PHASE_TIMES, as_ctx_grid_cta_phases): how far the
slowest CTA lags, and whether it depends on the SM.  usage: cta_phases.py [WORKLOAD] [ITERS]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2002_11710_b200 import airsched as A
    from paper_2002_11710_b200 import instgen
    name = sys.argv[1] if len(sys.argv) > 1 else "surge"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    inst = instgen.generate(name)
    ctx = A.Ctx(0)
    h = A.Instance(inst)
    p, m, _ = A.as_init_greedy(ctx, h)
    prm = A.params(mode=1, tenure=instgen.CONFIGS[name].tenure, max_iters=iters)
    with ctx.options(PHASE_TIMES=1):
        A.as_tabu_run(ctx, h, p, m, prm, want_best=False)
        ph = ctx.grid_phases()
        t, sm = ctx.grid_cta_phases()
    order = np.argsort(sm)
    half = len(t) // 2
    print(json.dumps({"workload": name, "iters": iters, "ctas": len(t), "phases_cta0": ph,
                      "tile_us": {"min": float(t.min()), "mean": float(t.mean()), "max": float(t.max()),
                                  "p10": float(np.percentile(t, 10)), "p90": float(np.percentile(t, 90))},
                      "by_sm_half_mean_us": [float(t[order[:half]].mean()), float(t[order[half:]].mean())],
                      "slowest": [(int(c), int(sm[c]), round(float(t[c]), 2)) for c in np.argsort(-t)[:8]],
                      "fastest": [(int(c), int(sm[c]), round(float(t[c]), 2)) for c in np.argsort(t)[:8]],
                      "per_cta_us": [round(float(x), 2) for x in t], "smid": sm.tolist()}), flush=True)


if __name__ == "__main__":
    main()
