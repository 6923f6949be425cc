#!/usr/bin/env python
"""the paper's experimental protocol (§5, P:423-429,
Tables) on synthetic data with this engine.

For n = 12, 15, ..., 33 missions and the paper's fleet (12 vehicles: 8
helicopters + 4 planes, one per base): an Ontario-like instance with
deadlines inside 24 h, the Alg. 1 start, 10 runs each of NS and TS (runs differ
by their seeded kick, the analogue of the paper's random permutation vectors,
P:269), U / L / A objective in hours, the exact optimum of the arc model
(tools/exact.py: scipy HiGHS, the stand-in for Gurobi, with a time limit; status
reported; --mps-dir also writes each instance's model as MPS for an external
solver), and the A-gap.  Runtimes are GPU device times per run.
Writes a markdown table and (--json) the rows with every run's raw result, the
start schedule and the parameters, from which tests/test_gpu_protocol.py re-runs
run 1 of each size on the CPU oracle (this tool itself never touches oracle/).

    python tools/paper_protocol.py --out profiles/r02/paper_protocol.md
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]

import exact  # noqa: E402
from paper_2002_11710_b200 import airsched as A  # noqa: E402
from paper_2002_11710_b200 import instgen  # noqa: E402


def paper_instance(n, seed):
    cfg = instgen.Config(f"paper{n}", n, 8, 4, 8, 4, 40, "ontario", 6, 1000, 10)
    return instgen.generate(cfg, seed=seed)


def ilp(inst, time_limit):
    t0 = time.perf_counter()
    opt = exact.solve(inst, time_limit=time_limit)
    return opt, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "paper_protocol.md"))
    ap.add_argument("--json", default=None, help="also write the rows as JSON lines")
    ap.add_argument("--mps-dir", default=None, help="write each instance's model (MPS) here")
    ap.add_argument("--runs", type=int, default=10)
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--ilp-time", type=float, default=120.0)
    ap.add_argument("--sizes", default="12,15,18,21,24,27,30,33")
    args = ap.parse_args()
    ctx = A.Ctx(0)
    rows = []
    for n in [int(x) for x in args.sizes.split(",")]:
        inst = paper_instance(n, 2002117100 + 100 + n)
        h = A.Instance(inst)
        p, m, nrep = A.as_init_greedy(ctx, h)
        start = h.check(p, m)[1]
        R = args.runs
        seeds = np.arange(1, R + 1, dtype=np.uint64)
        out = {}
        for name, mode in (("NS", A.AS_MODE_NS), ("TS", A.AS_MODE_TABU)):
            res = np.zeros(R, A.RESULT_DTYPE)
            prm = A.params(mode=mode, tenure=10, max_iters=args.iters, kick=4)
            A.as_batch_run(ctx, h, R, p, m, prm, seeds, results=res)
            ms = ctx.last_kernel_ms
            objs = res["best_obj"] / 3600.0
            out[name] = dict(U=float(objs.max()), L=float(objs.min()), A=float(objs.mean()), ms=ms,
                             iters=int(res["iters_done"].mean()), raw=res["best_obj"].tolist())

        if args.mps_dir:
            os.makedirs(args.mps_dir, exist_ok=True)
            exact.export_mps(inst, os.path.join(args.mps_dir, f"paper_n{n}.mps"))
        opt, t_ilp = ilp(inst, args.ilp_time)
        rows.append(dict(n=n, seed=2002117100 + 100 + n, start_h=start / 3600.0,
                         opt_h=None if opt is None else opt / 3600.0, t_ilp=t_ilp,
                         start_ptr=p.tolist(), start_ms=m.tolist(), iters=args.iters, tenure=10, kick=4, **out))
        print(json.dumps({k: (v if not isinstance(v, dict) else {kk: vv for kk, vv in v.items() if kk != "raw"})
                          for k, v in rows[-1].items()}), flush=True)
    lines = ["# Paper protocol (§5) on synthetic instances — SURVEY §8(f) f4", "",
             "12 vehicles (8 helicopter + 4 plane, one per base), Ontario-like geography, deadlines within 24 h; "
             f"Alg. 1 start; {args.runs} runs per algorithm (seeded 4-relocate kicks), {args.iters} iterations, "
             "tabu tenure 10; objective in hours (P:427). Optimum: arc ILP (Eqs. obj_s, con1-con13) solved by scipy "
             f"HiGHS with a {args.ilp_time:.0f} s limit (test-only stand-in for Gurobi); '—' = not proven in the limit. "
             "GPU time = one as_batch_run of all runs on one B200.", "",
             "| missions | start (h) | optimum (h) | ILP s | NS U / L / A (h) | TS U / L / A (h) | NS A-gap | TS A-gap | "
             "GPU ms NS / TS |", "|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        opt = r["opt_h"]
        g = (lambda a: f"{abs(100 * (a - opt) / opt) if abs(a - opt) < 1e-9 else 100 * (a - opt) / opt:.2f} %") if opt else (lambda a: "—")
        lines.append(f"| {r['n']} | {r['start_h']:.3f} | {opt:.3f} | {r['t_ilp']:.1f} | " if opt else
                     f"| {r['n']} | {r['start_h']:.3f} | — | {r['t_ilp']:.1f} | ")
        lines[-1] += (f"{r['NS']['U']:.3f} / {r['NS']['L']:.3f} / {r['NS']['A']:.3f} | "
                      f"{r['TS']['U']:.3f} / {r['TS']['L']:.3f} / {r['TS']['A']:.3f} | {g(r['NS']['A'])} | "
                      f"{g(r['TS']['A'])} | {r['NS']['ms']:.1f} / {r['TS']['ms']:.1f} |")
    lines += ["", "Paper (Tables P:446-481, its own data on an i9-7920X / GTX 1080 Ti): TS A-gap 1.6-6.3 %, NS A-gap "
              "2.0-7.1 %, Gurobi stuck beyond 27 missions, CUDA variants 0.5-0.7 s per run.", ""]
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    open(args.out, "w").write("\n".join(lines))
    if args.json:
        with open(args.json, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
