"""Extended parity evidence for the bench's C3 launch (4096 runs x 1000 TS iterations, shared Alg. 1 start,
seeds 1..4096, kick 8, device-resident buffers): K runs spread over the batch, each equal to the oracle run
(best/final objective, best iteration, kicks, best schedule).  usage: c3_parity_sample.py [K]
(the committed test, tests/test_gpu_fulllength.py, checks 64 runs)"""
import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import oracle
    from paper_2002_11710_b200 import airsched as A
    from paper_2002_11710_b200 import instgen
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    inst = instgen.generate("batched")
    O = oracle.Oracle(inst)
    ctx = A.Ctx(0)
    h = A.Instance(inst)
    c = instgen.CONFIGS["batched"]
    p, m, _ = A.as_init_greedy(ctx, h)
    R, iters = c.n_runs, c.max_iters
    dev = torch.device("cuda:0")
    tp, tm = torch.from_numpy(p).to(dev), torch.from_numpy(m).to(dev)
    ts = torch.from_numpy(np.arange(1, R + 1, dtype=np.uint64).view(np.int64)).to(dev)
    tres = torch.zeros((R, 40), dtype=torch.uint8, device=dev)
    tbp = torch.zeros((R, inst.n_vehicles + 1), dtype=torch.int32, device=dev)
    tbm = torch.zeros((R, inst.n_missions), dtype=torch.int32, device=dev)
    prm = A.params(mode=1, tenure=c.tenure, max_iters=iters, kick=c.kick)
    A.as_batch_run(ctx, h, R, tp, tm, prm, ts, shared_start=True, results=tres, best_ptr_out=tbp,
                   best_missions_out=tbm)
    torch.cuda.synchronize()
    res = tres.cpu().numpy().view(A.RESULT_DTYPE).reshape(R)
    bp, bm = tbp.cpu().numpy(), tbm.cpu().numpy()
    sample = sorted(set(np.linspace(0, R - 1, K).astype(int).tolist()))

    def one(r):
        return r, O.search_par(p, m, mode=1, tenure=c.tenure, max_iters=iters, seed=r + 1, kick=c.kick, threads=1,
                               memo=True, trace=False)

    bad = []
    with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
        for r, o in ex.map(one, sample):
            ok = (res[r]["best_obj"] == o["best_obj"] and res[r]["final_obj"] == o["final_obj"] and
                  res[r]["best_iter"] == o["best_iter"] and res[r]["kicks_applied"] == o["kicks_applied"])
            ptr, ms = o["best"]
            ok = ok and all((bm[r][bp[r][v]:bp[r][v + 1]] == ms[ptr[v]:ptr[v + 1]]).all() and
                            bp[r][v + 1] - bp[r][v] == ptr[v + 1] - ptr[v] for v in range(inst.n_vehicles))
            if not ok:
                bad.append(r)
    print(json.dumps({"workload": "C3 bench launch (4096 runs x 1000 TS iterations)", "runs_checked": len(sample),
                      "mismatches": bad, "all_equal": not bad}))


if __name__ == "__main__":
    main()
