"""Full-length, bit-exact trace parity on the large configs (BASELINE.json north_star:
"every chosen move ... and the final schedule ... on all 5 configs").

C4 (n=500, V=40): TS 20,000 iterations and NS to its local optimum.
C5 (n=4000, V=100, 32.4 M indices per iteration): TS 1,000 iterations and NS
(up to 1,000 iterations).  The CUDA path runs through the C ABI (as_tabu_run /
as_nbhd_run on the whole-GPU kernel) with full traces; the oracle side is
oracle.search_par, the chunk-parallel / memoised driver of the same oracle
arithmetic, itself pinned to the plain or_search in tests/test_oracle_driver.py.
Compared: every iteration's (index, delta, cur, best, class), the final tabu
expiry matrix, the best schedule, and the run counters.
"""
import os

import numpy as np
import pytest

from paper_2002_11710_b200 import instgen

pytestmark = [pytest.mark.gpu, pytest.mark.fulllength]


@pytest.fixture(scope="module")
def A():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2002_11710_b200 import airsched
    return airsched


@pytest.fixture(scope="module")
def ctx(A):
    return A.Ctx(0)


def routes_of(ptr, ms):
    return [list(map(int, ms[ptr[v]:ptr[v + 1]])) for v in range(len(ptr) - 1)]


def compare_full(A, ctx, O, h, p, m, mode, tenure, iters):
    prm = A.params(mode=mode, tenure=tenure, max_iters=iters, trace_level=1)
    run = A.as_tabu_run if mode == 1 else A.as_nbhd_run
    g = run(ctx, h, p, m, prm, want_trace=True, want_tabu=(mode == 1))
    o = O.search_par(p, m, mode=mode, tenure=tenure, max_iters=iters, threads=os.cpu_count(), memo=True)
    gt, ot = g["trace"], o["trace"]
    assert g["iters_done"] == o["iters_done"] and g["stop_reason"] == o["stop_reason"]
    bad = np.flatnonzero(gt["idx"] != ot["idx"])
    assert bad.size == 0, f"first divergence at iteration {bad[0]}"
    for k in ("delta", "cur", "best", "cls"):
        assert (gt[k] == ot[k]).all(), k
    if mode == 1:
        assert (g["tabu"] == o["E"]).all()
    assert g["best_obj"] == o["best_obj"] and g["final_obj"] == o["final_obj"] and g["best_iter"] == o["best_iter"]
    assert g["start_obj"] == o["start_obj"]
    assert routes_of(*g["best"]) == routes_of(*o["best"])
    return g, o


def start(A, ctx, h, O):
    p, m, _ = A.as_init_greedy(ctx, h)
    st, (op, om), _, _ = O.greedy()
    assert st == 0 and (p == op).all() and (m == om).all()
    return p, m


def test_large_c4_full_length(A, ctx, oracle_mod):
    inst = instgen.generate("large")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start(A, ctx, h, O)
    c = instgen.CONFIGS["large"]
    g, _ = compare_full(A, ctx, O, h, p, m, 1, c.tenure, c.max_iters)
    assert g["iters_done"] == c.max_iters
    g, _ = compare_full(A, ctx, O, h, p, m, 0, 0, c.max_iters)
    assert g["stop_reason"] == 1          # NS reached its local optimum


def test_surge_c5_full_length(A, ctx, oracle_mod):
    inst = instgen.generate("surge")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start(A, ctx, h, O)
    c = instgen.CONFIGS["surge"]
    g, _ = compare_full(A, ctx, O, h, p, m, 1, c.tenure, c.max_iters)
    assert g["iters_done"] == c.max_iters
    compare_full(A, ctx, O, h, p, m, 0, 0, c.max_iters)


def test_bench_configuration_64_runs(A, ctx, oracle_mod):
    """BASELINE configs[2] in bench.py's exact launch configuration (4096 runs x 1000
    iterations, shared Alg. 1 start, seeds 1..4096, kick 8, device-resident buffers):
    64 runs spread over the batch (every CTA position and warp slot class) equal the
    oracle run for run: best/final objective, best iteration, kicks, best schedule."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    inst = instgen.generate("batched")
    O = oracle_mod.Oracle(inst)
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
    assert (res["iters_done"] == iters).all()
    sample = sorted(set(np.linspace(0, R - 1, 58).astype(int).tolist()) |
                    {1, 27, 28, 29, 895, 896, 2047, 4095})

    def one(r):
        return r, O.search_par(p, m, mode=1, tenure=c.tenure, max_iters=iters, seed=r + 1, kick=c.kick,
                               threads=1, memo=True, trace=False)

    with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
        outs = list(ex.map(one, sample))
    assert len(outs) >= 64
    for r, o in outs:
        assert res[r]["best_obj"] == o["best_obj"] and res[r]["final_obj"] == o["final_obj"], r
        assert res[r]["best_iter"] == o["best_iter"] and res[r]["kicks_applied"] == o["kicks_applied"], r
        assert routes_of(bp[r], bm[r]) == routes_of(*o["best"]), r


def test_large_c4_nowait_full_length(A, ctx, oracle_mod):
    """f3 at C4's full length: the no-wait variant of C4 on the whole-GPU kernel (k_grid<..., NW>), TS for
    all 20,000 iterations and NS to its local optimum, against the oracle's no-wait trajectory."""
    import dataclasses
    inst = dataclasses.replace(instgen.generate("large"), no_wait=1)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start(A, ctx, h, O)
    c = instgen.CONFIGS["large"]
    g, _ = compare_full(A, ctx, O, h, p, m, 1, c.tenure, c.max_iters)
    assert g["iters_done"] == c.max_iters
    g, _ = compare_full(A, ctx, O, h, p, m, 0, 0, c.max_iters)
    assert g["stop_reason"] == 1
