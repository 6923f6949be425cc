"""GPU parity for Algorithm 1 on the device and the batched randomized starts
(reading #41): every start against the oracle's
or_greedy_seeded (routes, status, repairs), bit-exact; then the starts feed
as_batch_run on the device."""
import dataclasses

import numpy as np
import pytest

from paper_2002_11710_b200 import instgen

pytestmark = pytest.mark.gpu


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


def _compare_batch(A, ctx, O, inst, seeds, mode, max_repairs=50):
    h = A.Instance(inst)
    ptr, ms, status, nrep = A.as_init_greedy_batch(ctx, h, len(seeds), seeds=seeds, insert_mode=mode,
                                                   max_repairs=max_repairs)
    n_ok = 0
    for r, s in enumerate(seeds):
        st, (p, m), nr, _ = O.greedy(insert_mode=mode, max_repairs=max_repairs, seed=int(s))
        assert (status[r] == 0) == (st == 0), f"start {r} (seed {s}): status {status[r]} vs oracle {st}"
        if st == 0:
            assert routes_of(ptr[r], ms[r]) == routes_of(p, m), f"start {r} (seed {s})"
            assert nrep[r] == nr
            n_ok += 1
        else:
            assert ptr[r][-1] == 0
    return n_ok, nrep


@pytest.mark.parametrize("cfg,no_wait", [("tiny", 0), ("ontario", 0), ("batched", 0), ("ontario", 1),
                                         ("batched", 1)])
def test_greedy_batch_parity(A, ctx, oracle_mod, cfg, no_wait):
    inst = dataclasses.replace(instgen.generate(cfg), no_wait=no_wait)
    O = oracle_mod.Oracle(inst)
    seeds = np.array([0] + list(range(1, 64)) + [2**63 + 5, 2**64 - 1], dtype=np.uint64)
    for mode in (0, 1):
        n_ok, _ = _compare_batch(A, ctx, O, inst, seeds, mode)
        if mode == 1:
            assert n_ok >= len(seeds) // 2


def test_greedy_batch_repairs(A, ctx, oracle_mod):
    """Seeded starts that need Alg. 1's repair step, found by a seed scan,
    with and without a repair budget."""
    found = 0
    for iseed in range(200):
        cfg = instgen.Config("r", 12, 2, 1, 1, 1, 8, "ontario", 4, 10, 3)
        inst = instgen.generate(cfg, seed=iseed)
        O = oracle_mod.Oracle(inst)
        seeds = np.arange(0, 32, dtype=np.uint64)
        reps = [O.greedy(insert_mode=1, seed=int(s))[2] for s in seeds]
        if max(reps) == 0:
            continue
        found += 1
        _, nrep = _compare_batch(A, ctx, O, inst, seeds, 1)
        assert nrep.max() >= 1
        _compare_batch(A, ctx, O, inst, seeds, 1, max_repairs=0)
        if found >= 4:
            break
    assert found >= 1


@pytest.mark.parametrize("cfg", ["large", "surge"])
def test_greedy_large(A, ctx, oracle_mod, cfg):
    inst = instgen.generate(cfg)
    O = oracle_mod.Oracle(inst)
    _compare_batch(A, ctx, O, inst, np.array([0, 7], np.uint64), 1)
    gp, gm, gn = A.as_init_greedy(ctx, A.Instance(inst), insert_mode=0)
    st, (p, m), nr, _ = O.greedy(insert_mode=0)
    assert st == 0 and routes_of(gp, gm) == routes_of(p, m) and gn == nr


def test_greedy_state_in_global(A, ctx, oracle_mod, monkeypatch, ctxopt):
    ctxopt(GREEDY_GLOBAL=1)
    for cfg in ("ontario", "batched"):
        inst = instgen.generate(cfg)
        O = oracle_mod.Oracle(inst)
        _compare_batch(A, ctx, O, inst, np.arange(0, 40, dtype=np.uint64), 1)


def test_greedy_starts_feed_batch_run(A, ctx, oracle_mod):
    """Device-resident pipeline: as_init_greedy_batch -> as_batch_run (per-run starts,
    shared_start = 0), sampled runs against the oracle from the oracle's own starts."""
    import torch
    inst = instgen.generate("batched")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    c = instgen.CONFIGS["batched"]
    R, iters = 256, 120
    dev = torch.device("cuda:0")
    seeds = torch.arange(1000, 1000 + R, dtype=torch.int64, device=dev)
    tp = torch.zeros((R, inst.n_vehicles + 1), dtype=torch.int32, device=dev)
    tm = torch.zeros((R, inst.n_missions), dtype=torch.int32, device=dev)
    tst = torch.zeros(R, dtype=torch.int32, device=dev)
    A.as_init_greedy_batch(ctx, h, R, seeds=seeds, insert_mode=1, ptr_out=tp, ms_out=tm, status_out=tst,
                           nrep_out=torch.zeros(R, dtype=torch.int32, device=dev))
    tres = torch.zeros((R, 40), dtype=torch.uint8, device=dev)
    prm = A.params(mode=1, tenure=c.tenure, max_iters=iters)
    A.as_batch_run(ctx, h, R, tp, tm, prm, seeds, shared_start=False, results=tres)
    torch.cuda.synchronize()
    res = tres.cpu().numpy().view(A.RESULT_DTYPE).reshape(R)
    status = tst.cpu().numpy()
    starts = set()
    for r in (0, 1, 100, R - 1):
        st, (p, m), _, _ = O.greedy(insert_mode=1, seed=1000 + r)
        if st != 0:
            assert status[r] != 0 and res[r]["stop_reason"] == A.AS_STOP_INFEASIBLE_START
            continue
        o = O.search(p, m, mode=1, tenure=c.tenure, max_iters=iters, seed=1000 + r)
        assert res[r]["start_obj"] == O.objective(p, m)
        assert res[r]["best_obj"] == o["best_obj"] and res[r]["iters_done"] == o["iters_done"]
        assert res[r]["best_iter"] == o["best_iter"]
        starts.add(int(res[r]["start_obj"]))
    assert len(starts) >= 2
    assert ((status != 0) == (res["stop_reason"] == A.AS_STOP_INFEASIBLE_START)).all()
