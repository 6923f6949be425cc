"""GPU parity for the no-wait model variant (reading #40).

With no_wait the vehicle departs a mission on arrival, so a move shifts every
later arrival of a route; the CUDA path checks the shifted stretches against
their slack (engine.cuh nw_*), the oracle re-simulates each candidate route
(oracle.c or_route_feasible).  Same bar as the waiting model: bit-exact.

Instances: the generator's configurations with no_wait = 1, some with their
deadlines scaled down (w' = max(1, floor(s w))) so the time constraints bind;
states come from the oracle's own no-wait trajectories, most of which are
infeasible under the waiting rule (so the waiting-model arithmetic cannot pass
these tests by accident).
"""
import dataclasses

import numpy as np
import pytest

from e1 import e1_instance
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


def nowait(cfg, scale=1.0):
    inst = instgen.generate(cfg)
    w = np.maximum(1, np.floor(inst.deadline_s * scale)).astype(np.int32)
    return dataclasses.replace(inst, no_wait=1, deadline_s=w)


def decode_key(key):
    if key == 0xFFFFFFFFFFFFFFFF:
        return (-1, 0, -1)
    return (key >> 63, int(((key >> 32) & 0x7FFFFFFF) - (1 << 30)), key & 0xFFFFFFFF)


def routes_of(ptr, ms):
    return [list(map(int, ms[ptr[v]:ptr[v + 1]])) for v in range(len(ptr) - 1)]


def nw_states(O, tenure, n_ts=(5, 23, 60), kicks=(3, 9)):
    st, (p, m), _, _ = O.greedy()
    assert st == 0
    out = [(p, m)]
    for it in n_ts:
        out.append(O.search(p, m, mode=1, tenure=tenure, max_iters=it, trace=False)["final"])
    for s in kicks:
        out.append(O.kick(p, m, s, 12)[1])
    return out


def test_e1_nowait_eval(A, ctx, oracle_mod):
    """E1 with deadlines (3000, 2000, 3000): idx 2 (v0 = [m1, m0, m2]) is feasible
    only without waiting (tests/test_oracle.py::test_e1_nowait_golden, by hand)."""
    base = e1_instance()
    base.deadline_s = np.array([3000, 2000, 3000], np.int32)
    ptr, ms = np.array([0, 3, 3], np.int32), np.array([0, 1, 2], np.int32)
    inst = dataclasses.replace(base, no_wait=1)
    d, f, key = A.as_eval_moves(ctx, A.Instance(inst), ptr, ms, mode=A.AS_MODE_NS)
    od, of, ok = oracle_mod.Oracle(inst).eval_moves(ptr, ms, mode=0)
    assert (d == od).all() and (f == of).all() and decode_key(key) == ok
    assert d[2] == 200 and f[2] & 2
    # under the waiting rule the start itself is infeasible (m0 departs at 3000 > w_m1 - 700)
    with pytest.raises(A.AirschedError) as e:
        A.as_eval_moves(ctx, A.Instance(dataclasses.replace(base, no_wait=0)), ptr, ms, mode=A.AS_MODE_NS)
    assert e.value.status == A.AS_ERR_INFEASIBLE_START


@pytest.mark.parametrize("cfg,scale", [("tiny", 1.0), ("tiny", 0.5), ("tiny", 0.3), ("ontario", 1.0),
                                       ("batched", 1.0), ("batched", 0.5)])
def test_nowait_eval_parity(A, ctx, oracle_mod, cfg, scale):
    inst = nowait(cfg, scale)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    rng = np.random.default_rng(17)
    n_wait_infeasible = 0
    Ow = oracle_mod.Oracle(dataclasses.replace(inst, no_wait=0))
    for p, m in nw_states(O, instgen.CONFIGS[cfg].tenure):
        n_wait_infeasible += not Ow.feasible(p, m)
        obj = O.objective(p, m)
        for mode in (0, 1):
            E, it, best = None, 0, obj
            if mode == 1:
                it = int(rng.integers(5, 40))
                E = rng.integers(-1, it + 8, size=(inst.n_missions, inst.n_vehicles)).astype(np.int32)
                best = obj - int(rng.integers(0, 2000))
            od, of, ok = O.eval_moves(p, m, mode=mode, E=E, it=it, best_obj=best)
            gd, gf, key = A.as_eval_moves(ctx, h, p, m, mode=mode, tabu_expiry=E, iter=it, best_obj=best)
            assert (gf == of).all(), f"flags differ at {np.flatnonzero(gf != of)[:10]}"
            assert (gd == od).all()
            assert decode_key(key) == ok
    assert n_wait_infeasible >= 1


def _compare_run(A, ctx, O, h, p, m, mode, tenure, iters, digest=False, seed=0, kick=0):
    prm = A.params(mode=mode, tenure=tenure, max_iters=iters, trace_level=2 if digest else 1, seed=seed, kick=kick)
    g = A.as_tabu_run(ctx, h, p, m, prm, want_trace=True, want_digest=digest, want_tabu=(mode == 1))
    o = O.search(p, m, mode=mode, tenure=tenure, max_iters=iters, digest=digest, seed=seed, kick=kick)
    ot, gt = o["trace"], g["trace"]
    assert g["iters_done"] == o["iters_done"] and g["stop_reason"] == o["stop_reason"]
    assert (gt["idx"] == ot["idx"]).all(), f"first divergence at it {np.flatnonzero(gt['idx'] != ot['idx'])[:1]}"
    assert (gt["delta"] == ot["delta"]).all() and (gt["cur"] == ot["cur"]).all()
    assert (gt["best"] == ot["best"]).all() and (gt["cls"] == ot["cls"]).all()
    if digest:
        assert (g["digest"] == ot["digest"]).all()
    if mode == 1:
        assert (g["tabu"] == o["E"]).all()
    assert g["best_obj"] == o["best_obj"] and g["final_obj"] == o["final_obj"] and g["best_iter"] == o["best_iter"]
    assert g["kicks_applied"] == o["kicks_applied"]
    assert routes_of(*g["best"]) == routes_of(*o["best"])
    assert O.feasible(*g["best"])
    return g


@pytest.mark.parametrize("cfg,scale,iters,digest", [("tiny", 1.0, 200, True), ("tiny", 0.3, 200, True),
                                                    ("ontario", 1.0, 1500, True), ("batched", 0.5, 600, False)])
def test_nowait_run_parity(A, ctx, oracle_mod, cfg, scale, iters, digest):
    inst = nowait(cfg, scale)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    st, (p, m), _, _ = O.greedy()
    t = instgen.CONFIGS[cfg].tenure
    _compare_run(A, ctx, O, h, p, m, 1, t, iters, digest=digest)
    _compare_run(A, ctx, O, h, p, m, 0, 0, iters)
    _compare_run(A, ctx, O, h, p, m, 1, t, iters // 2, seed=99, kick=8)


def test_nowait_large_prefix(A, ctx, oracle_mod):
    inst = nowait("large")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    st, (p, m), _, _ = O.greedy()
    _compare_run(A, ctx, O, h, p, m, 1, 10, 15)


def test_nowait_batch_parity(A, ctx, oracle_mod):
    inst = nowait("batched", 0.5)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    c = instgen.CONFIGS["batched"]
    st, (p, m), _, _ = O.greedy()
    R, iters = 64, 150
    seeds = np.arange(1, R + 1, dtype=np.uint64)
    res = np.zeros(R, A.RESULT_DTYPE)
    bp = np.zeros((R, inst.n_vehicles + 1), np.int32)
    bm = np.zeros((R, inst.n_missions), np.int32)
    prm = A.params(mode=1, tenure=c.tenure, max_iters=iters, kick=c.kick)
    best_run = A.as_batch_run(ctx, h, R, p, m, prm, seeds, shared_start=True, results=res, best_ptr_out=bp,
                              best_missions_out=bm, want_best_run=True)
    assert best_run == int(np.lexsort((np.arange(R), res["best_obj"]))[0])
    for r in (0, 5, R - 1):
        o = O.search(p, m, mode=1, tenure=c.tenure, max_iters=iters, seed=int(seeds[r]), kick=c.kick)
        assert res[r]["best_obj"] == o["best_obj"] and res[r]["iters_done"] == o["iters_done"]
        assert res[r]["best_iter"] == o["best_iter"] and res[r]["kicks_applied"] == o["kicks_applied"]
        assert routes_of(bp[r], bm[r]) == routes_of(*o["best"])


def test_nowait_greedy_parity(A, ctx, oracle_mod):
    n_fail = n_ok = 0
    for cfg, scale in [("tiny", 1.0), ("tiny", 0.3), ("ontario", 1.0), ("ontario", 0.5), ("batched", 0.5),
                       ("large", 1.0)]:
        inst = nowait(cfg, scale)
        O = oracle_mod.Oracle(inst)
        h = A.Instance(inst)
        for mode in (0, 1):
            st, (p, m), nrep, _ = O.greedy(insert_mode=mode)
            if st != 0:
                n_fail += 1
                with pytest.raises(A.AirschedError):
                    A.as_init_greedy(ctx, h, insert_mode=mode)
                continue
            n_ok += 1
            gp, gm, gn = A.as_init_greedy(ctx, h, insert_mode=mode)
            assert routes_of(gp, gm) == routes_of(p, m) and gn == nrep
    assert n_ok >= 6 and n_fail >= 1


def test_nowait_unsupported_paths(A, ctx, oracle_mod, monkeypatch, ctxopt):
    inst = nowait("tiny")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    st, (p, m), _, _ = O.greedy()
    with pytest.raises(A.AirschedError) as e:
        A.as_tabu_run(ctx, h, p, m, A.params(mode=1, tenure=3, max_iters=10, sweep=1))
    assert e.value.status == A.AS_ERR_UNSUPPORTED
    ctxopt(SHARDED=1)
    with pytest.raises(A.AirschedError) as e:
        A.as_tabu_run(ctx, h, p, m, A.params(mode=1, tenure=3, max_iters=10))
    assert e.value.status == A.AS_ERR_UNSUPPORTED


@pytest.mark.parametrize("cfg,scale,iters", [("tiny", 1.0, 200), ("tiny", 0.3, 200), ("ontario", 1.0, 800),
                                             ("batched", 0.5, 400), ("ontario", 0.6, 600)])
def test_nowait_batch_kernel_single_runs(A, ctx, oracle_mod, cfg, scale, iters, ctxopt):
    """f3 on the batched kernel (one run per warp, exact no-wait evaluation of every move):
    single runs forced onto it -- full traces, final tabu matrix, best schedule, TS (plain and
    kicked) and NS, against the oracle."""
    ctxopt(BATCH_KERNEL=1)
    inst = nowait(cfg, scale)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    st, (p, m), _, _ = O.greedy()
    assert st == 0
    t = instgen.CONFIGS[cfg].tenure
    _compare_run(A, ctx, O, h, p, m, 1, t, iters)
    _compare_run(A, ctx, O, h, p, m, 0, 0, iters)
    _compare_run(A, ctx, O, h, p, m, 1, t, iters // 2, seed=17, kick=8)


def test_nowait_batch_kernel_traces(A, ctx, oracle_mod, ctxopt):
    """A whole no-wait batch on the batched kernel (option BATCH_KERNEL=1; the default for no-wait
    batches is the per-run kernel): per-run traces of sampled runs equal the oracle's."""
    ctxopt(BATCH_KERNEL=1)
    inst = nowait("ontario", 0.7)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    st, (p, m), _, _ = O.greedy()
    R, iters = 96, 300
    seeds = np.arange(1, R + 1, dtype=np.uint64)
    res = np.zeros(R, A.RESULT_DTYPE)
    tr = np.zeros((R, iters), A.TRACE_DTYPE)
    for mode, tenure in ((1, 10), (0, 0)):
        prm = A.params(mode=mode, tenure=tenure, max_iters=iters, kick=6, trace_level=1)
        A.as_batch_run(ctx, h, R, p, m, prm, seeds, shared_start=True, results=res, trace_out=tr)
        for r in (0, 31, 32, 95):
            o = O.search(p, m, mode=mode, tenure=tenure, max_iters=iters, seed=int(seeds[r]), kick=6)
            k = o["iters_done"]
            assert res[r]["iters_done"] == k and res[r]["best_obj"] == o["best_obj"]
            assert (tr[r]["idx"][:k] == o["trace"]["idx"]).all() and (tr[r]["cur"][:k] == o["trace"]["cur"]).all()


@pytest.mark.parametrize("cfg,scale,iters,opts", [
    ("tiny", 1.0, 200, {"GRID": 1}),
    ("tiny", 0.3, 200, {"GRID": 1, "GRID_BLOCKS": 1}),
    ("ontario", 1.0, 800, {"GRID": 1}),
    ("ontario", 0.6, 600, {"GRID": 1, "GRID_T_GLOBAL": 1, "GRID_G": 3}),
    ("batched", 0.5, 400, {"GRID": 1, "GRID_T_GLOBAL": 1, "GRID_E_GLOBAL": 1}),
    ("batched", 0.5, 300, {"GRID": 1, "GRID_COMPACT": 0, "GRID_G": 7}),
    ("large", 1.0, 40, {"GRID": 1}),
])
def test_nowait_grid_runs(A, ctx, oracle_mod, cfg, scale, iters, opts, ctxopt):
    """f3 on the whole-GPU kernel (k_grid<..., NW>: general scorers with the engine's exact
    no-wait evaluation, whole-route refresh of the two changed routes): full traces, final tabu
    matrix, best schedule, TS (plain and kicked) and NS, against the oracle -- shared and global
    tables, one CTA and the whole grid, compact and full tile lists."""
    ctxopt(**opts)
    inst = nowait(cfg, scale)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    st, (p, m), _, _ = O.greedy()
    assert st == 0
    t = instgen.CONFIGS[cfg].tenure
    _compare_run(A, ctx, O, h, p, m, 1, t, iters)
    _compare_run(A, ctx, O, h, p, m, 0, 0, iters)
    _compare_run(A, ctx, O, h, p, m, 1, t, max(iters // 2, 1), seed=17, kick=8)


def test_nowait_grid_surge_prefix(A, ctx, oracle_mod):
    """C5-sized no-wait instance (n=4000, V=100) on the whole-GPU kernel (it holds no on-chip copy
    for the per-CTA kernel): the first TS and NS iterations equal the oracle's (chunk-parallel
    driver of the same arithmetic, tests/test_oracle_driver.py)."""
    import os
    inst = nowait("surge")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    st, (p, m), _, _ = O.greedy()
    assert st == 0
    for mode, tenure, iters in ((1, 10, 4), (0, 0, 3)):
        prm = A.params(mode=mode, tenure=tenure, max_iters=iters, trace_level=1)
        g = A.as_tabu_run(ctx, h, p, m, prm, want_trace=True, want_tabu=(mode == 1))
        o = O.search_par(p, m, mode=mode, tenure=tenure, max_iters=iters, threads=os.cpu_count(), memo=True)
        assert g["iters_done"] == o["iters_done"] and g["stop_reason"] == o["stop_reason"]
        for k in ("idx", "delta", "cur", "best", "cls"):
            assert (g["trace"][k] == o["trace"][k]).all(), k
        if mode == 1:
            assert (g["tabu"] == o["E"]).all()
        assert routes_of(*g["best"]) == routes_of(*o["best"])
