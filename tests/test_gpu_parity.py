"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact.

Every comparison is element by element on seeded synthetic inputs
(paper_2002_11710_b200/instgen.py).  Integer work => the bar is exact equality
(BASELINE.json north_star: "bit-exact").  The selection key is compared by
decoding (class, delta, idx) from the key and comparing with the oracle's
selected move.
"""
import json
import os

import numpy as np
import pytest

from e1 import e1_instance
from paper_2002_11710_b200 import instgen

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "e1.json")))


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


def decode_key(key):
    if key == 0xFFFFFFFFFFFFFFFF:
        return (-1, 0, -1)
    return (key >> 63, int(((key >> 32) & 0x7FFFFFFF) - (1 << 30)), key & 0xFFFFFFFF)


def routes_of(ptr, ms):
    return [list(map(int, ms[ptr[v]:ptr[v + 1]])) for v in range(len(ptr) - 1)]


def start_of(O, inst):
    st, (p, m), _, _ = O.greedy()
    if st != 0:
        p, m = inst.planted_ptr, inst.planted_missions
    return p, m


def states_for(O, inst, n_ts=(5, 23), kicks=(3, 9)):
    p, m = start_of(O, inst)
    out = [(p, m)]
    for it in n_ts:
        out.append(O.search(p, m, mode=1, tenure=3, max_iters=it, trace=False)["final"])
    for s in kicks:
        out.append(O.kick(p, m, s, 12)[1])
    return out


# ----------------------------------------------------------------- E1 golden --
def test_e1_eval_golden(A, ctx, oracle_mod):
    I = e1_instance()
    h = A.Instance(I)
    ptr, ms = np.array([0, 3, 3], np.int32), np.array([0, 1, 2], np.int32)
    d, f, key = A.as_eval_moves(ctx, h, ptr, ms, mode=A.AS_MODE_NS)
    for k, mv in GOLD["moves"].items():
        assert d[int(k)] == mv["delta"] and bool(f[int(k)] & 2) == mv["feasible"]
    assert int((f & 1).sum()) == GOLD["valid_count"]
    assert decode_key(key) == (0, -1160, 9)


def test_e1_runs_golden(A, ctx):
    I = e1_instance()
    h = A.Instance(I)
    ptr, ms = np.array([0, 3, 3], np.int32), np.array([0, 1, 2], np.int32)
    g = GOLD["ts_tenure2"]
    r = A.as_tabu_run(ctx, h, ptr, ms, A.params(mode=1, tenure=2, max_iters=4, trace_level=1), want_trace=True)
    tr = r["trace"]
    assert list(tr["idx"]) == g["idx"] and list(tr["delta"]) == g["delta"]
    assert list(tr["cur"]) == g["cur"] and list(tr["best"]) == g["best"] and list(tr["cls"]) == g["cls"]
    rn = A.as_nbhd_run(ctx, h, ptr, ms, A.params(mode=0, max_iters=10, trace_level=1), want_trace=True)
    assert list(rn["trace"]["idx"]) == GOLD["ns"]["idx"] and rn["best_obj"] == 640 and rn["stop_reason"] == 1
    rs = A.as_tabu_run(ctx, h, ptr, ms, A.params(mode=1, tenure=2, max_iters=8, strict_tabu_stop=1))
    assert rs["iters_done"] == 2 and rs["stop_reason"] == 2
    gp, gm, nrep = A.as_init_greedy(ctx, h)
    assert routes_of(gp, gm) == GOLD["greedy_tail"]["routes"]


# ------------------------------------------------------- as_eval_moves parity --
@pytest.mark.parametrize("cfg", ["tiny", "ontario", "batched", "large"])
def test_eval_moves_parity(A, ctx, oracle_mod, cfg):
    inst = instgen.generate(cfg)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    rng = np.random.default_rng(11)
    states = states_for(O, inst) if cfg != "large" else states_for(O, inst, n_ts=(3,), kicks=(5,))
    for si, (p, m) in enumerate(states):
        obj = O.objective(p, m)
        for mode in (0, 1):
            E = None
            it = 0
            best = obj
            if mode == 1:
                it = int(rng.integers(5, 40))
                E = rng.integers(-1, it + 8, size=(inst.n_missions, inst.n_vehicles)).astype(np.int32)
                best = obj - int(rng.integers(0, 2000))
            od, of, (bc, bd, bi) = O.eval_moves(p, m, mode=mode, E=E, it=it, best_obj=best)
            gd, gf, key = A.as_eval_moves(ctx, h, p, m, mode=mode, tabu_expiry=E, iter=it, best_obj=best)
            assert (gf == of).all(), f"flags differ at {np.flatnonzero(gf != of)[:10]}"
            assert (gd == od).all(), f"delta differs at {np.flatnonzero(gd != od)[:10]}"
            assert decode_key(key) == (bc, bd, bi) if bc >= 0 else key == 0xFFFFFFFFFFFFFFFF


def test_eval_moves_surge_sampled(A, ctx, oracle_mod):
    """Full C5 size (n=4000, V=100, 32.4 M indices): GPU dump vs oracle on a
    seeded sample of indices (every row touched), plus the selected key against
    a full oracle scan."""
    inst = instgen.generate("surge")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    p2, m2 = O.kick(p, m, 77, 40)[1]
    rng = np.random.default_rng(5)
    N = h.move_space_size
    idx = np.unique(np.concatenate([rng.integers(0, N, 200000), np.arange(0, N, 4001)]))
    E = rng.integers(-1, 30, size=(inst.n_missions, inst.n_vehicles)).astype(np.int32)
    obj = O.objective(p2, m2)
    od, of = O.eval_indices(p2, m2, idx, mode=1, E=E, it=20, best_obj=obj - 100)
    gd, gf, key = A.as_eval_moves(ctx, h, p2, m2, mode=1, tabu_expiry=E, iter=20, best_obj=obj - 100)
    assert (gf[idx] == of).all() and (gd[idx] == od).all()
    assert int((gf & 1).sum()) == h.valid_moves_per_iter


def test_partial_schedule_eval(A, ctx, oracle_mod):
    inst = instgen.generate("ontario")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    keep = [x for x in m if x % 3 != 0]
    routes = [[x for x in r if x in set(keep)] for r in routes_of(p, m)]
    pp = np.zeros(len(routes) + 1, np.int32)
    pp[1:] = np.cumsum([len(r) for r in routes])
    mm = np.array([x for r in routes for x in r], np.int32)
    od, of, ob = O.eval_moves(pp, mm, mode=0)
    gd, gf, key = A.as_eval_moves(ctx, h, pp, mm, mode=0)
    assert (gd == od).all() and (gf == of).all() and decode_key(key) == ob


# ------------------------------------------------------------- run parity --
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
    assert g["start_obj"] == o["start_obj"] and g["kicks_applied"] == o["kicks_applied"]
    assert routes_of(*g["best"]) == routes_of(*o["best"])
    return g


@pytest.mark.parametrize("cfg,iters,digest", [("tiny", 200, True), ("ontario", 5000, True), ("batched", 1000, False)])
def test_tabu_run_parity(A, ctx, oracle_mod, cfg, iters, digest):
    inst = instgen.generate(cfg)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    c = instgen.CONFIGS[cfg]
    _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters, digest=digest)
    _compare_run(A, ctx, O, h, p, m, 0, 0, iters)


def test_large_run_parity_prefix(A, ctx, oracle_mod):
    """C4 (n=500, V=40) at full size, the first iterations of TS and NS."""
    inst = instgen.generate("large")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    _compare_run(A, ctx, O, h, p, m, 1, 10, 40)
    _compare_run(A, ctx, O, h, p, m, 0, 0, 40)


def test_kicked_runs_parity(A, ctx, oracle_mod):
    inst = instgen.generate("batched")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    for seed in (1, 2, 4096):
        _compare_run(A, ctx, O, h, p, m, 1, 10, 300, seed=seed, kick=8)


def test_batch_run_parity(A, ctx, oracle_mod):
    """as_batch_run in the bench's launch configuration (shared start, per-run
    seeds, kick 8), with sampled runs checked against the oracle."""
    import torch
    inst = instgen.generate("batched")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    c = instgen.CONFIGS["batched"]
    p, m = start_of(O, inst)
    R, iters = 512, 200
    seeds = np.arange(1, R + 1, dtype=np.uint64)
    res = np.zeros(R, A.RESULT_DTYPE)
    bp = np.zeros((R, inst.n_vehicles + 1), np.int32)
    bm = np.zeros((R, inst.n_missions), np.int32)
    tr = np.zeros((R, iters), A.TRACE_DTYPE)
    prm = A.params(mode=1, tenure=c.tenure, max_iters=iters, kick=c.kick, trace_level=1)
    best_run = A.as_batch_run(ctx, h, R, p, m, prm, seeds, shared_start=True, results=res, best_ptr_out=bp,
                              best_missions_out=bm, trace_out=tr, want_best_run=True)
    assert best_run == int(np.lexsort((np.arange(R), res["best_obj"]))[0])
    for r in (0, 1, 77, 300, R - 1):
        o = O.search(p, m, mode=1, tenure=c.tenure, max_iters=iters, seed=int(seeds[r]), kick=c.kick)
        assert res[r]["best_obj"] == o["best_obj"] and res[r]["iters_done"] == o["iters_done"]
        assert res[r]["kicks_applied"] == o["kicks_applied"] and res[r]["best_iter"] == o["best_iter"]
        assert (tr[r]["idx"][:o["iters_done"]] == o["trace"]["idx"]).all()
        assert routes_of(bp[r], bm[r]) == routes_of(*o["best"])
    # device-resident inputs/outputs (the bench's timed configuration)
    dev = torch.device("cuda:0")
    tp, tm = torch.from_numpy(p).to(dev), torch.from_numpy(m).to(dev)
    ts = torch.from_numpy(seeds.view(np.int64)).to(dev)
    tres = torch.zeros((R, 40), dtype=torch.uint8, device=dev)
    A.as_batch_run(ctx, h, R, tp, tm, prm, ts, shared_start=True, results=tres)
    torch.cuda.synchronize()
    res2 = tres.cpu().numpy().view(A.RESULT_DTYPE).reshape(R)
    assert (res2 == res).all()


def test_greedy_parity(A, ctx, oracle_mod):
    for cfg in instgen.CONFIGS:
        inst = instgen.generate(cfg)
        O = oracle_mod.Oracle(inst)
        h = A.Instance(inst)
        for mode in (0, 1):
            st, (p, m), nrep, _ = O.greedy(insert_mode=mode)
            if st != 0:
                with pytest.raises(A.AirschedError):
                    A.as_init_greedy(ctx, h, insert_mode=mode)
                continue
            gp, gm, gn = A.as_init_greedy(ctx, h, insert_mode=mode)
            assert routes_of(gp, gm) == routes_of(p, m) and gn == nrep


def test_greedy_repair_parity(A, ctx, oracle_mod):
    """Instances where Alg. 1 needs its repair step -- found by seed scan."""
    found = 0
    for seed in range(400):
        cfg = instgen.Config("r", 12, 2, 1, 1, 1, 8, "ontario", 4, 10, 3)
        inst = instgen.generate(cfg, seed=seed)
        O = oracle_mod.Oracle(inst)
        st, (p, m), nrep, _ = O.greedy()
        if nrep == 0:
            continue
        found += 1
        h = A.Instance(inst)
        if st != 0:
            with pytest.raises(A.AirschedError):
                A.as_init_greedy(ctx, h)
        else:
            gp, gm, gn = A.as_init_greedy(ctx, h)
            assert routes_of(gp, gm) == routes_of(p, m) and gn == nrep
        if found >= 5:
            break


# ------------------------------------------------------------- edge cases --
def test_edge_cases(A, ctx, oracle_mod):
    base = instgen.generate("tiny")
    # zero missions
    empty = instgen.Instance(base.travel_s, base.class_is_heli, base.base_location, base.vehicle_base,
                             base.vehicle_class, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32),
                             np.zeros(0, np.uint8))
    h = A.Instance(empty)
    p = np.zeros(base.n_vehicles + 1, np.int32)
    r = A.as_tabu_run(ctx, h, p, np.zeros(0, np.int32), A.params(max_iters=10))
    assert r["best_obj"] == 0 and r["stop_reason"] == A.AS_STOP_NO_MOVE and r["iters_done"] == 0
    # one mission, one vehicle
    one_cfg = instgen.Config("one", 1, 1, 0, 1, 0, 4, "ontario", 3, 10, 2)
    one = instgen.generate(one_cfg, seed=3)
    O = oracle_mod.Oracle(one)
    h = A.Instance(one)
    g = A.as_tabu_run(ctx, h, one.planted_ptr, one.planted_missions, A.params(max_iters=5))
    o = O.search(one.planted_ptr, one.planted_missions, max_iters=5)
    assert g["best_obj"] == o["best_obj"] and g["stop_reason"] == o["stop_reason"]
    # infeasible start -> AS_ERR_INFEASIBLE_START
    inst = instgen.generate("ontario")
    h = A.Instance(inst)
    bad_ptr = np.array([0] + [inst.n_missions] * inst.n_vehicles, np.int32)
    bad_ms = np.argsort(inst.deadline_s)[::-1].astype(np.int32)   # everything on vehicle 0, reversed
    with pytest.raises(A.AirschedError) as e:
        A.as_tabu_run(ctx, h, bad_ptr, bad_ms, A.params(max_iters=5))
    assert e.value.status == A.AS_ERR_INFEASIBLE_START
    # paper-only move set (inter-route relocate only)
    O = oracle_mod.Oracle(inst)
    p, m = start_of(O, inst)
    _compare_run_mask(A, ctx, O, A.Instance(inst), p, m)


def _compare_run_mask(A, ctx, O, h, p, m):
    prm = A.params(mode=1, tenure=10, max_iters=300, move_mask=A.AS_MOVE_INTER_RELOCATE, trace_level=1)
    g = A.as_tabu_run(ctx, h, p, m, prm, want_trace=True)
    o = O.search(p, m, mode=1, tenure=10, max_iters=300, mask=1)
    assert (g["trace"]["idx"] == o["trace"]["idx"]).all() and g["best_obj"] == o["best_obj"]


@pytest.mark.parametrize("cfg,runs,iters", [("tiny", 64, 200), ("ontario", 64, 300), ("large", 6, 30)])
def test_batch_kernel_parity_configs(A, ctx, oracle_mod, cfg, runs, iters):
    """The one-run-per-warp batch kernel on every instance shape it accepts, NS and TS,
    with per-run seeds; sampled runs compared with the oracle trace by trace."""
    inst = instgen.generate(cfg)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    c = instgen.CONFIGS[cfg]
    p, m = start_of(O, inst)
    seeds = np.arange(1, runs + 1, dtype=np.uint64)
    for mode in (1, 0):
        res = np.zeros(runs, A.RESULT_DTYPE)
        tr = np.zeros((runs, iters), A.TRACE_DTYPE)
        bp = np.zeros((runs, inst.n_vehicles + 1), np.int32)
        bm = np.zeros((runs, inst.n_missions), np.int32)
        prm = A.params(mode=mode, tenure=c.tenure, max_iters=iters, kick=4, trace_level=1)
        A.as_batch_run(ctx, h, runs, p, m, prm, seeds, shared_start=True, results=res, best_ptr_out=bp,
                       best_missions_out=bm, trace_out=tr)
        for r in sorted({0, runs // 2, runs - 1}):
            o = O.search(p, m, mode=mode, tenure=c.tenure, max_iters=iters, seed=int(seeds[r]), kick=4)
            k = o["iters_done"]
            assert res[r]["iters_done"] == k and res[r]["stop_reason"] == o["stop_reason"]
            assert (tr[r]["idx"][:k] == o["trace"]["idx"]).all()
            assert (tr[r]["cur"][:k] == o["trace"]["cur"]).all() and (tr[r]["cls"][:k] == o["trace"]["cls"]).all()
            assert res[r]["best_obj"] == o["best_obj"] and routes_of(bp[r], bm[r]) == routes_of(*o["best"])


def test_batch_per_run_starts(A, ctx, oracle_mod):
    """Distinct start schedules per run (shared_start = 0)."""
    inst = instgen.generate("ontario")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    starts = [O.kick(p, m, s, 10)[1] for s in range(1, 9)]
    R = len(starts)
    sp = np.stack([s[0] for s in starts]).astype(np.int32)
    sm = np.stack([s[1] for s in starts]).astype(np.int32)
    res = np.zeros(R, A.RESULT_DTYPE)
    prm = A.params(mode=1, tenure=10, max_iters=150)
    A.as_batch_run(ctx, h, R, sp, sm, prm, np.zeros(R, np.uint64), shared_start=False, results=res)
    for r in range(R):
        o = O.search(sp[r], sm[r], mode=1, tenure=10, max_iters=150)
        assert res[r]["best_obj"] == o["best_obj"] and res[r]["best_iter"] == o["best_iter"]
    # an infeasible start in a batch reports stop_reason 3 and the call still succeeds
    sm2 = sm.copy()
    sm2[3] = sm2[3][::-1]
    sp2 = sp.copy()
    sp2[3] = np.array([0] + [inst.n_missions] * inst.n_vehicles, np.int32)
    A.as_batch_run(ctx, h, R, sp2, sm2, prm, np.zeros(R, np.uint64), shared_start=False, results=res)
    assert res[3]["stop_reason"] == A.AS_STOP_INFEASIBLE_START
    assert res[0]["stop_reason"] == A.AS_STOP_MAX_ITERS


@pytest.mark.parametrize("cfg,iters", [("tiny", 200), ("ontario", 400), ("batched", 300)])
def test_grid_kernel_forced_small(A, ctx, oracle_mod, cfg, iters, monkeypatch, ctxopt):
    """The cooperative whole-GPU kernel (k_grid) forced onto small instances:
    many tiles per row group, most warps idle -- the trace must not change."""
    ctxopt(GRID=1)
    inst = instgen.generate(cfg)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    c = instgen.CONFIGS[cfg]
    _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters, seed=3, kick=5)
    _compare_run(A, ctx, O, h, p, m, 0, 0, iters)
    ctxopt(GRID_G=3)
    _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters)
    ctxopt(GRID_T_GLOBAL=1)   # table in global memory: row-local reads
    _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters)
    ctxopt(GRID_E_GLOBAL=1)   # tabu matrix (and its transpose) in global memory
    _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters, seed=5, kick=4)


def test_surge_run_parity_prefix(A, ctx, oracle_mod):
    """C5 (n=4000, V=100, 32.4 M indices per iteration) on the whole-GPU kernel:
    the first TS and NS iterations against the oracle."""
    inst = instgen.generate("surge")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    _compare_run(A, ctx, O, h, p, m, 1, 10, 3)
    _compare_run(A, ctx, O, h, p, m, 0, 0, 2)
    with ctx.options(GRID_SWAP_REC=0):   # the swap rows' dynamic part computed by the whole warp
        _compare_run(A, ctx, O, h, p, m, 1, 10, 3)


# ------------------------------------------------- sharded single instance (C5) --
@pytest.mark.parametrize("cfg,iters,emulate", [("tiny", 200, 1), ("ontario", 400, 3), ("large", 30, 8),
                                               ("surge", 2, 8)])
def test_sharded_path_parity(A, ctx, oracle_mod, cfg, iters, emulate, monkeypatch, ctxopt):
    """The sharded path's kernels (replica in global memory, per-iteration
    eval -> MIN -> apply in a CUDA graph).  With `emulate` > 1 the slices of
    that many ranks are scored one after another on this GPU (no kernel waits
    on another) -- the move sequence must equal the oracle's."""
    ctxopt(SHARDED=1)
    ctxopt(SHARD_EMULATE=int(emulate))
    ctxopt(SHARD_K=7)
    inst = instgen.generate(cfg)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    c = instgen.CONFIGS[cfg]
    _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters, seed=9, kick=3)
    if cfg != "surge":
        _compare_run(A, ctx, O, h, p, m, 0, 0, iters)


def test_sharded_nccl_one_rank(A, ctx, oracle_mod):
    """The real NCCL path (ncclAllReduce MIN on ncclUint64 inside the captured
    graph) with a one-rank communicator on this GPU."""
    comm = A.Comm(ctx, 1, 0, A.as_comm_unique_id())
    inst = instgen.generate("ontario")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    for mode in (1, 0):
        prm = A.params(mode=mode, tenure=10, max_iters=500, trace_level=1)
        g = A.as_tabu_run(ctx, h, p, m, prm, want_trace=True, comm=comm)
        o = O.search(p, m, mode=mode, tenure=10, max_iters=500)
        assert g["iters_done"] == o["iters_done"] and g["stop_reason"] == o["stop_reason"]
        assert (g["trace"]["idx"] == o["trace"]["idx"]).all() and g["best_obj"] == o["best_obj"]
        assert routes_of(*g["best"]) == routes_of(*o["best"])


def test_batch_gather_best(A, ctx, oracle_mod):
    """Best run of a batch (device MIN of (best_obj, run)) and its schedule; with and
    without a one-rank NCCL communicator (allreduce + broadcast path)."""
    inst = instgen.generate("ontario")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    R = 40
    seeds = np.arange(1, R + 1, dtype=np.uint64)
    res = np.zeros(R, A.RESULT_DTYPE)
    bp = np.zeros((R, inst.n_vehicles + 1), np.int32)
    bm = np.zeros((R, inst.n_missions), np.int32)
    prm = A.params(mode=1, tenure=10, max_iters=120, kick=6)
    for comm in (None, A.Comm(ctx, 1, 0, A.as_comm_unique_id())):
        A.as_batch_run(ctx, h, R, p, m, prm, seeds, results=res, best_ptr_out=bp, best_missions_out=bm, comm=comm)
        g = A.as_batch_gather_best(ctx, h, R, bp, bm, comm=comm)
        want = int(np.lexsort((np.arange(R), res["best_obj"]))[0])
        assert g["best_run"] == want and g["best_obj"] == res[want]["best_obj"]
        assert routes_of(*g["best"]) == routes_of(bp[want], bm[want])
        assert O.objective(*g["best"]) == g["best_obj"] and O.feasible(*g["best"])


def test_per_cta_kernel_still_exact(A, ctx, oracle_mod, monkeypatch, ctxopt):
    """k_search (one run per CTA, int32 layout) -- the path for tabu digests and
    for instances outside the compact layout -- forced for a plain run."""
    ctxopt(ONE_CTA=0)
    ctxopt(GRID=0)
    inst = instgen.generate("ontario")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    _compare_run(A, ctx, O, h, p, m, 1, 10, 800, seed=2, kick=4)
    _compare_run(A, ctx, O, h, p, m, 0, 0, 800)


def test_bench_configuration_sampled_runs(A, ctx, oracle_mod):
    """BASELINE configs[2] at full size in bench.py's launch configuration: 4096 runs
    x 1000 iterations, shared start from Alg. 1, seeds 1..4096, kick 8, device-resident
    inputs and outputs; sampled runs must equal the oracle run for run."""
    import torch
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
    for r in (0, 1234, 4095):
        o = O.search(p, m, mode=1, tenure=c.tenure, max_iters=iters, seed=r + 1, kick=c.kick, trace=False)
        assert res[r]["best_obj"] == o["best_obj"] and res[r]["final_obj"] == o["final_obj"]
        assert res[r]["best_iter"] == o["best_iter"] and res[r]["kicks_applied"] == o["kicks_applied"]
        assert routes_of(bp[r], bm[r]) == routes_of(*o["best"])


@pytest.mark.parametrize("cfg,steps", [("tiny", 200), ("ontario", 1500), ("batched", 1500), ("large", 600)])
def test_sweep_mode_parity(A, ctx, oracle_mod, cfg, steps):
    """f1 (paper-literal Alg. 2 / 3 sweep) on the batched kernel: single runs and a batch
    with per-run permutation seeds, against the oracle step by step."""
    inst = instgen.generate(cfg)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    c = instgen.CONFIGS[cfg]
    for mode in (0, 1):
        prm = A.params(mode=mode, tenure=c.tenure, max_iters=steps, trace_level=1, sweep=1)
        g = A.as_tabu_run(ctx, h, p, m, prm, want_trace=True)
        o = O.sweep(p, m, mode=mode, tenure=c.tenure, max_steps=steps)
        k = o["iters_done"]
        assert g["iters_done"] == k and g["stop_reason"] == o["stop_reason"] and g["best_obj"] == o["best_obj"]
        gi = g["trace"]["idx"].astype(np.int64)
        gi[gi == 0xFFFFFFFF] = -1
        assert (gi == o["trace"]["idx"]).all() and (g["trace"]["cur"] == o["trace"]["cur"]).all()
        assert routes_of(*g["best"]) == routes_of(*o["best"])
    R = 8
    seeds = np.arange(11, 11 + R, dtype=np.uint64)
    res = np.zeros(R, A.RESULT_DTYPE)
    prm = A.params(mode=1, tenure=c.tenure, max_iters=steps, sweep=1)
    A.as_batch_run(ctx, h, R, p, m, prm, seeds, results=res)
    for r in (0, R - 1):
        o = O.sweep(p, m, mode=1, tenure=c.tenure, max_steps=steps, seed=int(seeds[r]))
        assert res[r]["best_obj"] == o["best_obj"] and res[r]["iters_done"] == o["iters_done"]
        assert res[r]["best_iter"] == o["best_iter"]


def _asymmetric(cfg, seed=5):
    """The configuration with a seeded asymmetric travel-time table (T[c][a][b] !=
    T[c][b][a]); the kernels then read the transposed padded copy (score.cuh)."""
    inst = instgen.generate(cfg)
    rng = np.random.default_rng(seed)
    T = inst.travel_s.astype(np.int64)
    T = T + rng.integers(0, 120, size=T.shape)
    for c in range(T.shape[0]):
        np.fill_diagonal(T[c], 0)
    inst.travel_s = T.astype(np.int32)
    return inst


@pytest.mark.parametrize("cfg,iters", [("ontario", 400), ("batched", 300), ("large", 25)])
def test_asymmetric_table_parity(A, ctx, oracle_mod, cfg, iters, monkeypatch):
    """Every scorer path (one-CTA and whole-GPU k_grid, k_batch, the sharded kernels)
    on an asymmetric table, where T and its transpose differ."""
    inst = _asymmetric(cfg)
    assert any((inst.travel_s[c] != inst.travel_s[c].T).any() for c in range(inst.travel_s.shape[0]))
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    c = instgen.CONFIGS[cfg]
    _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters, seed=4, kick=4)
    _compare_run(A, ctx, O, h, p, m, 0, 0, iters)
    with ctx.options(GRID=1):
        _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters)
        with ctx.options(GRID_T_GLOBAL=1):   # row-local reads of the global table (TR)
            _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters)
            _compare_run(A, ctx, O, h, p, m, 0, 0, iters)
    with ctx.options(SHARDED=1, SHARD_EMULATE=3):
        _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters)
    R = 40
    seeds = np.arange(1, R + 1, dtype=np.uint64)
    res = np.zeros(R, A.RESULT_DTYPE)
    prm = A.params(mode=1, tenure=c.tenure, max_iters=iters, kick=c.kick or 4)
    A.as_batch_run(ctx, h, R, p, m, prm, seeds, shared_start=True, results=res)
    for r in (0, R - 1):
        o = O.search(p, m, mode=1, tenure=c.tenure, max_iters=iters, seed=int(seeds[r]), kick=c.kick or 4)
        assert res[r]["best_obj"] == o["best_obj"] and res[r]["iters_done"] == o["iters_done"]
        assert res[r]["best_iter"] == o["best_iter"]
    d, f, key = A.as_eval_moves(ctx, h, p, m, mode=0)
    od, of, ok = O.eval_moves(p, m, mode=0)
    assert (d == od).all() and (f == of).all()


def test_batch_run_jobs(A, ctx, oracle_mod):
    """as_batch_run_jobs: several instances (different n, V, tables) in ONE launch, each CTA
    staging its job's instance; sampled runs of every job against the oracle, packed best
    schedules, traces, the best-run reduction, and the unsupported cases."""
    import dataclasses
    insts = [instgen.generate("tiny"), instgen.generate("ontario"), instgen.generate("batched"), _asymmetric("ontario", 9)]
    cfg = instgen.Config("j", 30, 4, 2, 3, 2, 20, "ontario", 5, 10, 3)
    insts += [instgen.generate(cfg, seed=s) for s in (1, 2)]
    runs = [8, 20, 40, 5, 3, 30]
    jobs, starts = [], []
    for inst, nr in zip(insts, runs):
        O = oracle_mod.Oracle(inst)
        p, m = start_of(O, inst)
        starts.append((O, p, m))
        jobs.append((A.Instance(inst), p, m, nr))
    total = sum(runs)
    iters = 120
    seeds = np.arange(101, 101 + total, dtype=np.uint64)
    for mode in (1, 0):
        prm = A.params(mode=mode, tenure=5, max_iters=iters, kick=3, trace_level=1)
        res = np.zeros(total, A.RESULT_DTYPE)
        bp = np.zeros(sum(nr * (inst.n_vehicles + 1) for inst, nr in zip(insts, runs)), np.int32)
        bm = np.zeros(sum(nr * inst.n_missions for inst, nr in zip(insts, runs)), np.int32)
        tr = np.zeros((total, iters), A.TRACE_DTYPE)
        best = A.as_batch_run_jobs(ctx, jobs, prm, seeds, results=res, best_ptr_out=bp, best_missions_out=bm,
                                   trace_out=tr, want_best_run=True)
        assert best == int(np.lexsort((np.arange(total), res["best_obj"]))[0])
        run0 = bpo = bmo = 0
        for (O, p, m), inst, nr in zip(starts, insts, runs):
            V, n = inst.n_vehicles, inst.n_missions
            for r in sorted({0, nr - 1}):
                g = run0 + r
                o = O.search(p, m, mode=mode, tenure=5, max_iters=iters, seed=int(seeds[g]), kick=3)
                assert res[g]["best_obj"] == o["best_obj"] and res[g]["iters_done"] == o["iters_done"]
                assert res[g]["best_iter"] == o["best_iter"] and res[g]["kicks_applied"] == o["kicks_applied"]
                assert (tr[g]["idx"][:o["iters_done"]] == o["trace"]["idx"]).all()
                ptr = bp[bpo + r * (V + 1): bpo + (r + 1) * (V + 1)]
                ms = bm[bmo + r * n: bmo + (r + 1) * n]
                assert routes_of(ptr, ms) == routes_of(*o["best"])
            run0 += nr
            bpo += nr * (V + 1)
            bmo += nr * n
    # device-resident starts and results
    import torch
    dev = torch.device("cuda:0")
    djobs = [(h, torch.from_numpy(p).to(dev), torch.from_numpy(m).to(dev), nr) for (h, p, m, nr) in jobs]
    tres = torch.zeros((total, 40), dtype=torch.uint8, device=dev)
    prm = A.params(mode=1, tenure=5, max_iters=iters, kick=3)
    A.as_batch_run_jobs(ctx, djobs, prm, torch.from_numpy(seeds.view(np.int64)).to(dev), results=tres)
    torch.cuda.synchronize()
    res2 = tres.cpu().numpy().view(A.RESULT_DTYPE).reshape(total)
    res1 = np.zeros(total, A.RESULT_DTYPE)
    A.as_batch_run_jobs(ctx, jobs, prm, seeds, results=res1)
    assert (res1 == res2).all()
    # the same runs through the single-instance entry point
    run0 = 0
    for (h, p, m, nr) in jobs:
        r3 = np.zeros(nr, A.RESULT_DTYPE)
        A.as_batch_run(ctx, h, nr, p, m, prm, seeds[run0:run0 + nr], results=r3)
        assert (r3 == res1[run0:run0 + nr]).all()
        run0 += nr
    # unsupported: the no-wait variant and > 2 classes
    nw = dataclasses.replace(insts[1], no_wait=1)
    with pytest.raises(A.AirschedError) as e:
        A.as_batch_run_jobs(ctx, [(A.Instance(nw), starts[1][1], starts[1][2], 2)], prm)
    assert e.value.status == A.AS_ERR_UNSUPPORTED


def test_state_too_large_for_shared_memory(A, oracle_mod):
    """When no on-chip kernel can hold an instance's state, as_tabu_run runs the sharded
    kernels on one rank (state in global memory).  Forced here by capping the usable shared
    memory of a fresh context; the trace must still equal the oracle's."""
    small = A.Ctx(0)
    small.set_option("SMEM_LIMIT", 12000)
    inst = instgen.generate("ontario")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    _compare_run(A, small, O, h, p, m, 1, 10, 400, seed=6, kick=3)
    _compare_run(A, small, O, h, p, m, 0, 0, 400)


def test_largest_single_instance(A, ctx, oracle_mod):
    """n = 9000 missions, V = 100 (state ~330 KB: beyond shared memory, so the one-rank sharded
    path; 171 M indices per iteration).  Checked at this size: the first selected move equals the
    evaluation dump's minimum (itself parity-tested), the oracle re-evaluates that move to the
    same delta and feasibility, and the best schedule is feasible with the reported objective."""
    cfg = instgen.Config("max", 9000, 67, 33, 17, 8, 400, "disaster", 20, 5, 10)
    inst = instgen.generate(cfg, seed=77)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = inst.planted_ptr, inst.planted_missions
    r = A.as_tabu_run(ctx, h, p, m, A.params(mode=1, tenure=10, max_iters=5, trace_level=1), want_trace=True)
    assert r["iters_done"] == 5
    d, f, key = A.as_eval_moves(ctx, h, p, m, mode=1, tabu_expiry=np.full((inst.n_missions, inst.n_vehicles), -1, np.int32),
                                iter=0, best_obj=O.objective(p, m))
    c0, dl0, i0 = decode_key(key)
    tr = r["trace"]
    assert (int(tr["idx"][0]), int(tr["delta"][0]), int(tr["cls"][0])) == (i0, dl0, c0)
    od, of = O.eval_indices(p, m, np.array([i0], np.int64), mode=1, E=None, it=0, best_obj=O.objective(p, m))
    assert od[0] == dl0 and of[0] & 2
    bp, bm = r["best"]
    assert O.feasible(bp, bm) and O.objective(bp, bm) == r["best_obj"]
    assert r["best_obj"] == int(tr["best"][-1])


@pytest.mark.parametrize("cfg,iters", [("ontario", 400), ("large", 30), ("surge", 2)])
def test_sharded_fused_one_rank(A, ctx, oracle_mod, cfg, iters, monkeypatch, ctxopt):
    """The fused sharded kernel (k_grid per rank; the 8-byte winner exchanged through NVLink
    stores into an NCCL symmetric window + an LSA barrier inside the kernel), run with a
    one-rank communicator on this GPU: its tile slice, exchange and apply against the oracle."""
    ctxopt(SHARD_FUSED_1=1)
    comm = A.Comm(ctx, 1, 0, A.as_comm_unique_id())
    inst = instgen.generate(cfg)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    ctx.upload(h)
    p, m = start_of(O, inst)
    c = instgen.CONFIGS[cfg]
    for mode in ((1,) if cfg == "surge" else (1, 0)):
        prm = A.params(mode=mode, tenure=c.tenure, max_iters=iters, trace_level=1, seed=3, kick=2)
        l0 = ctx.kernel_launches
        g = A.as_tabu_run(ctx, h, p, m, prm, want_trace=True, want_tabu=(mode == 1), comm=comm)
        assert ctx.kernel_launches - l0 <= 3   # one persistent kernel (+ CSR of the best), not per-iteration graphs
        o = O.search(p, m, mode=mode, tenure=c.tenure, max_iters=iters, seed=3, kick=2)
        assert g["iters_done"] == o["iters_done"] and g["stop_reason"] == o["stop_reason"]
        assert (g["trace"]["idx"] == o["trace"]["idx"]).all() and (g["trace"]["cur"] == o["trace"]["cur"]).all()
        assert g["best_obj"] == o["best_obj"] and g["best_iter"] == o["best_iter"]
        if mode == 1:
            assert (g["tabu"] == o["E"]).all()
        assert routes_of(*g["best"]) == routes_of(*o["best"])


def test_solver_one_call(A, oracle_mod):
    """paper_2002_11710_b200.solver.solve: the best of a batch equals the oracle's run with that
    seed, and the schedule is feasible with the reported objective (both start kinds)."""
    from paper_2002_11710_b200 import solver
    inst = instgen.generate("ontario")
    O = oracle_mod.Oracle(inst)
    out = solver.solve(inst, runs=32, iters=300, tenure=10, kick=6)
    ptr, ms = np.zeros(inst.n_vehicles + 1, np.int32), []
    for v, r in enumerate(out["routes"]):
        ptr[v + 1] = ptr[v] + len(r)
        ms += r
    ms = np.array(ms, np.int32)
    assert O.feasible(ptr, ms) and O.objective(ptr, ms) == out["objective"]
    st, (p, m), _, _ = O.greedy(insert_mode=1)
    o = O.search(p, m, mode=1, tenure=10, max_iters=300, seed=out["seed"], kick=6)
    assert o["best_obj"] == out["objective"] and routes_of(*o["best"]) == out["routes"]
    assert out["objective"] == int(out["results"]["best_obj"].min())
    out2 = solver.solve(inst, runs=32, iters=300, starts="seeded", mode="ns")
    st, (p2, m2), _, _ = O.greedy(insert_mode=1, seed=out2["seed"])
    o2 = O.search(p2, m2, mode=0, max_iters=300, seed=out2["seed"])
    assert o2["best_obj"] == out2["objective"]


def test_jobs_and_greedy_degenerate(A, ctx, oracle_mod):
    """Degenerate jobs: an instance with no missions, one with one mission and one vehicle,
    next to a normal one; and Alg. 1 batches on them."""
    base = instgen.generate("tiny")
    empty = instgen.Instance(base.travel_s, base.class_is_heli, base.base_location, base.vehicle_base,
                             base.vehicle_class, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32),
                             np.zeros(0, np.uint8))
    one = instgen.generate(instgen.Config("one", 1, 1, 0, 1, 0, 4, "ontario", 3, 10, 2), seed=3)
    insts = [empty, one, base]
    jobs = []
    for inst in insts:
        h = A.Instance(inst)
        ptr, ms, status, nrep = A.as_init_greedy_batch(ctx, h, 4, seeds=np.arange(4, dtype=np.uint64), insert_mode=1)
        O = oracle_mod.Oracle(inst)
        for r in range(4):
            st, (op, om), nr, _ = O.greedy(insert_mode=1, seed=r)
            assert (status[r] == 0) == (st == 0)
            if st == 0:
                assert routes_of(ptr[r], ms[r][:inst.n_missions]) == routes_of(op, om)
        jobs.append((h, ptr[0], ms[0][:inst.n_missions], 3))
    prm = A.params(mode=1, tenure=3, max_iters=50, kick=2)
    res = np.zeros(9, A.RESULT_DTYPE)
    A.as_batch_run_jobs(ctx, jobs, prm, np.arange(1, 10, dtype=np.uint64), results=res)
    assert (res["best_obj"][:3] == 0).all() and (res["stop_reason"][:3] == A.AS_STOP_NO_MOVE).all()
    for j, inst in enumerate(insts[1:], start=1):
        O = oracle_mod.Oracle(inst)
        h, p, m, _ = jobs[j]
        for r in range(3):
            o = O.search(p, m, mode=1, tenure=3, max_iters=50, seed=3 * j + r + 1, kick=2)
            assert res[3 * j + r]["best_obj"] == o["best_obj"] and res[3 * j + r]["iters_done"] == o["iters_done"]


@pytest.mark.parametrize("cfg,iters", [("ontario", 300), ("large", 40)])
def test_grid_phase_times(A, ctx, oracle_mod, cfg, iters, ctxopt):
    """AS_OPT_PHASE_TIMES: the whole-GPU kernel's per-iteration latency breakdown (CTA 0, %globaltimer)
    covers every iteration, sums to about the kernel time, and leaves the trace unchanged."""
    inst = instgen.generate(cfg)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    ctxopt(PHASE_TIMES=1, GRID=1)
    g = _compare_run(A, ctx, O, h, p, m, 1, 10, iters)
    ph = ctx.grid_phases()
    assert ph["iterations"] == g["iters_done"] == iters
    per_it = ph["own_tiles_us"] + ph["cta_wait_us"] + ph["reduce_barrier_us"] + ph["apply_us"]
    assert 0 < per_it * iters / 1e3 <= ctx.last_kernel_ms * 1.05
    assert min(ph["own_tiles_us"], ph["reduce_barrier_us"], ph["apply_us"]) > 0
    # per CTA: every CTA's tile phase is measured and fits in the iteration; SM ids distinct and in range
    t, sm = ctx.grid_cta_phases()
    assert len(t) >= 1 and (t > 0).all() and (t <= per_it * 1.05).all()
    assert len(set(sm.tolist())) == len(sm) and sm.min() >= 0


def test_global_node_cost_table(A, oracle_mod):
    """C5's table is read from global memory; with the node-cost table TD[c][x][t] (default) one gather of
    each relocate and swap becomes a coalesced row read.  A context without it (AS_OPT_NODE_COSTS=0,
    set before the upload) must give the same trace, and both equal the oracle's."""
    inst = instgen.generate("surge")
    O = oracle_mod.Oracle(inst)
    p, m = start_of(O, inst)
    out = []
    iters = 6
    for node_costs in (1, 0):
        c = A.Ctx(0)
        c.set_option("NODE_COSTS", node_costs)
        h = A.Instance(inst)
        c.upload(h)
        prm = A.params(mode=1, tenure=10, max_iters=iters, trace_level=1)
        out.append(A.as_tabu_run(c, h, p, m, prm, want_trace=True, want_tabu=True))
    o = O.search_par(p, m, mode=1, tenure=10, max_iters=iters, memo=True)
    for g in out:
        for k in ("idx", "delta", "cur", "best", "cls"):
            assert (g["trace"][k] == o["trace"][k]).all(), k
        assert (g["tabu"] == o["E"]).all() and routes_of(*g["best"]) == routes_of(*o["best"])


@pytest.mark.parametrize("cfg,iters,opts,blocks", [
    ("ontario", 600, {}, 16),                                   # the automatic choice for C2
    ("ontario", 400, {"GRID_CLUSTER": 8}, 8),
    ("tiny", 200, {"GRID": 1, "GRID_CLUSTER": 2}, 2),
    ("batched", 200, {}, 16),
    ("batched", 150, {"GRID_CLUSTER": 4, "GRID_G": 3}, 4),
])
def test_cluster_mode_parity(A, ctx, oracle_mod, cfg, iters, opts, blocks, ctxopt, capfd):
    """The whole-GPU kernel as ONE thread-block cluster (small instances: every CTA's key stored into every
    CTA's shared memory, one cluster barrier per iteration): TS (plain and kicked) and NS traces, tabu
    matrix and best schedule equal the oracle's; the verbose line names the path and its CTA count."""
    inst = instgen.generate(cfg)
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    p, m = start_of(O, inst)
    c = instgen.CONFIGS[cfg]
    ctxopt(VERBOSE=1, **opts)
    capfd.readouterr()
    _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters)
    err = capfd.readouterr().err
    import re
    got = [int(x) for x in re.findall(r"k_grid/cluster \(blocks (\d+),", err)]
    assert got, err
    if opts:
        assert got[-1] == blocks, err
    else:   # automatic: 16, or 8 if a 16-CTA cluster does not fit this GPU
        assert got[-1] in (8, 16), err
        blocks = got[-1]
    _compare_run(A, ctx, O, h, p, m, 0, 0, iters)
    _compare_run(A, ctx, O, h, p, m, 1, c.tenure, iters // 2, seed=11, kick=6)
    with ctx.options(PHASE_TIMES=1):   # the phase timers on the same path: every CTA of the cluster recorded
        g = _compare_run(A, ctx, O, h, p, m, 1, c.tenure, 50)
        ph = ctx.grid_phases()
        t, sm = ctx.grid_cta_phases()
    assert ph["iterations"] == g["iters_done"] == 50 and ph["own_tiles_us"] > 0
    assert len(t) == blocks and (t > 0).all()
