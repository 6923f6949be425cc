"""Randomised GPU parity (every kernel path against the oracle, bit-exact) on
seeded random instances outside the generator's shapes: 1-3 matrix layers
(3 -> the int32 per-CTA kernel), zero-length pickup->delivery legs (the general
scorers instead of the FAST ones), asymmetric tables, tight and loose deadlines,
helicopter-only missions, small flight limits, 0..40 missions, 1..8 vehicles,
and the no-wait variant."""
import os

import numpy as np
import pytest

from paper_2002_11710_b200 import instgen

pytestmark = pytest.mark.gpu

# longer sweeps on demand: AIRSCHED_FUZZ_SCALE multiplies the trial counts, AIRSCHED_FUZZ_SEED shifts the seeds
SCALE = max(1, int(os.environ.get("AIRSCHED_FUZZ_SCALE", "1")))
SEED = int(os.environ.get("AIRSCHED_FUZZ_SEED", "0"))


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


def random_instance(rng, no_wait=0):
    NL = int(rng.integers(2, 30))
    NC = int(rng.integers(1, 4))
    V = int(rng.integers(1, 9))
    n = int(rng.integers(0, 41))
    T = rng.integers(0, 3000, size=(NC, NL, NL)).astype(np.int64)
    if rng.random() < 0.5:                      # symmetric, as a distance table would be
        T = np.minimum(T, T.transpose(0, 2, 1))
    T[rng.random(T.shape) < 0.05] = 0          # zero legs
    for c in range(NC):
        np.fill_diagonal(T[c], 0)
    B = int(rng.integers(1, min(NL, 5) + 1))
    base_loc = rng.choice(NL, B, replace=False).astype(np.int32)
    cls_heli = (rng.random(NC) < 0.6).astype(np.uint8)
    cls_heli[0] = 1
    vb = rng.integers(0, B, V).astype(np.int32)
    vc = rng.integers(0, NC, V).astype(np.int32)
    pick = rng.integers(0, NL, n).astype(np.int32)
    dele = np.where(rng.random(n) < 0.1, pick, rng.integers(0, NL, n)).astype(np.int32)
    day = 86400
    tight = rng.random() < 0.5
    w = rng.integers(3000 if tight else 20000, day, n).astype(np.int32)
    heli = (rng.random(n) < 0.25).astype(np.uint8)
    P = int(rng.integers(8000, 40000))
    return instgen.Instance(T.astype(np.int32), cls_heli, base_loc, vb, vc, pick, dele, w, heli,
                            flight_limit_s=P, day_length_s=day, no_wait=no_wait)


def feasible_start(O):
    for mode in (1, 0):
        st, (p, m), _, _ = O.greedy(insert_mode=mode)
        if st == 0:
            return p, m
    return None


def compare_run(A, ctx, O, h, p, m, mode, tenure, iters, seed=0, kick=0, digest=False):
    prm = A.params(mode=mode, tenure=tenure, max_iters=iters, trace_level=2 if digest else 1, seed=seed, kick=kick)
    g = A.as_tabu_run(ctx, h, p, m, prm, want_trace=True, want_digest=digest, want_tabu=(mode == 1))
    o = O.search(p, m, mode=mode, tenure=tenure, max_iters=iters, seed=seed, kick=kick, digest=digest)
    assert g["iters_done"] == o["iters_done"] and g["stop_reason"] == o["stop_reason"]
    assert (g["trace"]["idx"] == o["trace"]["idx"]).all()
    assert (g["trace"]["cur"] == o["trace"]["cur"]).all() and (g["trace"]["cls"] == o["trace"]["cls"]).all()
    if digest:
        assert (g["digest"] == o["trace"]["digest"]).all()
    if mode == 1:
        assert (g["tabu"] == o["E"]).all()
    assert g["best_obj"] == o["best_obj"] and g["best_iter"] == o["best_iter"]
    assert g["kicks_applied"] == o["kicks_applied"]
    assert routes_of(*g["best"]) == routes_of(*o["best"])


# kernel selections: default policy, per-CTA int32 kernel, whole-GPU kernel on 1 and on all CTAs,
# the batched kernel for a single run, the sharded kernels with 2 emulated ranks
PATHS = {
    "default": {},
    "k_search": {"GRID": 0, "ONE_CTA": 0},
    "k_grid_1cta": {"GRID": 1, "GRID_BLOCKS": 1},
    "k_grid_all": {"GRID": 1},
    "k_grid_tglobal": {"GRID": 1, "GRID_T_GLOBAL": 1, "GRID_G": 2},
    "k_grid_teglobal": {"GRID": 1, "GRID_T_GLOBAL": 1, "GRID_E_GLOBAL": 1},
    "k_grid_tglobal_g20": {"GRID": 1, "GRID_T_GLOBAL": 1, "GRID_E_GLOBAL": 1, "GRID_G": 20},   # > SR_ROWS rows
    "k_grid_tglobal_norec": {"GRID": 1, "GRID_T_GLOBAL": 1, "GRID_SWAP_REC": 0},
    "k_grid_cluster4": {"GRID": 1, "GRID_CLUSTER": 4},
    "k_batch": {"BATCH_KERNEL": 1},
    "sharded2": {"SHARDED": 1, "SHARD_EMULATE": 2, "SHARD_K": 3},
}


@pytest.mark.parametrize("path", list(PATHS))
def test_fuzz_runs(A, ctx, oracle_mod, path, ctxopt):
    ctxopt(**PATHS[path])
    rng = np.random.default_rng(20021171 + list(PATHS).index(path) + SEED)
    done = 0
    for trial in range(120 * SCALE):
        inst = random_instance(rng)
        O = oracle_mod.Oracle(inst)
        start = feasible_start(O)
        if start is None:
            continue
        p, m = start
        h = A.Instance(inst)
        tenure = int(rng.integers(0, 6))
        if path == "sharded2" and inst.travel_s.shape[0] > 2:   # compact layout only (<= 2 classes)
            with pytest.raises(A.AirschedError) as e:
                A.as_tabu_run(ctx, h, p, m, A.params(mode=1, tenure=tenure, max_iters=5))
            assert e.value.status == A.AS_ERR_UNSUPPORTED
            continue
        # tabu digests force the per-CTA kernel, so they are requested on that path only
        compare_run(A, ctx, O, h, p, m, 1, tenure, 80, seed=int(rng.integers(1, 1000)), kick=int(rng.integers(0, 4)),
                    digest=(path == "k_search"))
        compare_run(A, ctx, O, h, p, m, 0, 0, 80)
        done += 1
        if done >= 40 * SCALE:
            break
    assert done >= 20 * SCALE


def test_fuzz_eval_and_batch(A, ctx, oracle_mod):
    rng = np.random.default_rng(7117 + SEED)
    done = 0
    for trial in range(80 * SCALE):
        inst = random_instance(rng)
        O = oracle_mod.Oracle(inst)
        start = feasible_start(O)
        if start is None:
            continue
        p, m = start
        h = A.Instance(inst)
        states = [(p, m), O.search(p, m, mode=1, tenure=2, max_iters=15, trace=False)["final"],
                  O.kick(p, m, 5, 6)[1]]
        for sp, sm in states:
            for mode in (0, 1):
                E, it, best = None, 0, O.objective(sp, sm)
                if mode == 1 and inst.n_missions:
                    it = int(rng.integers(1, 20))
                    E = rng.integers(-1, it + 4, size=(inst.n_missions, inst.n_vehicles)).astype(np.int32)
                    best -= int(rng.integers(0, 500))
                od, of, ok = O.eval_moves(sp, sm, mode=mode, E=E, it=it, best_obj=best)
                gd, gf, key = A.as_eval_moves(ctx, h, sp, sm, mode=mode, tabu_expiry=E, iter=it, best_obj=best)
                assert (gf == of).all() and (gd == od).all()
        R = 12
        seeds = np.arange(1, R + 1, dtype=np.uint64)
        res = np.zeros(R, A.RESULT_DTYPE)
        prm = A.params(mode=1, tenure=3, max_iters=30, kick=3)
        A.as_batch_run(ctx, h, R, p, m, prm, seeds, results=res)
        for r in (0, R - 1):
            o = O.search(p, m, mode=1, tenure=3, max_iters=30, seed=int(seeds[r]), kick=3)
            assert res[r]["best_obj"] == o["best_obj"] and res[r]["iters_done"] == o["iters_done"]
            assert res[r]["best_iter"] == o["best_iter"] and res[r]["kicks_applied"] == o["kicks_applied"]
        done += 1
        if done >= 25 * SCALE:
            break
    assert done >= 12 * SCALE


def test_fuzz_nowait_and_greedy(A, ctx, oracle_mod):
    rng = np.random.default_rng(99173 + SEED)
    done = 0
    for trial in range(80 * SCALE):
        inst = random_instance(rng, no_wait=1)
        O = oracle_mod.Oracle(inst)
        h = A.Instance(inst)
        seeds = np.arange(0, 8, dtype=np.uint64)
        ptr, ms, status, nrep = A.as_init_greedy_batch(ctx, h, len(seeds), seeds=seeds, insert_mode=1)
        for r, s in enumerate(seeds):
            st, (op, om), nr, _ = O.greedy(insert_mode=1, seed=int(s))
            assert (status[r] == 0) == (st == 0)
            if st == 0:
                assert routes_of(ptr[r], ms[r]) == routes_of(op, om) and nrep[r] == nr
        start = feasible_start(O)
        if start is None:
            continue
        p, m = start
        compare_run(A, ctx, O, h, p, m, 1, 3, 40, seed=5, kick=2, digest=True)
        compare_run(A, ctx, O, h, p, m, 0, 0, 40)
        with ctx.options(GRID=1):   # the whole-GPU kernel's no-wait form (compact layouts)
            compare_run(A, ctx, O, h, p, m, 1, 3, 40, seed=7, kick=2)
        with ctx.options(GRID=1, GRID_T_GLOBAL=1, GRID_E_GLOBAL=1, GRID_G=3):
            compare_run(A, ctx, O, h, p, m, 1, 2, 30)
        d, f, key = A.as_eval_moves(ctx, h, p, m, mode=0)
        od, of, ok = O.eval_moves(p, m, mode=0)
        assert (d == od).all() and (f == of).all()
        done += 1
        if done >= 20 * SCALE:
            break
    assert done >= 10 * SCALE
