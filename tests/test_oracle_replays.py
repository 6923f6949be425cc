"""Pins for the oracle's search-side functions by independent replay (-m "not gpu").

Each test runs the oracle (oracle/oracle.c) and a pure-Python replay written from
DESIGN.md's readings (tests/replay.py, on tests/pins.py's arc-form route check)
on the same seeded inputs and requires identical results.  The cases are chosen
so the rule under test actually fires: kicks whose 64 draws all fail, greedy
starts that need the repair (and hit its budget), seeded sweeps with several
permutations.  A plausible slip in oracle.c -- drawing modulo the whole move
space, not breaking after a successful kick draw, a second repair retry, a
Fisher-Yates range off by one, a wrong stream order -- fails one of them."""
import dataclasses

import numpy as np
import pytest

import replay
from paper_2002_11710_b200 import instgen


def routes_of(ptr, ms):
    return [list(map(int, ms[ptr[v]:ptr[v + 1]])) for v in range(len(ptr) - 1)]


def csr(routes):
    ptr = np.zeros(len(routes) + 1, np.int32)
    ptr[1:] = np.cumsum([len(r) for r in routes])
    ms = np.array([m for r in routes for m in r], np.int32)
    return ptr, ms


def tiny(n, V, seed, F=6, n_plane=None):
    n_plane = max(1, V // 3) if n_plane is None else n_plane
    cfg = instgen.Config("t", n, V - n_plane, n_plane, 1, 1, F, "ontario", 4, 50, 3)
    return instgen.generate(cfg, seed=seed)


def test_splitmix_python_matches_published_vector(oracle_mod):
    """The replay's generator against the same published vector the oracle's is
    pinned to (seed 1234567, Vigna's splitmix64.c)."""
    s, out = 1234567, []
    for _ in range(5):
        s, z = replay.splitmix64(s)
        out.append(z)
    assert out == [6457827717110365317, 3203168211198807973, 9817491932198370423, 4593380528125082431,
                   16408922859458223821]


# ------------------------------------------------------------------ O12 kick --
def test_kick_replay(oracle_mod):
    """O12: z mod n(n+V), up to 64 draws per kick, first VALID and FEASIBLE applied."""
    cases = 0
    skipped_kicks = 0
    for inst in (instgen.generate("batched"), instgen.generate("tiny"), tiny(6, 3, 41), tiny(9, 4, 42)):
        O = oracle_mod.Oracle(inst)
        M = replay.Model(inst)
        ptr, ms = inst.planted_ptr, inst.planted_missions
        for seed in range(1, 25 if inst.n_missions < 50 else 8):
            for k in (1, 3, 8):
                got_k, st = O.kick(ptr, ms, seed, k)
                exp_k, exp = replay.kick(M, routes_of(ptr, ms), seed, k)
                assert got_k == exp_k and routes_of(*st) == exp, (inst.n_missions, seed, k)
                skipped_kicks += k - exp_k
                cases += 1
    assert cases > 100
    # a tightened instance where whole kicks run out of draws (the 64-draw rule fires):
    # every deadline set to its arrival in the start schedule, so that schedule stays
    # feasible with zero slack and almost every relocate breaks a deadline
    inst = tiny(6, 3, 41)
    st0, (p0, m0), _, _ = oracle_mod.Oracle(inst).greedy(insert_mode=1)
    assert st0 == 0
    routes0 = routes_of(p0, m0)
    M = replay.Model(inst)
    w = inst.deadline_s.astype(np.int64).copy()
    for k, r in enumerate(routes0):
        prev, dep = inst.n_missions + k, 0
        for m in r:
            w[m] = dep + int(M.d[prev, m, int(inst.vehicle_class[k])])   # arrival; departure at w
            prev, dep = m, int(w[m])
    tight = dataclasses.replace(inst)
    tight.deadline_s = w.astype(np.int32)
    Ot = oracle_mod.Oracle(tight)
    Mt = replay.Model(tight)
    assert Ot.feasible(p0, m0)
    for seed in range(1, 40):
        got_k, st = Ot.kick(p0, m0, seed, 6)
        exp_k, exp = replay.kick(Mt, routes0, seed, 6)
        assert got_k == exp_k and routes_of(*st) == exp, seed
        skipped_kicks += 6 - exp_k
    assert skipped_kicks > 0, "no kick exhausted its 64 draws: the skip rule was not exercised"


# ------------------------------------------------------- O13 repair branch ----
def test_greedy_repair_replay(oracle_mod):
    """O13 with the repair: one NS iteration over the assigned missions (every move
    kind), one retry, the max_repairs budget (reading #22).
    Seeded 7-mission starts; the ones that needed a repair are replayed under
    several budgets.  The repairs picked cover relocates and swaps."""
    n_cases = n_fail = n_budget = 0
    kinds = set()
    for iseed in range(5000, 5400):
        inst = tiny(7, 3, iseed, F=8)
        if iseed % 2:       # f3 no-wait instances: intra-route repairs become feasible
            inst = dataclasses.replace(inst, no_wait=1)
        O = oracle_mod.Oracle(inst)
        M = replay.Model(inst)
        n = inst.n_missions
        for gseed in range(0, 12):
            for mode in (0, 1):
                st, _, nrep, order = O.greedy(insert_mode=mode, seed=gseed)
                if nrep == 0:
                    continue
                for max_rep in ((0, 1, 50) if n_cases < 40 else (50,)):
                    st, (p, m), nrep, order = O.greedy(insert_mode=mode, seed=gseed, max_repairs=max_rep)
                    est, eroutes, erep, picked = replay.greedy(M, order, mode, max_rep)
                    assert (st, nrep) == (est, erep), (iseed, gseed, mode, max_rep)
                    if st == 0:
                        assert routes_of(p, m) == eroutes
                    n_fail += st != 0
                    n_budget += max_rep == 0 and st != 0
                    kinds.update(("swap" if i >= n * (n + inst.n_vehicles) else "relocate") +
                                 ("-intra" if intra else "") for i, intra in picked)
                n_cases += 1
        if n_cases >= 160 and {"swap", "relocate", "relocate-intra"} <= kinds:
            break
    assert n_cases >= 160 and n_fail > 0 and n_budget > 0
    assert {"swap", "relocate", "relocate-intra"} <= kinds, kinds


def test_greedy_repair_replay_larger(oracle_mod):
    """The repair on the C1 ('tiny') and a 12-mission instance with shuffled orders."""
    checked = 0
    for inst in (instgen.generate("tiny"), tiny(12, 4, 77, F=8)):
        O = oracle_mod.Oracle(inst)
        M = replay.Model(inst)
        for gseed in range(1, 30):
            st, (p, m), nrep, order = O.greedy(insert_mode=0, seed=gseed, max_repairs=3)
            if nrep == 0 and checked > 4:
                continue
            est, eroutes, erep, _ = replay.greedy(M, order, 0, 3)
            assert (st, nrep) == (est, erep)
            if st == 0:
                assert routes_of(p, m) == eroutes
            checked += 1
    assert checked > 4


# ------------------------------------------------------- f1 seeded sweep ------
@pytest.mark.parametrize("seed", [0, 1, 7, 123456789])
def test_sweep_replay(oracle_mod, seed):
    """f1 (reading #39): vehicle permutation then per-route snapshot permutations from
    one SplitMix64 stream, one CurrentMin step per (i, j)."""
    for inst in (tiny(6, 3, 310, F=10), tiny(8, 4, 311, F=10), instgen.generate("tiny")):
        O = oracle_mod.Oracle(inst)
        M = replay.Model(inst)
        st, (p, m), _, _ = O.greedy(insert_mode=1)
        assert st == 0
        for mode, tenure in ((0, 0), (1, 2), (1, 5)):
            got = O.sweep(p, m, mode=mode, tenure=tenure, max_steps=60, seed=seed)
            exp = replay.sweep(M, routes_of(p, m), mode, tenure, 60, seed)
            for key in ("idx", "delta", "cur", "best"):
                assert (got["trace"][key] == exp["trace"][key]).all(), (key, mode, seed)
            assert got["best_obj"] == exp["best_obj"] and got["stop_reason"] == exp["stop_reason"]
            assert got["iters_done"] == exp["iters_done"]


def test_sweep_seed_changes_order(oracle_mod):
    inst = tiny(8, 4, 311, F=10)
    O = oracle_mod.Oracle(inst)
    st, (p, m), _, _ = O.greedy(insert_mode=1)
    traces = {tuple(O.sweep(p, m, mode=1, tenure=2, max_steps=40, seed=s)["trace"]["idx"].tolist())
              for s in range(0, 6)}
    assert len(traces) >= 3


# ----------------------------------------------- O10/O11 full search replay ---
@pytest.mark.parametrize("mode,tenure,seed,kick", [(1, 2, 0, 0), (1, 5, 9, 3), (0, 0, 4, 2), (1, 0, 0, 0)])
def test_search_replay(oracle_mod, mode, tenure, seed, kick):
    """The global-best NS / TS loop (with the kick in front) against the replay."""
    for inst in (tiny(6, 3, 320, F=10), instgen.generate("tiny")):
        O = oracle_mod.Oracle(inst)
        M = replay.Model(inst)
        st, (p, m), _, _ = O.greedy(insert_mode=1)
        got = O.search(p, m, mode=mode, tenure=tenure, max_iters=25, seed=seed, kick=kick)
        exp = replay.search(M, routes_of(p, m), mode, tenure, 25, seed, kick)
        assert got["kicks_applied"] == exp["kicks_applied"]
        for key in ("idx", "delta", "cur", "best", "cls"):
            assert (got["trace"][key] == exp["trace"][key]).all(), key
        assert got["best_obj"] == exp["best_obj"] and routes_of(*got["best"]) == exp["best"]
        assert got["stop_reason"] == exp["stop_reason"]
        if mode == 1:
            E = got["E"]
            for (mm, v), e in exp["E"].items():
                assert E[mm, v] == e
            assert int((E >= 0).sum()) == len([e for e in exp["E"].values() if e >= 0])


# ------------------------------------------------------- or_eval_index_list ---
def test_eval_indices_equals_eval_moves(oracle_mod):
    """or_eval_index_list (the C5 sampled check's oracle) == or_eval_moves on every
    index, in NS and TS modes, with live tabu state, aspiration thresholds and masks."""
    for name in ("tiny", "ontario"):
        inst = instgen.generate(name)
        O = oracle_mod.Oracle(inst)
        st, (p, m), _, _ = O.greedy()
        tr = O.search(p, m, mode=1, tenure=7, max_iters=15)
        states = [((p, m), None, 0), (tr["final"], tr["E"], 15)]
        N = O.move_space_size()
        idx = np.arange(N, dtype=np.int64)
        rng = np.random.default_rng(3)
        n_tabu = 0
        for (pp, mm), E, it in states:
            obj = O.objective(pp, mm)
            for mode in (0, 1):
                for mask in (0xF, 0x1, 0x5):
                    for best in (obj, obj - 500, obj + 10 ** 6):
                        d, f, _ = O.eval_moves(pp, mm, mode=mode, E=E, it=it, best_obj=best, mask=mask)
                        di, fi = O.eval_indices(pp, mm, idx, mode=mode, E=E, it=it, best_obj=best, mask=mask)
                        assert (d == di).all() and (f == fi).all()
                        sel = rng.permutation(N)[: N // 3]
                        ds, fs = O.eval_indices(pp, mm, sel, mode=mode, E=E, it=it, best_obj=best, mask=mask)
                        assert (ds == d[sel]).all() and (fs == f[sel]).all()
                        if E is not None and mode == 1:
                            n_tabu += int((f & oracle_mod.FLAG_TABU).sum())
    assert n_tabu > 0          # the comparison covered the tabu branch
