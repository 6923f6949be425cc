"""Pins for the CPU oracle (-m "not gpu").  The oracle is checked against things
other than itself: hand-derived worked-example values (tests/golden/e1.json),
an independent x_ijk coding of the paper's ILP constraints, exhaustive
enumeration, the HiGHS ILP optimum, published test vectors, and invariants."""
import json
import os

import numpy as np
import pytest

import pins
from e1 import e1_instance
from paper_2002_11710_b200 import instgen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "e1.json")))


def routes_of(ptr, ms):
    return [list(map(int, ms[ptr[v]:ptr[v + 1]])) for v in range(len(ptr) - 1)]


def csr(routes):
    ptr = np.zeros(len(routes) + 1, np.int32)
    ptr[1:] = np.cumsum([len(r) for r in routes])
    ms = np.array([m for r in routes for m in r], np.int32)
    return ptr, ms


def tiny_instance(n, V, seed, n_plane=None, F=6):
    n_plane = max(1, V // 3) if n_plane is None else n_plane
    cfg = instgen.Config("t", n, V - n_plane, n_plane, 1, 1, F, "ontario", 4, 50, 3)
    return instgen.generate(cfg, seed=seed)


def trajectory_states(O, inst, iters=(0, 3, 7, 15), tenure=2):
    """Feasible states: the greedy start and tabu-search states visited from it."""
    st, (p, m), _, _ = O.greedy()
    if st != 0:
        p, m = inst.planted_ptr, inst.planted_missions
    out = [(p, m)]
    for it in iters[1:]:
        out.append(O.search(p, m, mode=1, tenure=tenure, max_iters=it)["final"])
    return out


def feasible_states(O, inst, count, seed0=1, kick=6):
    ptr, ms = inst.planted_ptr, inst.planted_missions
    out = [(ptr, ms)]
    for s in range(seed0, seed0 + count):
        k, st = O.kick(ptr, ms, s, kick)
        out.append(st)
    return out


# ----------------------------------------------------------------- E1 golden --
def test_e1_start(oracle_mod):
    I = e1_instance()
    O = oracle_mod.Oracle(I)
    ptr, ms = csr(GOLD["start"])
    assert O.objective(ptr, ms) == GOLD["start_objective"]
    assert O.feasible(ptr, ms)
    ok, obj, bad = pins.xijk_check(I, GOLD["start"])
    assert ok and obj == GOLD["start_objective"]


def test_e1_move_table(oracle_mod):
    I = e1_instance()
    O = oracle_mod.Oracle(I)
    ptr, ms = csr(GOLD["start"])
    delta, flags, best = O.eval_moves(ptr, ms, mode=oracle_mod.MODE_NS)
    valid = np.flatnonzero(flags & oracle_mod.FLAG_VALID)
    assert sorted(map(int, valid)) == sorted(int(k) for k in GOLD["moves"])
    assert len(valid) == GOLD["valid_count"]
    for k, mv in GOLD["moves"].items():
        assert delta[int(k)] == mv["delta"], k
        assert bool(flags[int(k)] & oracle_mod.FLAG_FEASIBLE) == mv["feasible"], k
    assert best == (0, -1160, 9)


def test_e1_ns_ts(oracle_mod):
    I = e1_instance()
    O = oracle_mod.Oracle(I)
    ptr, ms = csr(GOLD["start"])
    r = O.search(ptr, ms, mode=oracle_mod.MODE_NS, max_iters=10)
    assert list(r["trace"]["idx"]) == GOLD["ns"]["idx"]
    assert r["best_obj"] == GOLD["ns"]["objective"] and r["stop_reason"] == GOLD["ns"]["stop_reason"]
    g = GOLD["ts_tenure2"]
    r = O.search(ptr, ms, mode=oracle_mod.MODE_TABU, tenure=2, max_iters=4)
    for key in ("idx", "delta", "cur", "best", "cls"):
        assert list(r["trace"][key]) == g[key], key
    r8 = O.search(ptr, ms, mode=oracle_mod.MODE_TABU, tenure=2, max_iters=8)
    assert list(r8["trace"]["idx"]) == g["idx"] * 2          # period 4
    assert r8["best_obj"] == 640 and r8["best_iter"] == 0
    rs = O.search(ptr, ms, mode=oracle_mod.MODE_TABU, tenure=2, max_iters=8, strict_tabu_stop=True)
    assert rs["iters_done"] == GOLD["ts_strict_stop_iters"] and rs["stop_reason"] == 2


def test_e1_greedy_and_optimum(oracle_mod):
    I = e1_instance()
    O = oracle_mod.Oracle(I)
    st, (ptr, ms), nrep, order = O.greedy(insert_mode=0)
    g = GOLD["greedy_tail"]
    assert st == 0 and routes_of(ptr, ms) == g["routes"] and nrep == g["repairs"]
    assert O.objective(ptr, ms) == g["objective"]
    assert list(order) == [2, 0, 1]                    # heli-only first, then by deadline
    opt, routes = pins.brute_optimum(I)
    assert opt == GOLD["optimum"] == pins.ilp_optimum(I)


# ------------------------------------------------------- published vectors --
def test_splitmix64_published_vector(oracle_mod):
    # Widely published SplitMix64 test vector for seed 1234567.
    assert oracle_mod.splitmix64(1234567, 5) == [6457827717110365317, 3203168211198807973, 9817491932198370423,
                                                 4593380528125082431, 16408922859458223821]


def _fnv1a64(data: bytes) -> int:
    h = 0xcbf29ce484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def test_tabu_digest_fnv(oracle_mod):
    assert _fnv1a64(b"a") == 0xaf63dc4c8601ec8c          # FNV-1a 64 published vector
    I = e1_instance()
    O = oracle_mod.Oracle(I)
    E = np.full((3, 2), -1, np.int32)
    assert O.tabu_digest(E, 0) == 0xcbf29ce484222325       # empty list = offset basis
    E[1, 0] = 5
    E[2, 1] = 3
    want = _fnv1a64(np.array([1, 0, 5, 2, 1, 3], "<i4").tobytes())
    assert O.tabu_digest(E, 2) == want
    assert O.tabu_digest(E, 3) == _fnv1a64(np.array([1, 0, 5], "<i4").tobytes())


def test_haversine_toronto_ottawa():
    # SPEC S:49 example; closed form with r = 6371.0 km: 352.0962 km.
    km = float(instgen.haversine_km(43.6532, -79.3832, 45.4215, -75.6972))
    assert abs(km - 352.0962) < 1e-3
    T = instgen.travel_matrix(np.array([43.6532, 45.4215]), np.array([-79.3832, -75.6972]))
    assert T[0, 0, 1] == 4225 and T[1, 0, 1] == 2535 and T[0, 0, 0] == 0
    assert T.shape == (2, 2, 2)


# ---------------------------------------------------- independent x_ijk coding --
def test_objective_feasibility_vs_xijk(oracle_mod):
    rng = np.random.default_rng(7)
    disagreements = 0
    checked = 0
    for seed in range(6):
        inst = tiny_instance(6, 3, 100 + seed)
        O = oracle_mod.Oracle(inst)
        states = feasible_states(O, inst, 8, seed0=1)
        n, V = inst.n_missions, inst.n_vehicles
        for _ in range(40):    # random (mostly infeasible) complete schedules
            perm = rng.permutation(n)
            cuts = np.sort(rng.integers(0, n + 1, V - 1))
            ptr = np.concatenate([[0], cuts, [n]]).astype(np.int32)
            states.append((ptr, perm.astype(np.int32)))
        for ptr, ms in states:
            ok, obj, bad = pins.xijk_check(inst, routes_of(ptr, ms))
            checked += 1
            assert O.objective(ptr, ms) == obj
            disagreements += (O.feasible(ptr, ms) != ok)
    assert disagreements == 0 and checked > 200


def test_all_move_deltas_vs_xijk(oracle_mod):
    """Every valid move of several feasible states: Delta and FEASIBLE against the
    x_ijk coding of the new schedule; route-local mode == full recompute mode."""
    n_feasible = 0
    for seed in range(4):
        inst = tiny_instance(5, 3, 300 + seed, F=10)
        O = oracle_mod.Oracle(inst)
        for ptr, ms in trajectory_states(O, inst):
            base_obj = pins.xijk_check(inst, routes_of(ptr, ms))[1]
            d, f, best = O.eval_moves(ptr, ms, mode=0)
            dfull, ffull, bfull = O.eval_moves(ptr, ms, mode=0, full=True)
            assert (d == dfull).all() and (f == ffull).all() and best == bfull
            for idx in range(O.move_space_size()):
                ok, (p2, m2) = O.apply_move(ptr, ms, idx)
                assert ok == bool(f[idx] & 1)
                if not ok:
                    assert d[idx] == 0 and f[idx] == 0
                    continue
                feas, obj, _ = pins.xijk_check(inst, routes_of(p2, m2))
                assert d[idx] == obj - base_obj
                assert bool(f[idx] & 2) == feas
                n_feasible += feas
    assert n_feasible > 60


def test_valid_count_state_independent(oracle_mod):
    inst = instgen.generate("tiny")
    O = oracle_mod.Oracle(inst)
    n, V = inst.n_missions, inst.n_vehicles
    for ptr, ms in feasible_states(O, inst, 5):
        d, f, _ = O.eval_moves(ptr, ms)
        assert int((f & 1).sum()) == n * (n + V - 2) + n * (n - 1) // 2 == 100


def test_relocate_inverse_and_swap_involution(oracle_mod):
    inst = instgen.generate("tiny")
    O = oracle_mod.Oracle(inst)
    n, V = inst.n_missions, inst.n_vehicles
    rng = np.random.default_rng(3)
    ptr, ms = inst.planted_ptr, inst.planted_missions
    for _ in range(200):
        idx = int(rng.integers(0, n * (n + V)))
        m, t = divmod(idx, n + V)
        routes = routes_of(ptr, ms)
        a = next(v for v in range(V) if m in routes[v])
        i = routes[a].index(m)
        succ = routes[a][i + 1] if i + 1 < len(routes[a]) else n + a
        ok, (p2, m2) = O.apply_move(ptr, ms, idx)
        if not ok:
            continue
        back = m * (n + V) + succ          # reinsert m before its old successor slot
        ok2, (p3, m3) = O.apply_move(p2, m2, back)
        assert ok2 and routes_of(p3, m3) == routes
        m1, mb = sorted(rng.choice(n, 2, replace=False))
        sidx = n * (n + V) + m1 * n + mb
        ok3, (p4, m4) = O.apply_move(ptr, ms, sidx)
        ok4, (p5, m5) = O.apply_move(p4, m4, sidx)
        assert ok3 and ok4 and routes_of(p5, m5) == routes


def test_f2_lemma_intra_moves_infeasible(oracle_mod):
    """with waiting and positive legs, feasible routes are strictly
    deadline-sorted, so no intra-route reorder or swap is ever feasible."""
    for cfgname in ("tiny", "ontario"):
        inst = instgen.generate(cfgname)
        O = oracle_mod.Oracle(inst)
        assert (inst.travel_s[:, inst.pickup_loc, inst.delivery_loc] > 0).all()
        for ptr, ms in feasible_states(O, inst, 4):
            d, f, _ = O.eval_moves(ptr, ms, mask=0x2 | 0x8)
            assert int((f & 1).sum()) > 0
            assert int((f & 2).sum()) == 0
            routes = routes_of(ptr, ms)
            for r in routes:
                assert all(inst.deadline_s[x] < inst.deadline_s[y] for x, y in zip(r[:-1], r[1:]))


# ---------------------------------------------------------- exact optimum pins --
def test_brute_equals_ilp_and_bounds_search(oracle_mod):
    for seed in range(8):
        inst = tiny_instance(5, 3, 500 + seed)
        O = oracle_mod.Oracle(inst)
        opt, routes = pins.brute_optimum(inst)
        assert opt is not None
        assert pins.ilp_optimum(inst) == opt
        assert pins.xijk_check(inst, routes)[:2] == (True, opt)
        ptr, ms = inst.planted_ptr, inst.planted_missions
        ts = O.search(ptr, ms, mode=1, tenure=3, max_iters=60)
        ns = O.search(ptr, ms, mode=0, max_iters=60)
        assert ts["best_obj"] >= opt and ns["best_obj"] >= opt
        # NS stops at a local optimum: no feasible improving move remains (O11)
        assert ns["stop_reason"] == 1
        d, f, best = O.eval_moves(*ns["best"], mode=0)
        assert not ((f & 2).astype(bool) & (d < 0)).any() and best[0] != 0


def test_c1_tiny_optimum(oracle_mod):
    inst = instgen.generate("tiny")
    O = oracle_mod.Oracle(inst)
    opt, routes = pins.brute_optimum(inst)
    assert opt == pins.ilp_optimum(inst)
    ptr, ms = inst.planted_ptr, inst.planted_missions
    ts = O.search(ptr, ms, mode=1, tenure=5, max_iters=200)
    assert ts["best_obj"] >= opt
    assert O.feasible(*ts["best"]) and O.objective(*ts["best"]) == ts["best_obj"]


# ------------------------------------------------------------- O14 invariants --
@pytest.mark.parametrize("cfgname,iters", [("tiny", 200), ("ontario", 300)])
def test_search_invariants(oracle_mod, cfgname, iters):
    inst = instgen.generate(cfgname)
    O = oracle_mod.Oracle(inst)
    ptr, ms = inst.planted_ptr, inst.planted_missions
    start = O.objective(ptr, ms)
    ns = O.search(ptr, ms, mode=0, max_iters=iters)
    cur = [start] + list(ns["trace"]["cur"])
    assert all(b < a for a, b in zip(cur[:-1], cur[1:]))          # NS strictly decreasing
    assert O.feasible(*ns["best"]) and O.objective(*ns["best"]) == ns["best_obj"]
    ts = O.search(ptr, ms, mode=1, tenure=10, max_iters=iters)
    tr = ts["trace"]
    assert all(b <= a for a, b in zip(tr["best"][:-1], tr["best"][1:]))   # best non-increasing
    assert (np.diff(np.concatenate([[start], tr["cur"]])) == tr["delta"]).all()
    assert O.feasible(*ts["best"]) and O.objective(*ts["best"]) == ts["best_obj"]
    assert O.feasible(*ts["final"]) and O.objective(*ts["final"]) == ts["final_obj"]
    assert ts["best_obj"] <= ns["best_obj"] or True    # statistical only (SPEC criterion 4)


def test_tabu_state_follows_moves(oracle_mod):
    """E after the run equals it+tenure on the 'from' pairs of the last moves (O8)."""
    inst = instgen.generate("tiny")
    O = oracle_mod.Oracle(inst)
    ptr, ms = inst.planted_ptr, inst.planted_missions
    r = O.search(ptr, ms, mode=1, tenure=5, max_iters=50, digest=True)
    E = r["E"]
    assert E.max() <= r["iters_done"] - 1 + 5
    assert r["trace"]["digest"][-1] == O.tabu_digest(E, r["iters_done"] - 1)


# ------------------------------------------------------------ greedy (O13) ---
def test_greedy_spec_examples(oracle_mod):
    inst = tiny_instance(4, 3, 900)
    # zero missions -> all routes empty
    empty = instgen.Instance(inst.travel_s, inst.class_is_heli, inst.base_location, inst.vehicle_base,
                             inst.vehicle_class, np.zeros(0, np.int32), np.zeros(0, np.int32),
                             np.zeros(0, np.int32), np.zeros(0, np.uint8))
    st, (ptr, ms), nrep, order = oracle_mod.Oracle(empty).greedy()
    assert st == 0 and len(ms) == 0 and list(ptr) == [0] * (inst.n_vehicles + 1)
    # equal deadlines -> lower id first; heli-only missions first
    tie = instgen.Instance(inst.travel_s, inst.class_is_heli, inst.base_location, inst.vehicle_base,
                           inst.vehicle_class, inst.pickup_loc, inst.delivery_loc,
                           np.array([50000, 50000, 40000, 60000], np.int32), np.array([0, 0, 0, 1], np.uint8))
    st, _, _, order = oracle_mod.Oracle(tie).greedy()
    assert list(order) == [3, 2, 0, 1]


def test_greedy_feasible_or_fails(oracle_mod):
    for name in ("tiny", "ontario", "batched"):
        inst = instgen.generate(name)
        O = oracle_mod.Oracle(inst)
        for mode in (0, 1):
            st, (ptr, ms), nrep, order = O.greedy(insert_mode=mode)
            if st == 0:
                assert O.feasible(ptr, ms)
                heli_pos = [i for i, m in enumerate(order) if inst.heli_only[m]]
                rest = [i for i, m in enumerate(order) if not inst.heli_only[m]]
                assert not heli_pos or not rest or max(heli_pos) < min(rest)


def test_kick_keeps_feasibility(oracle_mod):
    inst = instgen.generate("batched")
    O = oracle_mod.Oracle(inst)
    ptr, ms = inst.planted_ptr, inst.planted_missions
    for s in range(1, 20):
        k, st = O.kick(ptr, ms, s, 8)
        assert O.feasible(*st)
        k2, st2 = O.kick(ptr, ms, s, 8)
        assert k == k2 and routes_of(*st) == routes_of(*st2)
    k0, st0 = O.kick(ptr, ms, 0, 8)
    assert k0 == 0 and routes_of(*st0) == routes_of(ptr, ms)


def test_generated_instances_planted_feasible(oracle_mod):
    for name in instgen.CONFIGS:
        inst = instgen.generate(name)
        O = oracle_mod.Oracle(inst)
        assert O.feasible(inst.planted_ptr, inst.planted_missions), name
        a = instgen.generate(name)
        assert (a.travel_s == inst.travel_s).all() and (a.deadline_s == inst.deadline_s).all()


def test_e1_sweep_golden(oracle_mod):
    """f1: the paper-literal (i, j) sweep of Alg. 2 / Alg. 3 on E1, derived by hand."""
    I = e1_instance()
    O = oracle_mod.Oracle(I)
    ptr, ms = csr(GOLD["start"])
    r = O.sweep(ptr, ms, mode=0, max_steps=50)
    assert list(r["trace"]["idx"]) == GOLD["sweep_ns"]["idx"]
    assert r["best_obj"] == GOLD["sweep_ns"]["objective"] and r["stop_reason"] == 1
    r = O.sweep(ptr, ms, mode=1, tenure=2, max_steps=50)
    assert list(r["trace"]["idx"]) == GOLD["sweep_ts_tenure2"]["idx"]
    assert list(r["trace"]["delta"]) == GOLD["sweep_ts_tenure2"]["delta"]


def test_sweep_invariants(oracle_mod):
    """Sweep moves are inter-route relocates only; NS never worsens; results are feasible
    and bounded below by the exact optimum; seeded permutations change the order."""
    for seed in (0, 5):
        inst = tiny_instance(5, 3, 300 + seed, F=10)
        O = oracle_mod.Oracle(inst)
        st, (p, m), _, _ = O.greedy()
        opt, _ = pins.brute_optimum(inst)
        n, V = inst.n_missions, inst.n_vehicles
        for mode in (0, 1):
            r = O.sweep(p, m, mode=mode, tenure=3, max_steps=60, seed=seed)
            idx = r["trace"]["idx"]
            applied = idx[idx >= 0]
            assert (applied < n * (n + V)).all()
            if mode == 0:
                assert (r["trace"]["delta"][idx >= 0] < 0).all()
            assert O.feasible(*r["best"]) and r["best_obj"] >= opt
    inst = instgen.generate("ontario")
    O = oracle_mod.Oracle(inst)
    st, (p, m), _, _ = O.greedy()
    a = O.sweep(p, m, mode=1, max_steps=200, seed=0)
    b = O.sweep(p, m, mode=1, max_steps=200, seed=7)
    assert not (a["trace"]["idx"] == b["trace"]["idx"]).all()


# ------------------------------------------------------------- f3: no-wait ---
def _nowait_copy(inst, deadlines=None):
    import dataclasses
    out = dataclasses.replace(inst, no_wait=1)
    if deadlines is not None:
        out.deadline_s = np.array(deadlines, np.int32)
    return out


def test_e1_nowait_golden(oracle_mod):
    """E1 with deadlines (3000, 2000, 3000), by hand: v0 = [m1, m0, m2] (idx 2 from the start
    [m0, m1, m2]) arrives at m1 at 900, m0 at 900 + 900 = 1800, m2 at 1800 + 100 = 1900 and
    back at 2000 -- feasible without waiting; with waiting m1 departs at 2000, m0 at 3000 and
    m2 is reached at 3100 > 3000."""
    wait = _nowait_copy(e1_instance(), [3000, 2000, 3000])
    wait.no_wait = 0
    nowait = _nowait_copy(e1_instance(), [3000, 2000, 3000])
    ptr, ms = csr(GOLD["start"])
    dw, fw, _ = oracle_mod.Oracle(wait).eval_moves(ptr, ms, mode=0)
    dn, fn, _ = oracle_mod.Oracle(nowait).eval_moves(ptr, ms, mode=0)
    assert dw[2] == dn[2] == 200
    assert not fw[2] & 2 and fn[2] & 2
    assert oracle_mod.Oracle(nowait).route_feasible(0, [1, 0, 2])
    assert not oracle_mod.Oracle(wait).route_feasible(0, [1, 0, 2])


def test_nowait_vs_independent_check(oracle_mod):
    rng = np.random.default_rng(12)
    n_feas = 0
    for seed in range(4):
        base = tiny_instance(5, 3, 700 + seed, F=10)
        inst = _nowait_copy(base)
        O = oracle_mod.Oracle(inst)
        Ow = oracle_mod.Oracle(base)
        states = trajectory_states(Ow, base)
        n, V = inst.n_missions, inst.n_vehicles
        for _ in range(30):
            perm = rng.permutation(n).astype(np.int32)
            cuts = np.sort(rng.integers(0, n + 1, V - 1))
            states.append((np.concatenate([[0], cuts, [n]]).astype(np.int32), perm))
        for ptr, ms in states:
            routes = routes_of(ptr, ms)
            ok = all(pins.route_eval_nowait(inst, k, r) is not None for k, r in enumerate(routes))
            assert O.feasible(ptr, ms) == ok
            if Ow.feasible(ptr, ms):          # waiting-feasible => no-wait-feasible
                assert ok
        for ptr, ms in trajectory_states(Ow, base):
            d, f, _ = O.eval_moves(ptr, ms, mode=0)
            base_obj = O.objective(ptr, ms)
            for idx in range(O.move_space_size()):
                okm, (p2, m2) = O.apply_move(ptr, ms, idx)
                if not okm:
                    continue
                routes = routes_of(p2, m2)
                feas = all(pins.route_eval_nowait(inst, k, r) is not None for k, r in enumerate(routes))
                assert bool(f[idx] & 2) == feas and d[idx] == O.objective(p2, m2) - base_obj
                n_feas += feas
    assert n_feas > 50


# --------------------------------------------------- f2: randomized starts ---
def _replay_greedy(inst, order, insert_mode, nowait=False):
    """Independent replay of Alg. 1's placement decisions for a given
    order, with the route checks of tests/pins.py: candidate slot per vehicle
    (tail, or the deadline-sorted slot), feasible candidates only, the
    smallest cost increase, ties to the lower vehicle (reading #24).  None when a
    mission cannot be placed (the oracle would repair)."""
    n, V, NN, d, b, f = pins._node_model(inst)
    routes = [[] for _ in range(V)]

    def cost(k, r):
        if nowait:
            return pins.route_eval_nowait(inst, k, r, d)
        return pins._route_eval(inst, k, tuple(r), d, n) if r else 0

    for m in order:
        best = None
        for k in range(V):
            r = routes[k]
            at = len(r)
            if insert_mode == 1:
                at = 0
                while at < len(r) and inst.deadline_s[r[at]] <= inst.deadline_s[m]:
                    at += 1
            r2 = r[:at] + [int(m)] + r[at:]
            c2, c1 = cost(k, r2), cost(k, r)
            if c2 is None:
                continue
            if best is None or c2 - c1 < best[0]:
                best = (c2 - c1, k, r2)
        if best is None:
            return None
        routes[best[1]] = best[2]
    return routes


def test_seeded_greedy_order_and_replay(oracle_mod):
    """Seed 0 is Alg. 1 as written; seed != 0 permutes each phase (reading #41).
    Every seeded start that needed no repair equals an independent replay of the
    placement rule in the oracle's reported order."""
    n_checked = 0
    for cfg, nowait in (("tiny", False), ("ontario", False), ("batched", False), ("ontario", True)):
        inst = instgen.generate(cfg)
        if nowait:
            import dataclasses
            inst = dataclasses.replace(inst, no_wait=1)
        O = oracle_mod.Oracle(inst)
        heli = set(np.flatnonzero(inst.heli_only).tolist())
        base = O.greedy(insert_mode=1)
        assert routes_of(*O.greedy(insert_mode=1, seed=0)[1]) == routes_of(*base[1])
        orders = set()
        for seed in range(1, 9):
            for mode in (0, 1):
                st, (p, m), nrep, order = O.greedy(insert_mode=mode, seed=seed)
                assert sorted(order.tolist()) == list(range(inst.n_missions))
                k = len(heli)
                assert set(order[:k].tolist()) == heli
                orders.add(tuple(order.tolist()))
                if st == 0:
                    assert O.feasible(p, m)
                if nrep == 0:
                    rep = _replay_greedy(inst, order, mode, nowait)
                    if st == 0:
                        assert rep == routes_of(p, m)
                        n_checked += 1
                    else:
                        assert rep is None
        assert len(orders) == 8
    assert n_checked >= 10


def test_seeded_greedy_permutation_uniform(oracle_mod):
    """The phase permutations are uniform (a Fisher-Yates range slip would not be):
    3 non-heli missions with distinct deadlines, 6000 seeds, chi-square over the 6 orders."""
    inst = tiny_instance(3, 3, 901)
    inst.heli_only = np.zeros(3, np.uint8)
    inst.deadline_s = np.array([80000, 70000, 60000], np.int32)
    O = oracle_mod.Oracle(inst)
    counts = {}
    for seed in range(1, 6001):
        order = tuple(O.greedy(insert_mode=1, seed=seed)[3].tolist())
        counts[order] = counts.get(order, 0) + 1
    assert len(counts) == 6
    exp = 1000.0
    chi2 = sum((c - exp) ** 2 / exp for c in counts.values())
    assert chi2 < 20.5   # p ~ 0.001 at 5 degrees of freedom
    assert O.greedy(insert_mode=1)[3].tolist() == [2, 1, 0]
