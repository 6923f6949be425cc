"""Independent replays of the oracle's search-side rules (test helpers).

Pure Python on top of tests/pins.py's link-local route check (`pins._route_eval`,
a second coding of con6-con9 from the arc form of the ILP).  Nothing
here imports or calls oracle/ or the CUDA path: the canonical move index, the
move semantics, the SplitMix64 generator and every decision rule are written
out again from DESIGN.md's readings and the paper's text, so that a slip in
oracle.c (a wrong modulus, a missing break, a wrong Fisher-Yates range, a
dropped retry) fails a comparison.

Move space: relocate block idx = m(n+V) + t,
t < n inserts m before mission t (as the routes stand after removing m), t = n+v
appends to vehicle v; VALID iff m (and t < n) assigned, t != m and t is not m's
successor slot.  Swap block idx = n(n+V) + m1*n + m2, VALID iff m1 < m2, both
assigned.  Mask bits 1 inter-relocate, 2 intra-relocate, 4 inter-swap, 8
intra-swap.
"""
from __future__ import annotations

import numpy as np

import pins

MASK64 = (1 << 64) - 1


def splitmix64(state: int):
    """SplitMix64 (Steele, Lea & Flood 2014): returns (new_state, output)."""
    state = (state + 0x9E3779B97F4A7C15) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return state, z ^ (z >> 31)


class Model:
    """Routes as Python lists; costs and feasibility from pins' arc form."""

    def __init__(self, inst):
        self.inst = inst
        self.n, self.V, _, self.d, _, _ = pins._node_model(inst)

    def route(self, k, r):
        """Cost of route k, or None if infeasible (empty route: 0).  Instances with
        no_wait (f3, reading #40) use pins' no-wait clock instead of the arc form."""
        if getattr(self.inst, "no_wait", 0):
            return pins.route_eval_nowait(self.inst, k, list(r), self.d)
        return pins._route_eval(self.inst, k, tuple(r), self.d, self.n) if r else 0

    def where(self, routes):
        veh, pos = {}, {}
        for k, r in enumerate(routes):
            for i, m in enumerate(r):
                veh[m], pos[m] = k, i
        return veh, pos

    def apply(self, routes, idx, mask=0xF):
        """Returns (a, b, new routes list, placed pairs, from pairs) or None if not VALID."""
        n, V = self.n, self.V
        veh, pos = self.where(routes)
        if idx < n * (n + V):
            m, t = divmod(idx, n + V)
            if m not in veh:
                return None
            a = veh[m]
            ra = list(routes[a])
            succ = ra[pos[m] + 1] if pos[m] + 1 < len(ra) else n + a
            if t == m or t == succ:
                return None
            if t < n:
                if t not in veh:
                    return None
                b = veh[t]
            else:
                b = t - n
            if not mask & (1 if a != b else 2):
                return None
            ra.remove(m)
            new = [list(r) for r in routes]
            new[a] = ra
            rb = ra if a == b else list(routes[b])
            at = rb.index(t) if t < n else len(rb)
            rb.insert(at, m)
            new[b] = rb
            return a, b, new, [(m, b)], [(m, a)]
        k = idx - n * (n + V)
        m1, m2 = divmod(k, n)
        if not m1 < m2 or m1 not in veh or m2 not in veh:
            return None
        a, b = veh[m1], veh[m2]
        if not mask & (4 if a != b else 8):
            return None
        new = [list(r) for r in routes]
        new[a][pos[m1]] = m2
        new[b][pos[m2]] = m1
        return a, b, new, [(m1, b), (m2, a)], [(m1, a), (m2, b)]

    def evaluate(self, routes, idx, mask=0xF):
        """(delta, feasible, placed pairs, new routes, from pairs) of a VALID move, else None."""
        mv = self.apply(routes, idx, mask)
        if mv is None:
            return None
        a, b, new, placed, frm = mv
        touched = {a, b}
        before = sum(self.route(k, routes[k]) for k in touched)
        after = [self.route(k, new[k]) for k in touched]
        feas = all(c is not None for c in after)
        delta = (sum(after) - before) if feas else None
        return delta, feas, placed, new, frm

    def objective(self, routes):
        return sum(self.route(k, r) for k, r in enumerate(routes))


def kick(model: Model, routes, seed: int, kick_count: int):
    """O12 as DESIGN.md reading #27/#34 states it: seed 0 = no kick; for each of
    `kick_count` kicks draw up to 64 relocate-block indices z mod n(n+V) from one
    SplitMix64 stream, apply the first VALID and FEASIBLE one (every move kind),
    and skip this kick after 64 failed draws."""
    routes = [list(r) for r in routes]
    if seed == 0 or model.n == 0:
        return 0, routes
    s = seed
    R = model.n * (model.n + model.V)
    applied = 0
    for _ in range(kick_count):
        for _try in range(64):
            s, z = splitmix64(s)
            ev = model.evaluate(routes, z % R)
            if ev is not None and ev[1]:
                routes = ev[3]
                applied += 1
                break
    return applied, routes


def ns_iteration(model: Model, routes):
    """One NS iteration over the (possibly partial) schedule: the lowest-index
    move with the smallest negative delta among the feasible ones (reading #17,
    #26), every move kind; None when none improves."""
    n, V = model.n, model.V
    best = None
    for idx in range(n * (n + V) + n * n):
        ev = model.evaluate(routes, idx)
        if ev is None or not ev[1] or ev[0] >= 0:
            continue
        if best is None or ev[0] < best[0]:
            a, b = model.apply(routes, idx)[:2]
            best = (ev[0], idx, ev[3], a == b)
    return best


def greedy(model: Model, order, insert_mode: int, max_repairs: int):
    """Algorithm 1 in the given placement order with the repair rule of
    reading #22: when no vehicle can take mission m, fail if nothing is assigned
    yet or the repair budget is spent; otherwise perform ONE NS iteration
    over the assigned missions ("mission swaps from Algorithm 2"; "only
    performs a single iteration"), fail if it finds no improving move, and
    retry m once (fail if the retry fails).  Returns (status, routes, repairs,
    [(index, same-route) of each repair move])."""
    inst = model.inst
    routes = [[] for _ in range(model.V)]
    repairs = 0
    assigned = 0
    picked = []

    def place(m):
        best = None
        for k in range(model.V):
            r = routes[k]
            at = len(r)
            if insert_mode == 1:
                at = 0
                while at < len(r) and inst.deadline_s[r[at]] <= inst.deadline_s[m]:
                    at += 1
            r2 = r[:at] + [int(m)] + r[at:]
            c2 = model.route(k, r2)
            if c2 is None:
                continue
            inc = c2 - model.route(k, r)
            if best is None or inc < best[0]:
                best = (inc, k, r2)
        return best

    for m in order:
        m = int(m)
        b = place(m)
        if b is None:
            if assigned == 0 or repairs >= max_repairs:
                return 3, routes, repairs, picked
            step = ns_iteration(model, routes)
            if step is None:
                return 3, routes, repairs, picked
            routes = step[2]
            picked.append((step[1], step[3]))
            repairs += 1
            b = place(m)
            if b is None:
                return 3, routes, repairs, picked
        routes[b[1]] = b[2]
        assigned += 1
    return 0, routes, repairs, picked


def fisher_yates(items, s):
    """In-place SplitMix64 Fisher-Yates from the top: for x = L-1 .. 1 swap x with
    y = z mod (x+1).  Returns the new generator state."""
    for x in range(len(items) - 1, 0, -1):
        s, z = splitmix64(s)
        y = z % (x + 1)
        items[x], items[y] = items[y], items[x]
    return s


def sweep(model: Model, routes, mode: int, tenure: int, max_steps: int, seed: int):
    """f1, the paper-literal Alg. 2 / Alg. 3 sweep as DESIGN.md reading #39 states
    it.  Per sweep: a permutation of the vehicles ("random index permutation
    vectors"; identity when seed = 0); per vehicle i a snapshot of its route at the
    start of its turn, permuted likewise; per mission j of the snapshot one step:
    CurrentMin = the best (delta, idx) FEASIBLE inter-route relocate of j
    that is admissible (NS: delta < 0; TS: (j, target) not tabu, i.e. E < step, or
    cur + delta < best); applied when not empty (P:331 / P:408); TS then sets
    E[j][from] = step + tenure.  Stops after max_steps steps or a sweep
    without a move.  Returns dict(trace idx/delta/cur/best, best_obj, stop_reason)."""
    n, V = model.n, model.V
    routes = [list(r) for r in routes]
    E = {}
    cur = model.objective(routes)
    best = cur
    s = seed
    step = 0
    tr = dict(idx=[], delta=[], cur=[], best=[])
    stop_reason = 0
    while step < max_steps:
        moved = False
        perm = list(range(V))
        if seed:
            s = fisher_yates(perm, s)
        for i in perm:
            snap = list(routes[i])
            if seed:
                s = fisher_yates(snap, s)
            for j in snap:
                cand = None
                for t in range(n + V):
                    idx = j * (n + V) + t
                    ev = model.evaluate(routes, idx, mask=1)
                    if ev is None or not ev[1]:
                        continue
                    delta, _, placed, new, frm = ev
                    if mode == 1:
                        tabu = any(E.get(p, -1) >= step for p in placed)
                        adm = (not tabu) or cur + delta < best
                    else:
                        adm = delta < 0
                    if adm and (cand is None or delta < cand[0]):
                        cand = (delta, idx, new, frm)
                if cand is not None:
                    routes = cand[2]
                    cur += cand[0]
                    moved = True
                    if mode == 1:
                        E[cand[3][0]] = step + tenure
                    best = min(best, cur)
                tr["idx"].append(cand[1] if cand else -1)
                tr["delta"].append(cand[0] if cand else 0)
                tr["cur"].append(cur)
                tr["best"].append(best)
                step += 1
                if step >= max_steps:
                    break
            if step >= max_steps:
                break
        if step >= max_steps:
            break
        if not moved:
            stop_reason = 1 if mode == 0 else 2
            break
    return dict(trace={k: np.array(v, np.int64) for k, v in tr.items()}, best_obj=best, final=routes,
                stop_reason=stop_reason, iters_done=step)


def search(model: Model, routes, mode: int, tenure: int, max_iters: int, seed: int = 0, kick_count: int = 0,
           strict_tabu_stop: bool = False):
    """O10/O11 in north_star's global-best form (readings #16-#21, #26,
    #29): per iteration the whole move space; ADMISSIBLE = FEASIBLE and (NS) delta
    < 0 or (TS) not tabu or cur + delta < best; the smallest delta, lowest index,
    among the admissible, else (by-default class) among the feasible; NS stops on
    the by-default class, TS on no feasible move; TS writes E[from pairs] = it +
    tenure.  Small instances only (pure Python)."""
    n, V = model.n, model.V
    k_applied, routes = kick(model, routes, seed, kick_count)
    E = {}
    cur = model.objective(routes)
    best = cur
    best_routes = [list(r) for r in routes]
    tr = dict(idx=[], delta=[], cur=[], best=[], cls=[])
    stop = 0
    for it in range(max_iters):
        adm = dflt = None
        for idx in range(n * (n + V) + n * n):
            ev = model.evaluate(routes, idx)
            if ev is None or not ev[1]:
                continue
            delta, _, placed, new, frm = ev
            if mode == 1:
                ok = not any(E.get(p, -1) >= it for p in placed) or cur + delta < best
            else:
                ok = delta < 0
            if ok:
                if adm is None or delta < adm[0]:
                    adm = (delta, idx, new, frm)
            elif dflt is None or delta < dflt[0]:
                dflt = (delta, idx, new, frm)
        pick, cls = (adm, 0) if adm is not None else (dflt, 1)
        if pick is None:
            stop = 2
            break
        if cls == 1 and (mode == 0 or strict_tabu_stop):
            stop = 1 if mode == 0 else 2
            break
        routes = pick[2]
        cur += pick[0]
        if mode == 1:
            for p in pick[3]:
                E[p] = it + tenure
        if cur < best:
            best = cur
            best_routes = [list(r) for r in routes]
        for key, val in zip(("idx", "delta", "cur", "best", "cls"), (pick[1], pick[0], cur, best, cls)):
            tr[key].append(val)
    return dict(trace={k: np.array(v, np.int64) for k, v in tr.items()}, best_obj=best, best=best_routes,
                final=routes, stop_reason=stop, kicks_applied=k_applied, E=E)
