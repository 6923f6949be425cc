"""Independent pins for the oracle (test helpers; no code shared with oracle/ or the CUDA path).

* `xijk_check` expands a route schedule into the paper's decision variables
  x_ijk and u_i and tests Eqs. obj_s, con1-con13 (§3) as
  written (con8 read additively, reading #3).  It is a second coding of the
  model: link-local constraints on arcs, not the oracle's clock simulation.
* `brute_optimum` enumerates, for every vehicle and every subset of missions,
  every order of that subset (exhaustive, no pruning), and combines vehicles by
  a subset DP.  Exact for tiny instances.
* `ilp_optimum` builds the arc ILP (Eqs. obj_s, con1-con13) and solves it with
  scipy's HiGHS `milp` -- the test-only stand-in for Gurobi.
"""
from __future__ import annotations

import itertools

import numpy as np


def _node_model(inst):
    """Nodes 0..n-1 = missions, n+k = base node of vehicle k (reading #12)."""
    n, V = inst.n_missions, inst.n_vehicles
    vloc = inst.base_location[inst.vehicle_base]
    end = np.concatenate([inst.delivery_loc, vloc]).astype(np.int64)
    L = inst.n_classes
    NN = n + V
    d = np.zeros((NN, NN, L), np.int64)         # d_ijl (reading #1)
    for l in range(L):
        T = inst.travel_s[l].astype(np.int64)
        for i in range(NN):
            for j in range(NN):
                if j < n:
                    d[i, j, l] = T[end[i], inst.pickup_loc[j]] + T[inst.pickup_loc[j], inst.delivery_loc[j]]
                else:
                    d[i, j, l] = T[end[i], vloc[j - n]]
    b = np.array([0 if inst.class_is_heli[c] else 1 for c in inst.vehicle_class], np.int64)  # b_k
    f = np.array([0 if h else 1 for h in inst.heli_only], np.int64)                            # f_n
    return n, V, NN, d, b, f


def xijk_check(inst, routes):
    """routes: list of V mission lists.  Returns (feasible, objective, violated-constraint names)."""
    n, V, NN, d, b, f = _node_model(inst)
    x = np.zeros((NN, NN, V), np.int64)
    u = np.zeros(n, np.int64)
    for k, r in enumerate(routes):
        if not r:
            continue
        seq = [n + k] + list(r) + [n + k]
        for i, j in zip(seq[:-1], seq[1:]):
            x[i, j, k] += 1
        for pos, m in enumerate(r):
            u[m] = pos + 1                      # MTZ order variable
    l_of = [int(inst.vehicle_class[k]) for k in range(V)]  # l = b_k layer; class index is the layer
    bad = []
    obj = int(sum(x[:, :, k].ravel() @ d[:, :, l_of[k]].ravel() for k in range(V)))  # obj_s
    w = np.concatenate([inst.deadline_s.astype(np.int64), np.full(V, inst.day_length_s, np.int64)])
    for j in range(n):                                         # con1
        if x[:, j, :].sum() != 1:
            bad.append("con1")
    for i in range(n):                                         # con2
        if x[i, :, :].sum() != 1:
            bad.append("con2")
    for k in range(V):
        for node in range(NN):                                 # con3
            if x[:, node, k].sum() != x[node, :, k].sum():
                bad.append("con3")
        if (x[:, :, k].sum(axis=0) > 1).any():                 # con4
            bad.append("con4")
        if (x[:, :, k].sum(axis=1) > 1).any():                 # con5
            bad.append("con5")
        if (x[:, :, k] * d[:, :, l_of[k]]).sum() > inst.flight_limit_s:   # con6
            bad.append("con6")
        for i in range(NN):
            for j in range(NN):
                if not x[i, j, k]:
                    continue
                if i >= n and j < n and d[i, j, l_of[k]] > w[j]:          # con7: from a base, clock 0
                    bad.append("con7")
                if i < n and d[i, j, l_of[k]] + w[i] > w[j]:              # con8, additive
                    bad.append("con8")
                if i < n and b[k] - f[i] > 0:                             # con9
                    bad.append("con9")
                if i >= n and j >= n:                                     # con11
                    bad.append("con11")
                if (i >= n and i != n + k) or (j >= n and j != n + k):    # leave/return own base
                    bad.append("own-base")
        for i in range(n):                                     # con10 MTZ
            for j in range(n):
                if i != j and u[i] - u[j] + n * x[i, j, k] > n - 1:
                    bad.append("con10")
    if any(not (1 <= u[i] <= n) for i in range(n) if x[i].sum()):   # con13
        bad.append("con13")
    return (not bad), obj, bad


def _route_eval(inst, k, order, d, n):
    """Cost and feasibility of one route from the arc constraints (link-local form)."""
    l = int(inst.vehicle_class[k])
    if inst.heli_only[list(order)].any() and not inst.class_is_heli[l]:
        return None
    seq = [n + k] + list(order) + [n + k]
    cost = 0
    for i, j in zip(seq[:-1], seq[1:]):
        dij = int(d[i, j, l])
        wi = 0 if i >= n else int(inst.deadline_s[i])
        wj = int(inst.day_length_s) if j >= n else int(inst.deadline_s[j])
        if wi + dij > wj:
            return None
        cost += dij
    if cost > inst.flight_limit_s:
        return None
    return cost


def brute_optimum(inst):
    """Exhaustive optimum (every order of every subset per vehicle, subset DP over vehicles)."""
    n, V, NN, d, b, f = _node_model(inst)
    full = (1 << n) - 1
    best_route = []   # per vehicle: dict mask -> (cost, order)
    for k in range(V):
        table = {0: (0, ())}
        for size in range(1, n + 1):
            for subset in itertools.combinations(range(n), size):
                mask = sum(1 << m for m in subset)
                best = None
                for order in itertools.permutations(subset):
                    c = _route_eval(inst, k, order, d, n)
                    if c is not None and (best is None or c < best[0]):
                        best = (c, order)
                if best is not None:
                    table[mask] = best
        best_route.append(table)
    INF = None
    # dp over vehicles: dp[mask] = min cost covering exactly mask with vehicles 0..k
    dp = {0: (0, [])}
    for k in range(V):
        nd = {}
        for mask, (c0, rs) in dp.items():
            for sub, (c1, order) in best_route[k].items():
                if sub & mask:
                    continue
                m2 = mask | sub
                c = c0 + c1
                if m2 not in nd or c < nd[m2][0]:
                    nd[m2] = (c, rs + [list(order)])
        dp = nd
    if full not in dp:
        return INF, None
    return dp[full]


def ilp_optimum(inst, time_limit=60.0):
    """Arc ILP of Eqs. obj_s, con1-con13 solved by scipy HiGHS (test-only Gurobi stand-in)."""
    from scipy.optimize import Bounds, LinearConstraint, milp
    from scipy.sparse import lil_matrix

    n, V, NN, d, b, f = _node_model(inst)
    w = np.concatenate([inst.deadline_s.astype(np.int64), np.full(V, inst.day_length_s, np.int64)])
    arcs = []   # (i, j, k)
    for k in range(V):
        l = int(inst.vehicle_class[k])
        nodes = list(range(n)) + [n + k]            # own base only (con11)
        for i in nodes:
            for j in nodes:
                if i == j:
                    continue
                if i >= n and j >= n:
                    continue
                dij = int(d[i, j, l])
                wi = 0 if i >= n else int(w[i])     # con7 / con8 (x fixed to 0 when violated)
                if wi + dij > w[j]:
                    continue
                if (i < n and b[k] - f[i] > 0) or (j < n and b[k] - f[j] > 0):   # con9
                    continue
                if dij > inst.flight_limit_s:
                    continue
                arcs.append((i, j, k))
    nx = len(arcs)
    nvar = nx + n
    c = np.zeros(nvar)
    for a, (i, j, k) in enumerate(arcs):
        c[a] = d[i, j, int(inst.vehicle_class[k])]
    rows, lo, hi = [], [], []
    A = lil_matrix((4 * n + 2 * V * NN + V + V + n * n * V + 10, nvar))
    r = 0

    def add(coefs, lb, ub):
        nonlocal r
        for col, val in coefs:
            A[r, col] += val
        lo.append(lb); hi.append(ub); r += 1

    into = {j: [] for j in range(NN)}
    outof = {i: [] for i in range(NN)}
    for a, (i, j, k) in enumerate(arcs):
        into[j].append(a)
        outof[i].append(a)
    for j in range(n):                                   # con1
        add([(a, 1) for a in into[j]], 1, 1)
    for i in range(n):                                   # con2
        add([(a, 1) for a in outof[i]], 1, 1)
    for k in range(V):
        for node in list(range(n)) + [n + k]:            # con3
            add([(a, 1) for a in into[node] if arcs[a][2] == k] + [(a, -1) for a in outof[node] if arcs[a][2] == k], 0, 0)
        add([(a, 1) for a in outof[n + k] if arcs[a][2] == k], 0, 1)            # con5 at the base
        add([(a, float(c[a])) for a in range(nx) if arcs[a][2] == k], -np.inf, inst.flight_limit_s)  # con6
    for a, (i, j, k) in enumerate(arcs):                 # con10 MTZ
        if i < n and j < n:
            add([(nx + i, 1), (nx + j, -1), (a, n)], -np.inf, n - 1)
    A = A[:r].tocsr()
    integrality = np.ones(nvar)
    lb = np.concatenate([np.zeros(nx), np.ones(n)])
    ub = np.concatenate([np.ones(nx), np.full(n, max(n, 1))])
    res = milp(c, constraints=LinearConstraint(A, lo, hi), integrality=integrality, bounds=Bounds(lb, ub),
               options={"time_limit": time_limit})
    if res.status != 0 or res.x is None:
        return None
    return int(round(res.fun))


def route_eval_nowait(inst, k, order, d=None):
    """Independent no-wait route check (f3): the clock carries the arrival time;
    every arrival <= its deadline, return <= day, flight <= p, compatibility.
    d: the node model's d (from _node_model), recomputed when None."""
    n = inst.n_missions
    if d is None:
        d = _node_model(inst)[3]
    l = int(inst.vehicle_class[k])
    if len(order) and inst.heli_only[list(order)].any() and not inst.class_is_heli[l]:
        return None
    if not len(order):
        return 0
    seq = [n + k] + list(order) + [n + k]
    clock, cost = 0, 0
    for i, j in zip(seq[:-1], seq[1:]):
        dij = int(d[i, j, l])
        clock += dij
        cost += dij
        wj = int(inst.day_length_s) if j >= n else int(inst.deadline_s[j])
        if clock > wj:
            return None
    if cost > inst.flight_limit_s:
        return None
    return cost
