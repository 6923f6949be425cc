"""Exact optimum and MPS export of the paper's model.

The arc formulation of Eqs. obj_s, con1-con13 (§3) for a synthetic
instance, with the readings of DESIGN.md §2 (con8 additive, #3; con7 from a base with clock 0,
#4; heli polarity, #9; vehicles as routing units that leave and return to their own base, #12).
Variables: x_i_j_k (vehicle k travels node i -> node j; nodes 0..n-1 are missions, n+k is
vehicle k's base) and u_i (MTZ order, con10/con13).  Arcs that violate con7, con8, con9 or the
own-base rule (con11) are kept as columns and fixed to 0 by their bounds, so the file
holds the whole model.  `solve` runs scipy's HiGHS `milp` (the stand-in for Gurobi);
`export_mps` writes fixed-format MPS with deterministic names for any external MILP solver.

This is a tool, not the search path: nothing in paper_2002_11710_b200/ imports it.
"""
from __future__ import annotations

import numpy as np


def _node_costs(inst):
    """d[i, j, l] (reading #1) over mission and base nodes."""
    n, V = inst.n_missions, inst.n_vehicles
    vloc = inst.base_location[inst.vehicle_base]
    end = np.concatenate([inst.delivery_loc, vloc]).astype(np.int64)
    NN = n + V
    d = np.zeros((NN, NN, inst.n_classes), np.int64)
    for l in range(inst.n_classes):
        T = inst.travel_s[l].astype(np.int64)
        pick, dele = inst.pickup_loc.astype(np.int64), inst.delivery_loc.astype(np.int64)
        to_m = T[end][:, pick] + T[pick, dele][None, :]
        to_b = T[end][:, vloc]
        d[:, :n, l] = to_m
        d[:, n:, l] = to_b
    return d


def build_model(inst):
    """Columns, objective, constraint rows and bounds of the model.
    Returns dict(names, c, rows=[(name, [(col, coef)], lo, hi)], lb, ub, integer)."""
    n, V = inst.n_missions, inst.n_vehicles
    NN = n + V
    d = _node_costs(inst)
    w = np.concatenate([inst.deadline_s.astype(np.int64), np.full(V, inst.day_length_s, np.int64)])
    heli_cls = [bool(inst.class_is_heli[c]) for c in range(inst.n_classes)]
    names, c, lb, ub = [], [], [], []
    col = {}
    for k in range(V):
        l = int(inst.vehicle_class[k])
        for i in range(NN):
            for j in range(NN):
                if i == j or (i >= n and j >= n):
                    continue
                if (i >= n and i != n + k) or (j >= n and j != n + k):
                    continue            # only vehicle k's own base node (con11)
                dij = int(d[i, j, l])
                wi = 0 if i >= n else int(w[i])
                ok = wi + dij <= int(w[j])                                  # con7 / con8
                ok &= not ((i < n and inst.heli_only[i] and not heli_cls[l]) or
                           (j < n and inst.heli_only[j] and not heli_cls[l]))   # con9
                ok &= dij <= inst.flight_limit_s
                col[(i, j, k)] = len(names)
                names.append(f"x_{i}_{j}_{k}")
                c.append(float(dij))
                lb.append(0.0)
                ub.append(1.0 if ok else 0.0)
    nx = len(names)
    for i in range(n):
        names.append(f"u_{i}")
        c.append(0.0)
        lb.append(1.0)
        ub.append(float(max(n, 1)))
    rows = []
    into = {j: [] for j in range(NN)}
    outof = {i: [] for i in range(NN)}
    for (i, j, k), a in col.items():
        into[j].append(a)
        outof[i].append(a)
    for j in range(n):                                                   # con1
        rows.append((f"con1_{j}", [(a, 1.0) for a in into[j]], 1.0, 1.0))
    for i in range(n):                                                   # con2
        rows.append((f"con2_{i}", [(a, 1.0) for a in outof[i]], 1.0, 1.0))
    for k in range(V):
        l = int(inst.vehicle_class[k])
        for node in list(range(n)) + [n + k]:                            # con3 flow
            rows.append((f"con3_{node}_{k}", [(a, 1.0) for a in into[node] if _k(names[a]) == k] +
                         [(a, -1.0) for a in outof[node] if _k(names[a]) == k], 0.0, 0.0))
        rows.append((f"con5_{k}", [(a, 1.0) for a in outof[n + k] if _k(names[a]) == k], 0.0, 1.0))  # one tour
        rows.append((f"con6_{k}", [(a, c[a]) for (i, j, kk), a in col.items() if kk == k],
                     -np.inf, float(inst.flight_limit_s)))                # con6
    for (i, j, k), a in col.items():                                     # con10 MTZ
        if i < n and j < n:
            rows.append((f"con10_{i}_{j}_{k}", [(nx + i, 1.0), (nx + j, -1.0), (a, float(n))], -np.inf, float(n - 1)))
    return dict(names=names, c=np.array(c), rows=rows, lb=np.array(lb), ub=np.array(ub), nx=nx)


def _k(name):
    return int(name.rsplit("_", 1)[1])


def solve(inst, time_limit=60.0):
    """Optimum objective (integer seconds) by scipy HiGHS, or None if not proven in the limit."""
    from scipy.optimize import Bounds, LinearConstraint, milp
    from scipy.sparse import lil_matrix
    M = build_model(inst)
    nv = len(M["names"])
    if inst.n_missions == 0:
        return 0
    A = lil_matrix((len(M["rows"]), nv))
    lo, hi = [], []
    for r, (_, coefs, a, b) in enumerate(M["rows"]):
        for j, v in coefs:
            A[r, j] += v
        lo.append(a)
        hi.append(b)
    res = milp(M["c"], constraints=LinearConstraint(A.tocsr(), lo, hi), integrality=np.ones(nv),
               bounds=Bounds(M["lb"], M["ub"]), options={"time_limit": time_limit})
    if res.status != 0 or res.x is None:
        return None
    return int(round(res.fun))


def export_mps(inst, path):
    """Fixed-format MPS of build_model (rows N obj, E/L/G/ranged via RANGES; integer markers)."""
    M = build_model(inst)
    names, c, rows = M["names"], M["c"], M["rows"]
    cols = {j: [] for j in range(len(names))}
    rtype = {}
    rng = {}
    rhs = {}
    for name, coefs, lo, hi in rows:
        for j, v in coefs:
            cols[j].append((name, v))
        if lo == hi:
            rtype[name], rhs[name] = "E", lo
        elif np.isinf(lo):
            rtype[name], rhs[name] = "L", hi
        elif np.isinf(hi):
            rtype[name], rhs[name] = "G", lo
        else:
            rtype[name], rhs[name], rng[name] = "G", lo, hi - lo
    out = [f"NAME          AIRSCHED_{inst.n_missions}x{inst.n_vehicles}", "ROWS", " N  obj"]
    out += [f" {rtype[name]}  {name}" for name, _, _, _ in rows]
    out.append("COLUMNS")
    out.append("    MARKER                 'MARKER'                 'INTORG'")
    for j, nm in enumerate(names):
        if c[j] != 0:
            out.append(f"    {nm}  obj  {c[j]:.12g}")
        for rn, v in cols[j]:
            out.append(f"    {nm}  {rn}  {v:.12g}")
        if c[j] == 0 and not cols[j]:
            out.append(f"    {nm}  obj  0")
    out.append("    MARKER                 'MARKER'                 'INTEND'")
    out.append("RHS")
    for name, _, _, _ in rows:
        if rhs[name] != 0:
            out.append(f"    RHS  {name}  {rhs[name]:.12g}")
    if rng:
        out.append("RANGES")
        for name, v in rng.items():
            out.append(f"    RNG  {name}  {v:.12g}")
    out.append("BOUNDS")
    for j, nm in enumerate(names):
        if M["lb"][j] == M["ub"][j]:
            out.append(f" FX BND  {nm}  {M['lb'][j]:.12g}")
        else:
            if M["lb"][j] != 0:
                out.append(f" LO BND  {nm}  {M['lb'][j]:.12g}")
            out.append(f" UP BND  {nm}  {M['ub'][j]:.12g}")
    out.append("ENDATA")
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")
    return path


def read_mps(path):
    """Minimal reader of the files export_mps writes (for round-trip tests): returns
    (names, c, rows=[(name, {col: coef}, lo, hi)], lb, ub)."""
    sect = None
    rtype, order, coefs, c, rhs, rng, lb, ub, names = {}, [], {}, {}, {}, {}, {}, {}, []
    for line in open(path):
        if not line.strip():
            continue
        if not line.startswith(" "):
            sect = line.split()[0]
            continue
        t = line.split()
        if sect == "ROWS":
            if t[0] != "N":
                rtype[t[1]] = t[0]
                order.append(t[1])
                coefs[t[1]] = {}
        elif sect == "COLUMNS":
            if t[1] == "'MARKER'":
                continue
            if t[0] not in c:
                names.append(t[0])
                c[t[0]] = 0.0
                lb[t[0]], ub[t[0]] = 0.0, np.inf
            if t[1] == "obj":
                c[t[0]] = float(t[2])
            else:
                coefs[t[1]][t[0]] = float(t[2])
        elif sect == "RHS":
            rhs[t[1]] = float(t[2])
        elif sect == "RANGES":
            rng[t[1]] = float(t[2])
        elif sect == "BOUNDS":
            kind, nm, v = t[0], t[2], float(t[3])
            if kind == "FX":
                lb[nm] = ub[nm] = v
            elif kind == "LO":
                lb[nm] = v
            elif kind == "UP":
                ub[nm] = v
    rows = []
    for r in order:
        b = rhs.get(r, 0.0)
        if rtype[r] == "E":
            lo, hi = b, b
        elif rtype[r] == "L":
            lo, hi = -np.inf, b
        else:
            lo, hi = b, (b + rng[r]) if r in rng else np.inf
        rows.append((r, coefs[r], lo, hi))
    return names, np.array([c[nm] for nm in names]), rows, np.array([lb[nm] for nm in names]), \
        np.array([ub[nm] for nm in names])
