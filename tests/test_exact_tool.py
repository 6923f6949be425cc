"""f4 exact tool (tools/exact.py): the arc model's optimum by HiGHS and its MPS export,
pinned to exhaustive enumeration (tests/pins.py brute_optimum) and to the test-side ILP
coding (pins.ilp_optimum); MPS round trip; con9 fixings; the empty instance."""
import os
import sys

import numpy as np
import pytest

import pins
from e1 import e1_instance
from paper_2002_11710_b200 import instgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import exact  # noqa: E402


def tiny(n, V, seed, F=6):
    cfg = instgen.Config("t", n, V - max(1, V // 3), max(1, V // 3), 1, 1, F, "ontario", 4, 50, 3)
    return instgen.generate(cfg, seed=seed)


def solve_mps(path):
    from scipy.optimize import Bounds, LinearConstraint, milp
    from scipy.sparse import lil_matrix
    names, c, rows, lb, ub = exact.read_mps(path)
    if not names:                 # objective-only model (no missions): nothing to decide
        return 0
    idx = {nm: j for j, nm in enumerate(names)}
    A = lil_matrix((len(rows), len(names)))
    lo, hi = [], []
    for r, (_, co, a, b) in enumerate(rows):
        for nm, v in co.items():
            A[r, idx[nm]] = v
        lo.append(a)
        hi.append(b)
    res = milp(c, constraints=LinearConstraint(A.tocsr(), lo, hi), integrality=np.ones(len(names)),
               bounds=Bounds(lb, ub))
    assert res.status == 0
    return int(round(res.fun))


@pytest.mark.parametrize("case", ["e1", "t5a", "t5b", "t6"])
def test_exact_equals_brute_force_and_mps_round_trip(tmp_path, case):
    inst = {"e1": e1_instance, "t5a": lambda: tiny(5, 3, 601), "t5b": lambda: tiny(5, 2, 602),
            "t6": lambda: tiny(6, 3, 603, F=8)}[case]()
    brute, _ = pins.brute_optimum(inst)
    assert brute is not None
    assert exact.solve(inst) == brute == pins.ilp_optimum(inst)
    path = exact.export_mps(inst, str(tmp_path / f"{case}.mps"))
    assert solve_mps(path) == brute


def test_mps_con9_fixings_and_names(tmp_path):
    inst = tiny(6, 3, 604, F=8)
    inst.heli_only = np.array([1, 0, 1, 0, 0, 0], np.uint8)
    M = exact.build_model(inst)
    plane = [k for k in range(inst.n_vehicles) if not inst.class_is_heli[inst.vehicle_class[k]]]
    assert plane
    for j, nm in enumerate(M["names"][:M["nx"]]):
        _, i, jj, k = nm.split("_")
        i, jj, k = int(i), int(jj), int(k)
        if k in plane and ((i < 6 and inst.heli_only[i]) or (jj < 6 and inst.heli_only[jj])):
            assert M["ub"][j] == 0.0, nm          # con9: plane x heli-only arcs fixed at 0
    a = open(exact.export_mps(inst, str(tmp_path / "a.mps"))).read()
    b = open(exact.export_mps(inst, str(tmp_path / "b.mps"))).read()
    assert a == b and "x_0_1_0" in a and "u_0" in a       # deterministic naming


def test_mps_zero_missions(tmp_path):
    inst = tiny(1, 2, 605)
    import dataclasses
    z = dataclasses.replace(inst, pickup_loc=inst.pickup_loc[:0], delivery_loc=inst.delivery_loc[:0],
                            deadline_s=inst.deadline_s[:0], heli_only=inst.heli_only[:0])
    assert exact.solve(z) == 0
    M = exact.build_model(z)
    assert not any(r[0].startswith(("con1_", "con2_", "con10_")) for r in M["rows"])
    assert solve_mps(exact.export_mps(z, str(tmp_path / "z.mps"))) == 0
