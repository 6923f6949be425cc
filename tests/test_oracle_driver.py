"""The parallel / memoised search driver (or_search_par) against the plain one
(or_search): identical traces, tabu matrices and best schedules (-m "not gpu").
or_search_par is what the full-length GPU parity checks of C4 and C5 run
(tests/test_gpu_fulllength.py), so it is pinned here to the plain definition
on every config, both modes, kicks, strict stops and several chunk counts."""
import numpy as np
import pytest

from paper_2002_11710_b200 import instgen


def same(a, b):
    assert a["iters_done"] == b["iters_done"] and a["stop_reason"] == b["stop_reason"]
    for k in ("idx", "delta", "cur", "best", "cls"):
        assert (a["trace"][k] == b["trace"][k]).all(), k
    assert a["best_obj"] == b["best_obj"] and a["final_obj"] == b["final_obj"]
    assert a["best_iter"] == b["best_iter"] and a["kicks_applied"] == b["kicks_applied"]
    for k in ("best", "final"):
        assert all((x == y).all() for x, y in zip(a[k], b[k])), k
    assert (a["E"] == b["E"]).all()


@pytest.mark.parametrize("name,iters", [("tiny", 200), ("ontario", 400), ("batched", 150), ("large", 12)])
def test_par_driver_equals_plain(oracle_mod, name, iters):
    inst = instgen.generate(name)
    O = oracle_mod.Oracle(inst)
    st, (p, m), _, _ = O.greedy()
    assert st == 0
    cfg = instgen.CONFIGS[name]
    runs = [dict(mode=1, tenure=cfg.tenure), dict(mode=0)]
    if name in ("tiny", "batched"):
        runs += [dict(mode=1, tenure=cfg.tenure, seed=5, kick=8), dict(mode=1, tenure=0, strict_tabu_stop=True)]
    for kw in runs:
        ref = O.search(p, m, max_iters=iters, **kw)
        for threads, memo in ((1, False), (3, True), (7, True), (16, False)):
            got = O.search_par(p, m, max_iters=iters, threads=threads, memo=memo, **kw)
            same(got, ref)


def test_par_driver_masks_and_tiny_instances(oracle_mod):
    """Move masks and 2-5 mission instances (empty routes, routes emptied by a move)."""
    for n, V, seed in ((2, 2, 11), (3, 3, 12), (5, 3, 13), (5, 4, 14)):
        cfg = instgen.Config("t", n, V - 1, 1, 1, 1, 6, "ontario", 4, 50, 3)
        inst = instgen.generate(cfg, seed=seed)
        O = oracle_mod.Oracle(inst)
        p, m = inst.planted_ptr, inst.planted_missions
        for mask in (0xF, 0x1, 0x5, 0x3):
            for mode in (0, 1):
                ref = O.search(p, m, mode=mode, tenure=2, max_iters=40, mask=mask)
                got = O.search_par(p, m, mode=mode, tenure=2, max_iters=40, mask=mask, threads=4, memo=True)
                same(got, ref)


@pytest.mark.parametrize("name,scale,iters", [("ontario", 0.6, 300), ("batched", 0.5, 120)])
def test_par_driver_nowait(oracle_mod, name, scale, iters):
    """The no-wait variant (f3): a move's feasibility then depends on the whole of its two routes
    (arrival shifts), still only on those -- the memo stays valid; traces equal the plain driver's."""
    import dataclasses
    inst = instgen.generate(name)
    w = np.maximum(1, np.floor(inst.deadline_s * scale)).astype(np.int32)
    inst = dataclasses.replace(inst, no_wait=1, deadline_s=w)
    O = oracle_mod.Oracle(inst)
    st, (p, m), _, _ = O.greedy()
    assert st == 0
    for kw in (dict(mode=1, tenure=instgen.CONFIGS[name].tenure), dict(mode=0),
               dict(mode=1, tenure=5, seed=3, kick=6)):
        ref = O.search(p, m, max_iters=iters, **kw)
        for threads, memo in ((3, True), (8, False)):
            same(O.search_par(p, m, max_iters=iters, threads=threads, memo=memo, **kw), ref)
