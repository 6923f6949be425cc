"""C-ABI boundary tests that need no GPU: the library loads, exports every
symbol include/airsched.h declares, validates instances, and its host-side
schedule check agrees with the oracle.  (No compute calls without a GPU.)"""
import os
import re

import numpy as np
import pytest

from paper_2002_11710_b200 import instgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def A():
    from paper_2002_11710_b200 import _build
    _build.build()
    from paper_2002_11710_b200 import airsched
    return airsched


def header_symbols():
    src = open(os.path.join(ROOT, "include", "airsched.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(as_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(A):
    syms = header_symbols()
    assert len(syms) >= 18
    out = os.popen(f"nm -D --defined-only {A.LIB_PATH}").read()
    exported = set(re.findall(r"\bT (as_[a-z0-9_]+)", out))
    assert set(syms) <= exported, set(syms) - exported
    assert set(A.SYMBOLS) == set(syms)
    assert b"sm_100a" in A.lib.as_version()


def test_sass_is_sm100a(A):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {A.LIB_PATH}").read()
    assert "sm_100a" in out


def test_instance_validation(A):
    inst = instgen.generate("tiny")
    h = A.Instance(inst)
    n, V = inst.n_missions, inst.n_vehicles
    assert h.move_space_size == n * (n + V) + n * n == 152
    assert h.valid_moves_per_iter == 100
    bad = instgen.generate("tiny")
    bad.travel_s = bad.travel_s.copy()
    bad.travel_s[0, 1, 1] = 5
    with pytest.raises(A.AirschedError) as e:
        A.Instance(bad)
    assert e.value.status == A.AS_ERR_INVALID_ARG and "diagonal" in str(e.value)
    bad = instgen.generate("tiny")
    bad.deadline_s = bad.deadline_s.copy()
    bad.deadline_s[2] = 0
    with pytest.raises(A.AirschedError):
        A.Instance(bad)
    bad = instgen.generate("tiny")
    bad.vehicle_class = np.array([0, 0, 7], np.int32)
    with pytest.raises(A.AirschedError):
        A.Instance(bad)


def test_schedule_check_matches_oracle(A, oracle_mod):
    rng = np.random.default_rng(2)
    for cfg in ("tiny", "ontario"):
        inst = instgen.generate(cfg)
        h = A.Instance(inst)
        O = oracle_mod.Oracle(inst)
        states = [(inst.planted_ptr, inst.planted_missions)]
        n, V = inst.n_missions, inst.n_vehicles
        for _ in range(30):
            perm = rng.permutation(n).astype(np.int32)
            cuts = np.sort(rng.integers(0, n + 1, V - 1))
            states.append((np.concatenate([[0], cuts, [n]]).astype(np.int32), perm))
        for p, m in states:
            f, obj = h.check(p, m)
            assert obj == O.objective(p, m) and f == O.feasible(p, m)
    with pytest.raises(A.AirschedError):
        h.check(np.array([0, 1] + [1] * (V - 1), np.int32), np.array([n + 5], np.int32))


def test_nowait_schedule_check_matches_oracle(A, oracle_mod):
    """f3 (no-wait variant): the host check against the oracle on random states and
    on the oracle's own no-wait trajectory (states infeasible under waiting)."""
    import dataclasses
    rng = np.random.default_rng(3)
    n_diff = 0
    for cfg in ("tiny", "ontario"):
        inst = dataclasses.replace(instgen.generate(cfg), no_wait=1)
        wait = instgen.generate(cfg)
        h, hw = A.Instance(inst), A.Instance(wait)
        O = oracle_mod.Oracle(inst)
        st, (p, m), _, _ = O.greedy()
        states = [(p, m)] + [O.search(p, m, mode=1, tenure=5, max_iters=k, trace=False)["final"] for k in (5, 30)]
        n, V = inst.n_missions, inst.n_vehicles
        for _ in range(30):
            perm = rng.permutation(n).astype(np.int32)
            cuts = np.sort(rng.integers(0, n + 1, V - 1))
            states.append((np.concatenate([[0], cuts, [n]]).astype(np.int32), perm))
        for p, m in states:
            f, obj = h.check(p, m)
            assert obj == O.objective(p, m) and f == O.feasible(p, m)
            n_diff += f != hw.check(p, m)[0]
    assert n_diff >= 1
    bad = dataclasses.replace(instgen.generate("tiny"), no_wait=2)
    with pytest.raises(A.AirschedError) as e:
        A.Instance(bad)
    assert e.value.status == A.AS_ERR_INVALID_ARG


def test_ctx_without_gpu_fails_loudly(A):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(A.AirschedError) as e:
        A.Ctx(0, 0)
    assert e.value.status == A.AS_ERR_DEVICE


def test_option_enum_matches_binding(A):
    """as_ctx_set_option: the binding's option names are the header's AS_OPT_* enum in order."""
    import re
    hdr = open(os.path.join(ROOT, "include", "airsched.h")).read()
    block = hdr[hdr.index("AS_OPT_SMEM_LIMIT = 0"):hdr.index("AS_OPT_COUNT")]
    names = re.findall(r"AS_OPT_([A-Z_0-9]+)", block)
    assert names == A.OPTIONS


def test_library_reads_no_environment():
    """Dispatch is explicit (as_ctx_set_option): the library's own sources read no
    environment variable (the statically linked CUDA runtime has its own)."""
    import glob
    for f in glob.glob(os.path.join(ROOT, "paper_2002_11710_b200", "csrc", "*")):
        assert "getenv" not in open(f).read(), f


def test_schedule_handles(A, oracle_mod):
    """as_schedule_from_routes / as_schedule_get / as_schedule_destroy (host only): a validated copy of the
    routes with the objective and feasibility the oracle gives (Eq. obj_s, con6-con9); partial schedules
    only on request; the rules of as_schedule_check on bad input."""
    inst = instgen.generate("ontario")
    O = oracle_mod.Oracle(inst)
    h = A.Instance(inst)
    st, (p, m), _, _ = O.greedy()
    s = A.Schedule(h, p, m)
    gp, gm, obj, feas = s.get()
    assert (gp == p).all() and (gm == m).all()
    assert feas and obj == O.objective(p, m) and h.check(p, m) == (True, obj)
    # a partial schedule: the last mission of the last non-empty route left out
    V = inst.n_vehicles
    v = max(u for u in range(V) if p[u + 1] > p[u])
    pp = p.copy()
    pp[v + 1:] -= 1
    mm = np.delete(m, p[v + 1] - 1)
    with pytest.raises(A.AirschedError):
        A.Schedule(h, pp, mm)
    s2 = A.Schedule(h, pp, mm, allow_partial=True)
    gp2, gm2, obj2, feas2 = s2.get()
    assert (gp2 == pp).all() and (gm2 == mm).all() and not feas2
    assert obj2 == h.check(pp, mm)[1]
    # a mission listed twice
    bad = m.copy()
    bad[1] = bad[0]
    with pytest.raises(A.AirschedError) as e:
        A.Schedule(h, p, bad)
    assert e.value.status == A.AS_ERR_INVALID_ARG
    # every route empty: a partial schedule with objective 0
    empty = np.zeros(V + 1, np.int32)
    s3 = A.Schedule(h, empty, np.zeros(0, np.int32), allow_partial=True)
    assert s3.get()[2] == 0
