"""CPU oracle for arXiv 2002.11710's neighbourhood / tabu search (ctypes wrapper).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  The product
path (paper_2002_11710_b200/) never imports it, and this package never imports
the product's binding or loads its library: the only thing both sides share is
the seeded input generator (paper_2002_11710_b200/instgen.py), which holds none
of the method's arithmetic.

The arithmetic lives in oracle.c (plain C, definitions written out; see its
header for the paper citations).  This wrapper only converts schedules between
CSR form (route_ptr[V+1], route_missions[n]) and the oracle's per-vehicle lists.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MODE_NS, MODE_TABU = 0, 1
FLAG_VALID, FLAG_FEASIBLE, FLAG_TABU, FLAG_ADMISSIBLE, FLAG_BYDEFAULT = 1, 2, 4, 8, 16


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-pthread", "-o", _LIB, _SRC])
    return _LIB


class _Inst(C.Structure):
    _fields_ = [("NL", C.c_int32), ("NC", C.c_int32), ("T", C.c_void_p), ("class_is_heli", C.c_void_p),
                ("V", C.c_int32), ("veh_loc", C.c_void_p), ("veh_cls", C.c_void_p), ("n", C.c_int32),
                ("pick", C.c_void_p), ("dele", C.c_void_p), ("w", C.c_void_p), ("heli", C.c_void_p),
                ("P", C.c_int32), ("DAY", C.c_int32), ("no_wait", C.c_int32)]


class _Params(C.Structure):
    _fields_ = [("mode", C.c_int32), ("tenure", C.c_int32), ("max_iters", C.c_int32), ("kick", C.c_int32),
                ("strict_tabu_stop", C.c_int32), ("want_digest", C.c_int32), ("mask", C.c_uint32),
                ("seed", C.c_uint64)]


class _Result(C.Structure):
    _fields_ = [("best_obj", C.c_int64), ("final_obj", C.c_int64), ("start_obj", C.c_int64),
                ("best_iter", C.c_int32), ("iters_done", C.c_int32), ("stop_reason", C.c_int32),
                ("kicks_applied", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.or_route_cost.restype = C.c_int64
        _lib.or_objective.restype = C.c_int64
        _lib.or_move_space_size.restype = C.c_int64
        _lib.or_splitmix64_next.restype = C.c_uint64
        _lib.or_tabu_digest.restype = C.c_uint64
        _lib.or_tabu_digest.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
        _lib.or_kick.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32]
        _lib.or_apply_move.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_uint32,
                                       C.c_void_p, C.c_void_p]
        _lib.or_eval_moves.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                       C.c_int64, C.c_uint32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class Oracle:
    """Holds one instance (keeps its numpy arrays alive for the C struct)."""

    def __init__(self, inst):
        self.inst = inst
        self._keep = dict(
            T=np.ascontiguousarray(inst.travel_s, np.int32),
            ch=np.ascontiguousarray(inst.class_is_heli, np.uint8),
            vloc=np.ascontiguousarray(inst.base_location[inst.vehicle_base], np.int32),
            vcls=np.ascontiguousarray(inst.vehicle_class, np.int32),
            pick=np.ascontiguousarray(inst.pickup_loc, np.int32),
            dele=np.ascontiguousarray(inst.delivery_loc, np.int32),
            w=np.ascontiguousarray(inst.deadline_s, np.int32),
            heli=np.ascontiguousarray(inst.heli_only, np.uint8))
        k = self._keep
        self.n = int(k["pick"].shape[0])
        self.V = int(k["vloc"].shape[0])
        self.c = _Inst(int(k["T"].shape[1]), int(k["T"].shape[0]), _p(k["T"]), _p(k["ch"]), self.V,
                       _p(k["vloc"]), _p(k["vcls"]), self.n, _p(k["pick"]), _p(k["dele"]), _p(k["w"]),
                       _p(k["heli"]), int(inst.flight_limit_s), int(inst.day_length_s),
                       int(getattr(inst, "no_wait", 0)))
        self.ref = C.byref(self.c)

    # ---- schedule conversion (CSR <-> per-vehicle lists) -------------------
    def to_lists(self, ptr, ms):
        n, V = self.n, self.V
        length = np.zeros(V, np.int32)
        r = np.zeros((V, max(n, 1)), np.int32)
        for v in range(V):
            seg = np.asarray(ms[ptr[v]:ptr[v + 1]], np.int32)
            length[v] = len(seg)
            r[v, :len(seg)] = seg
        return length, r

    def to_csr(self, length, r):
        ptr = np.zeros(self.V + 1, np.int32)
        ptr[1:] = np.cumsum(length)
        ms = np.concatenate([r[v, :length[v]] for v in range(self.V)] + [np.zeros(0, np.int32)]).astype(np.int32)
        return ptr, ms

    # ---- O3/O4 ---------------------------------------------------------------
    def objective(self, ptr, ms) -> int:
        length, r = self.to_lists(ptr, ms)
        return int(lib().or_objective(self.ref, _p(length), _p(r)))

    def feasible(self, ptr, ms) -> bool:
        length, r = self.to_lists(ptr, ms)
        return bool(lib().or_schedule_feasible(self.ref, _p(length), _p(r)))

    def route_cost(self, v, route) -> int:
        route = np.ascontiguousarray(route, np.int32)
        return int(lib().or_route_cost(self.ref, C.c_int32(v), _p(route), C.c_int32(len(route))))

    def route_feasible(self, v, route) -> bool:
        route = np.ascontiguousarray(route, np.int32)
        return bool(lib().or_route_feasible(self.ref, C.c_int32(v), _p(route), C.c_int32(len(route))))

    def move_space_size(self) -> int:
        return int(lib().or_move_space_size(self.ref))

    def apply_move(self, ptr, ms, idx, mask=0xF):
        length, r = self.to_lists(ptr, ms)
        lo, ro = np.zeros_like(length), np.zeros_like(r)
        ok = lib().or_apply_move(self.ref, _p(length), _p(r), int(idx), int(mask), _p(lo), _p(ro))
        return bool(ok), self.to_csr(lo, ro)

    # ---- O6-O9 -----------------------------------------------------------------
    def eval_moves(self, ptr, ms, mode=MODE_TABU, E=None, it=0, best_obj=None, mask=0xF, full=False):
        length, r = self.to_lists(ptr, ms)
        N = self.move_space_size()
        delta = np.zeros(N, np.int32)
        flags = np.zeros(N, np.uint8)
        if best_obj is None:
            best_obj = self.objective(ptr, ms)
        Ec = None if E is None else np.ascontiguousarray(E, np.int32)
        bc, bd, bi = C.c_int32(), C.c_int32(), C.c_int64()
        lib().or_eval_moves(self.ref, _p(length), _p(r), int(mode), _p(Ec), int(it), int(best_obj), int(mask),
                            int(bool(full)), _p(delta), _p(flags), C.byref(bc), C.byref(bd), C.byref(bi))
        return delta, flags, (bc.value, bd.value, bi.value)

    def eval_indices(self, ptr, ms, idx, mode=MODE_TABU, E=None, it=0, best_obj=None, mask=0xF):
        length, r = self.to_lists(ptr, ms)
        idx = np.ascontiguousarray(idx, np.int64)
        delta = np.zeros(len(idx), np.int32)
        flags = np.zeros(len(idx), np.uint8)
        if best_obj is None:
            best_obj = self.objective(ptr, ms)
        Ec = None if E is None else np.ascontiguousarray(E, np.int32)
        lib().or_eval_index_list(self.ref, _p(length), _p(r), int(mode), _p(Ec), int(it), C.c_int64(int(best_obj)),
                                 C.c_uint32(int(mask)), C.c_int64(len(idx)), _p(idx), _p(delta), _p(flags))
        return delta, flags

    # ---- O10-O12 ---------------------------------------------------------------
    def search(self, ptr, ms, mode=MODE_TABU, tenure=10, max_iters=100, seed=0, kick=0, mask=0xF,
               strict_tabu_stop=False, digest=False, trace=True):
        length, r = self.to_lists(ptr, ms)
        V, n = self.V, self.n
        bl, br = np.zeros_like(length), np.zeros_like(r)
        fl, fr = np.zeros_like(length), np.zeros_like(r)
        K = max(int(max_iters), 1)
        tr = dict(idx=np.zeros(K, np.int64), delta=np.zeros(K, np.int32), cur=np.zeros(K, np.int64),
                  best=np.zeros(K, np.int64), cls=np.zeros(K, np.int32), digest=np.zeros(K, np.uint64))
        E = np.zeros((max(n, 1), V), np.int32)
        prm = _Params(int(mode), int(tenure), int(max_iters), int(kick), int(bool(strict_tabu_stop)),
                      int(bool(digest)), int(mask), int(seed))
        res = _Result()
        tp = (lambda k: _p(tr[k])) if trace else (lambda k: None)
        lib().or_search(self.ref, _p(length), _p(r), C.byref(prm), _p(bl), _p(br), _p(fl), _p(fr), C.byref(res),
                        tp("idx"), tp("delta"), tp("cur"), tp("best"), tp("cls"), tp("digest"), _p(E))
        k = res.iters_done
        out = dict(best_obj=res.best_obj, final_obj=res.final_obj, start_obj=res.start_obj,
                   best_iter=res.best_iter, iters_done=k, stop_reason=res.stop_reason,
                   kicks_applied=res.kicks_applied, best=self.to_csr(bl, br), final=self.to_csr(fl, fr),
                   E=E[:n])
        if trace:
            out["trace"] = {key: val[:k].copy() for key, val in tr.items()}
        return out

    def search_par(self, ptr, ms, mode=MODE_TABU, tenure=10, max_iters=100, seed=0, kick=0, mask=0xF,
                   strict_tabu_stop=False, threads=None, memo=True, trace=True):
        """or_search driven over `threads` index chunks (+ memo of unchanged moves):
        the full-length parity driver for the large configs.  Same results as search()."""
        length, r = self.to_lists(ptr, ms)
        V, n = self.V, self.n
        threads = int(threads or os.cpu_count() or 1)
        bl, br = np.zeros_like(length), np.zeros_like(r)
        fl, fr = np.zeros_like(length), np.zeros_like(r)
        K = max(int(max_iters), 1)
        tr = dict(idx=np.zeros(K, np.int64), delta=np.zeros(K, np.int32), cur=np.zeros(K, np.int64),
                  best=np.zeros(K, np.int64), cls=np.zeros(K, np.int32))
        E = np.zeros((max(n, 1), V), np.int32)
        prm = _Params(int(mode), int(tenure), int(max_iters), int(kick), int(bool(strict_tabu_stop)), 0, int(mask),
                      int(seed))
        res = _Result()
        tp = (lambda k: _p(tr[k])) if trace else (lambda k: None)
        lib().or_search_par(self.ref, _p(length), _p(r), C.byref(prm), C.c_int32(threads), C.c_int32(int(bool(memo))),
                            _p(bl), _p(br), _p(fl), _p(fr), C.byref(res), tp("idx"), tp("delta"), tp("cur"),
                            tp("best"), tp("cls"), _p(E))
        k = res.iters_done
        out = dict(best_obj=res.best_obj, final_obj=res.final_obj, start_obj=res.start_obj,
                   best_iter=res.best_iter, iters_done=k, stop_reason=res.stop_reason,
                   kicks_applied=res.kicks_applied, best=self.to_csr(bl, br), final=self.to_csr(fl, fr),
                   E=E[:n])
        if trace:
            out["trace"] = {key: val[:k].copy() for key, val in tr.items()}
        return out

    def sweep(self, ptr, ms, mode=MODE_TABU, tenure=10, max_steps=100, seed=0):
        """f1: Alg. 2 / Alg. 3 as written -- one (vehicle, mission) step at a time."""
        length, r = self.to_lists(ptr, ms)
        bl, br = np.zeros_like(length), np.zeros_like(r)
        K = max(int(max_steps), 1)
        tr = dict(idx=np.zeros(K, np.int64), delta=np.zeros(K, np.int32), cur=np.zeros(K, np.int64),
                  best=np.zeros(K, np.int64))
        prm = _Params(int(mode), int(tenure), int(max_steps), 0, 0, 0, 1, int(seed))
        res = _Result()
        lib().or_sweep(self.ref, _p(length), _p(r), C.byref(prm), _p(bl), _p(br), C.byref(res), _p(tr["idx"]),
                       _p(tr["delta"]), _p(tr["cur"]), _p(tr["best"]))
        k = res.iters_done
        return dict(best_obj=res.best_obj, final_obj=res.final_obj, start_obj=res.start_obj, best_iter=res.best_iter,
                    iters_done=k, stop_reason=res.stop_reason, best=self.to_csr(bl, br),
                    trace={key: val[:k].copy() for key, val in tr.items()})

    def kick(self, ptr, ms, seed, kick):
        length, r = self.to_lists(ptr, ms)
        applied = lib().or_kick(self.ref, _p(length), _p(r), int(seed), int(kick))
        return int(applied), self.to_csr(length, r)

    def tabu_digest(self, E, it) -> int:
        Ec = np.ascontiguousarray(E, np.int32)
        return int(lib().or_tabu_digest(self.ref, _p(Ec), int(it)))

    # ---- O13 -------------------------------------------------------------------
    def greedy(self, insert_mode=0, max_repairs=50, seed=0):
        V, n = self.V, self.n
        length = np.zeros(V, np.int32)
        r = np.zeros((V, max(n, 1)), np.int32)
        nrep = C.c_int32()
        order = np.zeros(max(n, 1), np.int32)
        st = lib().or_greedy_seeded(self.ref, int(insert_mode), int(max_repairs), C.c_uint64(int(seed)), _p(length),
                                    _p(r), C.byref(nrep), _p(order))
        return int(st), self.to_csr(length, r), int(nrep.value), order[:n]


def splitmix64(seed: int, count: int):
    s = C.c_uint64(seed)
    return [int(lib().or_splitmix64_next(C.byref(s))) for _ in range(count)]
