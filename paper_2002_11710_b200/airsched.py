"""Thin Python binding of the C ABI in include/airsched.h (ctypes).

Argument marshalling only: every step of the search path runs in the CUDA
kernels of libairsched.so.  There is no CPU fallback -- importing this module
fails loudly when the library is missing.  Array arguments may be numpy arrays
(host) or torch tensors (host or CUDA); torch provides device memory, streams
and process groups only.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libairsched.so")

AS_OK, AS_ERR_INVALID_ARG, AS_ERR_INFEASIBLE_START, AS_ERR_INIT_FAILED, AS_ERR_DEVICE, AS_ERR_OOM, AS_ERR_COMM, \
    AS_ERR_UNSUPPORTED = range(8)
AS_MODE_NS, AS_MODE_TABU = 0, 1
AS_FLAG_VALID, AS_FLAG_FEASIBLE, AS_FLAG_TABU, AS_FLAG_ADMISSIBLE, AS_FLAG_BYDEFAULT = 1, 2, 4, 8, 16
AS_MOVE_INTER_RELOCATE, AS_MOVE_INTRA_RELOCATE, AS_MOVE_INTER_SWAP, AS_MOVE_INTRA_SWAP, AS_MOVE_ALL = 1, 2, 4, 8, 15
AS_KEY_NONE = 0xFFFFFFFFFFFFFFFF
AS_STOP_MAX_ITERS, AS_STOP_LOCAL_OPT, AS_STOP_NO_MOVE, AS_STOP_INFEASIBLE_START, AS_STOP_COMM_ABORT = 0, 1, 2, 3, 4
# as_ctx_set_option names (include/airsched.h AS_OPT_*), in enum order
OPTIONS = ["SMEM_LIMIT", "T_SMEM", "WINDOW", "BATCH_KERNEL", "GRID", "GRID_MIN", "ONE_CTA", "GRID_T_GLOBAL",
           "GRID_E_GLOBAL", "GRID_BLOCKS", "GRID_G", "VERBOSE", "RPC", "THREADS", "SHARDED", "GREEDY_GLOBAL",
           "SHARD_FUSED", "SHARD_FUSED_1", "SHARD_EMULATE", "SHARD_K", "XR_TIMEOUT_MS", "PHASE_TIMES",
           "NODE_COSTS", "GRID_COMPACT", "GRID_SWAP_REC",
           "GRID_WARPS", "GRID_CLUSTER"]
OPT_UNSET = -(1 << 63)

SYMBOLS = ["as_instance_create", "as_instance_destroy", "as_move_space_size", "as_valid_moves_per_iter",
           "as_schedule_check", "as_ctx_create", "as_ctx_set_stream", "as_ctx_destroy", "as_instance_upload",
           "as_init_greedy", "as_eval_moves", "as_tabu_run", "as_nbhd_run", "as_batch_run",
           "as_ctx_last_kernel_ms", "as_ctx_kernel_launches", "as_last_error", "as_version",
           "as_comm_unique_id", "as_comm_init", "as_comm_destroy", "as_shard_plan", "as_batch_gather_best",
           "as_init_greedy_batch", "as_batch_run_jobs", "as_ctx_set_option", "as_ctx_grid_phases",
           "as_ctx_grid_cta_phases", "as_schedule_from_routes", "as_schedule_get", "as_schedule_destroy"]


class AirschedError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"airsched status {status}: {msg}")
        self.status = status


class as_instance_desc(C.Structure):
    _fields_ = [("n_locations", C.c_int32), ("n_classes", C.c_int32), ("travel_s", C.c_void_p),
                ("class_is_heli", C.c_void_p), ("n_bases", C.c_int32), ("base_location", C.c_void_p),
                ("n_vehicles", C.c_int32), ("vehicle_base", C.c_void_p), ("vehicle_class", C.c_void_p),
                ("n_missions", C.c_int32), ("pickup_loc", C.c_void_p), ("delivery_loc", C.c_void_p),
                ("deadline_s", C.c_void_p), ("heli_only", C.c_void_p), ("flight_limit_s", C.c_int32),
                ("day_length_s", C.c_int32), ("no_wait", C.c_int32)]


class as_run_params(C.Structure):
    _fields_ = [("mode", C.c_int32), ("tenure", C.c_int32), ("max_iters", C.c_int32), ("kick", C.c_int32),
                ("move_mask", C.c_uint32), ("strict_tabu_stop", C.c_int32), ("trace_level", C.c_int32),
                ("seed", C.c_uint64), ("sweep", C.c_int32), ("reserved", C.c_int32)]


class as_job(C.Structure):
    _fields_ = [("inst", C.c_void_p), ("start_ptr", C.c_void_p), ("start_missions", C.c_void_p),
                ("n_runs", C.c_int32), ("reserved", C.c_int32)]


class as_run_result(C.Structure):
    _fields_ = [("best_obj", C.c_int64), ("final_obj", C.c_int64), ("start_obj", C.c_int64),
                ("best_iter", C.c_int32), ("iters_done", C.c_int32), ("stop_reason", C.c_int32),
                ("kicks_applied", C.c_int32)]


RESULT_DTYPE = np.dtype([("best_obj", "<i8"), ("final_obj", "<i8"), ("start_obj", "<i8"), ("best_iter", "<i4"),
                         ("iters_done", "<i4"), ("stop_reason", "<i4"), ("kicks_applied", "<i4")])
TRACE_DTYPE = np.dtype([("cur", "<i8"), ("best", "<i8"), ("idx", "<u4"), ("delta", "<i4"), ("cls", "<i4"),
                        ("it", "<i4")])
assert RESULT_DTYPE.itemsize == C.sizeof(as_run_result) == 40 and TRACE_DTYPE.itemsize == 32


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64, u32, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64
    sig = {
        "as_instance_create": (i32, [vp, vp]),
        "as_instance_destroy": (None, [vp]),
        "as_move_space_size": (i64, [vp]),
        "as_valid_moves_per_iter": (i64, [vp]),
        "as_schedule_check": (i32, [vp, vp, vp, vp, vp]),
        "as_schedule_from_routes": (i32, [vp, vp, vp, i32, vp]),
        "as_schedule_get": (i32, [vp, vp, vp, vp, vp, vp]),
        "as_schedule_destroy": (None, [vp]),
        "as_ctx_create": (i32, [i32, vp, vp]),
        "as_ctx_set_stream": (i32, [vp, vp]),
        "as_ctx_set_option": (i32, [vp, i32, i64]),
        "as_ctx_grid_phases": (i32, [vp, vp]),
        "as_ctx_grid_cta_phases": (i32, [vp, vp, vp, vp]),
        "as_ctx_destroy": (None, [vp]),
        "as_instance_upload": (i32, [vp, vp]),
        "as_init_greedy": (i32, [vp, vp, i32, i32, vp, vp, vp]),
        "as_init_greedy_batch": (i32, [vp, vp, i32, i32, i32, vp, vp, vp, vp, vp]),
        "as_batch_run_jobs": (i32, [vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp]),
        "as_eval_moves": (i32, [vp, vp, vp, vp, i32, vp, i32, i64, u32, vp, vp, vp]),
        "as_tabu_run": (i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "as_nbhd_run": (i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "as_batch_run": (i32, [vp, vp, vp, i32, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp]),
        "as_ctx_last_kernel_ms": (C.c_float, [vp]),
        "as_ctx_kernel_launches": (i64, [vp]),
        "as_last_error": (C.c_char_p, []),
        "as_comm_unique_id": (i32, [vp]),
        "as_comm_init": (i32, [vp, i32, i32, vp, vp]),
        "as_comm_destroy": (None, [vp]),
        "as_shard_plan": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp]),
        "as_batch_gather_best": (i32, [vp, vp, i32, vp, vp, vp, vp, vp, vp]),
        "as_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def _check(status):
    if status != AS_OK:
        raise AirschedError(status, lib.as_last_error().decode())


def _ptr(a):
    """Raw pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous()
        return a.data_ptr()
    raise TypeError(type(a))


class Instance:
    """as_instance handle built from arrays (e.g. instgen.Instance)."""

    def __init__(self, src):
        keep = dict(
            T=np.ascontiguousarray(src.travel_s, np.int32), ch=np.ascontiguousarray(src.class_is_heli, np.uint8),
            bl=np.ascontiguousarray(src.base_location, np.int32), vb=np.ascontiguousarray(src.vehicle_base, np.int32),
            vc=np.ascontiguousarray(src.vehicle_class, np.int32), pk=np.ascontiguousarray(src.pickup_loc, np.int32),
            dl=np.ascontiguousarray(src.delivery_loc, np.int32), w=np.ascontiguousarray(src.deadline_s, np.int32),
            h=np.ascontiguousarray(src.heli_only, np.uint8))
        k = keep
        d = as_instance_desc(k["T"].shape[1], k["T"].shape[0], _ptr(k["T"]), _ptr(k["ch"]), len(k["bl"]),
                             _ptr(k["bl"]), len(k["vb"]), _ptr(k["vb"]), _ptr(k["vc"]), len(k["pk"]), _ptr(k["pk"]),
                             _ptr(k["dl"]), _ptr(k["w"]), _ptr(k["h"]), int(src.flight_limit_s),
                             int(src.day_length_s), int(getattr(src, "no_wait", 0)))
        h = C.c_void_p()
        _check(lib.as_instance_create(C.byref(d), C.byref(h)))
        self.handle = h
        self.n = int(len(k["pk"]))
        self.V = int(len(k["vb"]))

    def __del__(self):
        if getattr(self, "handle", None):
            lib.as_instance_destroy(self.handle)
            self.handle = None

    @property
    def move_space_size(self) -> int:
        return int(lib.as_move_space_size(self.handle))

    @property
    def valid_moves_per_iter(self) -> int:
        return int(lib.as_valid_moves_per_iter(self.handle))

    def check(self, ptr, ms):
        f, o = C.c_int32(), C.c_int64()
        ptr = np.ascontiguousarray(ptr, np.int32)
        ms = np.ascontiguousarray(ms, np.int32)
        _check(lib.as_schedule_check(self.handle, _ptr(ptr), _ptr(ms), C.byref(f), C.byref(o)))
        return bool(f.value), int(o.value)


class Schedule:
    """as_schedule: an owned, validated copy of a CSR schedule with its objective and feasibility."""

    def __init__(self, inst, ptr, ms, allow_partial=False):
        ptr = np.ascontiguousarray(ptr, np.int32)
        ms = np.ascontiguousarray(ms, np.int32)
        h = C.c_void_p()
        _check(lib.as_schedule_from_routes(inst.handle, _ptr(ptr), _ptr(ms) if ms.size else None,
                                           1 if allow_partial else 0, C.byref(h)))
        self.handle = h
        self.V = inst.V

    def get(self):
        """(route_ptr, route_missions, objective, feasible)."""
        na, o, f = C.c_int32(), C.c_int64(), C.c_int32()
        _check(lib.as_schedule_get(self.handle, None, None, None, None, C.byref(na)))
        ptr = np.zeros(self.V + 1, np.int32)
        ms = np.zeros(max(na.value, 1), np.int32)
        _check(lib.as_schedule_get(self.handle, _ptr(ptr), _ptr(ms), C.byref(o), C.byref(f), None))
        return ptr, ms[:na.value], int(o.value), bool(f.value)

    def __del__(self):
        if getattr(self, "handle", None):
            lib.as_schedule_destroy(self.handle)
            self.handle = None


class Ctx:
    """as_ctx: one device + one CUDA stream (default: torch's current stream)."""

    def __init__(self, device: int = 0, stream=None):
        if stream is None:
            try:
                import torch
                stream = torch.cuda.current_stream(device).cuda_stream
            except Exception:  # noqa: BLE001 - no torch CUDA: legacy default stream
                stream = 0
        h = C.c_void_p()
        _check(lib.as_ctx_create(int(device), C.c_void_p(stream), C.byref(h)))
        self.handle = h
        self.device = device

    def __del__(self):
        if getattr(self, "handle", None):
            lib.as_ctx_destroy(self.handle)
            self.handle = None

    def set_stream(self, stream):
        _check(lib.as_ctx_set_stream(self.handle, C.c_void_p(stream)))

    def set_option(self, name: str, value):
        """as_ctx_set_option(AS_OPT_<name>, value); None = back to the automatic choice."""
        _check(lib.as_ctx_set_option(self.handle, OPTIONS.index(name), OPT_UNSET if value is None else int(value)))

    def grid_phases(self):
        """as_ctx_grid_phases: per-iteration latency (us) of the last whole-GPU run with PHASE_TIMES=1."""
        out = np.zeros(10, np.int64)
        _check(lib.as_ctx_grid_phases(self.handle, out.ctypes.data))
        it = max(int(out[4]), 1)
        us = lambda k: float(out[k]) / it / 1e3   # noqa: E731
        return {"own_tiles_us": us(0), "cta_wait_us": us(1), "reduce_barrier_us": us(2), "apply_us": us(3),
                "apply_parts_us": {"key_read": us(5), "split": us(6), "relink": us(7), "totals": us(8),
                                   "refresh": us(9)},
                "iterations": int(out[4])}

    def grid_cta_phases(self):
        """as_ctx_grid_cta_phases: per CTA of that run, its tile phase per iteration (us) and its SM id."""
        t = np.zeros(256, np.int64)
        sm = np.zeros(256, np.int32)
        nc = C.c_int32(0)
        _check(lib.as_ctx_grid_cta_phases(self.handle, t.ctypes.data, sm.ctypes.data, C.byref(nc)))
        it = max(self.grid_phases()["iterations"], 1)
        return t[:nc.value] / it / 1e3, sm[:nc.value].copy()

    def options(self, **kw):
        """Context manager: set options, restore the automatic choice on exit."""
        import contextlib

        @contextlib.contextmanager
        def cm():
            for k, v in kw.items():
                self.set_option(k, v)
            try:
                yield self
            finally:
                for k in kw:
                    self.set_option(k, None)
        return cm()

    def upload(self, inst: Instance):
        _check(lib.as_instance_upload(self.handle, inst.handle))

    @property
    def last_kernel_ms(self) -> float:
        return float(lib.as_ctx_last_kernel_ms(self.handle))

    @property
    def kernel_launches(self) -> int:
        return int(lib.as_ctx_kernel_launches(self.handle))


def as_comm_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(lib.as_comm_unique_id(C.byref(buf)))
    return bytes(buf)


class Comm:
    """as_comm: NCCL communicator over the ranks of a torch.distributed job.

    The 128-byte NCCL unique id is created on rank 0 and broadcast with
    torch.distributed (any backend, e.g. gloo or nccl) -- plumbing only."""

    def __init__(self, ctx: Ctx, nranks: int, rank: int, uid: bytes):
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(lib.as_comm_init(ctx.handle, int(nranks), int(rank), C.byref(buf), C.byref(h)))
        self.handle = h
        self.nranks, self.rank = nranks, rank

    @classmethod
    def from_torch_distributed(cls, ctx: Ctx, group=None):
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [as_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(ctx, world, rank, obj[0])

    def __del__(self):
        if getattr(self, "handle", None):
            lib.as_comm_destroy(self.handle)
            self.handle = None


def as_shard_plan(inst: Instance, nranks: int, rank: int, n_sm: int = 148):
    lo, hi, tot = C.c_int32(), C.c_int32(), C.c_int32()
    wr, wt = C.c_int64(), C.c_int64()
    _check(lib.as_shard_plan(inst.handle, int(nranks), int(rank), int(n_sm), C.byref(lo), C.byref(hi), C.byref(tot),
                             C.byref(wr), C.byref(wt)))
    return dict(tile_lo=lo.value, tile_hi=hi.value, tile_total=tot.value, weight=wr.value, weight_total=wt.value)


def params(mode=AS_MODE_TABU, tenure=10, max_iters=100, kick=0, move_mask=AS_MOVE_ALL, strict_tabu_stop=0,
           trace_level=0, seed=0, sweep=0) -> as_run_params:
    return as_run_params(int(mode), int(tenure), int(max_iters), int(kick), int(move_mask), int(strict_tabu_stop),
                         int(trace_level), int(seed), int(sweep), 0)


# ---------------------------------------------------------------- entry points --
def as_init_greedy(ctx: Ctx, inst: Instance, insert_mode=0, max_repairs=50):
    ptr = np.zeros(inst.V + 1, np.int32)
    ms = np.zeros(max(inst.n, 1), np.int32)
    nrep = C.c_int32()
    _check(lib.as_init_greedy(ctx.handle, inst.handle, int(insert_mode), int(max_repairs), _ptr(ptr), _ptr(ms),
                              C.byref(nrep)))
    return ptr, ms[:inst.n], int(nrep.value)


def as_init_greedy_batch(ctx: Ctx, inst: Instance, n_starts, seeds=None, insert_mode=1, max_repairs=50,
                         ptr_out=None, ms_out=None, status_out=None, nrep_out=None):
    """Marshalling for as_init_greedy_batch.  Without output arrays, host numpy
    arrays are allocated and returned; torch CUDA tensors stay on the device."""
    R = int(n_starts)
    if ptr_out is None:
        ptr_out = np.zeros((R, inst.V + 1), np.int32)
        ms_out = np.zeros((R, max(inst.n, 1)), np.int32)
        status_out = np.zeros(R, np.int32)
        nrep_out = np.zeros(R, np.int32)
    if isinstance(seeds, np.ndarray):
        seeds = np.ascontiguousarray(seeds, np.uint64)
    _check(lib.as_init_greedy_batch(ctx.handle, inst.handle, R, int(insert_mode), int(max_repairs), _ptr(seeds),
                                    _ptr(ptr_out), _ptr(ms_out), _ptr(status_out), _ptr(nrep_out)))
    return ptr_out, ms_out, status_out, nrep_out


def as_eval_moves(ctx: Ctx, inst: Instance, route_ptr, route_missions, mode=AS_MODE_TABU, tabu_expiry=None,
                  iter=0, best_obj=None, move_mask=AS_MOVE_ALL, delta_out=None, flags_out=None):
    route_ptr = np.ascontiguousarray(route_ptr, np.int32)
    route_missions = np.ascontiguousarray(route_missions, np.int32)
    if best_obj is None:
        best_obj = inst.check(route_ptr, route_missions)[1]
    N = inst.move_space_size
    if delta_out is None:
        delta_out = np.zeros(N, np.int32)
    if flags_out is None:
        flags_out = np.zeros(N, np.uint8)
    if tabu_expiry is not None and isinstance(tabu_expiry, np.ndarray):
        tabu_expiry = np.ascontiguousarray(tabu_expiry, np.int32)
    key = C.c_uint64()
    _check(lib.as_eval_moves(ctx.handle, inst.handle, _ptr(route_ptr), _ptr(route_missions), int(mode),
                             _ptr(tabu_expiry), int(iter), int(best_obj), int(move_mask), _ptr(delta_out),
                             _ptr(flags_out), C.byref(key)))
    return delta_out, flags_out, int(key.value)


def _run(fn, ctx, inst, route_ptr, route_missions, prm, want_best=True, want_trace=False, want_digest=False,
         want_tabu=False, comm=None):
    route_ptr = np.ascontiguousarray(route_ptr, np.int32)
    route_missions = np.ascontiguousarray(route_missions, np.int32)
    res = as_run_result()
    bp = np.zeros(inst.V + 1, np.int32) if want_best else None
    bm = np.zeros(max(inst.n, 1), np.int32) if want_best else None
    K = max(prm.max_iters, 1)
    tr = np.zeros(K, TRACE_DTYPE) if want_trace else None
    dg = np.zeros(K, np.uint64) if want_digest else None
    tb = np.zeros((max(inst.n, 1), inst.V), np.int32) if want_tabu else None
    args = [ctx.handle, comm.handle if comm is not None else None, inst.handle, _ptr(route_ptr), _ptr(route_missions),
            C.byref(prm), C.byref(res),
            _ptr(bp), _ptr(bm), _ptr(tr)]
    if fn is lib.as_tabu_run:
        args += [_ptr(dg), _ptr(tb)]
    _check(fn(*args))
    out = {f: getattr(res, f) for f, _ in as_run_result._fields_}
    if want_best:
        out["best"] = (bp, bm[:inst.n])
    if want_trace:
        out["trace"] = tr[:res.iters_done]
    if want_digest:
        out["digest"] = dg[:res.iters_done]
    if want_tabu:
        out["tabu"] = tb[:inst.n]
    return out


def as_tabu_run(ctx, inst, route_ptr, route_missions, prm, **kw):
    return _run(lib.as_tabu_run, ctx, inst, route_ptr, route_missions, prm, **kw)


def as_nbhd_run(ctx, inst, route_ptr, route_missions, prm, **kw):
    return _run(lib.as_nbhd_run, ctx, inst, route_ptr, route_missions, prm, **kw)


def as_batch_run_jobs(ctx, jobs, prm, seeds=None, results=None, best_ptr_out=None, best_missions_out=None,
                      trace_out=None, want_best_run=False, comm=None):
    """Marshalling for as_batch_run_jobs.  jobs: list of (Instance, start_ptr, start_missions, n_runs);
    runs are numbered job after job.  Returns the best run's number (or -1) when want_best_run."""
    keep = []
    arr = (as_job * len(jobs))()
    for j, (inst, sp, sm, nr) in enumerate(jobs):
        if isinstance(sp, np.ndarray):
            sp = np.ascontiguousarray(sp, np.int32)
            sm = np.ascontiguousarray(sm, np.int32)
        keep.append((sp, sm))
        arr[j] = as_job(inst.handle, _ptr(sp), _ptr(sm), int(nr), 0)
    if isinstance(seeds, np.ndarray):
        seeds = np.ascontiguousarray(seeds, np.uint64)
    best_run = C.c_int64(-1)
    _check(lib.as_batch_run_jobs(ctx.handle, comm.handle if comm is not None else None, len(jobs), arr, C.byref(prm),
                                 _ptr(seeds), _ptr(results), _ptr(best_ptr_out), _ptr(best_missions_out),
                                 _ptr(trace_out), C.byref(best_run) if want_best_run else None))
    return int(best_run.value)


def as_batch_gather_best(ctx, inst, n_runs, run_best_ptr=None, run_best_ms=None, comm=None):
    """Global best run over all ranks of the last as_batch_run, and (if the
    per-run best schedules are given) that run's schedule broadcast from its owner."""
    run, obj = C.c_int64(), C.c_int64()
    want = run_best_ptr is not None
    ptr = np.zeros(inst.V + 1, np.int32) if want else None
    ms = np.zeros(max(inst.n, 1), np.int32) if want else None
    _check(lib.as_batch_gather_best(ctx.handle, comm.handle if comm is not None else None, int(n_runs),
                                    _ptr(run_best_ptr), _ptr(run_best_ms), C.byref(run), C.byref(obj), _ptr(ptr),
                                    _ptr(ms)))
    out = dict(best_run=run.value, best_obj=obj.value)
    if want:
        out["best"] = (ptr, ms[:inst.n])
    return out


def as_batch_run(ctx, inst, n_runs, start_ptr, start_missions, prm, seeds, shared_start=True, results=None,
                 best_ptr_out=None, best_missions_out=None, trace_out=None, want_best_run=False, comm=None):
    """Marshalling for as_batch_run.  Arrays may be numpy (host) or torch CUDA tensors
    (device-resident; then the call only enqueues work on the ctx stream)."""
    best_run = C.c_int64(-1)
    if isinstance(seeds, np.ndarray):
        seeds = np.ascontiguousarray(seeds, np.uint64)
    _check(lib.as_batch_run(ctx.handle, comm.handle if comm is not None else None, inst.handle, int(n_runs),
                            _ptr(start_ptr), _ptr(start_missions),
                            int(bool(shared_start)), C.byref(prm), _ptr(seeds), _ptr(results), _ptr(best_ptr_out),
                            _ptr(best_missions_out), _ptr(trace_out), C.byref(best_run) if want_best_run else None))
    return int(best_run.value)
