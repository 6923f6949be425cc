#!/usr/bin/env python
"""Benchmark: move evaluations/s (and tabu iterations/s) of the B200 engine.

Default workload = BASELINE.json configs[2], the batched multi-start config the
1e10 moves/s target is quoted on: 4096 independent tabu runs of a
20-vehicle / 100-mission instance, 1000 iterations each, on one GPU (SURVEY
§8.0 C3).  One step = one `as_batch_run` call over the whole batch (every §8(a)
row: decode, gather, delta, feasibility, tabu/aspiration, key reduction,
on-device apply, loop control, per-run kick).  Under torchrun each rank runs its
own 4096 runs (seeds offset by rank): weak scaling, no data-path collective.

Contract keys: see the task statement; `--impl reference` times the CPU oracle
(the reference arm of this tier) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2002_11710_b200 import instgen  # noqa: E402

METRIC = "move evals/sec and tabu iters/sec per B200 (1/2/4/8 GPU), % roofline"
UNIT = "move evals/s"

# Algorithmic integer operations per scored move: the
# adds/compares/selects the formulas of §8(a) a3-a6 require per (m,t) pair or
# per swap pair, with the per-row removal part amortised.
OPS_RELOCATE = 23
OPS_SWAP = 37
# SURVEY §8(d) algorithmic on-chip work per move (what the method must touch, the m side
# amortised): relocate 2 T + target record + vehicle record + E = 36-40 B, ~40 instructions;
# swap 4 T + 2 records + 2 vehicles + 2 E = 72 B, ~80 instructions.
BYTES_RELOCATE, BYTES_SWAP = 38, 72
INSTR_RELOCATE, INSTR_SWAP = 40, 80
PROFILE_DIR = os.path.join(ROOT, "profiles", "r02")


def onchip_peaks():
    """Measured on-chip ceilings of this B200 (tools/onchip_peaks.cu, committed JSON)."""
    try:
        with open(os.path.join(PROFILE_DIR, "onchip_peaks.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def move_mix(inst):
    n, V = inst.n_missions, inst.n_vehicles
    return n * (n + V - 2), n * (n - 1) // 2


def onchip_roofline(relocs, swaps, t_s, f_mhz, n_gpus=1, workload=None):
    """Roofline of the move-evaluation kernel at the memory level that serves it (SURVEY §8(d):
    shared memory / L1 for the resident configs; HBM ~0 by design) and at instruction issue.
    achieved = algorithmic bytes (instructions) of the moves scored / device time; peak = the
    MEASURED shared-memory bandwidth (conflict-free LDS wavefronts, tools/onchip_peaks.cu) and
    the issue ceiling (4 SMSP x 32 lanes per SM cycle; measured INT mixes alongside), both at the
    SM clock sampled under load.  `bound` = the ceiling closer to saturation."""
    pk = onchip_peaks()
    f = f_mhz * 1e6
    smem_bpc = (pk.get("lds_seq") or {}).get("bytes_per_sm_cycle") or 128.0
    smem_peak = 148 * smem_bpc * f * n_gpus
    issue_peak = 148 * 128 * f * n_gpus
    b = relocs * BYTES_RELOCATE + swaps * BYTES_SWAP
    ins = relocs * INSTR_RELOCATE + swaps * INSTR_SWAP
    a_smem, a_issue = b / t_s, ins / t_s
    ops = relocs * OPS_RELOCATE + swaps * OPS_SWAP
    smem = {"achieved": a_smem / 1e9, "peak": smem_peak / 1e9, "unit": "GB/s", "frac": a_smem / smem_peak,
            "peak_basis": f"measured {smem_bpc:.1f} B per SM cycle (conflict-free LDS, profiles/r02/onchip_peaks.json)"
                          f" x 148 SMs x {f_mhz:.0f} MHz" + (f" x {n_gpus} GPUs" if n_gpus > 1 else "")}
    issue = {"achieved": a_issue / 1e9, "peak": issue_peak / 1e9, "unit": "Ginstr/s", "frac": a_issue / issue_peak,
             "peak_basis": f"148 SMs x 4 SMSP x 32 lanes x {f_mhz:.0f} MHz" + (f" x {n_gpus} GPUs" if n_gpus > 1 else ""),
             "measured_int_lanes_per_sm_cycle": {"alu_only": (pk.get("int_alu") or {}).get("lanes_per_sm_cycle"),
                                                 "alu_fma_mix": (pk.get("int_mix") or {}).get("lanes_per_sm_cycle")}}
    bound, main = ("smem", smem) if smem["frac"] >= issue["frac"] else ("issue", issue)
    roof = {"bound": bound, "achieved": main["achieved"], "peak": main["peak"], "unit": main["unit"],
            "frac": main["frac"], "traffic": measured_traffic(workload) if workload else None,
            "peak_basis": main["peak_basis"],
            "model": f"SURVEY 8(d) per move: relocate {BYTES_RELOCATE} B / {INSTR_RELOCATE} instr, swap {BYTES_SWAP} B / "
                     f"{INSTR_SWAP} instr; {relocs:.4g} relocates + {swaps:.4g} swaps scored",
            "smem": smem, "issue": issue,
            "op_count": {"achieved": ops / t_s / 1e9, "peak": issue_peak / 1e9, "unit": "Gop/s",
                         "frac": ops / t_s / issue_peak,
                         "basis": f"{OPS_RELOCATE}/{OPS_SWAP} algorithmic integer ops per relocate/swap move"}}
    prof = measured_profile(workload) if workload else {}
    if prof:   # hardware counters of the committed ncu capture of this workload's dominant kernel
        hw = {"source": prof.get("source"), "issue_slots_busy": prof.get("issue_slots_busy"),
              "alu_fma_pipe": [prof.get("alu_pipe"), prof.get("fma_pipe")],
              "fmaheavy_pipe": prof.get("fmaheavy_pipe")}   # IMAD's half-rate pipe
        if "shared_wavefronts" in prof and "duration_ms" in prof:
            gbps = prof["shared_wavefronts"] * 128 / (prof["duration_ms"] / 1e3) / 1e9
            hw["shared_wavefront_GBps"] = gbps
            hw["shared_wavefront_frac_of_measured_peak"] = gbps / (148 * smem_bpc * 1965e6 / 1e9)
            if "shared_bank_conflict_wavefronts" in prof:
                hw["bank_conflict_share"] = prof["shared_bank_conflict_wavefronts"] / prof["shared_wavefronts"]
        roof["ncu"] = hw
    return roof


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.times = []
        self.t_mark = None
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except Exception:  # noqa: BLE001
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)
                self.times.append(time.perf_counter())

    def mark(self):
        """Start of the timed region (samples before it are dropped if enough remain)."""
        self.t_mark = time.perf_counter()

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        if self.t_mark is not None:
            timed = [r for r, t in zip(self.rows, self.times) if t >= self.t_mark]
            if len(timed) >= 3:
                self.rows = timed
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def workload(name):
    cfg = instgen.CONFIGS[name]
    inst = instgen.generate(name)
    return cfg, inst


def cpu_oracle_leg(inst, cfg, start, runs, iters, threads):
    """The oracle as it stands, on `threads` host threads (ctypes releases the GIL)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    O = oracle.Oracle(inst)
    p, m = start

    def one(seed):
        r = O.search(p, m, mode=1, tenure=cfg.tenure, max_iters=iters, seed=seed, kick=cfg.kick, trace=False)
        return r["iters_done"]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        done = list(ex.map(one, range(1, runs + 1)))
    dt = time.perf_counter() - t0
    return sum(done), dt


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def gather_clocks(clocks, world):
    """Clock records of every rank -> one record (median of the ranks' medians, union of reasons)."""
    if world == 1:
        return clocks
    import torch.distributed as dist
    allc = [None] * world
    dist.all_gather_object(allc, clocks)
    sm = [c["sm_mhz"] for c in allc if c.get("sm_mhz")]
    mx = [c["sm_max_mhz"] for c in allc if c.get("sm_max_mhz")]
    return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted({r for c in allc for r in c.get("reasons", [])}),
            "samples": int(sum(c.get("samples", 0) for c in allc)), "per_rank_sm_mhz": [c.get("sm_mhz") for c in allc]}


def valid_moves(inst):
    n, V = inst.n_missions, inst.n_vehicles
    return n * (n + V - 2) + n * (n - 1) // 2


def batched_config(cfg, inst, R, iters, world):
    """`config` of the batched workload; the reference arm reports the same object."""
    return {"workload": f"C3 batched: {R} tabu runs/GPU of a {inst.n_vehicles}-vehicle/"
                        f"{inst.n_missions}-mission instance, {iters} iters, tenure {cfg.tenure}, kick {cfg.kick}",
            "runs_per_gpu": R, "iters_per_run": iters, "valid_moves_per_iter": valid_moves(inst),
            "instance_seed": inst.seed, "l2": "flushed between timed steps (256 MiB write)",
            "parallelism": f"runs sharded over {world} GPU(s)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg, inst = workload(args.workload)
    import oracle
    O = oracle.Oracle(inst)
    st, start, _, _ = O.greedy()
    if st != 0:
        start = (inst.planted_ptr, inst.planted_missions)
    cores = os.cpu_count() or 1
    runs, iters = cores * args.ref_runs_per_core, args.ref_iters
    for _ in range(args.warmup):
        cpu_oracle_leg(inst, cfg, start, max(1, cores), 5, cores)
    tot_it, tot_t = 0, 0.0
    for _ in range(args.steps):
        it, dt = cpu_oracle_leg(inst, cfg, start, runs, iters, cores)
        tot_it += it
        tot_t += dt
    value = tot_it * valid_moves(inst) / tot_t
    if cfg.n_runs > 1:   # the GPU arm's config; each step times a bounded sample of it (cpu_baseline.sample)
        config = batched_config(cfg, inst, args.runs or cfg.n_runs, args.iters or cfg.max_iters, 1)
    else:
        config = {"workload": f"{args.workload}: n={inst.n_missions}, V={inst.n_vehicles}, TS",
                  "valid_moves_per_iter": valid_moves(inst)}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": config,
            "tabu_iters_per_s": tot_it / tot_t,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"{runs} runs x {iters} TS iterations of the C3 instance per step"},
            "measured": {"runs_per_step": runs, "iters_per_run": iters, "launched_gpus": args.gpus,
                         "note": "the plain oracle on the host cores (rank 0 only); n_gpus 0: no GPU work"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2002_11710_b200 import airsched as A

    cfg, inst = workload(args.workload)
    R = args.runs or cfg.n_runs
    iters = args.iters or cfg.max_iters
    h = A.Instance(inst)
    stream = torch.cuda.current_stream(dev)
    ctx = A.Ctx(local, stream.cuda_stream)
    ctx.upload(h)
    p, m, nrep = A.as_init_greedy(ctx, h)
    start = (p, m)
    prm = A.params(mode=A.AS_MODE_TABU, tenure=cfg.tenure, max_iters=iters, kick=cfg.kick, trace_level=0)
    seeds_np = np.arange(1 + rank * R, 1 + (rank + 1) * R, dtype=np.uint64)
    # device-resident inputs and outputs for the kernel-timed value
    tp = torch.from_numpy(p).to(dev)
    tm = torch.from_numpy(m).to(dev)
    ts = torch.from_numpy(seeds_np.view(np.int64)).to(dev)
    tres = torch.zeros((R, 40), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    comm = A.Comm.from_torch_distributed(ctx) if world > 1 else None
    tbp = torch.zeros((R, inst.n_vehicles + 1), dtype=torch.int32, device=dev)
    tbm = torch.zeros((R, inst.n_missions), dtype=torch.int32, device=dev)

    def step():
        # every run's best schedule stays on the device; with N GPUs the best
        # (objective, run) is all-reduced with NCCL MIN inside the call
        A.as_batch_run(ctx, h, R, tp, tm, prm, ts, shared_start=True, results=tres, best_ptr_out=tbp,
                       best_missions_out=tbm, comm=comm)

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = ctx.kernel_launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    iters_total = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.mark()
    for k in range(args.steps):
        flush.zero_()                      # L2 flush between timed steps (outside the events)
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    clocks = gather_clocks(sampler.stop(), world)
    if world > 1:
        dist.barrier()
    launches = ctx.kernel_launches - launches0
    res = tres.cpu().numpy().view(A.RESULT_DTYPE).reshape(R)
    iters_total = int(res["iters_done"].sum()) * args.steps
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_ms = float(sum(step_ms))
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
        it_t = torch.tensor([iters_total], dtype=torch.int64, device=dev)
        dist.all_reduce(it_t, op=dist.ReduceOp.SUM)
        iters_all = int(it_t.item())
    else:
        iters_all = iters_total
    VM = valid_moves(inst)
    value = iters_all * VM / (t_ms / 1e3)
    # best over all runs of all ranks (reduced on the device by the library) and its schedule
    gb = A.as_batch_gather_best(ctx, h, R, tbp, tbm, comm=comm)

    # ---- e2e: the same call with pinned HOST buffers (H2D/D2H inside the timed region)
    hp = torch.from_numpy(p).pin_memory()
    hm = torch.from_numpy(m).pin_memory()
    hs = torch.from_numpy(seeds_np.view(np.int64)).pin_memory()
    hres = torch.zeros((R, 40), dtype=torch.uint8).pin_memory()
    e2e_ms = []
    for k in range(max(1, args.e2e_steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A.as_batch_run(ctx, h, R, hp, hm, prm, hs, shared_start=True, results=hres)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_iters = int(hres.numpy().view(A.RESULT_DTYPE)["iters_done"].sum())
    e2e_t = float(np.mean(e2e_ms))
    if world > 1:   # whole job: iterations summed over ranks / the slowest rank's wall time
        tt = torch.tensor([e2e_t, float(e2e_iters)], dtype=torch.float64, device=dev)
        mx = tt.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        e2e_t, e2e_iters = float(mx[0].item()), int(tt[1].item())
    e2e_value = e2e_iters * VM / (e2e_t / 1e3)
    h2d = p.nbytes + m.nbytes + seeds_np.nbytes
    d2h = R * 40

    # ---- roofline of the dominant kernel (k_batch: the step is k_batch + the tiny k_batch_best;
    # its share of the step is in the committed ncu launch list)
    f_mhz = clocks.get("sm_mhz") or 1965.0
    rl, sw = move_mix(inst)
    its_rank = iters_total if world == 1 else iters_all / world
    roof = onchip_roofline(its_rank * rl, its_rank * sw, t_ms / 1e3, f_mhz, 1, args.workload)

    sharded = None if args.no_sharded else sharded_c5(args, A, ctx, comm, world, rank, dev)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        import oracle  # noqa: F401  (cpu_baseline leg only)
        cores = os.cpu_count() or 1
        runs_cpu, iters_cpu = cores * 4, 100
        it_cpu, dt_cpu = cpu_oracle_leg(inst, cfg, start, runs_cpu, iters_cpu, cores)
        it1, dt1 = cpu_oracle_leg(inst, cfg, start, 2, iters_cpu, 1)
        cpu = {"value": it_cpu * VM / dt_cpu, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
               "single_thread_value": it1 * VM / dt1,
               "sample": f"{runs_cpu} runs x {iters_cpu} TS iterations (seeds 1..{runs_cpu}, kick {cfg.kick}) of the "
                         f"same instance on {cores} threads; single thread: 2 runs x {iters_cpu}"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": batched_config(cfg, inst, R, iters, world),
            "tabu_iters_per_s": iters_all / (t_ms / 1e3),
            "best_objective_s": gb["best_obj"], "best_run": gb["best_run"],
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "clocks": clocks, "roofline": roof, "cpu_baseline": cpu,
            "sharded_c5": sharded,
            "step_ms": step_ms}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def sharded_c5(args, A, ctx, comm, world, rank, dev):
    """Extra object: C5 (BASELINE configs[4], disaster surge, n=4000, V=100) as ONE instance
    whose move space is sharded over the N ranks (strong scaling; N=1: the whole-GPU kernel).
    Per rank one persistent k_grid scores its tile slice and exchanges the 8-byte winner with
    its peers through NVLink stores into an NCCL symmetric window (bounded wait); if that
    path fails on any rank, every rank falls back to the NCCL-graph path and the object says so.
    value = iterations x valid moves / device time (max over ranks); e2e = as_tabu_run with
    host buffers (start in, result + best schedule out), wall clock, max over ranks."""
    import torch
    import torch.distributed as dist
    cfg, inst = workload("surge")
    h = A.Instance(inst)
    ctx.upload(h)
    p, m, _ = A.as_init_greedy(ctx, h)
    iters = args.shard_iters
    prm = A.params(mode=A.AS_MODE_TABU, tenure=cfg.tenure, max_iters=iters)
    VM = valid_moves(inst)
    path = "k_grid on 1 GPU" if world == 1 else "fused: k_grid per rank, NVLink key exchange (symmetric window)"
    err = None
    ctx.set_option("XR_TIMEOUT_MS", 10000)

    def run(want_best=False):
        return A.as_tabu_run(ctx, h, p, m, prm, want_best=want_best, comm=comm)

    def agree(ok):
        if world == 1:
            return ok
        t = torch.tensor([0.0 if ok else 1.0], device=dev)
        dist.all_reduce(t)
        return t.item() == 0.0

    try:
        run()
        ok = True
    except A.AirschedError as e:   # noqa: PERF203
        ok, err = False, str(e)
    if not agree(ok):
        if world == 1:
            return {"error": err}
        ctx.set_option("SHARD_FUSED", 0)
        path = f"NCCL graphs (ncclAllReduce MIN per iteration); fused path failed: {err}"
        run()
    run()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(int(dev.index or 0))
    sampler.start()
    sampler.mark()
    ms, its = [], 0
    for _ in range(3):
        r = run()
        ms.append(ctx.last_kernel_ms)
        its += r["iters_done"]
    clocks = gather_clocks(sampler.stop(), world)
    t = sum(ms) / 1e3
    t0 = time.perf_counter()
    r = run(want_best=True)
    te = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([t, te], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t, te = float(tt[0].item()), float(tt[1].item())
    ctx.set_option("SHARD_FUSED", None)
    ctx.set_option("XR_TIMEOUT_MS", None)
    f_mhz = clocks.get("sm_mhz") or 1965.0
    rl, sw = move_mix(inst)
    roof = onchip_roofline(its * rl, its * sw, t, f_mhz, world, "surge")
    return {"workload": f"C5 surge: n={inst.n_missions}, V={inst.n_vehicles}, TS {iters} iters per step, "
                        f"one instance sharded over {world} GPU(s)", "scaling": "strong", "path": path,
            "value": its * VM / t, "unit": UNIT, "tabu_iters_per_s": its / t, "ms_per_step": 1e3 * t / 3,
            "steps": 3, "n_gpus": world, "valid_moves_per_iter": VM, "best_obj": r["best_obj"], "clocks": clocks,
            "e2e": {"value": r["iters_done"] * VM / te, "unit": UNIT, "h2d_bytes_per_step": int(p.nbytes + m.nbytes),
                    "d2h_bytes_per_step": int(40 + (inst.n_vehicles + 1 + inst.n_missions) * 4)},
            "roofline": roof}


def run_jobs(args):
    """Multi-instance batch (`--workload instances`): 148 distinct C3-shaped instances
    (20 vehicles / 100 missions, generator seeds C3 + 1..148) x 28 tabu runs each -- one
    CTA per instance, one wave on 148 SMs -- one `as_batch_run_jobs` call per step (each
    CTA stages the instance of its job).  Same metric as the default line; under
    torchrun every rank runs its own 4144 runs."""
    import torch
    import torch.distributed as dist
    from paper_2002_11710_b200 import airsched as A
    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    base = instgen.CONFIGS["batched"]
    n_inst = 148
    per = max(1, (args.runs or 4144) // n_inst)
    iters = args.iters or base.max_iters
    insts = [instgen.generate(base, seed=2002117103 + 1 + i) for i in range(n_inst)]
    stream = torch.cuda.current_stream(dev)
    ctx = A.Ctx(local, stream.cuda_stream)
    hs = [A.Instance(x) for x in insts]
    jobs, djobs = [], []
    for h, x in zip(hs, insts):
        ctx.upload(h)
        try:
            p, m, _ = A.as_init_greedy(ctx, h, insert_mode=1)
        except A.AirschedError:      # Alg. 1 can fail: the generator's planted schedule then
            p, m = x.planted_ptr, x.planted_missions
        jobs.append((h, p, m, per))
        djobs.append((h, torch.from_numpy(p).to(dev), torch.from_numpy(m).to(dev), per))
    R = n_inst * per
    seeds_np = np.arange(1 + rank * R, 1 + (rank + 1) * R, dtype=np.uint64)
    ts = torch.from_numpy(seeds_np.view(np.int64)).to(dev)
    tres = torch.zeros((R, 40), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    prm = A.params(mode=A.AS_MODE_TABU, tenure=base.tenure, max_iters=iters, kick=base.kick)
    comm = A.Comm.from_torch_distributed(ctx) if world > 1 else None

    def step():
        A.as_batch_run_jobs(ctx, djobs, prm, ts, results=tres, comm=comm)

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = ctx.kernel_launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.mark()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = ctx.kernel_launches - launches0
    res = tres.cpu().numpy().view(A.RESULT_DTYPE).reshape(R)
    moves = sum(int(res["iters_done"][j * per:(j + 1) * per].sum()) * valid_moves(insts[j]) for j in range(n_inst))
    t_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    if world > 1:
        tt = torch.tensor([t_ms, 0.0], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt[0].item())
    value = moves * args.steps * world / (t_ms / 1e3)
    # e2e: host starts, seeds and results (the marshalling copies them inside the call)
    hres = np.zeros(R, A.RESULT_DTYPE)
    e2e_ms = []
    for _ in range(max(1, args.e2e_steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A.as_batch_run_jobs(ctx, jobs, prm, seeds_np, results=hres, comm=comm)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_moves = sum(int(hres["iters_done"][j * per:(j + 1) * per].sum()) * valid_moves(insts[j]) for j in range(n_inst))
    f_mhz = clocks.get("sm_mhz") or 1965.0
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    h2d = sum(p.nbytes + m.nbytes for _, p, m, _ in jobs) + seeds_np.nbytes
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"{n_inst} distinct 20-vehicle/100-mission instances x {per} tabu runs/GPU, "
                                   f"{iters} iters, tenure {base.tenure}, kick {base.kick} (as_batch_run_jobs)",
                       "runs_per_gpu": R, "l2": "flushed between timed steps (256 MiB write)",
                       "parallelism": f"runs sharded over {world} GPU(s)"},
            "tabu_iters_per_s": int(res["iters_done"].sum()) * args.steps * world / (t_ms / 1e3),
            "e2e": {"value": e2e_moves * world / (float(np.mean(e2e_ms)) / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(R * 40)},
            "gpu_launches": int(launches), "clocks": clocks,
            "roofline": onchip_roofline(
                sum(int(res["iters_done"][j * per:(j + 1) * per].sum()) * move_mix(insts[j])[0] for j in range(n_inst))
                * args.steps, sum(int(res["iters_done"][j * per:(j + 1) * per].sum()) * move_mix(insts[j])[1]
                                  for j in range(n_inst)) * args.steps, t_ms / 1e3, f_mhz, 1, "instances"),
            "cpu_baseline": None}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def measured_profile(workload):
    """The committed ncu --set full capture of the dominant kernel for this workload
    (profiles/r02/traffic.json), or {}."""
    path = os.path.join(PROFILE_DIR, "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload) or {}
    except (OSError, ValueError):
        return {}


def measured_traffic(workload):
    """DRAM bytes per launch of the dominant kernel (ncu capture), or None."""
    rec = measured_profile(workload)
    return float(rec["bytes_per_launch"]) if "bytes_per_launch" in rec else None


def run_single(args):
    """Single-instance workloads (C1 tiny, C2 ontario, C4 large, C5 surge): one step =
    one as_tabu_run (or as_nbhd_run with --ns) of max_iters iterations from the
    Alg. 1 start; device time from CUDA events around the kernel launches.  Under
    torchrun (N > 1) the ONE instance's move space is sharded over the ranks with an
    8-byte NCCL MIN per iteration (strong scaling; time = max over ranks)."""
    import torch
    import torch.distributed as dist
    from paper_2002_11710_b200 import airsched as A
    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    cfg, inst = workload(args.workload)
    iters = args.iters or cfg.max_iters
    h = A.Instance(inst)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    ctx = A.Ctx(local, stream.cuda_stream)
    ctx.upload(h)
    p, m, _ = A.as_init_greedy(ctx, h)
    comm = A.Comm.from_torch_distributed(ctx) if world > 1 else None
    mode = A.AS_MODE_NS if args.ns else A.AS_MODE_TABU
    prm = A.params(mode=mode, tenure=cfg.tenure, max_iters=iters)

    def fn():
        f = A.as_nbhd_run if args.ns else A.as_tabu_run
        return f(ctx, h, p, m, prm, want_best=False, comm=comm)

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        fn()
    if world > 1:
        dist.barrier()
    sampler.mark()
    ms, its = [], 0
    t_wall = time.perf_counter()
    steps = 0
    # at least `steps` steps; with --min-seconds, more until the timed region lasts that long, so the
    # clock sampler (200 ms period) sees the kernels of sub-millisecond configs
    while steps < args.steps or time.perf_counter() - t_wall < args.min_seconds:
        r = fn()
        ms.append(ctx.last_kernel_ms)
        its += r["iters_done"]
        steps += 1
    clocks = gather_clocks(sampler.stop(), world)
    # per-iteration device latency by phase of the whole-GPU kernel (one extra, untimed run)
    phases = None
    try:
        with ctx.options(PHASE_TIMES=1):
            fn()
            phases = ctx.grid_phases()
    except A.AirschedError:   # the run did not use the whole-GPU kernel
        phases = None
    t = sum(ms) / 1e3
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    if rank != 0:
        dist.destroy_process_group()
        return 0
    VM = valid_moves(inst)
    line = {"metric": METRIC, "value": its * VM / t, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": f"{args.workload}: n={inst.n_missions}, V={inst.n_vehicles}, "
                                   f"{'NS' if args.ns else 'TS'} {iters} iters", "valid_moves_per_iter": VM,
                       "parallelism": f"move space sharded over {world} GPUs" if world > 1 else "1 GPU"},
            "tabu_iters_per_s": its / t, "iters_done_per_step": its / steps, "best_obj": r["best_obj"],
            "stop_reason": r["stop_reason"], "clocks": clocks, "gpu_launches": ctx.kernel_launches,
            "phases_per_iter": phases,
            "roofline": onchip_roofline(its * move_mix(inst)[0], its * move_mix(inst)[1], t,
                                        clocks.get("sm_mhz") or 1965.0, world, args.workload)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# (config, single-thread iterations, all-core iterations)
ORACLE_PLAN = [("tiny", 200, 200), ("ontario", 200, 400), ("batched", 100, 100), ("large", 5, 40), ("surge", 1, 3)]



def oracle_baselines(out):
    """cpu_baseline leg for every config: the oracle as it stands on this host,
    single thread (or_search) and all cores (independent runs for C3; or_search_par with memo
    off -- the same per-move arithmetic over one index chunk per core -- for the single-instance
    configs), bounded samples (a few iterations of C4/C5).  JSON lines to `out`."""
    import oracle  # noqa: F401  (cpu_baseline leg only)
    from concurrent.futures import ThreadPoolExecutor
    cores = os.cpu_count() or 1
    rows = []
    for name, it1, itn in ORACLE_PLAN:
        cfg = instgen.CONFIGS[name]
        inst = instgen.generate(name)
        O = oracle.Oracle(inst)
        st, (p, m), _, _ = O.greedy()
        n, V = inst.n_missions, inst.n_vehicles
        VM = n * (n + V - 2) + n * (n - 1) // 2
        t0 = time.perf_counter()
        r = O.search(p, m, mode=1, tenure=cfg.tenure, max_iters=it1, trace=False)
        t1 = time.perf_counter() - t0
        single = r["iters_done"] * VM / t1
        if cfg.n_runs > 1:
            runs = cores * 4

            def one(seed):
                return O.search(p, m, mode=1, tenure=cfg.tenure, max_iters=itn, seed=seed, kick=cfg.kick,
                                trace=False)["iters_done"]
            t0 = time.perf_counter()
            with ThreadPoolExecutor(max_workers=cores) as ex:
                its = sum(ex.map(one, range(1, runs + 1)))
            tn = time.perf_counter() - t0
            alln = its * VM / tn
            how = f"{runs} independent runs x {itn} TS iterations on {cores} threads"
        else:
            t0 = time.perf_counter()
            r = O.search_par(p, m, mode=1, tenure=cfg.tenure, max_iters=itn, threads=cores, memo=False, trace=False)
            tn = time.perf_counter() - t0
            alln = r["iters_done"] * VM / tn
            how = f"{itn} TS iterations, index range in {cores} chunks (or_search_par, memo off)"
        row = {"config": name, "n": n, "V": V, "valid_moves_per_iter": VM, "unit": "move evals/s",
               "single_thread": single, "single_thread_sample": f"{it1} TS iterations (or_search)",
               "all_cores": alln, "all_cores_sample": how, "cores": cores, "cpu_model": cpu_model(),
               "kind": "oracle (plain recompute per move, untuned)"}
        rows.append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")



def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch(args):
    """`--gpus N` without a torchrun environment: start N ranks (one per GPU) under
    torch.distributed.run on this node and return its exit code.  Refuses (exit 2)
    when fewer than N GPUs are visible (the dry mode needs none)."""
    if not args.dry and args.impl != "reference":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but only {have} GPU(s) visible", "n_gpus": args.gpus}),
                  flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    log(f"bench: launching {args.gpus} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def run_dry(args):
    """Launch-path check without GPUs: every rank joins a gloo group, all-reduces its
    rank, and rank 0 prints the world it saw (tests/test_bench_contract.py)."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([1.0, float(rank)])
        dist.all_reduce(t)
        ranks, rank_sum = int(t[0].item()), int(t[1].item())
        dist.destroy_process_group()
    else:
        ranks, rank_sum = 1, 0
    if rank == 0:
        print(json.dumps({"dry": True, "n_gpus": args.gpus, "world": world, "ranks_seen": ranks,
                          "rank_sum": rank_sum}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--workload", default="batched")
    ap.add_argument("--runs", type=int, default=0)
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--ref-runs-per-core", type=int, default=2)
    ap.add_argument("--ref-iters", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sharded", action="store_true", help="skip the extra sharded-C5 object")
    ap.add_argument("--shard-iters", type=int, default=200, help="TS iterations per step of the sharded C5 object")
    ap.add_argument("--traffic", type=float, default=None, help="dram bytes/launch from an ncu --set full capture")
    ap.add_argument("--ns", action="store_true", help="single-instance workloads: neighbourhood search")
    ap.add_argument("--min-seconds", type=float, default=0.0,
                    help="single-instance workloads: repeat steps until the timed region lasts this long")
    ap.add_argument("--dry", action="store_true", help="launch-path check on CPU (gloo), no GPU work")
    ap.add_argument("--oracle-baselines", default=None, metavar="PATH",
                    help="only the cpu_baseline leg, for every config: write JSON lines to PATH")
    args = ap.parse_args()
    launched = "WORLD_SIZE" in os.environ
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if not launched and args.gpus > 1:
        return relaunch(args)
    _, world, _ = dist_env()
    if launched and world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}", "n_gpus": args.gpus}), flush=True)
        return 2
    if args.dry:
        return run_dry(args)
    if args.oracle_baselines:
        oracle_baselines(args.oracle_baselines)
        return 0
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "instances":
        return run_jobs(args)
    if instgen.CONFIGS[args.workload].n_runs == 1:
        return run_single(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
