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
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": config,
            "tabu_iters_per_s": tot_it / tot_t,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{runs} runs x {iters} TS iterations of the C3 instance per step"},
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
    clocks = sampler.stop()
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
    e2e_value = e2e_iters * VM / (float(np.mean(e2e_ms)) / 1e3) * world
    h2d = p.nbytes + m.nbytes + seeds_np.nbytes
    d2h = R * 40

    # ---- roofline of the dominant kernel (k_batch: the step is k_batch + the tiny k_batch_best)
    ops = (inst.n_missions * (inst.n_missions + inst.n_vehicles - 2) * OPS_RELOCATE +
           inst.n_missions * (inst.n_missions - 1) // 2 * OPS_SWAP)
    f_mhz = clocks.get("sm_mhz") or 1965.0
    peak_gops = 148 * 128 * f_mhz * 1e6 / 1e9
    achieved_gops = (iters_total * ops) / (t_ms / 1e3) / 1e9 if world == 1 else (iters_all * ops) / (t_ms / 1e3) / world / 1e9
    roof = {"bound": "alu", "achieved": achieved_gops, "peak": peak_gops, "unit": "Gop/s",
            "frac": achieved_gops / peak_gops, "traffic": args.traffic if args.traffic is not None else
            measured_traffic(args.workload),
            "peak_basis": f"148 SM x 128 INT32/FP32 lanes x {f_mhz:.0f} MHz (median SM clock under load)"}
    prof = measured_profile(args.workload)
    if "issue_slots_busy" in prof:   # the issue-slot view of the same kernel (ncu): it is issue-bound
        roof["ncu_issue_slots_busy"] = prof["issue_slots_busy"]
        roof["ncu_alu_fma_pipe"] = [prof.get("alu_pipe"), prof.get("fma_pipe")]
    if "shared_wavefronts_pct_of_peak" in prof:   # the memory level that binds (HBM/L2 are ~0 by design)
        roof["ncu_shared_mem_pct_of_peak"] = prof["shared_wavefronts_pct_of_peak"]
        if "duration_ms" in prof and "shared_wavefronts" in prof:   # 128 B per shared-memory wavefront
            roof["ncu_shared_mem_GBps"] = prof["shared_wavefronts"] * 128 / (prof["duration_ms"] / 1e3) / 1e9

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
        cpu = {"value": it_cpu * VM / dt_cpu, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{runs_cpu} runs x {iters_cpu} TS iterations (seeds 1..{runs_cpu}, kick {cfg.kick}) of the same instance"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": batched_config(cfg, inst, R, iters, world),
            "tabu_iters_per_s": iters_all / (t_ms / 1e3),
            "best_objective_s": gb["best_obj"], "best_run": gb["best_run"],
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "clocks": clocks, "roofline": roof, "cpu_baseline": cpu,
            "step_ms": step_ms}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


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
    ops = sum(int(res["iters_done"][j * per:(j + 1) * per].sum()) *
              (insts[j].n_missions * (insts[j].n_missions + insts[j].n_vehicles - 2) * OPS_RELOCATE +
               insts[j].n_missions * (insts[j].n_missions - 1) // 2 * OPS_SWAP) for j in range(n_inst))
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
    peak = 148 * 128 * f_mhz * 1e6 / 1e9
    ach = ops * args.steps / (t_ms / 1e3) / 1e9
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
            "roofline": {"bound": "alu", "achieved": ach, "peak": peak, "unit": "Gop/s", "frac": ach / peak,
                         "traffic": None,
                         "peak_basis": f"148 SM x 128 INT32/FP32 lanes x {f_mhz:.0f} MHz (median SM clock under load)"},
            "cpu_baseline": None}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def measured_profile(workload):
    """The committed ncu --set full capture of the dominant kernel for this workload
    (profiles/r01/traffic.json), or {}."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01", "traffic.json")
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
    for _ in range(args.steps):
        r = fn()
        ms.append(ctx.last_kernel_ms)
        its += r["iters_done"]
    clocks = sampler.stop()
    t = sum(ms) / 1e3
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    if rank != 0:
        dist.destroy_process_group()
        return 0
    VM = valid_moves(inst)
    line = {"metric": METRIC, "value": its * VM / t, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": f"{args.workload}: n={inst.n_missions}, V={inst.n_vehicles}, "
                                   f"{'NS' if args.ns else 'TS'} {iters} iters", "valid_moves_per_iter": VM,
                       "parallelism": f"move space sharded over {world} GPUs" if world > 1 else "1 GPU"},
            "tabu_iters_per_s": its / t, "iters_done_per_step": its / args.steps, "best_obj": r["best_obj"],
            "stop_reason": r["stop_reason"], "clocks": clocks, "gpu_launches": ctx.kernel_launches}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
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
    ap.add_argument("--traffic", type=float, default=None, help="dram bytes/launch from an ncu --set full capture")
    ap.add_argument("--ns", action="store_true", help="single-instance workloads: neighbourhood search")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "instances":
        return run_jobs(args)
    if instgen.CONFIGS[args.workload].n_runs == 1:
        return run_single(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
