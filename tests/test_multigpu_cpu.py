"""Multi-GPU host logic on CPU (gloo, world_size 2): the move-space shard plan and
the 'fake sharding' of one iteration -- each rank takes the minimum packed key
over the canonical indices of its tiles (oracle values), a gloo all-reduce(MIN)
joins them, and the result must equal the single-process selection (O9).  This
is the partitioning math of the sharded C5 path; the NCCL plumbing itself is
exercised on the GPU with a one-rank communicator (tests/test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2002_11710_b200 import instgen

KR, KS = 4, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def tile_of(idx, n, V, G, ptr, ms):
    """Tile id of canonical index idx in the flat list of the sharded kernels."""
    S = n + V
    nTC = (S + 32 * KR - 1) // (32 * KR)
    nSC = (n - 1 + 32 * KS - 1) // (32 * KS) if n > 1 else 0
    nRG = (n + G - 1) // G
    n_reloc, n_swap = nTC * nRG, nSC * nRG
    if idx < n * S:
        m, t = divmod(idx, S)
        return (m // G) * nTC + t // (32 * KR)
    m1, m2 = divmod(idx - n * S, n)
    succ = {}
    for v in range(len(ptr) - 1):
        r = list(ms[ptr[v]:ptr[v + 1]])
        for a, b in zip(r[:-1], r[1:]):
            succ[a] = b
    if succ.get(m1) == m2:
        return n_reloc + n_swap + m1 // 32
    if succ.get(m2) == m1:
        return n_reloc + n_swap + m2 // 32
    j = (n - 1 - m2) // (32 * KS)
    return n_reloc + (m1 // G) * nSC + j


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        import oracle
        from paper_2002_11710_b200 import airsched as A
        inst = instgen.generate("ontario")
        h = A.Instance(inst)
        plans = [A.as_shard_plan(h, world, r, n_sm=148) for r in range(world)]
        mine = A.as_shard_plan(h, world, rank, n_sm=148)
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        assert gathered == plans
        # NCCL unique id exchange through torch.distributed (the Comm helper's path)
        obj = [A.as_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        assert len(set(ids)) == 1 and len(ids[0]) == 128
        # fake sharding of one iteration
        O = oracle.Oracle(inst)
        st, (p, m), _, _ = O.greedy()
        n, V = inst.n_missions, inst.n_vehicles
        G = max(1, (n * ((n + V + 127) // 128) + n * ((n - 1 + 63) // 64) // 2) // (4 * 148 * 24))
        rng = np.random.default_rng(4)
        E = rng.integers(-1, 12, size=(n, V)).astype(np.int32)
        obj0 = O.objective(p, m)
        d, f, best = O.eval_moves(p, m, mode=1, E=E, it=6, best_obj=obj0 - 50)
        lo, hi = mine["tile_lo"], mine["tile_hi"]
        key = np.iinfo(np.int64).max
        for idx in np.flatnonzero(f & 2):
            if lo <= tile_of(int(idx), n, V, G, p, m) < hi:
                cls = 0 if f[idx] & 8 else 1
                k = (cls << 62) | ((int(d[idx]) + (1 << 30)) << 31) | int(idx)   # same order, fits int64
                key = min(key, k)
        t = torch.tensor([key], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        k = int(t.item())
        got = (k >> 62, ((k >> 31) & ((1 << 31) - 1)) - (1 << 30), k & ((1 << 31) - 1))
        result_q.put((rank, got == best, got, best))
    finally:
        dist.destroy_process_group()


def test_gloo_shard_plan_and_fake_sharding():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    out = [q.get(timeout=5) for _ in range(world)]
    assert all(pr.exitcode == 0 for pr in procs)
    assert all(ok for _, ok, _, _ in out), out


def test_shard_plan_partitions_tiles():
    from paper_2002_11710_b200 import airsched as A
    for cfg in ("ontario", "large", "surge"):
        h = A.Instance(instgen.generate(cfg))
        for world in (1, 2, 4, 8):
            plans = [A.as_shard_plan(h, world, r) for r in range(world)]
            assert plans[0]["tile_lo"] == 0 and plans[-1]["tile_hi"] == plans[0]["tile_total"]
            for a, b in zip(plans[:-1], plans[1:]):
                assert a["tile_hi"] == b["tile_lo"]
            w = [pl["weight"] for pl in plans]
            assert sum(w) == plans[0]["weight_total"]
            if cfg == "surge":
                assert max(w) <= 1.02 * sum(w) / world     # balanced within 2 %
