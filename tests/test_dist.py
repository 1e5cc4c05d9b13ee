"""Multi-process host logic on CPU (gloo, world size 2): sharding covers the
global partition exactly and the single all-reduce of shard totals equals the
single-process result.  The per-shard simulation is the oracle here; on GPUs
the same code paths run with NCCL and the CUDA simulator."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2105_05821_b200.dist import Totals, all_reduce_totals, max_over_ranks, shard_range


def test_shard_range_covers_partition():
    for k in (1, 5, 7, 1024, 65536):
        for world in (1, 2, 3, 8):
            if world > k:
                continue
            spans = [shard_range(k, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == k
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from helpers import random_trace
    from oracle.oracle import Port

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = random_trace(11, 3000)
        k = 7
        r = Port().simulate(t, oracle=True, k=k, warmup=50)
        b, e = shard_range(k, rank, world)
        mine = [dict(zip(("instructions", "total_cycles", "sum_fetch", "delta", "drain_cycles",
                          "overflow_stall_cycles"), map(int, row[:6]))) for row in r["subs"][b:e]]
        tot = all_reduce_totals(Totals.of(mine))
        tmax = max_over_ranks(float(rank + 1))
        q.put((rank, tot.as_list(), tmax, int(r["total_cycles"]), int(r["subs"][:, 0].sum())))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_totals_reduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, tot, tmax, full_total, full_n in out:
        assert tot[0] == full_total and tot[1] == full_n == 3000
        assert tot[0] == tot[2] + tot[3] and tot[3] == tot[4] + tot[5]  # Eq. 1 identity survives the reduce
        assert tmax == 2.0
