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
    for k in (1, 2, 5, 7, 1024, 65536):
        for world in (1, 2, 3, 8):
            spans = [shard_range(k, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == k
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
            if world > k:  # extra ranks get an empty shard (and still join the all-reduce)
                assert sizes.count(0) == world - k


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


def _gpu_worker(rank, world, port, q, k, precision):
    """One rank of a world-`world` gloo group running the GPU library on its
    shard (every rank on cuda:0: the box has one GPU)."""
    import torch.distributed as dist

    from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig, read_model, read_trace
    from paper_2105_05821_b200.dist import simulate_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gold = __import__("conftest").GOLDEN
        t = read_trace(gold / "mix_3000_s4.trace")
        m = read_model(gold / "small_dataset.model")
        pc = ParallelConfig(k=k, sim=SimConfig(max_context=m.config.max_context))
        with GpuSimulator(0, precision) as g:
            g.load_model(m)
            b, e = shard_range(k, rank, world)
            from paper_2105_05821_b200.api import partition_starts

            starts = partition_starts(t.n, k) + [t.n]
            # the rank holds only its own slice of the trace (base = its first instruction)
            lo, hi = (starts[b], starts[e]) if b < e else (0, 0)
            res, tot = simulate_sharded(g, t.slice(lo, hi) if b < e else t.slice(0, 0), pc, rank, world,
                                        n_total=t.n, base=lo)
            subs = [[s.instructions, s.total_cycles, s.sum_fetch, s.delta, s.drain_cycles,
                     s.overflow_stall_cycles] for s in res.sub_results]
            pf = res.predicted_fetch.tolist() if res.predicted_fetch is not None else []
        q.put((rank, subs, pf, tot.as_list()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,k,precision", [(2, 5, "tf32x3"), (3, 2, "fp32")])
def test_gloo_gpu_shards_match_single_process(world, k, precision):
    """Each rank simulates its contiguous shard with the CUDA library from its
    own trace slice; concatenated, the shards reproduce the single-process
    sub-results and predicted fetch series bit-exactly, and the one
    all-reduce gives the single-process totals (parallel.cpp:83-92).  world 3,
    k 2 leaves one rank with no sub-traces (it still joins the collective)."""
    from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig, read_model, read_trace

    gold = __import__("conftest").GOLDEN
    t = read_trace(gold / "mix_3000_s4.trace")
    m = read_model(gold / "small_dataset.model")
    pc = ParallelConfig(k=k, sim=SimConfig(max_context=m.config.max_context))
    with GpuSimulator(0, precision) as g:
        g.load_model(m)
        full = g.simulate_parallel(t, pc)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q, k, precision)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    subs = [row for _, s, _, _ in out for row in s]
    pf = [v for _, _, f, _ in out for v in f]
    want = [[s.instructions, s.total_cycles, s.sum_fetch, s.delta, s.drain_cycles, s.overflow_stall_cycles]
            for s in full.sub_results]
    assert subs == want
    assert pf == full.predicted_fetch.tolist()
    for _, _, _, tot in out:
        assert tot[0] == full.total_cycles and tot[1] == t.n


def _failing_worker(rank, world, port, q):
    """Rank 1's shard simulation raises; every rank must raise, none may hang
    in the collective."""
    import torch.distributed as dist

    from paper_2105_05821_b200 import IlsimError, ParallelConfig
    from paper_2105_05821_b200.api import ParallelResult
    from paper_2105_05821_b200.dist import simulate_sharded
    from helpers import random_trace

    class FakeSim:
        def simulate_parallel(self, trace, pc, **kw):
            if rank == 1:
                raise IlsimError("device error on rank 1")
            return ParallelResult([], 0, 0, 0.0, None)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        try:
            simulate_sharded(FakeSim(), random_trace(3, 400), ParallelConfig(k=4), rank, world)
            q.put((rank, "no error"))
        except IlsimError as e:
            q.put((rank, str(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_rank_failure_reaches_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_failing_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[1] == "device error on rank 1"
    assert out[0] == "the simulation failed on 1 other rank(s)"
