"""Multi-GPU plumbing: one process per GPU, sub-traces sharded contiguously.

Sub-traces are independent (parallel.cpp:51-58; "no inter-GPU communication
is required during the simulation process"), so rank r
simulates sub-traces [shard_begin, shard_end) of the reference's global
partition (parallel.cpp:9-24) and owns one contiguous instruction range.  The
only collective is one all-reduce of the per-shard totals after the last
round (NCCL over NVLink on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

TOTAL_FIELDS = ("total_cycles", "instructions", "sum_fetch", "delta", "drain_cycles", "overflow_stall_cycles")


def shard_range(k: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of sub-traces for `rank` (first ranks take the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(k, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


@dataclass
class Totals:
    total_cycles: int = 0
    instructions: int = 0
    sum_fetch: int = 0
    delta: int = 0
    drain_cycles: int = 0
    overflow_stall_cycles: int = 0

    @staticmethod
    def of(subs) -> "Totals":
        t = Totals()
        if hasattr(subs, "array"):  # api.SubResults: sum the columns
            for f in TOTAL_FIELDS:
                setattr(t, f, int(subs.array[f].sum()))
            return t
        for s in subs:
            for f in TOTAL_FIELDS:
                setattr(t, f, getattr(t, f) + int(getattr(s, f) if not isinstance(s, dict) else s[f]))
        return t

    def as_list(self) -> list[int]:
        return [getattr(self, f) for f in TOTAL_FIELDS]

    @property
    def cpi(self) -> float:
        return self.total_cycles / self.instructions if self.instructions else 0.0


def _device(device):
    """The collective's tensor device: CPU tensors under gloo, else `device`."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_backend() == "gloo":
        return "cpu"
    return device


def all_reduce_totals(t: Totals, device=None, failed: bool = False, with_failures: bool = False):
    """Sum the shard totals over all ranks (exact: integer sums).  With
    ``with_failures`` the same collective also counts the ranks that report
    ``failed``, and ``(Totals, n_failed)`` is returned."""
    import torch
    import torch.distributed as dist

    v = torch.tensor(t.as_list() + [1 if failed else 0], dtype=torch.int64, device=_device(device))
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
    vals = [int(x) for x in v.tolist()]
    tot = Totals(*vals[:-1])
    return (tot, vals[-1]) if with_failures else tot


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank timing (multi-GPU times are the slowest rank's)."""
    import torch
    import torch.distributed as dist

    v = torch.tensor([x], dtype=torch.float64, device=_device(device))
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
    return float(v.item())


def simulate_sharded(sim, trace, pc, rank: int, world: int, *, oracle: bool = False, n_total: int | None = None,
                     base: int = 0, fetch_out=None):
    """Run this rank's shard of the global partition on its GPU and return
    (shard ParallelResult, global Totals).  ``trace`` is the whole trace, or
    (``n_total``/``base``) only the slice [base, base + trace.n) that holds
    this rank's instructions.  A rank with no sub-traces (world > k) still
    joins the one collective with zero totals, so no rank is left waiting."""
    from .api import GpuSimulator, ParallelResult
    from .errors import IlsimError

    n = trace.n if n_total is None else n_total
    k = GpuSimulator._num_sub(pc, n, False)
    shard = shard_range(k, rank, world)
    res, err = ParallelResult([], 0, 0, 0.0, None), None
    if shard[0] != shard[1]:
        try:
            res = sim.simulate_parallel(trace, pc, oracle=oracle, shard=shard, n_total=n_total, base=base,
                                        fetch_out=fetch_out)
        except Exception as e:  # still join the collective: no rank is left waiting in it
            err = e
    tot, n_failed = all_reduce_totals(Totals.of(res.sub_results), device="cuda", failed=err is not None,
                                      with_failures=True)
    if err is not None:
        raise err
    if n_failed:
        raise IlsimError(f"the simulation failed on {n_failed} other rank(s)")
    return res, tot
