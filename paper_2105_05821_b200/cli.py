"""``ilsim simulate`` on the GPU (tools/ilsim_main.cpp:126-186, 253-264).

  python -m paper_2105_05821_b200 simulate --trace T (--model M | --oracle) --report R
         [--parallel K] [--subtrace-size S] [--batch-max B] [--window W]
         [--phase-report P] [--throughput C] [--device D] [--precision tf32x3]
         [--warmup N] [--drain-trim]

Same files and console line as the reference: the summary CSV
(metrics.cpp:33-40), the phase-CPI CSV from the predicted fetch series
(metrics.cpp:18-31, 42-47; window n/100 by default), the throughput CSV
(parallel.cpp:95-105), "simulated N instructions: C cycles, cpi X (Ts)".
Errors print "error: <message>" and exit 1 (ilsim_main.cpp:285-288).
"""
from __future__ import annotations

import argparse
import sys
import time

import numpy as np

from .api import GpuSimulator, ParallelConfig, SimConfig, throughput_csv
from .errors import IlsimError
from .formats import trace_records


def phase_cpi(fetch: np.ndarray, window: int) -> tuple[list[float], bool]:
    """``phase_cpi`` (metrics.cpp:18-31): mean fetch latency per window."""
    if window < 1:
        raise IlsimError("phase_cpi: window must be >= 1")
    f = np.asarray(fetch, dtype=np.uint64)
    out, partial = [], False
    for start in range(0, f.size, window):
        chunk = f[start:start + window]
        out.append(float(chunk.sum()) / float(chunk.size))
        partial = partial or chunk.size < window
    return out, partial


def _g(x: float) -> str:
    """std::ostream default formatting of a double (6 significant digits)."""
    return f"{x:.6g}"


def sim_report_csv(r: dict) -> str:
    """``sim_report_csv`` (metrics.cpp:33-40)."""
    return ("instructions,total_cycles,cpi,sum_fetch,delta,drain_cycles,overflow_stall_cycles,empty\n"
            f"{r['instructions']},{r['total_cycles']},{_g(r['cpi'])},{r['sum_fetch']},{r['delta']},"
            f"{r['drain_cycles']},{r['overflow_stall_cycles']},{1 if r['empty'] else 0}\n")


def phase_cpi_csv(cpi: list[float]) -> str:
    """``phase_cpi_csv`` (metrics.cpp:42-47)."""
    return "window_index,cpi\n" + "".join(f"{i},{_g(c)}\n" for i, c in enumerate(cpi))


def cmd_simulate(a) -> int:
    n_trace = trace_records(a.trace)[1]  # header checks; the records are unpacked on the GPU
    sim = SimConfig()
    with GpuSimulator(a.device, a.precision) as g:
        if not a.oracle:
            if not a.model:
                raise IlsimError("simulate requires --model or --oracle")
            g.load_model(a.model)
            sim.max_context = g.model.config.max_context
        t0 = time.perf_counter()
        if a.parallel > 1 or a.subtrace_size > 0:
            pc = ParallelConfig(k=a.parallel, subtrace_size=a.subtrace_size, batch_max=a.batch_max, sim=sim,
                                warmup=a.warmup, drain_trim=a.drain_trim, write_ring=a.write_ring)
            g.load_trace_file(a.trace, pc, oracle=a.oracle)
            pr = g.run(pc, oracle=a.oracle)
            subs, n, total, cpi, fetch = pr.sub_results, pr.instructions, pr.total_cycles, pr.cpi, pr.predicted_fetch
        else:
            pc = ParallelConfig(k=1, sim=sim, write_ring=a.write_ring)
            g.load_trace_file(a.trace, pc, sequential=True, oracle=a.oracle)
            r = g.run(pc, sequential=True, oracle=a.oracle).sub_results[0]
            subs, n, total, cpi, fetch = [r], r.instructions, r.total_cycles, r.cpi, r.predicted_fetch
        seconds = time.perf_counter() - t0
    agg = {"instructions": n, "total_cycles": total, "cpi": cpi,
           "sum_fetch": sum(s.sum_fetch for s in subs), "delta": sum(s.delta for s in subs),
           "drain_cycles": sum(s.drain_cycles for s in subs),
           "overflow_stall_cycles": sum(s.overflow_stall_cycles for s in subs), "empty": n_trace == 0}
    with open(a.report, "w") as f:
        f.write(sim_report_csv(agg))
    w = a.window if a.window > 0 else max(1, n_trace // 100)
    if fetch is not None and len(fetch) > 0:
        cpis, _ = phase_cpi(fetch, w)
        with open(a.phase_report or a.report + ".phase.csv", "w") as f:
            f.write(phase_cpi_csv(cpis))
    if a.throughput:
        with open(a.throughput, "w") as f:
            f.write(throughput_csv([(max(a.parallel, 1), n, seconds)]))
    print(f"simulated {n} instructions: {total} cycles, cpi {_g(cpi)} ({_g(seconds)}s)")
    return 0


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="ilsim-gpu")
    sub = p.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("simulate", help="instruction-centric trace simulation on the GPU")
    s.add_argument("--trace", required=True)
    s.add_argument("--model", default="")
    s.add_argument("--oracle", action="store_true", help="use recorded ground-truth latencies")
    s.add_argument("--parallel", type=int, default=1, help="number of sub-traces")
    s.add_argument("--subtrace-size", type=int, default=0, help="instructions per sub-trace")
    s.add_argument("--batch-max", type=int, default=4096, help="max predictor batch size")
    s.add_argument("--window", type=int, default=0, help="phase CPI window (default: n/100)")
    s.add_argument("--report", required=True, help="summary csv")
    s.add_argument("--phase-report", default="", help="phase CPI csv (default: <report>.phase.csv)")
    s.add_argument("--throughput", default="", help="throughput csv")
    s.add_argument("--device", type=int, default=0, help="CUDA device")
    s.add_argument("--precision", default="tf32x3", choices=["fp32", "tf32x3", "tf32", "bf16", "fp8"])
    s.add_argument("--warmup", type=int, default=0, help="extension: warm-up instructions per sub-trace")
    s.add_argument("--drain-trim", action="store_true", help="extension: count only the last sub-trace's drain")
    s.add_argument("--write-ring", type=int, default=0,
                   help="write-queue ring entries per sub-trace (0 = auto: grows on overflow)")
    a = p.parse_args(argv)
    try:
        return cmd_simulate(a)
    except (IlsimError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
