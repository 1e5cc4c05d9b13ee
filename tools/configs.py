"""Runs BASELINE.json's other configurations on one GPU and prints JSON lines
(the bench line covers c2).  Synthetic traces / random-init weights as bench.py.

  python tools/configs.py [--only c1,c3,c4,c5] [--precision tf32x3]

c1  FC-only predictor (paper FC2), one sub-trace (sequential), 1M
    instructions, GPU fp32 path, against the CPU run of the same config
    (tests/golden/scale/c1_k1_ref.json, tools/cpu_long_refs.py).
c3  per-GPU shard of the 8-GPU config: 100M instructions / 65,536 sub-traces
    over 8 GPUs = 12.5M instructions as 8,192 sub-traces per GPU, with parity
    against the reference fixture (tools/scale_parity.py).
c4  memory-heavy regime (store head active, long queues, full contexts).
c5  sub-trace count sweep x warm-up overlap x drain-trim: MIPS vs CPI error
    against the K=1 run with the same weights (acceptance_main.cpp:326-334).
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig  # noqa: E402
from paper_2105_05821_b200.formats import CnnConfig  # noqa: E402
from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace  # noqa: E402


def emit(d):
    print(json.dumps(d), flush=True)


def run(g, t, pc, reps=2):
    g.load_trace(t, pc)
    r = None
    for _ in range(reps):
        r = g.run(pc)
    return r


def _k1_ref(which):
    p = ROOT / "tests" / "golden" / "scale" / f"{which}_k1_ref.json"
    return json.loads(p.read_text()) if p.exists() else None


def c1(args):
    """FC-only predictor, one sub-trace, 1M instructions: the GPU fp32 path vs
    the CPU run of the same configuration (tools/cpu_long_refs.py c1)."""
    from oracle.oracle import Port
    from scale_parity import block_hashes, model_digest, trace_digest

    t = synthetic_trace(args.c1_n, 101)
    port = Port()
    cfg = CnnConfig.preset_fc2()
    m = synthetic_model(synthetic_trace(200_000, 101), 1, config=cfg)
    g = GpuSimulator(0, "fp32")
    g.load_model(m)
    pc = ParallelConfig(k=1, sim=SimConfig(max_context=cfg.max_context))
    r = run(g, t, pc, reps=1)
    path = "persistent cooperative kernel (seq_fc.cu, 1 launch)" if r.launches == 1 else \
        f"launch-per-layer rounds ({r.launches} launches)"
    out = {"config": "c1", "predictor": "FC2 5550-1024-33 (5,716,992 mults)", "precision": "fp32 (SIMT)",
           "path": path, "instructions": t.n, "sub_traces": 1, "gpu_mips": t.n / (r.device_ms / 1e3) / 1e6,
           "us_per_instruction": 1e3 * r.device_ms / t.n, "gpu_cpi": r.cpi}
    ref = _k1_ref("c1")
    if ref and ref["instructions"] == t.n and ref["trace_digest"] == trace_digest(t) and \
            ref["model_digest"] == model_digest(m):
        got = block_hashes(r.predicted_fetch)
        out.update(cpu_ref_cpi=ref["cpi"], cpu_ref_mips=ref["cpu_mips"], cpu_ref_impl=ref["impl"],
                   cpi_error_percent=100.0 * (r.cpi - ref["cpi"]) / ref["cpi"],
                   fetch_block_identical_frac=float((got == np.array(ref["fetch_blocks"], np.uint64)).mean()),
                   gpu_over_cpu=out["gpu_mips"] / ref["cpu_mips"])
    emit(out)


def c3(args):
    from scale_parity import compare

    n, k = 12_500_992, 8192  # rank 0's shard of the 100M / 65,536 partition (1526 instructions each)
    t = synthetic_trace(n, 101)
    m = synthetic_model(synthetic_trace(200_000, 101), 1)
    g = GpuSimulator(0, args.precision)
    g.load_model(m)
    r = run(g, t, ParallelConfig(k=k, sim=SimConfig(max_context=m.config.max_context)))
    emit({"config": "c3 (per-GPU shard)", "precision": args.precision, "instructions": n, "sub_traces": k,
          "rounds": r.rounds, "mips_per_gpu": n / (r.device_ms / 1e3) / 1e6,
          "us_per_round": 1e3 * r.device_ms / r.rounds, "cpi": r.cpi, "parity": compare("c3s", r, t, m),
          "note": "8 GPUs run 8 such shards with no communication until one all-reduce of the totals"})


def c4(args):
    from scale_parity import compare

    n, k = 2_000_000, 1024
    t = synthetic_trace(n, 101, kind="memory")
    m = synthetic_model(synthetic_trace(200_000, 101, kind="memory"), 1, regime="memory")
    g = GpuSimulator(0, args.precision)
    g.load_model(m)
    r = run(g, t, ParallelConfig(k=k, sim=SimConfig(max_context=m.config.max_context)))
    emit({"config": "c4 memory-heavy", "precision": args.precision, "instructions": n, "sub_traces": k,
          "mips": n / (r.device_ms / 1e3) / 1e6, "us_per_round": 1e3 * r.device_ms / r.rounds, "cpi": r.cpi,
          "overflow_stall_cycles": sum(s.overflow_stall_cycles for s in r.sub_results),
          "drain_cycles": sum(s.drain_cycles for s in r.sub_results), "parity": compare("c4", r, t, m)})


def seq(args):
    """simulate_trace with the C3 (K = 1) on the c2 trace, fp32: the persistent
    kernel (seq_c3_kernel) against the reference's own single-thread
    simulate_trace of the same trace and weights (the c5 K = 1 fixture,
    tools/cpu_long_refs.py c5): CPI error and fetch-block identity."""
    from scale_parity import block_hashes, model_digest, trace_digest

    n = args.c5_n
    t = synthetic_trace(n, 101)
    m = synthetic_model(synthetic_trace(200_000, 101), 1)
    g = GpuSimulator(0, "fp32")
    g.load_model(m)
    r = run(g, t, ParallelConfig(k=1, sim=SimConfig(max_context=m.config.max_context)), reps=1)
    out = {"config": "sequential C3 (simulate_trace, K = 1)", "precision": "fp32",
           "path": "persistent cooperative kernel (seq_c3_kernel, 1 launch)" if r.launches == 1 else
                   f"launch-per-layer rounds ({r.launches} launches)",
           "instructions": n, "gpu_mips": n / (r.device_ms / 1e3) / 1e6, "us_per_instruction": 1e3 * r.device_ms / n,
           "gpu_cpi": r.cpi}
    ref = _k1_ref("c5")
    if ref and ref["instructions"] == n and ref["trace_digest"] == trace_digest(t) and \
            ref["model_digest"] == model_digest(m):
        got = block_hashes(r.predicted_fetch)
        out.update(ref_cpi=ref["cpi"], ref_mips=ref["cpu_mips"], ref_impl=ref["impl"],
                   cpi_error_percent=100.0 * (r.cpi - ref["cpi"]) / ref["cpi"],
                   fetch_block_identical_frac=float((got == np.array(ref["fetch_blocks"], np.uint64)).mean()),
                   gpu_over_cpu=out["gpu_mips"] / ref["cpu_mips"])
    emit(out)


def c5(args):
    """Sub-trace count sweep on the c2 trace (10M instructions) up to 1M
    sub-traces x warm-up overlap x drain-trim: owned-instruction MIPS vs the
    CPI error against the reference's K = 1 run of the same trace and weights
    (tools/cpu_long_refs.py c5; acceptance_main.cpp:326-334)."""
    n = args.c5_n
    t = synthetic_trace(n, 101)
    m = synthetic_model(synthetic_trace(200_000, 101), 1)
    g = GpuSimulator(0, args.precision)
    g.load_model(m)
    mc = m.config.max_context
    ref = _k1_ref("c5")
    if ref and ref["instructions"] == n:
        ref_cpi, ref_src = ref["cpi"], ref["impl"]
    else:
        r1 = run(g, t, ParallelConfig(k=1, sim=SimConfig(max_context=mc)), reps=1)
        ref_cpi, ref_src = r1.cpi, f"GPU {args.precision} K=1"
    emit({"config": "c5 reference", "instructions": n, "sub_traces": 1, "cpi": ref_cpi, "source": ref_src})
    for k in (1024, 4096, 16384, 65536, 262144, 1048576):
        if k > n:
            continue
        for w in (0, 110, 500):
            for trim in (False, True):
                pc = ParallelConfig(k=k, warmup=w, drain_trim=trim, sim=SimConfig(max_context=mc))
                r = run(g, t, pc, reps=1)
                emit({"config": "c5", "precision": args.precision, "instructions": n, "sub_traces": k, "warmup": w,
                      "drain_trim": trim, "mips_owned": n / (r.device_ms / 1e3) / 1e6, "rounds": r.rounds,
                      "us_per_round": 1e3 * r.device_ms / r.rounds,
                      "cpi": r.cpi, "cpi_error_pct_vs_k1": 100.0 * (r.cpi - ref_cpi) / ref_cpi})


def rb7(args):
    """A paper-scale model (RB7-like: 7 residual 384-channel conv blocks,
    84 MFLOPs per instruction) through the same kernels: the generic
    per-layer tensor-core path (split-K for the wide layers)."""
    n, k = args.rb7_n, 1024
    t = synthetic_trace(n, 101)
    cfg = CnnConfig.preset_rb7()
    m = synthetic_model(synthetic_trace(200_000, 101), 1, config=cfg)
    g = GpuSimulator(0, args.precision)
    g.load_model(m)
    r = run(g, t, ParallelConfig(k=k, sim=SimConfig(max_context=cfg.max_context)), reps=1)
    mflop = 84_361_728
    emit({"config": "rb7-like (f2)", "precision": args.precision, "instructions": n, "sub_traces": k,
          "mips": n / (r.device_ms / 1e3) / 1e6, "us_per_round": 1e3 * r.device_ms / r.rounds, "cpi": r.cpi,
          "mflop_per_instruction": mflop / 1e6,
          "achieved_tflops": n * mflop / (r.device_ms / 1e3) / 1e12})


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--only", default="c1,c3,c4,c5")
    p.add_argument("--precision", default="tf32x3")
    p.add_argument("--c1-n", type=int, default=1_000_000)
    p.add_argument("--c5-n", type=int, default=10_000_000)
    p.add_argument("--rb7-n", type=int, default=200_000)
    args = p.parse_args()
    for name in args.only.split(","):
        globals()[name.strip()](args)


if __name__ == "__main__":
    main()
