"""Benchmark: simulated MIPS of the SimNet parallel sub-trace simulation path.

Workload (BASELINE.json configs[1], "c2"): C3 CNN latency predictor, synthetic
10M-instruction trace, 1024 sub-traces per GPU.  One "step" = one complete
simulation of the trace (all 9,766 rounds of K1 context -> K2 inference ->
K3 decode/clock) with the trace resident in HBM.  N>1 (torchrun, one process
per GPU): weak scaling, each rank simulates its own 10M-instruction slice as
1024 sub-traces; the cycle/instruction totals are summed with one NCCL
all-reduce at the end (the only collective on this path).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation of the path
(oracle/_ref: the reference sources compiled from /root/reference, with the
Eigen-free restated forward) on the host cores, on a bounded sample of the
same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MFLOP_C3 = 2 * 1_073_408  # 2 x model_flops(preset_c3), cnn.cpp:319-333
CONV_MACS_C3 = 64 * 64 * 100 + 32 * 64 * 128 + 16 * 64 * 128  # conv0-2 multiplications per instruction (802,816)
N_INSTR = 10_000_000
K_SUB = 1024


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--precision", default=os.environ.get("SIMNET_PRECISION", "tf32x3"),
                   choices=["fp32", "tf32x3", "tf32", "bf16", "fp8"])
    p.add_argument("--instructions", dest="n", type=int, default=N_INSTR)
    p.add_argument("--k", type=int, default=K_SUB)
    p.add_argument("--regime", default="default", choices=["default", "memory"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-rounds", type=int, default=0, help="rounds in the CPU-baseline sample (0 = auto)")
    return p.parse_args()


def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def ncu_traffic(precision: str):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/ncu_traffic.json), or None."""
    try:
        return json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text()).get(precision)
    except (OSError, ValueError):
        return None


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        return {}


def workload(rank: int, n: int, regime: str):
    from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace

    kind = "memory" if regime == "memory" else "mix"
    trace = synthetic_trace(n, seed=101 + rank, kind=kind)
    model = synthetic_model(synthetic_trace(200_000, seed=101, kind=kind), seed=1, regime=regime)
    return trace, model


def pinned_trace(trace):
    """Copy the trace arrays into page-locked host memory (e2e H2D source)."""
    import torch

    from paper_2105_05821_b200.formats import Trace

    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    return Trace(pin(trace.pc), pin(trace.op), pin(trace.src), pin(trace.dst), pin(trace.has_data),
                 pin(trace.data_addr), pin(trace.data_size), pin(trace.hist), pin(trace.truth), trace.fetch_tick)


def trace_h2d_bytes(t) -> int:
    """Bytes ilsim_gpu_simulate_parallel copies host->device per step (CNN
    path: the recorded truth latencies are not uploaded)."""
    return int(t.pc.nbytes + t.op.nbytes + t.src.nbytes + t.dst.nbytes + t.data_addr.nbytes + t.hist.nbytes)


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref, else the oracle port) on a bounded sample
# ---------------------------------------------------------------------------
def cpu_reference(trace, model, k: int, rounds: int, repeats: int = 1):
    """Times the reference's simulate_parallel on the first rounds*k
    instructions as k sub-traces (same batch shape as the GPU run)."""
    from oracle.oracle import Port, Ref, ref_available

    from paper_2105_05821_b200.formats import write_model, write_trace

    n = rounds * k
    sample = trace.slice(0, n)
    threads = os.cpu_count() or 1
    secs = []
    if ref_available():
        kind = "reference"
        R = Ref()
        with tempfile.TemporaryDirectory() as td:
            tp, mp = Path(td) / "s.trace", Path(td) / "m.model"
            write_trace(tp, sample)
            write_model(mp, model)
            for _ in range(repeats):
                r = R.simulate(tp, mp, k=k, workers=threads, n_hint=n)
                secs.append(r["seconds"])
    else:
        kind = "port"
        P = Port()
        for _ in range(repeats):
            t0 = time.perf_counter()
            P.simulate(sample, model, k=k, threads=threads)
            secs.append(time.perf_counter() - t0)
    mips = n / statistics.median(secs) / 1e6
    return {"value": mips, "unit": "MIPS", "cores": threads, "kind": kind,
            "sample": f"{rounds} rounds x {k} sub-traces = {n} instructions of the same trace/model "
                      f"(simulate_parallel, OpenMP threads={threads}, timing scope as cmd_simulate)"}, secs


def run_reference_impl(args):
    rank, world, _ = dist_info()
    if rank != 0:
        return
    trace, model = workload(0, max(args.k * 64, 200_000), args.regime)
    rounds = args.cpu_rounds or 48
    per_step = []
    for i in range(args.warmup + args.steps):
        base, secs = cpu_reference(trace, model, args.k, rounds)
        if i >= args.warmup:
            per_step.append(secs[0])
    n = rounds * args.k
    mips = n * len(per_step) / sum(per_step) / 1e6
    line = {
        "metric": "simulated MIPS", "value": mips, "unit": "MIPS", "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(per_step), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"c2: C3 CNN, {args.k} sub-traces, {args.regime} regime (bounded CPU sample)",
                   "sub_traces": args.k, "instructions_per_step": n},
        "cpu_baseline": dict(base, value=mips),
        "e2e": {"value": mips, "unit": "MIPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our implementation
# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        run_reference_impl(args)
        return
    rank, world, local = dist_info()
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig

    trace, model = workload(rank, args.n, args.regime)
    g = GpuSimulator(local, args.precision)
    g.load_model(model)
    pc = ParallelConfig(k=args.k, sim=SimConfig(max_context=model.config.max_context))
    g.load_trace(trace, pc)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        g.run(pc)
    barrier()
    dev_ms, launches, results = [], 0, []
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r = g.run(pc)
            dev_ms.append(r.device_ms)
            launches += r.launches
            results.append(r)
        barrier()
        wall = time.perf_counter() - t0
    step_ms = sum(dev_ms) / len(dev_ms)
    # max over ranks of the device time, and the one collective: the totals
    from paper_2105_05821_b200.dist import Totals, all_reduce_totals, max_over_ranks

    tot = all_reduce_totals(Totals.of(r.sub_results), device="cuda")
    step_ms_max = max_over_ranks(step_ms, device="cuda")
    n_all = tot.instructions
    value = n_all / (step_ms_max / 1e3) / 1e6

    # kernel breakdown + roofline of the dominant kernel (instrumented pass:
    # events around every launch of every round, no graphs)
    prof = g.run(pc, profile=True)
    rounds = max(prof.rounds, 1)
    tc = args.precision != "fp32"
    if tc:  # fused round: front (K3 of the previous round + K1 + conv chain) -> FC1
        k_ms = {"round_front": prof.kernel_ms[0], "fc1": prof.kernel_ms[1]}
        dom_ms, dom_name = prof.kernel_ms[0], "round_front_kernel (K3 decode + K1 apply/gather + conv0-2 chain)"
        flops_launch = CONV_MACS_C3 * 2 * args.k
    else:
        k_ms = {"context": prof.kernel_ms[0], "inference": prof.kernel_ms[1], "decode": prof.kernel_ms[2]}
        dom_ms, dom_name = prof.kernel_ms[1], "K2 inference (SIMT fp32, all layers)"
        flops_launch = MFLOP_C3 * args.k
    launch_ms = dom_ms / rounds
    pk = peaks()
    if tc:
        div = {"bf16": 1.0, "fp8": 0.5}.get(args.precision, 2.0)
        peak_val = pk.get("bf16_tflops_sustained", 1365.8) / div
        peak_src = "MEASURED_PEAKS.json bf16_tflops_sustained" + {1.0: "", 0.5: " x 2 (fp8 e4m3 rate)"}.get(
            div, " / 2 (tf32 rate)")
        if args.precision == "tf32x3":
            peak_src += "; 3xTF32 issues 3 tensor ops per algorithmic op"
    else:
        sm_mhz = pk.get("sm_max_mhz", 1965.0)
        peak_val, peak_src = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12, "derived FFMA peak 148 SM x 128 FMA/clk x 2 x sm_max_mhz"
    achieved = flops_launch / (launch_ms / 1e3) / 1e12
    roofline = {"bound": "tensor" if tc else "fp32-ffma", "kernel": dom_name, "achieved": achieved, "peak": peak_val,
                "unit": "TFLOP/s", "frac": achieved / peak_val, "peak_source": peak_src,
                "algorithmic_flops_per_launch": flops_launch, "launch_us": 1e3 * launch_ms,
                "traffic": ncu_traffic(args.precision)}

    # e2e through the public C-ABI with host buffers (pinned), copies inside
    e2e_line = None
    if rank == 0 or world > 1:
        ptrace = pinned_trace(trace)
        # caller-owned, page-locked output for the predicted fetch series (the
        # C-ABI's caller-allocated buffer), allocated once outside the timed region
        fetch_out = torch.empty(max(trace.n, 1), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        e2e_s = []
        for _ in range(max(1, min(args.steps, 3))):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            g.simulate_parallel(ptrace, pc, fetch_out=fetch_out)
            e2e_s.append(time.perf_counter() - t1)
        e2e_t = max_over_ranks(statistics.median(e2e_s), device="cuda")
        h2d = trace_h2d_bytes(trace)
        d2h = args.k * 56 + trace.n * 4
        e2e_line = {"value": n_all / e2e_t / 1e6, "unit": "MIPS", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "scope": "ilsim_gpu_simulate_parallel: H2D trace + pack + rounds + "
                                                        "D2H sub-results and predicted fetch series (wall clock)"}

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu_base, _ = cpu_reference(trace, model, args.k, args.cpu_rounds or 48)
        except Exception as e:  # the baseline is reported, never the product
            cpu_base = {"value": None, "error": str(e)}
    if world > 1:
        torch.distributed.barrier()
    if rank != 0:
        return
    r0 = results[-1]
    line = {
        "metric": "simulated MIPS", "value": value, "unit": "MIPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision in ("fp32", "tf32x3") else ("e4m3" if args.precision == "fp8" else args.precision),
        "data": "synthetic trace + random-init C3 weights (reference init rule), resident in HBM",
        "config": {"workload": f"c2: C3 CNN predictor, {args.n} instructions x {world} GPU(s), {args.k} sub-traces per GPU",
                   "precision": args.precision, "regime": args.regime, "sub_traces": args.k * world,
                   "instructions": n_all, "rounds": r0.rounds,
                   "l2": "trace+state > 126 MB L2 per step (no flush needed)"},
        "cpi": tot.cpi,
        "wall_ms_per_step": 1e3 * wall / args.steps,
        "kernels_ms_per_step": k_ms,
        "roofline": roofline,
        "cpu_baseline": cpu_base,
        "e2e": e2e_line,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
