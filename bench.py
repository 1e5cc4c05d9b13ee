"""Benchmark: simulated MIPS of the SimNet parallel sub-trace simulation path.

Default workload (BASELINE.json configs[1], "c2"): C3 CNN latency predictor,
synthetic 10M-instruction trace, 1024 sub-traces per GPU.  One "step" = one
complete simulation of the trace (all 9,766 rounds of K1 context -> K2
inference -> K3 decode/clock) with the trace resident in HBM.  N>1 (torchrun,
one process per GPU): weak scaling, each rank simulates its own
10M-instruction slice as 1024 sub-traces; the cycle/instruction totals are
summed with one NCCL all-reduce at the end (the only collective on this path).

--config c3 (configs[2]): ONE global 100M-instruction trace partitioned into
65,536 sub-traces (parallel.cpp:9-24) and sharded contiguously over the N
ranks (strong scaling: at N=8 each GPU runs 8,192 sub-traces); each rank
builds and uploads only its own slice.  --config c4 (configs[3]): the
memory-heavy regime, 2M instructions, 1024 sub-traces.

`parity`: the GPU run's total cycles (and per-sub-trace totals and
predicted-fetch blocks) against the reference's own simulate_parallel run
once on the same workload (tests/golden/scale/, tools/scale_parity.py) — the
acceptance criterion of acceptance_main.cpp:326-334.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c3|c4]

--impl reference times the reference's own CPU implementation of the path
(oracle/_ref: the reference sources compiled from /root/reference, with the
Eigen-free restated forward) on the host cores, on a bounded steady-state
sample of the same workload; it never loads the product library.
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


DEFAULT_WEIGHTS = "synthetic"
TRAINED_MODEL = ROOT / "tests" / "golden" / "c3_trained.model"
WEIGHTS_DESC = {
    "synthetic": "random-init C3 weights (reference init rule, synth.py head-bias recipe)",
    "trained": "C3 trained on the reference's DES traces (tests/golden/c3_trained.model, tests/golden/train_c3.py)",
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--precision", default=os.environ.get("SIMNET_PRECISION", "tf32x3"),
                   choices=["fp32", "tf32x3", "tf32", "bf16", "fp8"])
    p.add_argument("--config", default="c2", choices=["c2", "c3", "c4"])
    p.add_argument("--instructions", dest="n", type=int, default=0, help="c2/c4 trace length (0 = the config's)")
    p.add_argument("--k", type=int, default=0, help="sub-traces per GPU (c2/c4) or global (c3); 0 = the config's")
    p.add_argument("--weights", default=os.environ.get("SIMNET_WEIGHTS", DEFAULT_WEIGHTS),
                   choices=["synthetic", "trained"],
                   help="synthetic: reference init rule + head-bias recipe (synth.py); trained: the C3 trained "
                        "on the reference's DES traces (tests/golden/c3_trained.model)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-rounds", type=int, default=0, help="rounds in the CPU-baseline sample (0 = auto)")
    a = p.parse_args()
    a.regime = "memory" if a.config == "c4" else "default"
    if a.config == "c3":
        from paper_2105_05821_b200.synth import C3_K, C3_N

        a.n, a.k = C3_N, a.k or C3_K
    else:
        a.n = a.n or (2_000_000 if a.config == "c4" else N_INSTR)
        a.k = a.k or K_SUB
    return a


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


NCU_TRAFFIC_SAMPLES = 1024  # the captures in profiles/ncu_traffic.json are launches over 1,024 sub-traces


def ncu_traffic(precision: str, samples: int = NCU_TRAFFIC_SAMPLES):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/ncu_traffic.json, a launch over
    1,024 sub-traces), scaled to a launch over `samples` sub-traces, or None."""
    try:
        v = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text()).get(precision)
    except (OSError, ValueError):
        return None
    return None if v is None else v * samples / NCU_TRAFFIC_SAMPLES


def tc_peaks():
    try:
        return json.loads((ROOT / "profiles" / "peaks_tc.json").read_text())["dense_tflops"]
    except (OSError, ValueError, KeyError):
        return {}


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        return {}


def model_for(regime: str, init_params=None, weights: str = "synthetic"):
    from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace

    if weights == "trained":
        from paper_2105_05821_b200.formats import read_model

        return read_model(TRAINED_MODEL)
    kind = "memory" if regime == "memory" else "mix"
    return synthetic_model(synthetic_trace(200_000, seed=101, kind=kind), seed=1, regime=regime,
                           init_params=init_params)


def workload(args, rank: int, world: int, init_params=None):
    """(trace or this rank's slice, model, n_total, base, shard, fixture name)."""
    from paper_2105_05821_b200.dist import shard_range
    from paper_2105_05821_b200.synth import c3_trace_slice, partition_start, synthetic_trace

    model = model_for(args.regime, init_params, args.weights)
    if args.config == "c3":
        sb, se = shard_range(args.k, rank, world)
        lo, hi = partition_start(args.n, args.k, sb), partition_start(args.n, args.k, se)
        fixture = "c3s" if (sb == 0 and se >= 8192 and args.k == 65_536 and args.weights == "synthetic") else None
        return c3_trace_slice(lo, hi), model, args.n, lo, (sb, se), fixture
    kind = "memory" if args.regime == "memory" else "mix"
    trace = synthetic_trace(args.n, seed=101 + rank, kind=kind)
    fixture = None
    if rank == 0 and args.k == K_SUB:
        fixture = {("c2", N_INSTR): "c2", ("c4", 2_000_000): "c4"}.get((args.config, args.n))
        if fixture and args.weights == "trained":
            fixture += "t"
    return trace, model, args.n, 0, None, fixture


def parity_of(args, fixture, result, trace, model):
    """GPU result vs the reference fixture (rank 0; c3: its first 8192 sub-traces)."""
    if fixture is None:
        return None
    sys.path.insert(0, str(ROOT / "tools"))
    from scale_parity import WORKLOADS, compare, model_digest, trace_digest
    from paper_2105_05821_b200.api import ParallelResult

    w = WORKLOADS[fixture]
    res, tr = result, trace
    if fixture == "c3s":  # rank 0's first 8192 sub-traces = the fixture's K=8192 run
        subs = result.sub_results[: w["k"]]
        n = sum(x.instructions for x in subs)
        res = ParallelResult(subs, sum(x.total_cycles for x in subs), n, 0.0,
                             None if result.predicted_fetch is None else result.predicted_fetch[:n])
        tr = trace.slice(0, n)
    try:
        return compare(fixture, res, tr, model)
    except Exception as e:  # parity is reported, never fatal to the bench line
        return {"fixture": fixture, "error": repr(e)}


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
def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sample_trace(trace, n_total: int, k: int, base: int, subs: int, rounds: int):
    """The first `rounds` instructions of each of the first `subs` sub-traces of
    the partition (n_total, k), concatenated: simulate_parallel(k=subs) on it
    runs exactly rounds 0..rounds-1 of those sub-traces."""
    from paper_2105_05821_b200.formats import Trace
    from paper_2105_05821_b200.synth import partition_start

    parts = []
    for i in range(subs):
        s0 = partition_start(n_total, k, i) - base
        parts.append(trace.slice(s0, s0 + rounds))
    return Trace.concat(parts)


def cpu_reference(trace, model, n_total: int, k: int, base: int = 0, r0: int = 0, r1: int = 0, subs: int = 0):
    """Steady-state host-CPU MIPS of the reference's simulate_parallel
    (oracle/_ref; the oracle port where it was not built): rounds r0..r1 of
    the first `subs` sub-traces, as (time of r1 rounds - time of r0 rounds),
    so the cold start with empty queues is excluded.  Timing scope as
    cmd_simulate (ilsim_main.cpp:145-170): trace and model already loaded."""
    from oracle.oracle import Port, Ref, ref_available

    from paper_2105_05821_b200.formats import write_model, write_trace

    threads = os.cpu_count() or 1
    subs = subs or min(k, 1024)
    r1 = r1 or max(64, min(288, (n_total // k) - 1))
    r0 = r0 or max(1, r1 // 9)
    secs = {}
    if ref_available():
        kind = "reference"
        R = Ref()
        with tempfile.TemporaryDirectory() as td:
            mp = Path(td) / "m.model"
            write_model(mp, model)
            for r in (r0, r1):
                tp = Path(td) / f"s{r}.trace"
                write_trace(tp, sample_trace(trace, n_total, k, base, subs, r))
                secs[r] = R.simulate(tp, mp, k=subs, workers=threads, n_hint=subs * r)["seconds"]
    else:
        kind = "port"
        P = Port()
        for r in (r0, r1):
            t = sample_trace(trace, n_total, k, base, subs, r)
            t0 = time.perf_counter()
            P.simulate(t, model, k=subs, threads=threads)
            secs[r] = time.perf_counter() - t0
    dt = max(secs[r1] - secs[r0], 1e-9)
    mips = (r1 - r0) * subs / dt / 1e6
    return {"value": mips, "unit": "MIPS", "cores": threads, "kind": kind, "cpu_model": cpu_model(),
            "sample": f"steady state: rounds {r0}..{r1} of the first {subs} sub-traces of the same workload "
                      f"({(r1 - r0) * subs} instructions; time(rounds 0..{r1}) - time(rounds 0..{r0}); "
                      f"simulate_parallel, OpenMP threads={threads}, timing scope as cmd_simulate)",
            "seconds": dt}


def cpu_single_thread_k1(trace, model, n: int = 2000):
    """the reference's sequential simulate_trace (K=1) on one
    host thread, first n instructions of the same trace."""
    from oracle.oracle import Ref, ref_available

    from paper_2105_05821_b200.formats import write_model, write_trace

    if not ref_available():
        return None
    with tempfile.TemporaryDirectory() as td:
        tp, mp = Path(td) / "t.trace", Path(td) / "m.model"
        write_trace(tp, trace.slice(0, n))
        write_model(mp, model)
        r = Ref().simulate(tp, mp, k=1, sequential=True, workers=1, n_hint=n)
    return {"value": n / r["seconds"] / 1e6, "unit": "MIPS", "cores": 1, "kind": "reference",
            "sample": f"simulate_trace (K=1) on the first {n} instructions"}


def product_library_loaded() -> bool:
    """Whether this process mapped libilsim_gpu.so (the reference arm must not)."""
    try:
        return "libilsim_gpu.so" in Path("/proc/self/maps").read_text()
    except OSError:
        return False


def run_reference_impl(args):
    rank, world, _ = dist_info()
    if rank != 0:
        return
    from oracle.oracle import Port

    # weights through the oracle's init (cnn.cpp:335-352): the product library is never loaded
    port = Port()
    if args.config == "c3":
        from paper_2105_05821_b200.synth import c3_trace_slice, partition_start

        subs = min(args.k, 1024)
        trace = c3_trace_slice(0, partition_start(args.n, args.k, subs))
        model = model_for(args.regime, port.init_params, args.weights)
    else:
        from paper_2105_05821_b200.synth import synthetic_trace

        trace = synthetic_trace(args.n, seed=101, kind="memory" if args.regime == "memory" else "mix")
        model = model_for(args.regime, port.init_params, args.weights)
    per_step, base = [], None
    for i in range(args.warmup + args.steps):
        b = cpu_reference(trace, model, args.n, args.k, r1=args.cpu_rounds)
        if i >= args.warmup:
            per_step.append(b)
            base = b
    vals = sorted(x["value"] for x in per_step)
    mips = statistics.median(vals)
    n_step = int(round(per_step[0]["value"] * per_step[0]["seconds"] * 1e6))
    line = {
        "metric": "simulated MIPS", "value": mips, "unit": "MIPS", "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(x["seconds"] for x in per_step),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "impl": "reference",
        "config": config_dict(args, world),  # the GPU arm's workload; each step times a bounded sample of it
        "instructions_per_step": n_step,
        "cpu_baseline": dict(base, value=mips, min=vals[0], max=vals[-1]),
        "single_thread_k1": cpu_single_thread_k1(trace, model),
        "e2e": {"value": mips, "unit": "MIPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_library_loaded": product_library_loaded(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our implementation
# ---------------------------------------------------------------------------
def config_dict(args, world: int) -> dict:
    """The workload both arms report (the reference arm times a bounded
    steady-state sample of it, described in its cpu_baseline.sample)."""
    n_all = args.n if args.config == "c3" else args.n * world
    k = args.k if args.config == "c3" else args.k * world
    return {"workload": workload_name(args, world), "precision": args.precision, "regime": args.regime,
            "weights": WEIGHTS_DESC[args.weights],
            "sub_traces": k, "instructions": n_all, "rounds": -(-args.n // args.k),
            "l2": "trace+state > 126 MB L2 per step (no flush needed)"}


def workload_name(args, world: int) -> str:
    if args.config == "c3":
        return (f"c3: C3 CNN predictor, one {args.n}-instruction trace as {args.k} sub-traces sharded over "
                f"{world} GPU(s)")
    reg = ", memory-heavy regime (store head active)" if args.config == "c4" else ""
    return f"{args.config}: C3 CNN predictor{reg}, {args.n} instructions x {world} GPU(s), {args.k} sub-traces per GPU"


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

    trace, model, n_total, base, shard, fixture = workload(args, rank, world)
    g = GpuSimulator(local, args.precision)
    g.load_model(model)
    pc = ParallelConfig(k=args.k, sim=SimConfig(max_context=model.config.max_context))
    g.load_trace(trace, pc, shard=shard, n_total=n_total, base=base)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        g.run(pc, shard=shard)
    barrier()
    dev_ms, launches, results = [], 0, []
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r = g.run(pc, shard=shard)
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
    prof = g.run(pc, profile=True, shard=shard)
    rounds = max(prof.rounds, 1)
    tc = args.precision != "fp32"
    if tc:  # fused round: front (K3 of the previous round + K1 + conv chain) -> FC1
        k_ms = {"round_front": prof.kernel_ms[0], "fc1": prof.kernel_ms[1]}
        dom_ms, dom_name = prof.kernel_ms[0], "round_front_kernel (K3 decode + K1 apply/gather + conv0-2 chain)"
        flops_launch = CONV_MACS_C3 * 2 * len(results[-1].sub_results)
    else:
        k_ms = {"context": prof.kernel_ms[0], "inference": prof.kernel_ms[1], "decode": prof.kernel_ms[2]}
        dom_ms, dom_name = prof.kernel_ms[1], "K2 inference (SIMT fp32, all layers)"
        flops_launch = MFLOP_C3 * len(results[-1].sub_results)
    launch_ms = dom_ms / rounds
    pk = peaks()
    if tc:
        # the tcgen05 dense pipe peak of this kind, measured on B200 by
        # tools/probes/tc_peak.py (profiles/peaks_tc.json, sustained: the front
        # runs inside a long step); fallback MEASURED_PEAKS.json bf16 (cuBLAS)
        kind = {"bf16": "bf16", "fp8": "fp8"}.get(args.precision, "tf32")
        tcp = tc_peaks().get(kind)
        if tcp:
            peak_val = tcp["sustained"]
            peak_src = f"profiles/peaks_tc.json {kind} dense sustained (tcgen05 M=128 N=256, tools/probes/tc_peak.py)"
        else:
            div = {"bf16": 1.0, "fp8": 0.5}.get(args.precision, 2.0)
            peak_val = pk.get("bf16_tflops_sustained", 1365.8) / div
            peak_src = "MEASURED_PEAKS.json bf16_tflops_sustained scaled (peaks_tc.json absent)"
        if args.precision == "tf32x3":
            peak_src += "; 3xTF32 issues 3 tf32 products per algorithmic multiply-add (fp32-faithful ceiling = peak / 3)"
    else:
        sm_mhz = pk.get("sm_max_mhz", 1965.0)
        peak_val, peak_src = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12, "derived FFMA peak 148 SM x 128 FMA/clk x 2 x sm_max_mhz"
    achieved = flops_launch / (launch_ms / 1e3) / 1e12
    roofline = {"bound": "tensor" if tc else "fp32-ffma", "kernel": dom_name, "achieved": achieved, "peak": peak_val,
                "unit": "TFLOP/s", "frac": achieved / peak_val, "peak_source": peak_src,
                "algorithmic_flops_per_launch": flops_launch, "launch_us": 1e3 * launch_ms,
                "frac_of_3xtf32_ceiling": achieved / (peak_val / 3) if args.precision == "tf32x3" else None,
                "traffic": ncu_traffic(args.precision, len(results[-1].sub_results))}

    # the same kernel against HBM: its DRAM bytes per launch (ncu capture,
    # cold caches: an upper bound) over the live launch time -- the K1 gather /
    # K3 decode half of the fused front is memory-latency-bound, not HBM-bound
    roofline_hbm = None
    if tc and roofline["traffic"]:
        hbm_peak = pk.get("hbm_gbs", 6549.8)
        ach = roofline["traffic"] / (launch_ms / 1e3) / 1e9
        roofline_hbm = {"bound": "hbm", "kernel": dom_name, "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                        "frac": ach / hbm_peak, "bytes_per_launch": roofline["traffic"],
                        "source": "dram bytes per launch from the committed ncu --set full capture "
                                  "(profiles/ncu_traffic.json) / the live event-timed launch"}

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
            g.simulate_parallel(ptrace, pc, fetch_out=fetch_out, shard=shard, n_total=n_total, base=base)
            e2e_s.append(time.perf_counter() - t1)
        e2e_t = max_over_ranks(statistics.median(e2e_s), device="cuda")
        h2d = trace_h2d_bytes(trace)
        d2h = len(results[-1].sub_results) * 56 + trace.n * 4
        e2e_line = {"value": n_all / e2e_t / 1e6, "unit": "MIPS", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "scope": "ilsim_gpu_simulate_parallel: H2D trace + pack + rounds + "
                                                        "D2H sub-results and predicted fetch series (wall clock)"}

    parity = parity_of(args, fixture, results[-1], trace, model) if rank == 0 else None
    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu_base = cpu_reference(trace, model, n_total, args.k, base, r1=args.cpu_rounds)
        except Exception as e:  # the baseline is reported, never the product
            cpu_base = {"value": None, "error": str(e)}
    if world > 1:
        torch.distributed.barrier()
    if rank != 0:
        return
    r0 = results[-1]
    line = {
        "metric": "simulated MIPS", "value": value, "unit": "MIPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms_max, "higher_is_better": True,
        "scaling": "strong" if args.config == "c3" else "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision in ("fp32", "tf32x3") else ("e4m3" if args.precision == "fp8" else args.precision),
        "data": f"synthetic trace + {WEIGHTS_DESC[args.weights]}, resident in HBM",
        "config": config_dict(args, world),
        "cpi": tot.cpi,
        "parity": parity,
        "wall_ms_per_step": 1e3 * wall / args.steps,
        "kernels_ms_per_step": k_ms,
        "roofline": roofline,
        "roofline_hbm": roofline_hbm,
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
