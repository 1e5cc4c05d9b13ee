"""Parity at BASELINE scale: the reference's own simulate_parallel
(oracle/_ref, /root/reference/proj/src/parallel.cpp:26-93 compiled unmodified,
with the Eigen-free restated forward) run ONCE in the CPU container on the
exact bench workloads, stored as small fixtures under tests/golden/scale/,
and compared with the GPU run inside bench.py / tools/configs.py.

  python tools/scale_parity.py make [--only c2,c4,c3s] [--threads 8]   (CPU, reference)
  python tools/scale_parity.py gpu  [--only ...] [--precisions tf32x3,fp32,tf32,bf16,fp8]

TEST INFRASTRUCTURE: `make` runs the CPU reference; the GPU side only reads
the committed fixtures (the GPU box has no /root/reference).

Workloads (the same generators and seeds bench.py / tools/configs.py use):
  c2   mix trace, 10M instructions, seed 101, K=1024, default-regime model
  c4   memory-heavy trace, 2M instructions, seed 101, K=1024, memory-regime model
  c3s  rank 0's shard of c3: c3 is 100M instructions as K=65,536 sub-traces
       (partition base 1525, rem 57,600), so sub-traces 0..8191 hold 1526
       instructions each = the first 12,500,992 instructions of the global
       trace, simulated as K=8192 (the same per-sub-trace results as the
       global partition, parallel.cpp:9-24)

Fixture contents: the reference's 7 per-sub-trace counters
({instructions, total, sum_fetch, delta, drain, overflow, empty}), its total
cycles, and a 64-bit hash of every 256-instruction block of predicted_fetch
(trace order), so the fraction of identical fetch blocks is measurable
without shipping 40 MB of latencies.  The criterion is the reference's
acceptance check (acceptance_main.cpp:326-334, cpi_error_percent in
include/ilsim/metrics.hpp:16-17): total cycles within 0.1% for the fp32
path; bf16 / fp8 report their CPI error separately.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
FIXDIR = ROOT / "tests" / "golden" / "scale"
BLOCK = 256

# c3: 100M instructions / 65,536 sub-traces -> the first 8192 sub-traces hold 1526 each
C3_SHARD_N = 8192 * 1526

WORKLOADS = {
    "c2": dict(n=10_000_000, k=1024, kind="mix", regime="default", seed=101),
    "c4": dict(n=2_000_000, k=1024, kind="memory", regime="memory", seed=101),
    "c3s": dict(n=C3_SHARD_N, k=8192, kind="mix", regime="default", seed=101),
    # the same workloads with the trained C3 (tests/golden/c3_trained.model, tests/golden/train_c3.py)
    "c2t": dict(n=10_000_000, k=1024, kind="mix", regime="trained", seed=101),
    "c4t": dict(n=2_000_000, k=1024, kind="memory", regime="trained", seed=101),
    "c3st": dict(n=C3_SHARD_N, k=8192, kind="mix", regime="trained", seed=101),
    # the paper-scale residual model (7 x 384-channel residual conv blocks, 84 MFLOPs per instruction)
    "rb7": dict(n=200_000, k=1024, kind="mix", regime="default", seed=101, config="rb7"),
}
TRAINED_MODEL = ROOT / "tests" / "golden" / "c3_trained.model"


def build_workload(name: str, init_params=None):
    """(trace, model, spec) exactly as the bench / configs build them."""
    from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace

    w = WORKLOADS[name]
    trace = synthetic_trace(w["n"], seed=w["seed"], kind=w["kind"])
    if w["regime"] == "trained":
        from paper_2105_05821_b200.formats import read_model

        model = read_model(TRAINED_MODEL)
    else:
        from paper_2105_05821_b200.formats import CnnConfig

        cfg = CnnConfig.preset_rb7() if w.get("config") == "rb7" else None
        model = synthetic_model(synthetic_trace(200_000, seed=101, kind=w["kind"]), seed=1, regime=w["regime"],
                                init_params=init_params, config=cfg)
    return trace, model, w


def trace_digest(t) -> str:
    h = hashlib.blake2b(digest_size=8)
    for a in (t.pc, t.op, t.src, t.dst, t.has_data, t.data_addr, t.hist):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def model_digest(m) -> str:
    h = hashlib.blake2b(digest_size=8)
    h.update(np.ascontiguousarray(m.params, np.float32).tobytes())
    h.update(np.ascontiguousarray(m.norm, np.float64).tobytes())
    return h.hexdigest()


_MULT = np.random.default_rng(0x5EED).integers(1, 2**63, BLOCK, dtype=np.uint64) * np.uint64(2) + np.uint64(1)


def block_hashes(pf: np.ndarray) -> np.ndarray:
    """u64 hash of each 256-instruction block of a predicted-fetch series."""
    n = pf.size
    nb = -(-n // BLOCK)
    v = np.zeros(nb * BLOCK, np.uint64)
    v[:n] = pf.astype(np.uint64) + np.uint64(1)
    with np.errstate(over="ignore"):
        return (v.reshape(nb, BLOCK) * _MULT[None, :]).sum(axis=1, dtype=np.uint64)


def fixture_path(name: str) -> Path:
    return FIXDIR / f"{name}.npz"


def load_fixture(name: str):
    p = fixture_path(name)
    if not p.exists():
        return None
    z = np.load(p, allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    return {"meta": meta, "subs": z["subs"], "blocks": z["blocks"]}


def compare(name: str, result, trace=None, model=None, *, digests=None) -> dict:
    """Parity of a GPU ParallelResult against the reference fixture."""
    fx = load_fixture(name)
    if fx is None:
        return {"fixture": None, "note": f"no reference fixture for {name}"}
    meta = fx["meta"]
    if digests is None and trace is not None:
        digests = (trace_digest(trace), model_digest(model))
    if digests is not None and (digests[0] != meta["trace_digest"] or digests[1] != meta["model_digest"]):
        return {"fixture": fixture_path(name).name, "error": "workload digest differs from the fixture's",
                "got": list(digests), "want": [meta["trace_digest"], meta["model_digest"]]}
    ref_total = int(meta["total_cycles"])
    got_total = int(result.total_cycles)
    ref_sub_total = fx["subs"][:, 1].astype(np.int64)
    got_sub_total = np.array([s.total_cycles for s in result.sub_results], np.int64)
    out = {
        "fixture": fixture_path(name).name,
        "reference": meta["reference"],
        "instructions": int(meta["instructions"]),
        "sub_traces": int(meta["k"]),
        "ref_total_cycles": ref_total,
        "gpu_total_cycles": got_total,
        "rel_err": (got_total - ref_total) / ref_total if ref_total else 0.0,
        "cpi_error_percent": 100.0 * (got_total - ref_total) / ref_total if ref_total else 0.0,
        "within_0p1pct": abs(got_total - ref_total) <= 1e-3 * ref_total,
    }
    if got_sub_total.size == ref_sub_total.size:
        rel = np.abs(got_sub_total - ref_sub_total) / np.maximum(ref_sub_total, 1)
        out["subtrace_identical_frac"] = float(np.mean(got_sub_total == ref_sub_total))
        out["subtrace_max_rel_err"] = float(rel.max()) if rel.size else 0.0
    if result.predicted_fetch is not None and result.predicted_fetch.size == int(meta["instructions"]):
        gb = block_hashes(np.asarray(result.predicted_fetch))
        out["fetch_block_identical_frac"] = float(np.mean(gb == fx["blocks"]))
        out["fetch_block"] = BLOCK
    return out


def make(names, threads: int):
    from oracle.oracle import Port, Ref

    from paper_2105_05821_b200.formats import write_model, write_trace

    FIXDIR.mkdir(parents=True, exist_ok=True)
    port = Port()
    R = Ref()
    for name in names:
        t0 = time.time()
        trace, model, w = build_workload(name, init_params=port.init_params)
        with tempfile.TemporaryDirectory() as td:
            tp, mp = Path(td) / "t.trace", Path(td) / "m.model"
            write_trace(tp, trace)
            write_model(mp, model)
            r = R.simulate(tp, mp, k=w["k"], workers=threads, n_hint=trace.n)
        meta = dict(w, workload=name, instructions=int(r["instructions"]), total_cycles=int(r["total_cycles"]),
                    trace_digest=trace_digest(trace), model_digest=model_digest(model), threads=threads,
                    seconds=r["seconds"], block=BLOCK,
                    reference="oracle/_ref: /root/reference/proj/src/{parallel,simcore,predictor,dataset,trace}.cpp "
                              "compiled unmodified + oracle/cnn_restated.cpp forward (Eigen absent)",
                    generator="tools/scale_parity.py make")
        np.savez_compressed(fixture_path(name), meta=np.array(json.dumps(meta)), subs=r["subs"].astype(np.uint64),
                            blocks=block_hashes(r["predicted_fetch"]))
        print(json.dumps({"workload": name, "total_cycles": meta["total_cycles"],
                          "cpi": meta["total_cycles"] / meta["instructions"], "ref_seconds": r["seconds"],
                          "wall_s": time.time() - t0}), flush=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("cmd", choices=["make", "gpu"])
    p.add_argument("--only", default="c2,c4,c3s")
    p.add_argument("--threads", type=int, default=0)
    p.add_argument("--precisions", default="tf32x3,fp32,tf32,bf16,fp8")
    a = p.parse_args()
    import os

    names = [s.strip() for s in a.only.split(",")]
    if a.cmd == "gpu":
        gpu_sweep(names, [s.strip() for s in a.precisions.split(",")])
    else:
        make(names, a.threads or os.cpu_count() or 1)



def gpu_sweep(names, precisions):
    """GPU side: every precision on every fixture workload, one JSON line each
    (the bf16 / fp8 / tf32 CPI errors against the reference that north_star
    asks to be reported separately)."""
    from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig

    for name in names:
        trace, model, w = build_workload(name)
        digests = (trace_digest(trace), model_digest(model))
        pc = ParallelConfig(k=w["k"], sim=SimConfig(max_context=model.config.max_context))
        for prec in precisions:
            with GpuSimulator(0, prec) as g:
                g.load_model(model)
                g.load_trace(trace, pc)
                r = g.run(pc)
            out = compare(name, r, digests=digests)
            out.update(workload=name, precision=prec, gpu_mips=trace.n / (r.device_ms / 1e3) / 1e6,
                       us_per_round=1e3 * r.device_ms / r.rounds)
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
