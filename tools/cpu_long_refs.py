"""Long CPU reference runs for BASELINE configs c1 and c5 (TEST / MEASUREMENT
INFRASTRUCTURE, CPU container; results committed under profiles/):

  c1  the FC-only predictor (FC2 5550-1024-33) on a synthetic 1M-instruction
      trace, one sub-trace (simulate_trace), CPU: the oracle port (the
      reference's validate_or_throw rejects zero conv layers, cnn.cpp:245, so
      the FC2 predictor has no reference implementation; the port defines it
      identically to the GPU path).  Also the GPU side's parity anchor.
  c5  the K = 1 (sequential) reference run of the c2 workload (10M
      instructions, C3): the accuracy baseline of the sub-trace count sweep
      (CPI error vs K = 1, acceptance_main.cpp:326-334), by the reference's
      own simulate_trace (oracle/_ref).

  python tools/cpu_long_refs.py c1|c5 [--n N]
"""
import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("which", choices=["c1", "c5"])
    p.add_argument("--n", type=int, default=0)
    a = p.parse_args()
    from oracle.oracle import Port, Ref

    from paper_2105_05821_b200.formats import CnnConfig, Model, write_model, write_trace
    from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace
    from scale_parity import block_hashes, model_digest, trace_digest

    port = Port()
    t0 = time.time()
    if a.which == "c1":
        n = a.n or 1_000_000
        t = synthetic_trace(n, 101)
        # the bench model recipe (synth.synthetic_model: reference init rule,
        # hidden biases zeroed, head gains / biases for a DES-like regime)
        m = synthetic_model(synthetic_trace(200_000, 101), 1, config=CnnConfig.preset_fc2(),
                            init_params=port.init_params)
        r = port.simulate(t, m, sequential=True, threads=1)
        out = {"config": "c1", "predictor": "FC2 5550-1024-33", "impl": "oracle port (1 thread)",
               "instructions": n, "total_cycles": r["total_cycles"], "cpi": r["total_cycles"] / n,
               "seconds": time.time() - t0, "cpu_mips": n / (time.time() - t0) / 1e6,
               "trace_digest": trace_digest(t), "model_digest": model_digest(m),
               "fetch_blocks": block_hashes(r["predicted_fetch"]).tolist()}
    else:
        n = a.n or 10_000_000
        t = synthetic_trace(n, 101)
        m = synthetic_model(synthetic_trace(200_000, 101), 1, init_params=port.init_params)
        R = Ref()
        with tempfile.TemporaryDirectory() as td:
            tp, mp = Path(td) / "t.trace", Path(td) / "m.model"
            write_trace(tp, t)
            write_model(mp, m)
            r = R.simulate(tp, mp, k=1, sequential=True, workers=1, n_hint=n)
        out = {"config": "c5 K=1 reference", "impl": "oracle/_ref simulate_trace (1 thread)", "instructions": n,
               "total_cycles": r["total_cycles"], "cpi": r["total_cycles"] / n, "seconds": r["seconds"],
               "cpu_mips": n / r["seconds"] / 1e6, "trace_digest": trace_digest(t), "model_digest": model_digest(m),
               "fetch_blocks": block_hashes(r["predicted_fetch"][:n]).tolist()}
    dst = ROOT / "tests" / "golden" / "scale" / f"{a.which}_k1_ref.json"
    dst.write_text(json.dumps(out))
    print(json.dumps({k: v for k, v in out.items() if k != "fetch_blocks"}))


if __name__ == "__main__":
    main()
