"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

Runs only where /root/reference exists (the build container): the reference's
own workload generator + DES make the traces, and the reference's simulate
path (oracle/_ref, compiled from /root/reference/proj/src) produces the
expected results.  The outputs are small and committed, so the GPU box (which
has no /root/reference) can pin the oracle port and the CUDA path against
them.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Ref  # noqa: E402
from paper_2105_05821_b200.formats import read_model, read_trace  # noqa: E402

OUT = Path(__file__).resolve().parent

# (name, DES workload kind, instructions, seed) — shapes follow the reference
# tests (test_parallel.cpp:16-24, test_simcore.cpp:48-59, 16 MiB footprint).
TRACES = [
    ("mix_3000_s4", "mix", 3000, 4),
    ("streaming_3000_s6", "streaming", 3000, 6),
    ("branchy_2000_s8", "branchy", 2000, 8),
    ("pointer_chase_2000_s3", "pointer-chase", 2000, 3),
]

# Oracle-latency cases: (k, subtrace_size, max_context, retire_bandwidth, per_cycle, sequential)
ORACLE_CASES = [
    (1, 0, 110, 8, False, True),
    (1, 0, 110, 8, False, False),
    (2, 0, 110, 8, False, False),
    (3, 0, 110, 8, False, False),
    (7, 0, 110, 8, False, False),
    (64, 0, 110, 8, False, False),
    (0, 250, 110, 8, False, False),
    (5, 0, 16, 2, False, False),
    (5, 0, 4, 1, False, False),
    (3, 0, 64, 3, True, False),
]

# CNN cases run with the small model (test_parallel.cpp:114-146 config) and a
# C3-shaped model regenerated from init_weights (too large to commit).
CNN_CASES = [(1, True), (5, False), (16, False)]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    R = Ref()
    gold: dict = {"traces": {}, "oracle": [], "cnn": [], "models": {}}
    for name, kind, n, seed in TRACES:
        path = OUT / f"{name}.trace"
        des_total = R.make_trace(kind, n, seed, path)
        gold["traces"][name] = {"kind": kind, "n": n, "seed": seed, "des_total": des_total,
                                "sha256": hashlib.sha256(path.read_bytes()).hexdigest()}
        for k, size, mc, bw, pcyc, seq in ORACLE_CASES:
            r = R.simulate(path, None, k=k, subtrace_size=size, max_context=mc, retire_bandwidth=bw,
                           per_cycle=pcyc, sequential=seq, n_hint=n)
            gold["oracle"].append({
                "trace": name, "k": k, "subtrace_size": size, "max_context": mc, "retire_bandwidth": bw,
                "per_cycle": pcyc, "sequential": seq, "total_cycles": r["total_cycles"],
                "subs": r["subs"].tolist(), "predicted_fetch_sha256": sha(r["predicted_fetch"][:n]),
            })

    # models: small (committed) with identity norm and with dataset norm
    mix = OUT / "mix_3000_s4.trace"
    small_id = OUT / "small_identity.model"
    small_ds = OUT / "small_dataset.model"
    R.make_model(None, small_id, conv=(16, 16, 16), fc_hidden=32, seed=33, identity=True)
    R.make_model(mix, small_ds, conv=(16, 16, 16), fc_hidden=32, seed=7, identity=False)
    with tempfile.TemporaryDirectory() as td:
        c3 = Path(td) / "c3.model"
        R.make_model(mix, c3, seed=1, identity=False)
        m = read_model(c3)
        gold["models"]["c3_mix_seed1"] = {"norm": m.norm.tolist(), "seed": 1, "params_sha256": sha(m.params)}
        models = {"small_identity": small_id, "small_dataset": small_ds, "c3_mix_seed1": c3}
        for mname, mpath in models.items():
            for tname in ("mix_3000_s4", "branchy_2000_s8", "pointer_chase_2000_s3"):
                tpath = OUT / f"{tname}.trace"
                n = read_trace(tpath).n
                for k, seq in CNN_CASES:
                    if mname == "c3_mix_seed1" and k == 1:
                        continue  # the K=1 C3 run is slow on CPU; K=5/16 cover it
                    r = R.simulate(tpath, mpath, k=k, sequential=seq, n_hint=n)
                    gold["cnn"].append({"trace": tname, "model": mname, "k": k, "sequential": seq,
                                        "total_cycles": r["total_cycles"], "subs": r["subs"].tolist(),
                                        "predicted_fetch_sha256": sha(r["predicted_fetch"][:n])})
            # captured request stream (inputs hashed) for input-tensor pinning
            cap = R.capture(mix, mpath, 400, k=5, width=5550)
            gold["cnn"].append({"trace": "mix_3000_s4", "model": mname, "capture": 400, "k": 5,
                                "inputs_sha256": sha(cap["inputs"]), "triples_sha256": sha(cap["triples"]),
                                "index_sha256": sha(cap["index"])})
    (OUT / "golden.json").write_text(json.dumps(gold, indent=1))
    print("wrote", OUT / "golden.json")


if __name__ == "__main__":
    main()
