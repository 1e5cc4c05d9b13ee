"""The BASELINE-scale reference fixtures (tests/golden/scale/, made by
tools/scale_parity.py from the reference's own simulate_parallel) and the
comparison the bench's `parity` key uses.  CPU only."""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))

import scale_parity as sp  # noqa: E402
from paper_2105_05821_b200.api import ParallelResult, SimResult  # noqa: E402


def _result_from(fx, pf=None):
    subs = [SimResult(int(r[1]), int(r[0]), 0.0, int(r[2]), int(r[3]), int(r[4]), int(r[5]), bool(r[6]))
            for r in fx["subs"]]
    return ParallelResult(subs, sum(s.total_cycles for s in subs), sum(s.instructions for s in subs), 0.0, pf)


@pytest.mark.parametrize("name", ["c2", "c4", "c3s"])
def test_fixture_is_consistent(name):
    fx = sp.load_fixture(name)
    assert fx is not None, f"missing fixture {name}"
    m, w = fx["meta"], sp.WORKLOADS[name]
    assert (m["n"], m["k"], m["kind"], m["regime"]) == (w["n"], w["k"], w["kind"], w["regime"])
    subs = fx["subs"]
    assert subs.shape == (w["k"], 7)
    assert int(subs[:, 0].sum()) == m["instructions"] == w["n"]
    assert int(subs[:, 1].sum()) == m["total_cycles"]
    # Eq. 1 identity per sub-trace: total = sum_fetch + delta, delta = drain + overflow
    assert np.all(subs[:, 1] == subs[:, 2] + subs[:, 3]) and np.all(subs[:, 3] == subs[:, 4] + subs[:, 5])
    assert fx["blocks"].size == -(-w["n"] // sp.BLOCK)


def test_compare_reports_exact_match_and_differences():
    fx = sp.load_fixture("c4")
    r = _result_from(fx)
    d = sp.fixture_path("c4")
    out = sp.compare("c4", r, digests=(fx["meta"]["trace_digest"], fx["meta"]["model_digest"]))
    assert out["rel_err"] == 0.0 and out["within_0p1pct"] and out["subtrace_identical_frac"] == 1.0, d
    r.sub_results[3].total_cycles += 50
    r.total_cycles += 50
    out = sp.compare("c4", r, digests=(fx["meta"]["trace_digest"], fx["meta"]["model_digest"]))
    assert out["gpu_total_cycles"] - out["ref_total_cycles"] == 50
    assert out["subtrace_identical_frac"] == 1.0 - 1.0 / 1024
    bad = sp.compare("c4", r, digests=("0", "0"))
    assert "error" in bad


def test_block_hash_detects_any_change():
    rng = np.random.default_rng(3)
    pf = rng.integers(0, 9, 1000).astype(np.uint32)
    h = sp.block_hashes(pf)
    assert h.size == 4
    for i in (0, 255, 256, 999):
        q = pf.copy()
        q[i] += 1
        d = sp.block_hashes(q) != h
        assert d.sum() == 1 and d[i // 256]


def test_c4_workload_reproduces_fixture_digest():
    """The generators are deterministic: the bench rebuilds the exact trace and
    weights the reference fixture was made from (weights via the oracle's init,
    identical to the library's, test_lib / test_oracle)."""
    from oracle.oracle import Port

    trace, model, _ = sp.build_workload("c4", init_params=Port().init_params)
    m = sp.load_fixture("c4")["meta"]
    assert sp.trace_digest(trace) == m["trace_digest"] and sp.model_digest(model) == m["model_digest"]
