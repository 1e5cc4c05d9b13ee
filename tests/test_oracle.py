"""The CPU oracle (oracle/port) pinned against the reference's own goldens and
against the reference library itself (oracle/_ref, compiled from
/root/reference/proj/src).  CPU only."""
import hashlib

import numpy as np
import pytest

from helpers import SUB, instr_trace, model_from_params, random_input, random_trace, small_config, tiny_config
from paper_2105_05821_b200.formats import CnnConfig, Model, identity_norm, read_model, read_trace

GOLD = __import__("conftest").GOLDEN


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sub(r, field, i=0):
    return int(r["subs"][i][SUB.index(field)])


# ---- test_simcore.cpp goldens (ScriptedPredictor == truth latencies) -------
def test_single_step(port):  # test_simcore.cpp:63-77
    r = port.simulate(instr_trace([False], [(5, 2, 0)]), oracle=True, sequential=True)
    assert (sub(r, "sum_fetch"), sub(r, "total_cycles"), sub(r, "delta")) == (5, 7, 2)


def test_worked_example(port):  # test_simcore.cpp:94-103
    r = port.simulate(instr_trace([False] * 3, [(5, 2, 0), (0, 3, 0), (1, 3, 0)]), oracle=True, sequential=True)
    assert sub(r, "sum_fetch") == 6 and sub(r, "drain_cycles") == 3 and sub(r, "delta") == 3
    assert sub(r, "total_cycles") == 9


@pytest.mark.parametrize("k,b,want", [(5, 2, 3), (8, 8, 1), (9, 8, 2), (16, 4, 4), (1, 3, 1)])
def test_drain_ready_entries(port, k, b, want):  # test_simcore.cpp:119-137
    r = port.simulate(instr_trace([False] * k, [(0, 0, 0)] * k), oracle=True, sequential=True, retire_bandwidth=b)
    assert sub(r, "drain_cycles") == want


def test_drain_one_entry(port):  # test_simcore.cpp:110-118
    r = port.simulate(instr_trace([False], [(0, 4, 0)]), oracle=True, sequential=True)
    assert sub(r, "drain_cycles") == 4


def test_store_write_queue(port):  # test_simcore.cpp:140-149
    r = port.simulate(instr_trace([True, False], [(1, 2, 6), (0, 1, 0)]), oracle=True, sequential=True)
    assert (sub(r, "total_cycles"), sub(r, "sum_fetch"), sub(r, "delta")) == (7, 1, 6)


def test_forced_stall(port):  # test_simcore.cpp:151-165
    r = port.simulate(instr_trace([False] * 6, [(0, 100, 0)] * 6), oracle=True, sequential=True, max_context=4)
    assert sub(r, "overflow_stall_cycles") == 100


def test_empty_trace(port):  # test_simcore.cpp:167-174
    r = port.simulate(instr_trace([], []), oracle=True, sequential=True)
    assert sub(r, "empty") == 1 and sub(r, "total_cycles") == 0


# ---- test_parallel.cpp goldens ---------------------------------------------
def test_partition(port):  # test_parallel.cpp:38-63
    assert port.partition(10, 1) == [0]
    assert port.partition(10, 2) == [0, 5]
    assert port.partition(10, 3) == [0, 4, 7]
    assert port.partition(10, 10) == list(range(10))
    for bad in (0, 11):
        with pytest.raises(Exception, match="out of range"):
            port.partition(10, bad)


def test_k_subtrace_consistency(port):  # test_parallel.cpp:98-112
    t = read_trace(GOLD / "mix_3000_s4.trace").slice(0, 100)
    port.simulate(t, oracle=True, k=4, subtrace_size=25)
    port.simulate(t, oracle=True, k=4, subtrace_size=30)
    with pytest.raises(Exception, match="inconsistent partition: k=4 but subtrace size 50 implies k=2"):
        port.simulate(t, oracle=True, k=4, subtrace_size=50)
    assert len(port.simulate(t, oracle=True, k=0, subtrace_size=50)["subs"]) == 2


def test_k1_equals_sequential_and_additivity(port):  # test_parallel.cpp:65-96
    t = read_trace(GOLD / "mix_3000_s4.trace")
    seq = port.simulate(t, oracle=True, sequential=True)
    k1 = port.simulate(t, oracle=True, k=1)
    assert np.array_equal(seq["subs"], k1["subs"])
    assert np.array_equal(seq["predicted_fetch"], k1["predicted_fetch"])
    for k in (2, 3, 7):
        r = port.simulate(t, oracle=True, k=k)
        assert r["subs"][:, 1].sum() == r["total_cycles"] and r["subs"][:, 0].sum() == t.n
        assert np.all(r["subs"][:, 1] == r["subs"][:, 2] + r["subs"][:, 3])  # Eq. 1 identity
        assert np.all(r["subs"][:, 3] == r["subs"][:, 4] + r["subs"][:, 5])


def test_validation_messages(port):  # parallel.cpp:40, simcore.cpp:13-18
    t = read_trace(GOLD / "mix_3000_s4.trace").slice(0, 50)
    with pytest.raises(Exception, match="batch_max must be >= 1"):
        port.simulate(t, oracle=True, k=2, batch_max=0)
    with pytest.raises(Exception, match="retire_bandwidth must be >= 1"):
        port.simulate(t, oracle=True, retire_bandwidth=0)


# ---- decode goldens (test_cnn.cpp:183-224) ---------------------------------
def _decode(port, head_vals, is_store=False, norm=None):
    cfg = small_config()
    m = model_from_params(cfg, np.zeros(cfg.param_count(), np.float32), norm)
    y = np.zeros((1, 33), np.float32)
    for i, v in head_vals.items():
        y[0, i] = v
    return port.decode(m, y, np.array([is_store], np.uint8))[0]


def test_decode_goldens(port):
    assert _decode(port, {3 + 3: 2.0})[0] == 3  # argmax c3
    assert _decode(port, {3 + 9: 5.0, 0: np.float32(np.log1p(20.4))})[0] == 20  # overflow -> regression
    assert _decode(port, {3 + 9: 5.0, 0: -3.0})[0] == 0  # clamps at 0
    assert _decode(port, {3: 1.5, 4: 1.5})[0] == 0  # tie -> smaller class
    t = _decode(port, {13: 3.0, 23 + 7: 3.0})
    assert t[1] == 1 and t[2] == 0  # exec floor, store masked
    assert _decode(port, {13: 3.0, 23 + 7: 3.0}, is_store=True)[2] == 7
    norm = identity_norm()
    norm[100], norm[103] = 1.0, 0.5
    assert _decode(port, {12: 5.0, 0: np.float32((np.log1p(18.0) - 1.0) / 0.5)}, norm=norm)[0] == 18


# ---- forward pins (test_cnn.cpp:126-168) -----------------------------------
def naive_forward(cfg: CnnConfig, p: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Straight-line double-precision forward (the test_cnn.cpp:29-79 oracle)."""
    a = np.zeros(cfg.input_channels * cfg.sequence_length)
    a[: x.size] = x
    cin, off = cfg.input_channels, 0
    for cout in cfg.conv_channels:
        W = p[off: off + cout * 2 * cin].astype(np.float64).reshape(2 * cin, cout).T
        off += cout * 2 * cin
        b = p[off: off + cout].astype(np.float64)
        off += cout
        cols = a.reshape(-1, 2 * cin)
        a = np.maximum(cols @ W.T + b, 0).reshape(-1)
        cin = cout
    W1 = p[off: off + cfg.fc_hidden * cfg.flat_dim].astype(np.float64).reshape(cfg.flat_dim, cfg.fc_hidden).T
    off += cfg.fc_hidden * cfg.flat_dim
    h = np.maximum(W1 @ a + p[off: off + cfg.fc_hidden], 0)
    off += cfg.fc_hidden
    W2 = p[off: off + cfg.output_dim * cfg.fc_hidden].astype(np.float64).reshape(cfg.fc_hidden, cfg.output_dim).T
    off += cfg.output_dim * cfg.fc_hidden
    return W2 @ h + p[off: off + cfg.output_dim]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_forward_matches_naive_double(port, seed):  # test_cnn.cpp:155-168
    cfg = CnnConfig.preset_c3()
    m = model_from_params(cfg, port.init_params(cfg, seed))
    x = np.random.default_rng(seed + 100).uniform(-1.5, 1.5, (4, 5550)).astype(np.float32)
    y, _ = port.forward(m, x, np.zeros(4, np.uint8))
    for i in range(4):
        want = naive_forward(cfg, m.params, x[i])
        assert np.all(np.abs(y[i] - want) <= 1e-6 * np.maximum(1.0, np.abs(want)) * 50)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_forward_tiny_pin(port, seed):
    """The reference's own forward pin, verbatim (test_cnn.cpp:155-168):
    CnnConfig::tiny(5, 16) with conv {7, 9}, init_weights(cfg, NormStats{},
    seed), random_input(cfg, seed + 100) from the reference Rng, every output
    within 1e-6 relative of the straight-line double forward."""
    cfg = tiny_config(5, 16, conv=(7, 9))
    m = model_from_params(cfg, port.init_params(cfg, seed))
    x = random_input(cfg, seed + 100)
    y, _ = port.forward(m, x[None, :], np.zeros(1, np.uint8))
    want = naive_forward(cfg, m.params, x)
    assert y.shape[1] == want.size
    assert np.all(np.abs(y[0] - want) <= 1e-6 * np.maximum(1.0, np.abs(want)))


def test_init_weights_matches_reference_rule(port, golden):  # cnn.cpp:335-352
    g = golden["models"]["c3_mix_seed1"]
    cfg = CnnConfig.preset_c3()
    assert sha(port.init_params(cfg, g["seed"])) == g["params_sha256"]


# ---- golden.json replay (fixtures made by the reference, make_golden.py) ----
def test_golden_oracle_cases(port, golden):
    traces = {name: read_trace(GOLD / f"{name}.trace") for name in golden["traces"]}
    for c in golden["oracle"]:
        t = traces[c["trace"]]
        r = port.simulate(t, oracle=True, k=c["k"], subtrace_size=c["subtrace_size"], max_context=c["max_context"],
                          retire_bandwidth=c["retire_bandwidth"], per_cycle=c["per_cycle"], sequential=c["sequential"])
        assert r["subs"].tolist() == c["subs"], c
        assert sha(r["predicted_fetch"]) == c["predicted_fetch_sha256"], c


def _golden_models(port, golden):
    c3cfg = CnnConfig.preset_c3()
    g = golden["models"]["c3_mix_seed1"]
    return {
        "small_identity": read_model(GOLD / "small_identity.model"),
        "small_dataset": read_model(GOLD / "small_dataset.model"),
        "c3_mix_seed1": Model(c3cfg, np.array(g["norm"]), port.init_params(c3cfg, g["seed"])),
    }


def test_golden_cnn_cases(port, golden):
    models = _golden_models(port, golden)
    for c in golden["cnn"]:
        t = read_trace(GOLD / f"{c['trace']}.trace")
        m = models[c["model"]]
        if "capture" in c:
            r = port.simulate(t, m, k=c["k"], capture=c["capture"], capture_inputs=True)
            assert sha(r["cap_inputs"]) == c["inputs_sha256"], c["model"]
            assert sha(r["cap_triples"]) == c["triples_sha256"], c["model"]
            continue
        r = port.simulate(t, m, k=c["k"], sequential=c["sequential"])
        assert r["subs"].tolist() == c["subs"], (c["model"], c["trace"], c["k"])
        assert sha(r["predicted_fetch"]) == c["predicted_fetch_sha256"]


# ---- port vs the reference library on fresh inputs ---------------------------
@pytest.mark.parametrize("kind,n,seed", [("mix", 4000, 11), ("streaming", 3000, 12), ("pointer-chase", 3000, 13),
                                         ("loop-kernel", 3000, 14), ("branchy", 3000, 15)])
def test_port_equals_reference(ref, port, tmp_path, kind, n, seed):
    path = tmp_path / "t.trace"
    des_total = ref.make_trace(kind, n, seed, path)
    t = read_trace(path)
    seq = port.simulate(t, oracle=True, sequential=True)
    # oracle vs DES (test_simcore.cpp:190-205): <= 0.5%
    assert abs(seq["total_cycles"] - des_total) <= 0.005 * des_total
    for k in (1, 3, 17, 256):
        a = port.simulate(t, oracle=True, k=k)
        b = ref.simulate(path, None, k=k, n_hint=n)
        assert np.array_equal(a["subs"], b["subs"]) and np.array_equal(a["predicted_fetch"], b["predicted_fetch"][:n])
    mpath = tmp_path / "m.model"
    ref.make_model(path, mpath, conv=(16, 16, 16), fc_hidden=32, seed=seed)
    m = read_model(mpath)
    for k in (1, 9):
        a = port.simulate(t, m, k=k)
        b = ref.simulate(path, mpath, k=k, n_hint=n)
        assert np.array_equal(a["subs"], b["subs"]) and np.array_equal(a["predicted_fetch"], b["predicted_fetch"][:n])
    ca = port.simulate(t, m, k=9, capture=300, capture_inputs=True)
    cb = ref.capture(path, mpath, 300, k=9)
    assert np.array_equal(ca["cap_inputs"], cb["inputs"]) and np.array_equal(ca["cap_triples"], cb["triples"])


def test_port_forward_equals_reference(ref, port, tmp_path):
    path = GOLD / "mix_3000_s4.trace"
    mpath = tmp_path / "c3.model"
    ref.make_model(path, mpath, seed=5)
    cap = ref.capture(path, mpath, 64, k=4)
    m = read_model(mpath)
    a_out, a_tri = port.forward(m, cap["inputs"], cap["is_store"])
    b_out, b_tri = ref.forward(mpath, cap["inputs"], cap["is_store"])
    assert np.array_equal(a_out, b_out) and np.array_equal(a_tri, b_tri)


def test_extensions_defaults_and_identities(port):
    """warm-up / drain-trim have no reference; check their definitions."""
    t = random_trace(5, 3000)
    base = port.simulate(t, oracle=True, k=6)
    same = port.simulate(t, oracle=True, k=6, warmup=0, drain_trim=False)
    assert np.array_equal(base["subs"], same["subs"])
    for w in (50, 500):
        r = port.simulate(t, oracle=True, k=6, warmup=w)
        s = r["subs"]
        assert s[:, 0].sum() == t.n
        assert np.all(s[:, 1] == s[:, 2] + s[:, 3]) and np.all(s[:, 3] == s[:, 4] + s[:, 5])
        assert r["subs"][0].tolist() == base["subs"][0].tolist()  # the first sub-trace has no history
        assert np.array_equal(r["predicted_fetch"], base["predicted_fetch"])  # truth latencies
    r = port.simulate(t, oracle=True, k=6, drain_trim=True)
    assert np.all(r["subs"][:-1, 4] == 0) and r["subs"][-1].tolist() == base["subs"][-1].tolist()


def test_trained_model_fixture(ref, port, tmp_path):
    """The trained C3 the benches can load (tests/golden/train_c3.py): a C3 in
    the reference's ILMD layout, its training report, and the port and the
    reference library agreeing bit for bit on its forward and on a free-running
    simulation."""
    import json

    mpath = GOLD / "c3_trained.model"
    m = read_model(mpath)
    c3 = CnnConfig.preset_c3()
    assert m.config.hash() == c3.hash() and m.params.size == c3.param_count()
    assert np.all(np.isfinite(m.params))
    rep = json.loads((GOLD / "c3_trained.json").read_text())
    assert set(rep["held_out"]) == {f"{k}_held" for k in rep["kinds"]} and rep["selected_epoch"] >= 0
    path = GOLD / "mix_3000_s4.trace"
    cap = ref.capture(path, mpath, 64, k=4)
    a_out, a_tri = port.forward(m, cap["inputs"], cap["is_store"])
    b_out, b_tri = ref.forward(mpath, cap["inputs"], cap["is_store"])
    assert np.array_equal(a_out, b_out) and np.array_equal(a_tri, b_tri)
    t = read_trace(path)
    a = port.simulate(t, m, k=9)
    b = ref.simulate(path, mpath, k=9, n_hint=t.n)
    assert np.array_equal(a["subs"], b["subs"]) and np.array_equal(a["predicted_fetch"], b["predicted_fetch"][:t.n])
