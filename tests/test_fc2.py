"""FC-only latency predictor (the paper's FC2; BASELINE config
c1).  The reference has no implementation (cnn.cpp:245 rejects zero conv
layers), so this is an extension defined identically in the oracle port and on
the GPU; parity is unpinned against the reference and pinned here against a
direct numpy statement of the two layers."""
import numpy as np
import pytest

from helpers import SUB, gpu_subs, random_trace
from paper_2105_05821_b200 import IlsimError, ParallelConfig, SimConfig, init_weights
from paper_2105_05821_b200.api import model_flops
from paper_2105_05821_b200.formats import CnnConfig, Model, identity_norm, read_model, write_model


def fc_config(mc=7, hidden=32):
    c = CnnConfig.preset_fc2(mc, hidden)
    return c


def test_fc2_preset_shape():
    c = CnnConfig.preset_fc2()
    assert c.flat_dim == 5550 and c.fc_hidden == 1024 and c.output_dim == 33
    assert c.param_count() == 5550 * 1024 + 1024 + 33 * 1024 + 33
    assert c.model_flops() == 5_716_992 == model_flops("fc2")  # 5.7 M mults


def test_fc2_forward_matches_numpy(port):
    cfg = fc_config()
    rng = np.random.default_rng(3)
    m = Model(cfg, identity_norm(), port.init_params(cfg, 5))
    width = cfg.flat_dim
    x = rng.normal(size=(40, width)).astype(np.float32)
    y, _ = port.forward(m, x, np.zeros(40, np.uint8))
    p = m.params.astype(np.float64)
    h, od = cfg.fc_hidden, cfg.output_dim
    w1 = p[: h * width].reshape(width, h).T  # column-major W[o + k*rows]
    b1 = p[h * width: h * width + h]
    off = h * width + h
    w2 = p[off: off + od * h].reshape(h, od).T
    b2 = p[off + od * h: off + od * h + od]
    want = (w2 @ np.maximum(w1 @ x.T.astype(np.float64) + b1[:, None], 0.0) + b2[:, None]).T
    assert np.max(np.abs(y - want) / np.maximum(1.0, np.abs(want))) < 1e-5


def test_fc2_model_file_roundtrip(tmp_path, port):
    cfg = fc_config()
    m = Model(cfg, identity_norm(), port.init_params(cfg, 9))
    write_model(tmp_path / "fc.model", m)
    r = read_model(tmp_path / "fc.model")
    assert r.config == cfg and np.array_equal(r.params, m.params)


def test_fc2_port_simulates(port):
    cfg = fc_config()
    m = Model(cfg, identity_norm(), port.init_params(cfg, 5))
    t = random_trace(4, 600)
    r = port.simulate(t, m, k=3)
    assert int(np.asarray(r["subs"])[:, SUB.index("instructions")].sum()) == 600
    assert r["total_cycles"] > 0


@pytest.mark.gpu
def test_fc2_gpu_matches_port(gpu, port):
    g = gpu("fp32")
    cfg = fc_config()
    m = Model(cfg, identity_norm(), port.init_params(cfg, 5))
    g.load_model(m)
    t = random_trace(4, 3000)
    want = port.simulate(t, m, k=16, capture=800, capture_inputs=True, capture_outputs=True)
    out, tri = g.predict(want["cap_inputs"], want["cap_is_store"])
    assert np.max(np.abs(out - want["cap_outputs"]) / np.maximum(1.0, np.abs(want["cap_outputs"]))) <= 2e-5
    pc = ParallelConfig(k=16, sim=SimConfig(max_context=cfg.max_context))
    g.load_trace(t, pc)
    r = g.run(pc)
    full = port.simulate(t, m, k=16)
    assert abs(r.total_cycles - full["total_cycles"]) <= 1e-3 * full["total_cycles"]
    assert np.mean(r.predicted_fetch == full["predicted_fetch"]) >= 0.999


@pytest.mark.gpu
def test_fc2_tensor_core_precision_rejected(gpu, port):
    g = gpu("tf32x3")
    cfg = fc_config()
    with pytest.raises(IlsimError, match="FC-only"):
        g.load_model(Model(cfg, identity_norm(), port.init_params(cfg, 5)))


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 2])
def test_fc2_persistent_kernel(gpu, port, k, monkeypatch):
    """K <= 2 with the paper-size FC2 (5550 -> 1024 -> 33, config c1's shape):
    the whole simulation is one persistent cooperative launch (seq_fc.cu), bit
    for bit the launch-per-layer rounds (SIMNET_NO_SEQ_FC), and the sequential
    run matches the oracle port's simulate_trace semantics."""
    g = gpu("fp32")
    cfg = CnnConfig.preset_fc2()
    m = Model(cfg, identity_norm(), port.init_params(cfg, 5))
    g.load_model(m)
    t = random_trace(6, 2501)  # K = 2: sub-traces of 1251 and 1250 (one finishes a round early)
    pc = ParallelConfig(k=k, sim=SimConfig(max_context=cfg.max_context))
    g.load_trace(t, pc)
    monkeypatch.delenv("SIMNET_NO_SEQ_FC", raising=False)
    a = g.run(pc)
    assert a.launches == 1  # the persistent kernel ran
    monkeypatch.setenv("SIMNET_NO_SEQ_FC", "1")
    b = g.run(pc)
    assert b.launches > 1000
    assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch)
    want = port.simulate(t, m, k=k)
    assert abs(a.total_cycles - want["total_cycles"]) <= 1e-3 * want["total_cycles"]
    assert np.mean(a.predicted_fetch == want["predicted_fetch"]) >= 0.999
