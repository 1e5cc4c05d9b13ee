"""CUDA path (through the C-ABI) vs the CPU oracle port and the reference
goldens.  Integer work (queues, clocks, gathered inputs) must be bit-exact;
the fp32 CNN is checked teacher-forced (per-instruction triples equal except
at documented near-ties) and free-running (total cycles within 0.1%)."""
import hashlib

import numpy as np
import pytest

from helpers import SUB, gpu_subs, instr_trace, random_trace, small_config
from paper_2105_05821_b200 import IlsimError, ParallelConfig, SimConfig, init_weights
from paper_2105_05821_b200.formats import CnnConfig, Model, read_model, read_trace

pytestmark = pytest.mark.gpu
GOLD = __import__("conftest").GOLDEN


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def pcfg(k=1, subtrace_size=0, batch_max=4096, mc=110, bw=8, per_cycle=False, warmup=0, drain_trim=False,
         write_ring=0):
    return ParallelConfig(k=k, subtrace_size=subtrace_size, batch_max=batch_max,
                          sim=SimConfig(max_context=mc, retire_bandwidth=bw, per_cycle_advance=per_cycle),
                          warmup=warmup, drain_trim=drain_trim, write_ring=write_ring)


def run_gpu(g, t, pc, *, oracle=True, sequential=False, shard=None):
    g.load_trace(t, pc, sequential=sequential, oracle=oracle, shard=shard)
    return g.run(pc, sequential=sequential, oracle=oracle, shard=shard)


# ---- scripted goldens (test_simcore.cpp:63-174) on the GPU -------------------
def test_scripted_goldens(gpu):
    g = gpu("fp32")
    r = g.simulate_trace(instr_trace([False], [(5, 2, 0)]), oracle=True)
    assert (r.sum_fetch, r.total_cycles, r.delta) == (5, 7, 2)
    r = g.simulate_trace(instr_trace([False] * 3, [(5, 2, 0), (0, 3, 0), (1, 3, 0)]), oracle=True)
    assert (r.sum_fetch, r.drain_cycles, r.delta, r.total_cycles) == (6, 3, 3, 9)
    for k, b, want in [(5, 2, 3), (8, 8, 1), (9, 8, 2), (16, 4, 4), (1, 3, 1)]:
        r = g.simulate_trace(instr_trace([False] * k, [(0, 0, 0)] * k), SimConfig(retire_bandwidth=b), oracle=True)
        assert r.drain_cycles == want
    r = g.simulate_trace(instr_trace([False], [(0, 4, 0)]), oracle=True)
    assert r.drain_cycles == 4
    r = g.simulate_trace(instr_trace([True, False], [(1, 2, 6), (0, 1, 0)]), oracle=True)
    assert (r.total_cycles, r.sum_fetch, r.delta) == (7, 1, 6)
    r = g.simulate_trace(instr_trace([False] * 6, [(0, 100, 0)] * 6), SimConfig(max_context=4), oracle=True)
    assert r.overflow_stall_cycles == 100
    r = g.simulate_trace(instr_trace([], []), oracle=True)
    assert r.empty and r.total_cycles == 0 and r.cpi == 0.0


# ---- golden.json oracle cases (made by the reference) -------------------------
def test_golden_oracle_cases(gpu, golden):
    g = gpu("fp32")
    traces = {name: read_trace(GOLD / f"{name}.trace") for name in golden["traces"]}
    for c in golden["oracle"]:
        t = traces[c["trace"]]
        pc = pcfg(c["k"], c["subtrace_size"], mc=c["max_context"], bw=c["retire_bandwidth"], per_cycle=c["per_cycle"])
        r = run_gpu(g, t, pc, sequential=c["sequential"])
        assert gpu_subs(r).tolist() == c["subs"], c
        assert sha(r.predicted_fetch) == c["predicted_fetch_sha256"], c


# ---- random traces / configurations vs the port (bit-exact) -------------------
def store_heavy(seed, n, lat_hi=1500):
    """Memory-heavy trace with scripted store-heavy truth latencies (the c4
    regime of SURVEY.md §6: long queues, frequent retire)."""
    t = random_trace(seed, n)
    rng = np.random.default_rng(seed + 1)
    st = rng.random(n) < 0.25
    t.op[:, 0] = np.where(st, 8, t.op[:, 0])
    t.op[:, 2] = st
    t.op[:, 1] = np.where(st, 0, t.op[:, 1])
    mem = (t.op[:, 1] | t.op[:, 2]) != 0
    t.has_data = mem.astype(np.uint8)
    t.data_addr = np.where(mem, 0x10000000 + rng.integers(0, 1 << 16, n) * 8, 0).astype(np.uint64)
    t.truth[:, 0] = np.where(rng.random(n) < 0.5, 0, rng.integers(1, 4, n))
    t.truth[:, 1] = rng.integers(1, 41, n)
    t.truth[:, 2] = np.where(st, rng.integers(100, lat_hi, n), 0)
    return t


CASES = [
    dict(k=1), dict(k=4), dict(k=33), dict(k=128), dict(k=7, mc=16, bw=2), dict(k=5, mc=4, bw=1),
    dict(k=9, mc=64, bw=3, per_cycle=True), dict(k=6, warmup=40), dict(k=6, warmup=300, drain_trim=True),
    dict(k=12, drain_trim=True), dict(k=0, subtrace_size=97), dict(k=3, mc=200),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_oracle_mode_vs_port(gpu, port, case):
    g = gpu("fp32")
    c = dict(CASES[case])
    for t in (random_trace(100 + case, 2500), store_heavy(200 + case, 2500)):
        pc = pcfg(**c)
        r = run_gpu(g, t, pc)
        want = port.simulate(t, oracle=True, k=pc.k, subtrace_size=pc.subtrace_size, max_context=pc.sim.max_context,
                             retire_bandwidth=pc.sim.retire_bandwidth, per_cycle=pc.sim.per_cycle_advance,
                             warmup=pc.warmup, drain_trim=pc.drain_trim)
        assert np.array_equal(gpu_subs(r), want["subs"]), c
        assert np.array_equal(r.predicted_fetch, want["predicted_fetch"]), c


def test_sequential_equals_k1_and_shards_compose(gpu, port):
    g = gpu("fp32")
    t = store_heavy(7, 4000)
    seq = run_gpu(g, t, pcfg(1), sequential=True)
    k1 = run_gpu(g, t, pcfg(1))
    assert np.array_equal(gpu_subs(seq), gpu_subs(k1))
    full = run_gpu(g, t, pcfg(7, warmup=100))
    parts = [run_gpu(g, t, pcfg(7, warmup=100), shard=s) for s in ((0, 3), (3, 5), (5, 7))]
    assert np.array_equal(np.concatenate([gpu_subs(p) for p in parts]), gpu_subs(full))
    assert np.array_equal(np.concatenate([p.predicted_fetch for p in parts]), full.predicted_fetch)


def test_write_ring_grows_on_auto(gpu, port):
    """The reference's write queue is an unbounded deque: with write_ring on
    auto (0) a queue longer than the default 2048-entry ring reruns with a
    larger ring and matches the port bit-exactly; an explicit write_ring is
    a hard bound (reported overflow)."""
    g = gpu("fp32")
    t = store_heavy(5, 12000, lat_hi=400)
    first = int(np.flatnonzero(t.op[:, 2])[0])
    t.truth[first, 2] = 50_000_000  # the head store blocks the in-order write queue
    assert int(t.op[:, 2].sum()) > 2048
    r = run_gpu(g, t, pcfg(1))
    want = port.simulate(t, oracle=True, k=1)
    assert gpu_subs(r).tolist() == want["subs"].tolist()
    assert np.array_equal(r.predicted_fetch, want["predicted_fetch"])
    with pytest.raises(IlsimError, match="write queue ring overflow"):
        run_gpu(g, t, pcfg(1, write_ring=2048))


def test_errors_and_validation(gpu):
    g = gpu("fp32")
    t = store_heavy(9, 3000, lat_hi=100000)
    with pytest.raises(IlsimError, match="write queue ring overflow"):
        run_gpu(g, t, pcfg(2, write_ring=4))
    with pytest.raises(IlsimError, match="batch_max must be >= 1"):
        run_gpu(g, t, pcfg(2, batch_max=0))
    with pytest.raises(IlsimError, match="inconsistent partition: k=4 but subtrace size 1000 implies k=3"):
        run_gpu(g, t, pcfg(4, subtrace_size=1000))
    with pytest.raises(IlsimError, match="retire_bandwidth must be >= 1"):
        run_gpu(g, t, pcfg(2, bw=0))
    with pytest.raises(IlsimError, match="out of range"):
        run_gpu(g, t.slice(0, 5), pcfg(6))
    g2 = gpu("fp32")
    t2 = random_trace(1, 100)
    r = run_gpu(g2, t2, pcfg(3))  # the context is still usable after an error
    assert r.instructions == 100


# ---- gathered input tensor: bit-exact vs the reference's next_request ----------
def c3_model(port, golden) -> Model:
    gm = golden["models"]["c3_mix_seed1"]
    cfg = CnnConfig.preset_c3()
    return Model(cfg, np.array(gm["norm"]), port.init_params(cfg, gm["seed"]))


@pytest.mark.parametrize("trace_name,k", [("mix_3000_s4", 5), ("pointer_chase_2000_s3", 16)])
def test_input_tensor_bit_exact(gpu, port, golden, trace_name, k):
    g = gpu("fp32")
    m = c3_model(port, golden)
    g.load_model(m)
    t = read_trace(GOLD / f"{trace_name}.trace")
    want = port.simulate(t, m, k=k, truth_with_inputs=True, capture=t.n, capture_inputs=True)
    rounds = want["cap_round"]
    for r in (0, 1, 7, 50, int(rounds.max())):
        rows = np.nonzero(rounds == r)[0]
        buf = g.capture_round(r, k)
        pc = pcfg(k)
        g.load_trace(t, pc, oracle=True)
        g.run(pc, truth_inputs=True)
        g.clear_capture()
        assert np.array_equal(buf[: rows.size], want["cap_inputs"][rows]), f"round {r}"


def test_input_tensor_store_heavy(gpu, port, golden):
    """Long queues (write queue > 110 entries): truncation + newest-first order."""
    g = gpu("fp32")
    m = c3_model(port, golden)
    g.load_model(m)
    t = store_heavy(31, 1500)
    k = 3
    want = port.simulate(t, m, k=k, truth_with_inputs=True, capture=t.n, capture_inputs=True)
    for r in (10, 200, 480):
        rows = np.nonzero(want["cap_round"] == r)[0]
        buf = g.capture_round(r, k)
        pc = pcfg(k)
        g.load_trace(t, pc, oracle=True)
        g.run(pc, truth_inputs=True)
        g.clear_capture()
        assert np.array_equal(buf[: rows.size], want["cap_inputs"][rows]), f"round {r}"


# ---- CNN: teacher-forced and free-running ------------------------------------
def tie_explained(y_ref, y_gpu, tri_ref, tri_gpu, cfg, norm):
    """Why a decoded triple differs, or None when the difference is NOT
    explained by the two forwards' output difference.  Absolute criteria
    (no tolerance relative to the decoded value):
      * a class flip needs the reference's top-2 logit gap to be at most
        twice that head's largest |y_gpu - y_ref| (each logit moved by at
        most that much, so only then can their order swap);
      * a regression-path flip (both in the overflow class) must be to the
        neighbouring integer, with the reference's de-normalised value within
        sigma * (v + 1) * |dr| (1st-order expm1 propagation of the actual
        regression output difference dr, x1.01) of the .5 rounding boundary.
    Returns the gap that excused it (logit gap or distance to .5)."""
    heads = [(3, cfg.class_fetch, 0), (3 + cfg.class_fetch, cfg.class_exec, 1),
             (3 + cfg.class_fetch + cfg.class_exec, cfg.class_store, 2)]
    gaps = []
    for h, (base, n, j) in enumerate(heads):
        if tri_ref[h] == tri_gpu[h]:
            continue
        lr = y_ref[base: base + n].astype(np.float64)
        lg = y_gpu[base: base + n].astype(np.float64)
        cls_r, cls_g = int(np.argmax(lr)), int(np.argmax(lg))
        if cls_r != cls_g:
            top = np.sort(lr)
            err = float(np.max(np.abs(lg - lr)))
            if top[-1] - top[-2] <= 2.0 * err:
                gaps.append(("logit", top[-1] - top[-2], err))
                continue
            return None
        # both overflow class: regression rounding
        sd, mu = norm[103 + j], norm[100 + j]
        v = max(0.0, float(np.expm1(min(float(y_ref[j]) * sd + mu, 22.0))))
        dr = abs(float(y_gpu[j]) - float(y_ref[j]))
        dist = abs(v - np.floor(v) - 0.5)
        if abs(int(tri_ref[h]) - int(tri_gpu[h])) == 1 and dist <= 1.01 * sd * (v + 1.0) * dr:
            gaps.append(("regression", dist, dr))
            continue
        return None
    return gaps


@pytest.mark.parametrize("precision,rtol,exact", [("fp32", 2e-5, True), ("tf32x3", 1e-4, True),
                                                  ("tf32", 3e-2, False), ("bf16", 1.5e-1, False)])
def test_teacher_forced_predict(gpu, port, golden, precision, rtol, exact):
    g = gpu(precision)
    m = c3_model(port, golden)
    g.load_model(m)
    t = read_trace(GOLD / "mix_3000_s4.trace")
    want = port.simulate(t, m, k=16, capture=1200, capture_inputs=True, capture_outputs=True)
    out, tri = g.predict(want["cap_inputs"], want["cap_is_store"])
    ref = want["cap_outputs"]
    err = np.abs(out - ref) / np.maximum(1.0, np.abs(ref))
    assert err.max() <= rtol, err.max()
    bad = [i for i in range(tri.shape[0]) if not np.array_equal(tri[i], want["cap_triples"][i])]
    # the device decode of the device outputs must itself be the reference decode
    assert np.array_equal(port.decode(m, out, want["cap_is_store"]), tri)
    if exact:
        excused = []
        for i in bad:
            why = tie_explained(ref[i], out[i], want["cap_triples"][i], tri[i], m.config, m.norm)
            assert why is not None, (i, ref[i], out[i], want["cap_triples"][i], tri[i])
            excused.append((i, why))
        print(f"{precision}: {len(excused)} of {tri.shape[0]} triples differ, all explained: {excused}")
        assert len(excused) <= 0.01 * tri.shape[0], excused
    else:  # reduced precision: decode agreement is reported, not required exact
        assert len(bad) <= 0.05 * tri.shape[0], len(bad)


@pytest.mark.parametrize("precision", ["fp32", "tf32x3"])
def test_free_running_cnn(gpu, port, golden, precision):
    g = gpu(precision)
    models = {"small_identity": read_model(GOLD / "small_identity.model"),
              "small_dataset": read_model(GOLD / "small_dataset.model"), "c3": c3_model(port, golden)}
    for name, m in models.items():
        g.load_model(m)
        for tname, k in (("mix_3000_s4", 5), ("branchy_2000_s8", 16), ("pointer_chase_2000_s3", 1)):
            t = read_trace(GOLD / f"{tname}.trace")
            pc = pcfg(k)
            r = run_gpu(g, t, pc, oracle=False)
            want = port.simulate(t, m, k=k)
            tot, wtot = r.total_cycles, want["total_cycles"]
            assert abs(tot - wtot) <= 1e-3 * wtot, (name, tname, tot, wtot)
            same = np.mean(r.predicted_fetch == want["predicted_fetch"])
            assert same >= 0.999, (name, tname, same)


def test_batch_and_chunk_invariance(gpu):
    """Per-request results must not depend on batch composition
    (predictor.hpp:25-26, test_parallel.cpp:114-146)."""
    g = gpu("fp32")
    cfg = small_config()
    g.load_model(init_weights(cfg, np.r_[np.zeros(50), np.ones(50), np.zeros(3), np.ones(3)], 33))
    t = random_trace(3, 4000)
    a = run_gpu(g, t, pcfg(5), oracle=False)
    b = run_gpu(g, t, pcfg(5, batch_max=2), oracle=False)
    assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch)


@pytest.mark.parametrize("precision", ["tf32x3", "bf16"])
def test_tensor_core_batch_tail_and_small_model(gpu, port, precision):
    """Ragged batches (samples not a multiple of the 128-row tile) and the
    16/16/16 model (one K chunk per conv) through the tcgen05 kernels."""
    g = gpu(precision)
    m = read_model(GOLD / "small_dataset.model")
    g.load_model(m)
    t = read_trace(GOLD / "branchy_2000_s8.trace")
    for k in (1, 3, 130):
        want = port.simulate(t, m, k=k, capture=min(t.n, 700), capture_inputs=True, capture_outputs=True)
        out, _ = g.predict(want["cap_inputs"], want["cap_is_store"])
        err = np.abs(out - want["cap_outputs"]) / np.maximum(1.0, np.abs(want["cap_outputs"]))
        assert err.max() <= (1e-4 if precision == "tf32x3" else 1.5e-1), (k, err.max())


# ---- fused round front (K1 + conv chain in one kernel) -----------------------
def _fused_cases(port, golden):
    m = c3_model(port, golden)
    return m, [(read_trace(GOLD / "mix_3000_s4.trace"), 5), (read_trace(GOLD / "branchy_2000_s8.trace"), 130),
               (store_heavy(31, 1500), 3), (read_trace(GOLD / "pointer_chase_2000_s3.trace"), 1)]


def _bench_like(regime="default", n=24_000):
    """The bench's synthetic workload shape at test size: head biases put many
    decodes on the overflow class (fp64 regression path) and contexts are long."""
    from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace
    kind = "memory" if regime == "memory" else "mix"
    return synthetic_model(synthetic_trace(20_000, 101, kind=kind), 1, regime=regime), synthetic_trace(n, 7, kind=kind)


@pytest.mark.parametrize("precision", ["tf32x3", "bf16"])
@pytest.mark.parametrize("regime", ["default", "memory"])
def test_fused_front_bench_workload(gpu, port, precision, regime):
    """Fused vs unfused bit-exact, and total cycles vs the CPU oracle, on the
    bench's own synthetic workload (frequent regression decodes, full contexts)."""
    g = gpu(precision)
    m, t = _bench_like(regime)
    g.load_model(m)
    pc = pcfg(64)
    g.load_trace(t, pc)
    a = g.run(pc)
    b = g.run(pc, fused=False)
    assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch)
    if precision == "tf32x3":
        want = port.simulate(t, m, k=64)
        assert abs(a.total_cycles - want["total_cycles"]) <= 1e-3 * want["total_cycles"]
        assert np.mean(a.predicted_fetch == want["predicted_fetch"]) >= 0.999


@pytest.mark.parametrize("precision", ["tf32x3", "bf16", "tf32"])
def test_fused_front_matches_unfused(gpu, port, golden, precision):
    """The fused round front (gather straight into the conv0 operand, skipped
    all-zero tiles) must reproduce the unfused tensor-core round bit for bit:
    every accumulator row depends only on its own input row."""
    g = gpu(precision)
    m, cases = _fused_cases(port, golden)
    g.load_model(m)
    for t, k in cases:
        pc = pcfg(k)
        g.load_trace(t, pc)
        a = g.run(pc, fused=True)
        b = g.run(pc, fused=False)
        assert np.array_equal(gpu_subs(a), gpu_subs(b)), (t.n, k)
        assert np.array_equal(a.predicted_fetch, b.predicted_fetch), (t.n, k)


@pytest.mark.parametrize("precision,geom", [("tf32x3", (64, 4096)), ("bf16", (64, 4096)), ("tf32x3", (48, 3000))])
def test_fused_front_inputs_bit_exact(gpu, port, golden, precision, geom):
    """Inputs gathered by the fused kernel (captured from its shared-memory
    operand as exact f32) equal the reference's next_request tensors for every
    round up to the first decode divergence from the CPU oracle.  geom: line /
    page size of the dependency flags (dataset.cpp:48-58); 48 / 3000 takes the
    division path, powers of two the shift path."""
    g = gpu(precision)
    m = c3_model(port, golden)
    g.load_model(m)
    line, page = geom
    for t, k in ((read_trace(GOLD / "mix_3000_s4.trace"), 5), (store_heavy(31, 1500), 3)):
        pc = pcfg(k)
        pc.sim.line_size, pc.sim.page_size = line, page
        g.load_trace(t, pc)
        got = g.run(pc)
        want = port.simulate(t, m, k=k, capture=t.n, capture_inputs=True, line_size=line, page_size=page)
        # rounds before the first differing fetch latency see identical queues
        diff = np.nonzero(got.predicted_fetch != want["predicted_fetch"])[0]
        idx = want["cap_index"]
        rounds = want["cap_round"]
        first_bad = int(rounds[np.isin(idx, diff)].min()) if diff.size else int(rounds.max()) + 1
        checked = 0
        for r in (0, 1, 7, 50, 200, 480, int(rounds.max())):
            if r >= first_bad:
                continue
            rows = np.nonzero(rounds == r)[0]
            buf = g.capture_round(r, k)
            g.run(pc)
            g.clear_capture()
            assert np.array_equal(buf[: rows.size], want["cap_inputs"][rows]), f"round {r}"
            checked += 1
        assert checked >= 2, (first_bad, precision)


@pytest.mark.parametrize("precision", ["tf32x3", "bf16"])
def test_fc1_tma_store_matches_direct_store(gpu, port, golden, precision, monkeypatch):
    """FC1's split-K partials and the front's flat output, staged in shared
    memory and TMA-stored, equal the per-thread direct stores bit for bit,
    including a partial last M tile / item (rows clipped by the tensor map);
    FC1 with A in tensor memory (3xTF32) equals A read from shared memory."""
    g = gpu(precision)
    m, _ = _fused_cases(port, golden)
    g.load_model(m)
    t = read_trace(GOLD / "branchy_2000_s8.trace")
    for k in (130, 300):
        pc = pcfg(k)
        g.load_trace(t, pc)
        toggles = ("SIMNET_FC1_DIRECT_STORE", "SIMNET_FLAT_DIRECT_STORE", "SIMNET_FC1_SS")
        for v in toggles:
            monkeypatch.delenv(v, raising=False)
        a = g.run(pc)
        for v in toggles:
            monkeypatch.setenv(v, "1")
        b = g.run(pc)
        assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch), k


@pytest.mark.parametrize("precision", ["tf32x3", "bf16"])
def test_fc1_tmem_a_multi_tile(gpu, port, precision, monkeypatch):
    """FC1 CTAs looping over several M tiles (K > 9 x 128 sub-traces) take A
    from tensor memory (3xTF32) and TMA-store their partial tiles through two
    staging buffers; results equal A read from shared memory and per-thread
    row stores, bit for bit (1500 sub-traces: CTAs with one and with two M
    tiles, a partial last tile clipped by the tensor map), and stay within
    0.1% of the CPU oracle."""
    g = gpu(precision)
    m, t = _bench_like("default", n=24_000)
    g.load_model(m)
    pc = pcfg(1500)
    g.load_trace(t, pc)
    toggles = ("SIMNET_FC1_SS", "SIMNET_FC1_MULTI_DIRECT")
    for v in toggles:
        monkeypatch.delenv(v, raising=False)
    a = g.run(pc)
    for v in toggles:
        monkeypatch.setenv(v, "1")
        b = g.run(pc)
        assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch), v
    if precision == "tf32x3":
        want = port.simulate(t, m, k=1500)
        assert abs(a.total_cycles - want["total_cycles"]) <= 1e-3 * want["total_cycles"]


@pytest.mark.parametrize("precision", ["tf32x3", "bf16"])
def test_chunked_rounds_match(gpu, port, golden, precision, monkeypatch):
    """Batches larger than one chunk (65536 sub-traces in production; 24 here)
    run chunk after chunk each round; results must not change."""
    g = gpu(precision)
    m, _ = _fused_cases(port, golden)
    g.load_model(m)
    t = read_trace(GOLD / "branchy_2000_s8.trace")
    pc = pcfg(100)
    g.load_trace(t, pc)
    a = g.run(pc)
    monkeypatch.setenv("SIMNET_CHUNK", "24")
    for fused in (True, False):
        b = g.run(pc, fused=fused)
        assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch)


@pytest.mark.parametrize("precision", ["fp32", "tf32x3", "bf16"])
def test_residual_c3(gpu, port, golden, precision):
    """c3-rb (residual blocks, cnn.cpp:54-57, 104-107): the SIMT path computes
    W in + P in, the tensor-core path folds P into W; both against the port."""
    g = gpu(precision)
    cfg = CnnConfig.preset_c3()
    cfg.residual_blocks = True
    gm = golden["models"]["c3_mix_seed1"]
    m = Model(cfg, np.array(gm["norm"]), port.init_params(cfg, 3))
    g.load_model(m)
    t = read_trace(GOLD / "mix_3000_s4.trace")
    want = port.simulate(t, m, k=16, capture=600, capture_inputs=True, capture_outputs=True)
    out, tri = g.predict(want["cap_inputs"], want["cap_is_store"])
    err = np.abs(out - want["cap_outputs"]) / np.maximum(1.0, np.abs(want["cap_outputs"]))
    assert err.max() <= {"fp32": 2e-5, "tf32x3": 1e-4, "bf16": 1.5e-1}[precision], err.max()
    if precision != "bf16":
        pc = pcfg(16)
        r = run_gpu(g, t, pc, oracle=False)
        full = port.simulate(t, m, k=16)
        assert abs(r.total_cycles - full["total_cycles"]) <= 1e-3 * full["total_cycles"]
        assert np.mean(r.predicted_fetch == full["predicted_fetch"]) >= 0.999


@pytest.mark.parametrize("extra", [dict(warmup=40), dict(warmup=300, drain_trim=True), dict(drain_trim=True),
                                   dict(bw=3), dict(mc=110, per_cycle=True)])
def test_fused_round_extensions_and_options(gpu, port, extra):
    """Warm-up overlap, drain-trim, retire bandwidth and per-cycle advance
    through the fused tensor-core round: bit-identical to the unfused round and
    within 0.1% of the CPU oracle."""
    g = gpu("tf32x3")
    m, t = _bench_like("default", n=12_000)
    g.load_model(m)
    pc = pcfg(48, **extra)
    g.load_trace(t, pc)
    a = g.run(pc)
    b = g.run(pc, fused=False)
    assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch)
    want = port.simulate(t, m, k=48, retire_bandwidth=pc.sim.retire_bandwidth,
                         per_cycle=pc.sim.per_cycle_advance, warmup=pc.warmup, drain_trim=pc.drain_trim)
    assert abs(a.total_cycles - want["total_cycles"]) <= 1e-3 * want["total_cycles"]


def test_sharded_fused_rounds_compose(gpu, port):
    """Shards (the multi-GPU partition) through the fused round reproduce the
    single-device run sub-trace for sub-trace."""
    g = gpu("tf32x3")
    m, t = _bench_like("default", n=12_000)
    g.load_model(m)
    full = run_gpu(g, t, pcfg(40, warmup=64), oracle=False)
    parts = [run_gpu(g, t, pcfg(40, warmup=64), oracle=False, shard=s) for s in ((0, 13), (13, 29), (29, 40))]
    got = np.concatenate([gpu_subs(p) for p in parts])
    assert np.array_equal(got, gpu_subs(full))
    assert np.array_equal(np.concatenate([p.predicted_fetch for p in parts]), full.predicted_fetch)


@pytest.mark.parametrize("oracle", [True, False])
def test_gpu_trace_ingest_matches_host_path(gpu, port, golden, oracle):
    """SNT1 records unpacked on the device (load_trace_file) = the host SoA path."""
    g = gpu("tf32x3")
    g.load_model(c3_model(port, golden))
    path = GOLD / "pointer_chase_2000_s3.trace"
    t = read_trace(path)
    for pc in (pcfg(7), pcfg(5, warmup=30)):
        g.load_trace(t, pc, oracle=oracle)
        a = g.run(pc, oracle=oracle)
        n = g.load_trace_file(str(path), pc, oracle=oracle)
        b = g.run(pc, oracle=oracle)
        assert n == t.n
        assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch)
    for shard in ((0, 3), (3, 7)):
        g.load_trace(t, pcfg(7), oracle=oracle, shard=shard)
        a = g.run(pcfg(7), oracle=oracle, shard=shard)
        g.load_trace_file(str(path), pcfg(7), oracle=oracle, shard=shard)
        b = g.run(pcfg(7), oracle=oracle, shard=shard)
        assert np.array_equal(gpu_subs(a), gpu_subs(b))


def test_fp8_fused_rounds(gpu, port):
    """fp8 (e4m3 operands, tcgen05 kind::f8f6f4) runs the fused rounds; its CPI
    error against the CPU oracle is reported (printed) and loosely bounded.
    Teacher-forced predict and unfused rounds refuse fp8 with an error."""
    g = gpu("fp8")
    m, t = _bench_like("default", n=12_000)
    g.load_model(m)
    pc = pcfg(48)
    g.load_trace(t, pc)
    r = g.run(pc)
    want = port.simulate(t, m, k=48)
    err = (r.total_cycles - want["total_cycles"]) / want["total_cycles"]
    same = float(np.mean(r.predicted_fetch == want["predicted_fetch"]))
    print(f"fp8: total cycles {r.total_cycles} vs oracle {want['total_cycles']} ({100 * err:+.2f}%), "
          f"{100 * same:.1f}% fetch latencies identical")
    assert abs(err) < 0.25 and r.instructions == t.n
    with pytest.raises(IlsimError):
        g.run(pc, fused=False)
    with pytest.raises(IlsimError):
        g.predict(np.zeros((1, 50 * 111), np.float32), np.zeros(1, np.uint8))


def test_run_into_caller_fetch_buffer(gpu, port, golden):
    """run(fetch_out=...) writes the predicted fetch series into a caller-owned
    buffer (the C-ABI contract), with the same values as a fresh array."""
    g = gpu("tf32x3")
    m, _ = _fused_cases(port, golden)
    g.load_model(m)
    t = read_trace(GOLD / "mix_3000_s4.trace")
    pc = pcfg(5)
    g.load_trace(t, pc)
    a = g.run(pc)
    buf = np.full(t.n + 7, 0xDEADBEEF, np.uint32)
    b = g.run(pc, fetch_out=buf)
    assert np.array_equal(a.predicted_fetch, b.predicted_fetch) and np.array_equal(buf[:t.n], a.predicted_fetch)
    assert np.all(buf[t.n:] == 0xDEADBEEF)
    with pytest.raises(IlsimError):
        g.run(pc, fetch_out=np.zeros(t.n, np.int64))


@pytest.mark.parametrize("extra", [dict(), dict(warmup=200, drain_trim=True), dict(k=3000),
                                   dict(shard=(300, 900), warmup=50)])
def test_overlapped_upload_matches_load_then_run(gpu, extra):
    """simulate_parallel on a large trace uploads it window by window (2-D
    copies over runs of equal-length sub-traces, packed per window) while the
    rounds run; results equal a full upload followed by the rounds, bit for bit."""
    from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace
    g = gpu("tf32x3")
    m = synthetic_model(synthetic_trace(20_000, 101), 1)
    g.load_model(m)
    t = synthetic_trace(1_100_000, 7)
    pc = pcfg(extra.get("k", 1024), warmup=extra.get("warmup", 0), drain_trim=extra.get("drain_trim", False))
    shard = extra.get("shard")
    a = g.simulate_parallel(t, pc, shard=shard)
    g.load_trace(t, pc, shard=shard, truth=False)
    b = g.run(pc, shard=shard)
    assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch)


@pytest.mark.parametrize("heads", [(6, 9, 12), (4, 4, 5), (20, 20, 20)])
def test_fc2_head_sizes(gpu, port, golden, heads):
    """Head sizes other than 10/10/10 (output_dim 30, 16 and 63: FC2's od % 8
    remainder is 6, 0 and 7, spread over the warps; 63 needs more than 48 KB
    of shared memory in the final decode): teacher-forced outputs vs the
    port, the fused round bit-identical to the unfused one and within 0.1% of
    the CPU oracle."""
    g = gpu("tf32x3")
    cfg = CnnConfig.preset_c3()
    cfg.class_fetch, cfg.class_exec, cfg.class_store = heads
    gm = golden["models"]["c3_mix_seed1"]
    m = Model(cfg, np.array(gm["norm"]), port.init_params(cfg, 5))
    g.load_model(m)
    t = read_trace(GOLD / "mix_3000_s4.trace")
    want = port.simulate(t, m, k=16, capture=600, capture_inputs=True, capture_outputs=True)
    out, _ = g.predict(want["cap_inputs"], want["cap_is_store"])
    assert out.shape[1] == cfg.output_dim
    err = np.abs(out - want["cap_outputs"]) / np.maximum(1.0, np.abs(want["cap_outputs"]))
    assert err.max() <= 1e-4, err.max()
    pc = pcfg(16)
    g.load_trace(t, pc)
    a = g.run(pc)
    b = g.run(pc, fused=False)
    assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch)
    full = port.simulate(t, m, k=16)
    assert abs(a.total_cycles - full["total_cycles"]) <= 1e-3 * full["total_cycles"]


# ---- the reference's decode goldens on the device decode functions ----------
def _decode_model(norm=None):
    from helpers import model_from_params

    cfg = small_config()
    return model_from_params(cfg, np.zeros(cfg.param_count(), np.float32), norm)


@pytest.mark.parametrize("path", [0, 1])
def test_decode_goldens_on_device(gpu, path):
    """test_cnn.cpp:183-224 replayed on decode.cuh (path 0) and the fused
    round's warp_decode_triple (path 1) through ilsim_gpu_decode_outputs."""
    from paper_2105_05821_b200.formats import identity_norm

    g = gpu("fp32")

    def dec(vals, is_store=False, norm=None):
        g.load_model(_decode_model(norm))
        y = np.zeros((1, 33), np.float32)
        for i, v in vals.items():
            y[0, i] = v
        return g.decode(y, np.array([is_store], np.uint8), path)[0]

    assert dec({3 + 3: 2.0})[0] == 3                                          # argmax at c_3
    assert dec({3 + 9: 5.0, 0: np.float32(np.log1p(20.4))})[0] == 20           # overflow -> regression
    assert dec({3 + 9: 5.0, 0: -3.0})[0] == 0                                  # clamps at 0
    assert dec({3: 1.5, 4: 1.5})[0] == 0                                       # exact tie -> smaller class
    t = dec({13: 3.0, 23 + 7: 3.0})
    assert t[1] == 1 and t[2] == 0                                             # exec floor 1, store masked
    assert dec({13: 3.0, 23 + 7: 3.0}, is_store=True)[2] == 7
    norm = identity_norm()
    norm[100], norm[103] = 1.0, 0.5
    assert dec({12: 5.0, 0: np.float32((np.log1p(18.0) - 1.0) / 0.5)}, norm=norm)[0] == 18


@pytest.mark.parametrize("path", [0, 1])
def test_decode_device_equals_port(gpu, port, path):
    """Bit-exact decode of the same head outputs on the device and in the
    port (cnn.cpp:388-417): ties, overflow-class regression near .5
    boundaries, NaN / inf logits and regressions, values past 22 and 4e9."""
    from paper_2105_05821_b200.formats import identity_norm

    rng = np.random.default_rng(7)
    n = 4096
    y = rng.normal(0, 2, (n, 33)).astype(np.float32)
    y[::7, 3:13] = 1.25                                   # full ties
    y[1::7, 12] = 50.0                                    # overflow class wins (fetch)
    y[2::7, 22] = 50.0                                    # exec
    y[3::7, 32] = 50.0                                    # store
    y[1::7, 0] = rng.uniform(-5, 30, y[1::7, 0].shape)    # includes clamp at 22 and 4e9
    y[2::7, 1] = np.float32(np.log1p(np.floor(rng.uniform(0, 900, y[2::7, 1].shape)) + 0.5))  # .5 boundaries
    y[3::7, 2] = np.nan                                   # NaN regression in the overflow class
    y[4::7, 3 + 4] = np.nan                               # NaN logit never wins
    y[5::7, 13:23] = -np.inf
    y[6::7, 23 + 9] = np.inf
    y[6::7, 2] = np.inf
    st = (rng.random(n) < 0.5).astype(np.uint8)
    norm = identity_norm()
    norm[100:103] = [0.7, 1.6, 0.4]
    norm[103:106] = [0.6, 0.9, 1.2]
    m = _decode_model(norm)
    g = gpu("fp32")
    g.load_model(m)
    got = g.decode(y, st, path)
    want = port.decode(m, y, st)
    assert np.array_equal(got, want), np.nonzero((got != want).any(1))[0][:10]


def test_forward_tiny_pin_gpu(gpu, port):
    """The reference's forward pin (test_cnn.cpp:155-168: tiny config with
    conv {7, 9}, init_weights(cfg, NormStats{}, seed), random_input from the
    reference Rng, 1e-6 relative vs the straight-line double forward) through
    ilsim_gpu_predict in fp32.  The device feature layout has 50 slots per
    column, so the config is tiny(50, 16) instead of tiny(5, 16)."""
    from helpers import model_from_params, random_input, tiny_config
    from test_oracle import naive_forward

    g = gpu("fp32")
    for seed in (1, 2, 3):
        cfg = tiny_config(50, 16, conv=(7, 9))
        m = model_from_params(cfg, port.init_params(cfg, seed))
        g.load_model(m)
        x = random_input(cfg, seed + 100)
        out, _ = g.predict(x[None, :], np.zeros(1, np.uint8))
        want = naive_forward(cfg, m.params, x)
        assert np.all(np.abs(out[0] - want) <= 1e-6 * np.maximum(1.0, np.abs(want))), (seed, out[0] - want)


@pytest.mark.parametrize("devices,k,precision", [([0], 5, "tf32x3"), ([0, 0], 5, "tf32x3"), ([0, 0, 0], 17, "fp32"),
                                                 ([0, 0, 0, 0], 3, "bf16")])
def test_device_group_matches_single_context(gpu, devices, k, precision):
    """ilsim_gpu_group_simulate_parallel (one host thread per listed device;
    the box has one GPU, so the shards share it) reproduces the single-context
    sub-results, predicted fetch series and totals bit-exactly for any device
    list, including a device with no sub-traces (test_parallel.cpp:114-146)."""
    from paper_2105_05821_b200 import GpuGroup

    t = read_trace(GOLD / "mix_3000_s4.trace")
    m = read_model(GOLD / "small_dataset.model")
    pc = pcfg(k, mc=m.config.max_context)
    g = gpu(precision)
    g.load_model(m)
    want = g.simulate_parallel(t, pc)
    with GpuGroup(devices, precision) as grp:
        grp.load_model(m)
        got = grp.simulate_parallel(t, pc)
        assert gpu_subs(got).tolist() == gpu_subs(want).tolist()
        assert np.array_equal(got.predicted_fetch, want.predicted_fetch)
        assert got.total_cycles == want.total_cycles and got.instructions == t.n
        o = grp.simulate_parallel(t, pc, oracle=True)
        assert o.instructions == t.n
        with pytest.raises(IlsimError, match="batch_max must be >= 1"):
            grp.simulate_parallel(t, pcfg(k, batch_max=0, mc=m.config.max_context))


# ---- a paper-scale residual model (RB7-like, 84 MFLOPs) through the same kernels
@pytest.mark.parametrize("precision,rtol", [("fp32", 1e-5), ("tf32x3", 1e-5), ("bf16", 5e-3)])
def test_rb7_teacher_forced_and_free_running(gpu, port, golden, precision, rtol):
    """Seven residual 384-channel conv blocks (CnnConfig.preset_rb7, the scale
    of the paper's RB7): the tensor-core path runs the wide layers split-K
    (K up to 768 per layer), the fp32 path SIMT.  Teacher-forced outputs vs
    the port's forward, and a free-running simulation vs the port."""
    g = gpu(precision)
    cfg = CnnConfig.preset_rb7()
    gm = golden["models"]["c3_mix_seed1"]
    m = Model(cfg, np.array(gm["norm"]), port.init_params(cfg, 3))
    g.load_model(m)
    t = read_trace(GOLD / "mix_3000_s4.trace").slice(0, 400)
    want = port.simulate(t, m, k=4, capture=200, capture_inputs=True, capture_outputs=True)
    out, tri = g.predict(want["cap_inputs"], want["cap_is_store"])
    ref = want["cap_outputs"]
    err = np.abs(out - ref) / np.maximum(1.0, np.abs(ref))
    print(f"rb7 {precision}: max rel err {err.max():.3g}, triples equal {np.mean((tri == want['cap_triples']).all(1)):.4f}")
    assert err.max() <= rtol, err.max()
    assert np.array_equal(port.decode(m, out, want["cap_is_store"]), tri)
    r = run_gpu(g, t, pcfg(4), oracle=False)
    tot, wtot = r.total_cycles, want["total_cycles"]
    print(f"rb7 {precision}: total cycles {tot} vs port {wtot} ({100 * (tot - wtot) / wtot:+.3f}%)")
    if precision != "bf16":
        assert abs(tot - wtot) <= 1e-3 * wtot, (tot, wtot)


# ---- parity at BASELINE scale against the reference's own runs --------------
@pytest.mark.parametrize("name,precision,exact,min_blocks", [
    ("c4", "fp32", True, 1.0), ("c2", "tf32x3", False, 0.99), ("c4", "tf32x3", False, 0.99),
    ("c2t", "fp32", True, 1.0), ("c2t", "tf32x3", False, 0.98), ("c4t", "fp32", True, 1.0),
    ("c4t", "tf32x3", False, 0.98), ("c3st", "fp32", True, 1.0), ("rb7", "fp32", True, 1.0),
    ("rb7", "tf32x3", False, 0.99)])
def test_scale_parity_against_reference_fixture(gpu, name, precision, exact, min_blocks):
    """The reference's simulate_parallel (oracle/_ref) was run once on the exact
    bench workloads (tools/scale_parity.py, tests/golden/scale/; c2t: the c2
    workload with the trained C3, tests/golden/train_c3.py): the fp32 path
    must reproduce every per-sub-trace counter and every predicted-fetch block;
    tf32x3 must be within 0.1% of the total cycles (acceptance_main.cpp:326-334)
    with >= 99% of the fetch blocks identical.  The trained C3 (c2t) has
    narrower decision margins, so the fp32 path's accumulation order matters:
    it follows the reference's restated forward (one fma chain per output;
    with FC1 in two 512-wide chunks it was +0.0004%, 99.9% of the blocks) and
    is bit-exact; tf32x3's rounding flips more decisions than with the
    synthetic weights: held to 0.1% with >= 98% of the blocks (-0.0105%, 98.9%)."""
    import sys

    sys.path.insert(0, str(GOLD.parents[1] / "tools"))
    from scale_parity import build_workload, compare, load_fixture

    trace, model, w = build_workload(name)
    g = gpu(precision)
    g.load_model(model)
    pc = pcfg(w["k"], mc=model.config.max_context)
    g.load_trace(trace, pc, truth=False)
    r = g.run(pc)
    out = compare(name, r, trace, model)
    print(name, precision, {k: out.get(k) for k in ("cpi_error_percent", "subtrace_identical_frac",
                                                     "fetch_block_identical_frac")})
    assert "error" not in out, out
    assert out["within_0p1pct"], out
    if exact:
        fx = load_fixture(name)
        assert gpu_subs(r).tolist() == fx["subs"].tolist()
        assert out["fetch_block_identical_frac"] == 1.0
    else:
        assert out["fetch_block_identical_frac"] >= min_blocks, out


@pytest.mark.parametrize("model_name", ["trained", "synthetic"])
def test_sequential_c3_persistent_kernel(gpu, port, model_name, monkeypatch):
    """The C3 at one sub-trace (simulate_trace with the CNN, fp32) runs as ONE
    persistent cooperative launch (seq_c3_kernel): bit for bit the
    launch-per-layer rounds (SIMNET_NO_SEQ_FC) and the oracle port's
    sequential simulation (the reference's restated forward order), with the
    trained C3's narrow margins as well."""
    import sys

    t = read_trace(GOLD / "mix_3000_s4.trace")
    if model_name == "trained":
        m = read_model(GOLD / "c3_trained.model")
    else:
        sys.path.insert(0, str(GOLD.parents[1]))
        from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace

        m = synthetic_model(synthetic_trace(50_000, 101), 1, init_params=port.init_params)
    g = gpu("fp32")
    g.load_model(m)
    pc = pcfg(1, mc=m.config.max_context)
    g.load_trace(t, pc)
    monkeypatch.delenv("SIMNET_NO_SEQ_FC", raising=False)
    a = g.run(pc)
    assert a.launches == 1  # the persistent kernel ran
    monkeypatch.setenv("SIMNET_NO_SEQ_FC", "1")
    b = g.run(pc)
    assert b.launches > 1000
    assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch)
    want = port.simulate(t, m, sequential=True)
    assert gpu_subs(a).tolist() == np.asarray(want["subs"]).tolist()
    assert np.array_equal(a.predicted_fetch, want["predicted_fetch"])


def test_device_group_concurrent_persistent_kernels(gpu):
    """Two group members on the same GPU, one sub-trace each, fp32 C3: both
    run the persistent cooperative kernel at once from their host threads
    (cooperative grids are gang-scheduled, so one waits for the other; every
    wait inside is bounded, so a scheduling problem would be an error, not a
    hang); results equal the single-context launch-per-layer run of K = 2."""
    from paper_2105_05821_b200 import GpuGroup

    t = read_trace(GOLD / "mix_3000_s4.trace").slice(0, 1200)
    m = read_model(GOLD / "c3_trained.model")
    pc = pcfg(2, mc=m.config.max_context)
    g = gpu("fp32")
    g.load_model(m)
    want = g.simulate_parallel(t, pc)
    with GpuGroup([0, 0], "fp32") as grp:
        grp.load_model(m)
        got = grp.simulate_parallel(t, pc)
        assert gpu_subs(got).tolist() == gpu_subs(want).tolist()
        assert np.array_equal(got.predicted_fetch, want.predicted_fetch)


def test_persistent_c3_error_paths(gpu, monkeypatch):
    """A sub-trace error inside the persistent C3 kernel (an explicit write
    ring too small for the store queue) ends the run with the same reported
    error as the launch-per-layer rounds (the kernel keeps its rounds in step
    and leaves; nothing hangs); with the ring on auto both paths rerun with a
    larger ring and agree."""
    t = store_heavy(5, 3000, lat_hi=400)
    m = read_model(GOLD / "c3_trained.model")
    g = gpu("fp32")
    g.load_model(m)
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("SIMNET_NO_SEQ_FC", env)
        else:
            monkeypatch.delenv("SIMNET_NO_SEQ_FC", raising=False)
        pc = pcfg(1, mc=m.config.max_context, write_ring=2)
        g.load_trace(t, pc)
        with pytest.raises(IlsimError, match="write queue ring overflow"):
            g.run(pc)
    monkeypatch.delenv("SIMNET_NO_SEQ_FC", raising=False)
    pc = pcfg(1, mc=m.config.max_context)
    g.load_trace(t, pc)
    a = g.run(pc)
    monkeypatch.setenv("SIMNET_NO_SEQ_FC", "1")
    b = g.run(pc)
    assert np.array_equal(gpu_subs(a), gpu_subs(b)) and np.array_equal(a.predicted_fetch, b.predicted_fetch)
