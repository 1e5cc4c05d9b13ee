"""Synthetic workloads for benchmarking (no reference code, no DES).

* :func:`synthetic_trace` — an annotated trace of the reference's record
  shape (trace.hpp:49-109): a static program of basic blocks walked with loop
  locality, per-static-instruction operand registers, strided / random data
  addresses inside a footprint, cache-level history fields and plausible
  truth latencies (used only in oracle mode).
* :func:`synthetic_model` — a C3 (or FC-style) model drawn with the
  reference's ``init_weights`` rule (cnn.cpp:335-352), NormStats estimated
  from the trace, and fc2 head biases set so the decoded latencies fall in a
  chosen regime: ``"default"`` (DES-like, ~30 context
  columns) or ``"memory"`` (store-heavy: P(F=0)~0.5, stores 100s of cycles,
  full 110-column contexts).
"""
from __future__ import annotations

import numpy as np

from .api import init_weights
from .formats import (OP_BRANCH, OP_FP_ALU, OP_FP_DIV, OP_FP_MULT, OP_INT_ALU, OP_INT_DIV, OP_INT_MULT, OP_LOAD,
                      OP_SIMD, OP_STORE, CnnConfig, Model, Trace)

MIXES = {
    # op-class weights in OpClass order (trace.hpp:15-26)
    "mix": [0.40, 0.04, 0.01, 0.05, 0.03, 0.01, 0.02, 0.22, 0.10, 0.12],
    "memory": [0.30, 0.02, 0.0, 0.05, 0.02, 0.0, 0.0, 0.30, 0.25, 0.06],
}


def synthetic_trace(n: int, seed: int = 101, kind: str = "mix", footprint: int = 16 << 20,
                    static_size: int = 8192) -> Trace:
    rng = np.random.default_rng(seed)
    mix = np.asarray(MIXES[kind], dtype=np.float64)
    mix /= mix.sum()
    # --- static program -------------------------------------------------
    S = static_size
    opc = rng.choice(10, size=S, p=mix)
    block_end = rng.random(S) < 0.12
    opc = np.where(block_end, OP_BRANCH, opc)
    sop = np.zeros((S, 13), np.uint8)
    sop[:, 0] = opc
    sop[:, 1] = opc == OP_LOAD
    sop[:, 2] = opc == OP_STORE
    sop[:, 3] = opc == OP_BRANCH
    sop[:, 4] = (opc == OP_BRANCH) & (rng.random(S) < 0.9)
    sop[:, 5] = (opc == OP_BRANCH) & ~sop[:, 4].astype(bool)
    sop[:, 6] = (opc == OP_BRANCH) & (rng.random(S) < 0.7)
    sop[:, 7] = (opc == OP_BRANCH) & (rng.random(S) < 0.05)
    sop[:, 8] = (opc == OP_BRANCH) & (rng.random(S) < 0.05)
    sop[:, 11] = (opc == OP_FP_ALU) | (opc == OP_FP_MULT) | (opc == OP_FP_DIV)
    sop[:, 12] = np.where(opc == OP_SIMD, 4, 0)
    nsrc = rng.integers(1, 4, S)
    ssrc = np.where(np.arange(8)[None, :] < nsrc[:, None], 1 + rng.integers(0, 48, (S, 8)), 0).astype(np.uint16)
    hasdst = (opc != OP_STORE) & (opc != OP_BRANCH)
    sdst = np.zeros((S, 6), np.uint16)
    sdst[:, 0] = np.where(hasdst, 1 + rng.integers(0, 48, S), 0)
    mem = (opc == OP_LOAD) | (opc == OP_STORE)
    sbase = (0x10000000 + rng.integers(0, footprint // 64, S) * 64).astype(np.uint64)
    sstride = rng.choice(np.array([0, 8, 8, 16, 64, 4096], np.uint64), S)
    chase = rng.random(S) < (0.5 if kind == "memory" else 0.15)
    # --- dynamic walk: basic blocks with loop locality ---------------------
    starts = np.flatnonzero(np.r_[True, block_end[:-1]])
    nb = starts.size
    ends = np.r_[starts[1:], S]
    avg = max(1, int(np.mean(ends - starts)))
    nblocks = n // avg + 64
    jump = rng.random(nblocks)
    step = np.where(jump < 0.55, 0, np.where(jump < 0.85, 1, rng.integers(-64, 64, nblocks)))
    seq = np.cumsum(step) % nb
    lens = (ends - starts)[seq]
    idx = np.repeat(starts[seq], lens) + (np.arange(lens.sum()) - np.repeat(np.cumsum(lens) - lens, lens))
    while idx.size < n:
        idx = np.r_[idx, idx[: n - idx.size]]
    idx = idx[:n]
    # --- per-dynamic fields ----------------------------------------------
    op = sop[idx]
    dmem = mem[idx]
    occ = np.zeros(n, np.int64)
    order = np.argsort(idx, kind="stable")
    counts = np.bincount(idx, minlength=S)
    first = np.cumsum(counts) - counts
    occ[order] = np.arange(n) - np.repeat(first, counts)
    rnd = (0x10000000 + rng.integers(0, footprint // 8, n) * 8).astype(np.uint64)
    strided = (sbase[idx] + (sstride[idx] * occ.astype(np.uint64)) % np.uint64(footprint)).astype(np.uint64)
    addr = np.where(dmem, np.where(chase[idx], rnd, strided), 0).astype(np.uint64)
    hist = np.zeros((n, 14), np.uint16)
    hist[:, 1] = np.where(rng.random(n) < 0.97, 1, rng.integers(2, 4, n))
    lvl = np.where(chase[idx], rng.choice([1, 2, 3], n, p=[0.4, 0.3, 0.3]), rng.choice([1, 2, 3], n, p=[0.9, 0.08, 0.02]))
    hist[:, 7] = np.where(dmem, lvl, 0)
    hist[:, 0] = np.where(op[:, 3] != 0, rng.random(n) < 0.06, 0)
    hist[:, 2:5] = np.where(rng.random((n, 1)) < 0.01, rng.integers(0, 3, (n, 3)), 0)
    hist[:, 8:11] = np.where(dmem[:, None] & (rng.random((n, 1)) < 0.03), rng.integers(0, 3, (n, 3)), 0)
    truth = np.zeros((n, 3), np.uint32)
    truth[:, 0] = rng.choice([0, 1, 2, 3, 8], n, p=[0.45, 0.35, 0.12, 0.05, 0.03])
    base_lat = np.array([1, 3, 20, 2, 4, 12, 3, 1, 1, 1], np.uint32)[op[:, 0]]
    truth[:, 1] = base_lat + np.where(dmem, np.array([0, 5, 29, 100], np.uint32)[lvl], 0)
    truth[:, 2] = np.where(op[:, 2] != 0, truth[:, 1] + rng.integers(1, 60, n), 0)
    return Trace(
        pc=(0x400000 + idx.astype(np.uint64) * 4).astype(np.uint64),
        op=np.ascontiguousarray(op),
        src=np.ascontiguousarray(ssrc[idx]),
        dst=np.ascontiguousarray(sdst[idx]),
        has_data=dmem.astype(np.uint8),
        data_addr=addr,
        data_size=np.where(dmem, 8, 0).astype(np.uint16),
        hist=hist,
        truth=truth,
        fetch_tick=np.cumsum(truth[:, 0], dtype=np.uint64),
    )


def norm_from_trace(t: Trace, sample: int = 200_000) -> np.ndarray:
    """NormStats-shaped statistics (dataset.cpp:142-178 form: per-slot mean,
    stdev floored at 1; log1p label stats floored at 0.25) estimated from the
    static slots of a trace sample; dynamic slots get fixed plausible values."""
    m = min(sample, t.n)
    raw = np.concatenate([t.op[:m], t.src[:m], t.dst[:m], t.hist[:m]], axis=1).astype(np.float64)
    norm = np.zeros(106)
    norm[:41] = raw.mean(0)
    norm[50:91] = np.maximum(1.0, raw.std(0))
    norm[41], norm[91] = 20.0, 25.0  # residence
    norm[42], norm[92] = 8.0, 12.0   # execution
    norm[43], norm[93] = 4.0, 20.0   # store
    norm[44:49], norm[94:99] = 0.3, 1.0
    norm[49], norm[99] = 0.0, 1.0
    norm[100:103] = [0.7, 1.6, 0.4]
    norm[103:106] = [0.6, 0.9, 1.2]
    return norm


# fc2 head biases (output order: 3 regression, 10 fetch, 10 exec, 10 store).
# Regression rows carry no weights, so the overflow class decodes to a fixed
# value: r = (log1p(v) - label_mean) / label_stdev with norm_from_trace's
# label statistics.  Chosen so that, with seed 1 on a synthetic trace, the
# "default" regime holds ~30 context columns (the DES traces' 29-32, SURVEY.md
# §6) and the "memory" regime ~70 with full 110-column windows and overflow
# stalls (the c4 regime).
def _reg(e: float, s: float) -> list[float]:
    return [0.0, (float(np.log1p(e)) - 1.6) / 0.9, (float(np.log1p(s)) - 0.4) / 1.2]


_REGIMES = {
    "default": dict(reg=_reg(30, 60), fetch=[0.9, 1.0, 0.5, 0.0, -1, -2, -2, -2, -3, -3],
                    exec_=[-3, 0.6, 0.8, 0.7, 0.6, 0.5, 0.4, 0.3, 0.2, 0.2],
                    store=[-3, -3, -1, 0, 0.2, 0.3, 0.3, 0.2, 0, 0.6]),
    "memory": dict(reg=_reg(40, 600), fetch=[4.5, 2.5, -1.0, -1.5, -2, -2, -2, -2, -3, -3],
                   exec_=[-3, 0.3, 0.5, 0.5, 0.5, 0.5, 0.5, 0.5, 0.5, 0.6],
                   store=[-3, -3, -3, -3, -3, -3, -3, -3, -3, 3]),
}
HEAD_GAIN = 200.0  # classification rows of fc2 are scaled by this (input sensitivity)


def synthetic_model(trace: Trace, seed: int = 1, regime: str = "default",
                    config: CnnConfig | None = None, init_params=None) -> Model:
    """``init_params(cfg, seed) -> f32[param_count]`` replaces the library's
    ``init_weights`` (the CPU reference arm draws the same weights through
    the oracle so that it never loads the product library)."""
    cfg = config or CnnConfig.preset_c3()
    if init_params is None:
        m = init_weights(cfg, norm_from_trace(trace), seed)
    else:
        n = cfg.param_count()
        m = Model(cfg, norm_from_trace(trace), np.asarray(init_params(cfg, seed), np.float32).copy(),
                  np.zeros(n, np.float32), np.zeros(n, np.float32), 0)
    p = m.params
    L = cfg.param_count()
    od, H = cfg.output_dim, cfg.fc_hidden
    # Zero the hidden biases: U(+-1) biases (cnn.cpp:346 draws biases with
    # cols == 1) otherwise swamp the input signal and every decode is constant.
    off, cin = 0, cfg.input_channels
    for cout in cfg.conv_channels:  # tensor table order (cnn.cpp:293-315): w, b (, p)
        off += cout * 2 * cin
        p[off: off + cout] = 0.0
        off += cout
        if cfg.residual_blocks:
            off += cout * 2 * cin
        cin = cout
    off += H * cfg.flat_dim
    p[off: off + H] = 0.0
    off += H
    W2 = p[off: off + od * H].reshape(H, od)  # column-major: element (o, k) at o + k*od
    W2[:, :3] = 0.0        # regression heads: constant de-normalised fallback values
    W2[:, 3:] *= HEAD_GAIN  # classification heads: input-dependent argmax around the biases
    r = _REGIMES[regime]
    b = np.r_[r["reg"], r["fetch"][: cfg.class_fetch], r["exec_"][: cfg.class_exec], r["store"][: cfg.class_store]]
    p[L - od:] = np.asarray(b, np.float32)
    return m


# ---------------------------------------------------------------------------
# c3 (BASELINE.json configs[2]): one global 100M-instruction trace partitioned
# into 65,536 sub-traces (partition, parallel.cpp:9-24: base 1525, rem 57,600).
# The trace is defined as 8 chunks, chunk j = synthetic_trace(len_j, 101 + j)
# holding global sub-traces [8192 j, 8192 (j + 1)) — one 8-GPU shard each — so
# a process builds only the chunks its shard touches.
# ---------------------------------------------------------------------------
C3_N, C3_K, C3_CHUNKS = 100_000_000, 65_536, 8


def partition_start(n: int, k: int, i: int) -> int:
    """First instruction of sub-trace i (parallel.cpp:9-24)."""
    base, rem = divmod(n, k)
    return i * base + min(i, rem)


def c3_chunk_bounds() -> list[int]:
    per = C3_K // C3_CHUNKS
    return [partition_start(C3_N, C3_K, per * j) for j in range(C3_CHUNKS)] + [C3_N]


def c3_trace_slice(lo: int, hi: int) -> Trace:
    """Instructions [lo, hi) of the c3 global trace."""
    b = c3_chunk_bounds()
    parts = []
    for j in range(C3_CHUNKS):
        a, e = max(lo, b[j]), min(hi, b[j + 1])
        if a < e:
            t = synthetic_trace(b[j + 1] - b[j], seed=101 + j)
            parts.append(t.slice(a - b[j], e - b[j]) if (a, e) != (b[j], b[j + 1]) else t)
    return Trace.concat(parts)
