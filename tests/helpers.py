"""Shared trace/model builders and backend runners for the test suite."""
from __future__ import annotations

import numpy as np

from paper_2105_05821_b200.formats import OP_INT_ALU, OP_STORE, CnnConfig, Model, Trace, identity_norm


def instr_trace(kinds: list[bool], script: list[tuple[int, int, int]]) -> Trace:
    """Trace of test_simcore.cpp:28-44 ``instr(store)`` records with scripted
    truth latencies (the ScriptedPredictor of test_simcore.cpp:14-26)."""
    n = len(kinds)
    op = np.zeros((n, 13), np.uint8)
    hist = np.zeros((n, 14), np.uint16)
    has = np.zeros(n, np.uint8)
    addr = np.zeros(n, np.uint64)
    size = np.zeros(n, np.uint16)
    for i, st in enumerate(kinds):
        op[i, 0] = OP_STORE if st else OP_INT_ALU
        op[i, 2] = 1 if st else 0
        hist[i, 1] = 1
        if st:
            has[i], addr[i], size[i] = 1, 0x10000, 8
            hist[i, 7] = 1
    truth = np.asarray(script, dtype=np.uint32).reshape(n, 3)
    ft = np.cumsum(truth[:, 0].astype(np.uint64))
    return Trace(np.full(n, 0x400000, np.uint64), op, np.zeros((n, 8), np.uint16), np.zeros((n, 6), np.uint16),
                 has, addr, size, hist, truth, ft)


def random_trace(seed: int, n: int) -> Trace:
    """``random_trace`` shape of test_trace.cpp:21-60 (numpy RNG, not bit-identical)."""
    rng = np.random.default_rng(seed)
    opc = rng.integers(0, 10, n)
    op = np.zeros((n, 13), np.uint8)
    op[:, 0] = opc
    op[:, 1] = opc == 7
    op[:, 2] = opc == 8
    op[:, 3] = opc == 9
    op[:, 6] = (opc == 9) & (rng.random(n) < 0.7)
    op[:, 11] = (opc >= 3) & (opc <= 5)
    op[:, 12] = np.where(opc == 6, 4, 0)
    mem = (opc == 7) | (opc == 8)
    pc = (0x400000 + rng.integers(0, 1 << 20, n) * 4).astype(np.uint64)
    addr = np.where(mem, 0x10000000 + rng.integers(0, 1 << 22, n), 0).astype(np.uint64)
    hist = np.zeros((n, 14), np.uint16)
    hist[:, 1] = rng.integers(1, 4, n)
    hist[:, 7] = np.where(mem, rng.integers(1, 4, n), 0)
    hist[:, 0] = np.where(opc == 9, rng.random(n) < 0.1, 0)
    truth = np.zeros((n, 3), np.uint32)
    truth[:, 0] = rng.integers(0, 4, n)
    truth[:, 1] = 1 + rng.integers(0, 40, n)
    truth[:, 2] = np.where(opc == 8, truth[:, 1] + rng.integers(0, 100, n), 0)
    return Trace(pc, op, rng.integers(0, 49, (n, 8)).astype(np.uint16), rng.integers(0, 49, (n, 6)).astype(np.uint16),
                 mem.astype(np.uint8), addr, np.where(mem, 8, 0).astype(np.uint16), hist, truth,
                 np.cumsum(truth[:, 0]).astype(np.uint64))


def small_config(max_context: int = 110) -> CnnConfig:
    """The untrained CNN of test_parallel.cpp:118-121 (16/16/16, fc 32)."""
    c = CnnConfig.preset_c3(max_context)
    c.conv_channels = [16, 16, 16]
    c.fc_hidden = 32
    return c


def model_from_params(cfg: CnnConfig, params: np.ndarray, norm: np.ndarray | None = None) -> Model:
    return Model(cfg, identity_norm() if norm is None else np.asarray(norm, np.float64),
                 np.asarray(params, np.float32))


SUB = ["instructions", "total_cycles", "sum_fetch", "delta", "drain_cycles", "overflow_stall_cycles", "empty"]


def gpu_subs(pr) -> np.ndarray:
    return np.array([[getattr(s, f) if f != "empty" else int(s.empty) for f in SUB] for s in pr.sub_results],
                    dtype=np.uint64)
