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


class RefRng:
    """The reference's ``Rng`` (common.hpp:27-66: xoshiro256** seeded by
    splitmix64), so test inputs are drawn exactly as the reference tests draw
    them (e.g. ``random_input``, test_cnn.cpp:16-21)."""

    M = (1 << 64) - 1

    @staticmethod
    def splitmix64(x: int) -> int:
        M = RefRng.M
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)

    def __init__(self, seed: int):
        self.s = []
        x = seed & self.M
        for _ in range(4):
            x = self.splitmix64(x)
            self.s.append(x)

    @staticmethod
    def _rotl(x: int, k: int) -> int:
        return ((x << k) | (x >> (64 - k))) & RefRng.M

    def next_u64(self) -> int:
        s, M = self.s, self.M
        result = (self._rotl((s[1] * 5) & M, 7) * 9) & M
        t = (s[1] << 17) & M
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return result

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def next_symmetric(self, a: float) -> np.float32:
        return np.float32((2.0 * self.next_double() - 1.0) * a)


def tiny_config(channels: int = 4, seq: int = 8, conv=(6, 6), fc_hidden: int = 8) -> CnnConfig:
    """``CnnConfig::tiny`` (cnn.cpp:283-291)."""
    c = CnnConfig.preset_c3(seq - 1)
    c.input_channels = channels
    c.max_context = seq - 1
    c.sequence_length = seq
    c.conv_channels = list(conv)
    c.fc_hidden = fc_hidden
    return c


def random_input(cfg: CnnConfig, seed: int) -> np.ndarray:
    """``random_input`` (test_cnn.cpp:16-21): input_channels x (max_context+1)
    values U[-1.5, 1.5] from the reference Rng."""
    r = RefRng(seed)
    return np.array([r.next_symmetric(1.5) for _ in range(cfg.input_channels * (cfg.max_context + 1))],
                    np.float32)
