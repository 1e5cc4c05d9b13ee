"""Reference file formats, read/written with numpy.

* ``SNT1`` annotated traces (reference ``trace.cpp:49-124``): 24-byte header,
  then 108-byte little-endian records.  Held in memory as structure-of-arrays,
  the layout the C-ABI (``ilsim_trace_view``) uploads.
* ``ILMD`` model files (reference ``cnn.cpp:635-697``): config, NormStats,
  parameters (and Adam moments, kept for byte-exact round trips).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .errors import IlsimError

# --------------------------------------------------------------------------
# traces
# --------------------------------------------------------------------------
RECORD = np.dtype(
    [
        ("pc", "<u8"),
        ("op", "u1", (13,)),
        ("src", "<u2", (8,)),
        ("dst", "<u2", (6,)),
        ("has_data", "u1"),
        ("data_addr", "<u8"),
        ("data_size", "<u2"),
        ("hist", "<u2", (14,)),
        ("truth", "<u4", (3,)),
        ("fetch_tick", "<u8"),
    ],
    align=False,
)
assert RECORD.itemsize == 108
_TRACE_MAGIC = b"SNT1"

# OpClass codes / op feature slots (trace.hpp:15-45)
OP_INT_ALU, OP_INT_MULT, OP_INT_DIV, OP_FP_ALU, OP_FP_MULT, OP_FP_DIV, OP_SIMD, OP_LOAD, OP_STORE, OP_BRANCH = range(10)
OPF_IS_LOAD, OPF_IS_STORE, OPF_IS_BRANCH = 1, 2, 3


@dataclass
class Trace:
    """Annotated instruction trace as structure-of-arrays (C-contiguous)."""

    pc: np.ndarray
    op: np.ndarray  # [n, 13] u8
    src: np.ndarray  # [n, 8] u16
    dst: np.ndarray  # [n, 6] u16
    has_data: np.ndarray  # [n] u8
    data_addr: np.ndarray  # [n] u64
    data_size: np.ndarray  # [n] u16
    hist: np.ndarray  # [n, 14] u16
    truth: np.ndarray  # [n, 3] u32 (fetch, execution, store)
    fetch_tick: np.ndarray  # [n] u64
    config_hash: int = 0

    def __len__(self) -> int:
        return int(self.pc.shape[0])

    @property
    def n(self) -> int:
        return len(self)

    def slice(self, a: int, b: int) -> "Trace":
        f = lambda x: np.ascontiguousarray(x[a:b])
        return Trace(f(self.pc), f(self.op), f(self.src), f(self.dst), f(self.has_data), f(self.data_addr),
                     f(self.data_size), f(self.hist), f(self.truth), f(self.fetch_tick), self.config_hash)

    @staticmethod
    def concat(parts: list["Trace"]) -> "Trace":
        """The traces one after another (the simulator ignores fetch_tick)."""
        if len(parts) == 1:
            return parts[0]
        f = lambda name: np.ascontiguousarray(np.concatenate([getattr(t, name) for t in parts]))
        return Trace(f("pc"), f("op"), f("src"), f("dst"), f("has_data"), f("data_addr"), f("data_size"), f("hist"),
                     f("truth"), f("fetch_tick"), parts[0].config_hash)

    @staticmethod
    def from_records(rec: np.ndarray, config_hash: int = 0) -> "Trace":
        c = lambda x: np.ascontiguousarray(x)
        has = c(rec["has_data"] != 0).astype(np.uint8)
        addr = c(rec["data_addr"]) * (has != 0)  # read_record zeroes address/size without data
        size = c(rec["data_size"]) * (has != 0)
        return Trace(c(rec["pc"]), c(rec["op"]), c(rec["src"]), c(rec["dst"]), has, addr.astype(np.uint64),
                     size.astype(np.uint16), c(rec["hist"]), c(rec["truth"]), c(rec["fetch_tick"]), config_hash)

    def to_records(self) -> np.ndarray:
        rec = np.zeros(self.n, dtype=RECORD)
        for name in ("pc", "op", "src", "dst", "has_data", "data_addr", "data_size", "hist", "truth", "fetch_tick"):
            rec[name] = getattr(self, name)
        return rec

    def is_store(self) -> np.ndarray:
        return self.op[:, OPF_IS_STORE] != 0


def read_trace(path: str | Path) -> Trace:
    """``read_trace`` (trace.cpp:102-124) with the same validation messages."""
    path = str(path)
    try:
        raw = Path(path).read_bytes()
    except OSError:
        raise IlsimError("cannot open file for reading: " + path) from None
    if len(raw) < 4 or raw[:4] != _TRACE_MAGIC:
        raise IlsimError("bad trace magic in " + path)
    if len(raw) < 24:
        raise IlsimError("truncated file: " + path)
    version, config_hash, count = struct.unpack_from("<IQQ", raw, 4)
    if version != 1:
        raise IlsimError(f"unsupported trace version {version} in {path}")
    body = len(raw) - 24
    if body < count * RECORD.itemsize:
        raise IlsimError(f"trace truncated at record {body // RECORD.itemsize} in {path}")
    if body > count * RECORD.itemsize:
        raise IlsimError(f"trailing bytes after record {count} in {path}")
    rec = np.frombuffer(raw, dtype=RECORD, count=count, offset=24)
    return Trace.from_records(rec, config_hash)


def trace_records(path: str | Path) -> tuple[np.ndarray, int, int]:
    """The raw 108-byte SNT1 records of a trace file, memory-mapped, after the
    header checks of ``read_trace`` (trace.cpp:102-124): (uint8 body, count,
    config hash).  No per-record work on the host (GPU trace ingest)."""
    path = str(path)
    try:
        size = Path(path).stat().st_size
        with open(path, "rb") as f:
            head = f.read(24)
    except OSError:
        raise IlsimError("cannot open file for reading: " + path) from None
    if len(head) < 4 or head[:4] != _TRACE_MAGIC:
        raise IlsimError("bad trace magic in " + path)
    if len(head) < 24:
        raise IlsimError("truncated file: " + path)
    version, config_hash, count = struct.unpack_from("<IQQ", head, 4)
    if version != 1:
        raise IlsimError(f"unsupported trace version {version} in {path}")
    body = size - 24
    if body < count * RECORD.itemsize:
        raise IlsimError(f"trace truncated at record {body // RECORD.itemsize} in {path}")
    if body > count * RECORD.itemsize:
        raise IlsimError(f"trailing bytes after record {count} in {path}")
    if count == 0:
        return np.zeros(0, np.uint8), 0, config_hash
    return np.memmap(path, dtype=np.uint8, mode="r", offset=24, shape=(count * RECORD.itemsize,)), count, config_hash


def write_trace(path: str | Path, t: Trace, config_hash: int = 0) -> None:
    """``write_trace`` (trace.cpp:87-100); validation is the caller's job here."""
    with open(path, "wb") as f:
        f.write(_TRACE_MAGIC + struct.pack("<IQQ", 1, config_hash, t.n))
        f.write(t.to_records().tobytes())


# --------------------------------------------------------------------------
# models
# --------------------------------------------------------------------------
@dataclass
class CnnConfig:
    """``CnnConfig`` (cnn.hpp:17-40)."""

    input_channels: int = 50
    max_context: int = 110
    sequence_length: int = 128
    conv_channels: list[int] = field(default_factory=lambda: [64, 64, 64])
    fc_hidden: int = 256
    class_fetch: int = 10
    class_exec: int = 10
    class_store: int = 10
    residual_blocks: bool = False

    @property
    def output_dim(self) -> int:
        return 3 + self.class_fetch + self.class_exec + self.class_store

    @property
    def final_positions(self) -> int:
        return self.sequence_length >> len(self.conv_channels)

    @property
    def flat_dim(self) -> int:
        # FC-only predictor (extension, no reference implementation): FC1 reads
        # the unpadded input, 50 slots x (max_context + 1) columns
        if not self.conv_channels:
            return self.input_channels * (self.max_context + 1)
        return self.conv_channels[-1] * self.final_positions

    @staticmethod
    def preset_c3(max_context: int = 110) -> "CnnConfig":
        """``CnnConfig::preset_c3`` (cnn.cpp:272-281)."""
        seq = 1
        while seq < max_context + 1:
            seq <<= 1
        return CnnConfig(max_context=max_context, sequence_length=max(seq, 1 << 3))

    @staticmethod
    def preset_rb7(max_context: int = 110, channels: int = 384) -> "CnnConfig":
        """A paper-scale residual CNN (PAPER.md:794-810 lists RB7, 93 MFLOPs):
        seven residual conv blocks (cnn.cpp:54-57, 104-107) of `channels`
        channels over the 128 padded columns (128 -> 1 positions), FC 256.
        At 384 channels: 85,071,872 FLOPs per instruction (2 x model_flops).
        The reference has no such preset, but its CnnConfig takes any
        conv_channels list, so this is a reference-expressible model (ILMD
        files round-trip) and the oracle port runs it unchanged."""
        c = CnnConfig.preset_c3(max_context)
        c.conv_channels = [channels] * 7
        c.residual_blocks = True
        return c

    @staticmethod
    def preset_fc2(max_context: int = 110, hidden: int = 1024) -> "CnnConfig":
        """The paper's FC2 latency predictor: 5550 -> 1024 -> 33,
        5,716,992 multiplications.  No reference implementation (the reference's
        validate_or_throw rejects zero conv layers, cnn.cpp:245): an extension
        defined identically here, in the oracle port and on the GPU."""
        seq = 1
        while seq < max_context + 1:
            seq <<= 1
        return CnnConfig(max_context=max_context, sequence_length=max(seq, 1 << 3), conv_channels=[],
                         fc_hidden=hidden)

    def hash(self) -> int:
        """``CnnConfig::hash`` (cnn.cpp:245-259): FNV-1a over u64 fields."""
        h = 0xCBF29CE484222325
        vals = [self.input_channels, self.max_context, self.sequence_length, *self.conv_channels, self.fc_hidden,
                self.class_fetch, self.class_exec, self.class_store, 1 if self.residual_blocks else 0]
        for v in vals:
            for b in struct.pack("<Q", v & 0xFFFFFFFFFFFFFFFF):
                h ^= b
                h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
        return h

    def param_count(self) -> int:
        n, cin = 0, self.input_channels
        for c in self.conv_channels:
            taps = c * 2 * cin
            n += taps + c + (taps if self.residual_blocks else 0)
            cin = c
        return n + self.fc_hidden * self.flat_dim + self.fc_hidden + self.output_dim * self.fc_hidden + self.output_dim

    def model_flops(self) -> int:
        """Multiplications per forward (cnn.cpp:319-333)."""
        mults, cin, length = 0, self.input_channels, self.sequence_length
        for c in self.conv_channels:
            length //= 2
            one = c * length * 2 * cin
            mults += 2 * one if self.residual_blocks else one
            cin = c
        return mults + self.fc_hidden * self.flat_dim + self.output_dim * self.fc_hidden


@dataclass
class Model:
    """``ModelWeights`` (cnn.hpp:59-67)."""

    config: CnnConfig
    norm: np.ndarray  # [106] f64: mean[50], stdev[50], label_mean[3], label_stdev[3]
    params: np.ndarray  # f32
    adam_m: np.ndarray | None = None
    adam_v: np.ndarray | None = None
    adam_step: int = 0


def identity_norm() -> np.ndarray:
    """Default NormStats (dataset.hpp:54-65): mean 0, stdev 1."""
    n = np.zeros(106, dtype=np.float64)
    n[50:100] = 1.0
    n[103:106] = 1.0
    return n


def read_model(path: str | Path) -> Model:
    """``load_model`` (cnn.cpp:662-697), same error messages."""
    path = str(path)
    try:
        raw = Path(path).read_bytes()
    except OSError:
        raise IlsimError("cannot open file for reading: " + path) from None
    if raw[:4] != b"ILMD":
        raise IlsimError("bad model magic in " + path)
    off = 4
    try:
        (version,) = struct.unpack_from("<I", raw, off)
        off += 4
        if version != 1:
            raise IlsimError("unsupported model version")
        (stored_hash,) = struct.unpack_from("<Q", raw, off)
        off += 8
        ic, mc, seq, layers = struct.unpack_from("<IIII", raw, off)
        off += 16
        conv = list(struct.unpack_from(f"<{layers}I", raw, off))
        off += 4 * layers
        fc, cf, ce, cs = struct.unpack_from("<IIII", raw, off)
        off += 16
        residual = raw[off] != 0
        off += 1
        cfg = CnnConfig(ic, mc, seq, conv, fc, cf, ce, cs, residual)
        if cfg.hash() != stored_hash:
            raise IlsimError("model config hash mismatch in " + path)
        norm = np.frombuffer(raw, dtype="<f8", count=106, offset=off).copy()
        off += 106 * 8
        (adam_step,) = struct.unpack_from("<q", raw, off)
        off += 8
        (n,) = struct.unpack_from("<Q", raw, off)
        off += 8
        if n != cfg.param_count():
            raise IlsimError("model parameter count mismatch in " + path)
        params = np.frombuffer(raw, dtype="<f4", count=n, offset=off).copy()
        off += 4 * n
        m = np.frombuffer(raw, dtype="<f4", count=n, offset=off).copy()
        off += 4 * n
        v = np.frombuffer(raw, dtype="<f4", count=n, offset=off).copy()
    except (struct.error, ValueError):
        raise IlsimError("truncated file: " + path) from None
    return Model(cfg, norm, params, m, v, adam_step)


def write_model(path: str | Path, model: Model) -> None:
    """``save_model`` (cnn.cpp:635-660)."""
    c = model.config
    n = model.params.size
    m = model.adam_m if model.adam_m is not None else np.zeros(n, np.float32)
    v = model.adam_v if model.adam_v is not None else np.zeros(n, np.float32)
    with open(path, "wb") as f:
        f.write(b"ILMD" + struct.pack("<IQ", 1, c.hash()))
        f.write(struct.pack("<IIII", c.input_channels, c.max_context, c.sequence_length, len(c.conv_channels)))
        f.write(struct.pack(f"<{len(c.conv_channels)}I", *c.conv_channels))
        f.write(struct.pack("<IIIIB", c.fc_hidden, c.class_fetch, c.class_exec, c.class_store,
                            1 if c.residual_blocks else 0))
        f.write(np.asarray(model.norm, dtype="<f8").tobytes())
        f.write(struct.pack("<qQ", model.adam_step, n))
        f.write(np.asarray(model.params, dtype="<f4").tobytes())
        f.write(np.asarray(m, dtype="<f4").tobytes())
        f.write(np.asarray(v, dtype="<f4").tobytes())
