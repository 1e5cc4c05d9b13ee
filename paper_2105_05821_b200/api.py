"""Host-side mirror of the reference's simulate interface, backed by the CUDA
library.

Reference surface mirrored (file:line under /root/reference/proj):

* ``SimConfig`` / ``SimResult`` / ``simulate_trace``       simcore.hpp:13-32, 94-95
* ``ParallelConfig`` / ``ParallelResult`` / ``partition`` /
  ``simulate_parallel`` / ``throughput_csv``              parallel.hpp:11-53
* ``LatencyPredictor::predict`` as ``GpuSimulator.predict`` predictor.hpp:19-29
* ``ilsim.simulate(...)`` dict result                     bindings/module.cpp:117-156, 191-194

Errors raise :class:`IlsimError` with the reference's messages.
"""
from __future__ import annotations

import ctypes as C
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import IlsimError
from .formats import CnnConfig, Model, Trace, read_model, read_trace

_ERRLEN = 1024


@dataclass
class SimConfig:
    """``SimConfig`` (simcore.hpp:13-20)."""

    max_context: int = 110
    retire_bandwidth: int = 8
    per_cycle_advance: bool = False
    record_fetch: bool = True
    line_size: int = 64
    page_size: int = 4096


@dataclass
class ParallelConfig:
    """``ParallelConfig`` (parallel.hpp:24-29) plus two opt-in extensions that
    have no reference implementation: ``warmup`` (each sub-trace first replays
    up to ``warmup`` preceding instructions, uncounted) and ``drain_trim``
    (only the last sub-trace's drain tail is counted)."""

    k: int = 1
    subtrace_size: int = 0
    batch_max: int = 4096
    sim: SimConfig = field(default_factory=SimConfig)
    warmup: int = 0
    drain_trim: bool = False
    write_ring: int = 0


@dataclass
class SimResult:
    """``SimResult`` (simcore.hpp:22-32)."""

    total_cycles: int = 0
    instructions: int = 0
    cpi: float = 0.0
    sum_fetch: int = 0
    delta: int = 0
    drain_cycles: int = 0
    overflow_stall_cycles: int = 0
    empty: bool = False
    predicted_fetch: np.ndarray | None = None


class SubResults(Sequence):
    """``ParallelResult::sub_results``: a sequence of ``SimResult`` over the
    C-ABI's ``ilsim_sub_result`` array, each built on first access (and kept,
    so edits stick). Building 65,536 Python objects up front cost ~0.2 s of a
    2 s c3 call; ``array`` is the raw structured array for vectorised use."""

    def __init__(self, array: np.ndarray, pf: np.ndarray | None):
        self.array = array
        self._pf = pf
        self._off = None
        self._cache: dict[int, SimResult] = {}

    def __len__(self) -> int:
        return len(self.array)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        i = int(i)
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        r = self._cache.get(i)
        if r is None:
            s = self.array[i]
            r = SimResult(int(s["total_cycles"]), int(s["instructions"]), 0.0, int(s["sum_fetch"]), int(s["delta"]),
                          int(s["drain_cycles"]), int(s["overflow_stall_cycles"]), bool(s["empty"]))
            r.cpi = 0.0 if r.instructions == 0 else r.total_cycles / r.instructions
            if self._pf is not None:
                if self._off is None:  # the sub-traces' fetch series are consecutive in trace order
                    self._off = np.concatenate(([0], np.cumsum(self.array["instructions"], dtype=np.uint64)))
                r.predicted_fetch = self._pf[int(self._off[i]):int(self._off[i + 1])]
            self._cache[i] = r
        return r

    def __eq__(self, other) -> bool:
        return isinstance(other, Sequence) and len(self) == len(other) and all(a == b for a, b in zip(self, other))


@dataclass
class ParallelResult:
    """``ParallelResult`` (parallel.hpp:31-38) for the simulated shard."""

    sub_results: list[SimResult]
    total_cycles: int
    instructions: int
    cpi: float
    predicted_fetch: np.ndarray | None
    device_ms: float = 0.0
    kernel_ms: tuple = (0.0, 0.0, 0.0, 0.0)
    launches: int = 0
    rounds: int = 0


def _err(buf) -> str:
    return buf.value.decode(errors="replace")


def _partition_array(n: int, k: int) -> np.ndarray:
    """``partition(n, k).starts`` as a uint64 array (no per-sub-trace Python ints)."""
    L = _lib.lib()
    starts = np.zeros(max(k, 1), dtype=np.uint64)
    err = C.create_string_buffer(_ERRLEN)
    if L.ilsim_gpu_partition(n, k, starts.ctypes.data, err, _ERRLEN) != 0:
        raise IlsimError(_err(err))
    return starts[:k]


def partition_starts(n: int, k: int) -> list[int]:
    """``partition(n, k).starts`` (parallel.cpp:9-24)."""
    return [int(s) for s in _partition_array(n, k)]


def _cnn_cfg(c: CnnConfig) -> _lib.CnnCfg:
    if len(c.conv_channels) > 8:
        raise IlsimError("at most 8 conv layers supported")
    cfg = _lib.CnnCfg()
    cfg.input_channels = c.input_channels
    cfg.max_context = c.max_context
    cfg.sequence_length = c.sequence_length
    cfg.n_conv = len(c.conv_channels)
    for i, ch in enumerate(c.conv_channels):
        cfg.conv[i] = ch
    cfg.fc_hidden = c.fc_hidden
    cfg.class_fetch = c.class_fetch
    cfg.class_exec = c.class_exec
    cfg.class_store = c.class_store
    cfg.residual = 1 if c.residual_blocks else 0
    return cfg


def model_flops(cfg: CnnConfig | str = "c3") -> int:
    """``model_flops`` (cnn.cpp:319-333): multiplications per forward."""
    if isinstance(cfg, str):
        name = cfg
        cfg = CnnConfig.preset_c3()
        if name == "c3-rb":
            cfg.residual_blocks = True
        elif name == "fc2":
            cfg = CnnConfig.preset_fc2()
        elif name != "c3":
            raise IlsimError("unknown preset: " + name)
    return int(_lib.lib().ilsim_gpu_model_flops(C.byref(_cnn_cfg(cfg))))


def init_weights(cfg: CnnConfig, norm: np.ndarray, seed: int) -> Model:
    """``init_weights`` (cnn.cpp:335-352)."""
    L = _lib.lib()
    c = _cnn_cfg(cfg)
    n = int(L.ilsim_gpu_param_count(C.byref(c)))
    params = np.zeros(n, dtype=np.float32)
    err = C.create_string_buffer(_ERRLEN)
    if L.ilsim_gpu_init_weights(C.byref(c), seed, params.ctypes.data, n, err, _ERRLEN) != 0:
        raise IlsimError(_err(err))
    return Model(cfg, np.asarray(norm, dtype=np.float64).copy(), params, np.zeros(n, np.float32),
                 np.zeros(n, np.float32), 0)


def trace_view(t: Trace, with_truth: bool = True, n_total: int | None = None, base: int = 0
               ) -> tuple[_lib.TraceView, list]:
    """C view of a trace (keeps the arrays alive via the returned list).
    ``n_total``/``base``: ``t`` holds only instructions [base, base + t.n) of
    a global trace of n_total instructions (a shard's slice)."""
    keep = [np.ascontiguousarray(a) for a in (t.pc, t.op, t.src, t.dst, t.has_data, t.data_addr, t.hist, t.truth)]
    v = _lib.TraceView()
    v.n = t.n if n_total is None else n_total
    v.base = base
    v.pc, v.op, v.src, v.dst, v.has_data, v.data_addr, v.hist = (a.ctypes.data for a in keep[:7])
    v.truth = keep[7].ctypes.data if with_truth else None
    return v, keep


class GpuSimulator:
    """One CUDA context (one GPU).  Stands in for ``CnnPredictor`` plus the
    ``simulate_parallel`` / ``simulate_trace`` drivers of the reference."""

    def __init__(self, device: int = 0, precision: str = "tf32x3"):
        if precision not in _lib.PREC:
            raise IlsimError("unknown precision: " + precision)
        self.L = _lib.lib()
        self.precision = precision
        opts = _lib.Options(device, _lib.PREC[precision])
        h = C.c_void_p()
        err = C.create_string_buffer(_ERRLEN)
        if self.L.ilsim_gpu_create(C.byref(opts), C.byref(h), err, _ERRLEN) != 0:
            raise IlsimError(_err(err))
        self._h = h
        self.model: Model | None = None

    def close(self) -> None:
        if getattr(self, "_h", None):
            self.L.ilsim_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise IlsimError(self.L.ilsim_gpu_last_error(self._h).decode(errors="replace"))

    # -- predictor --------------------------------------------------------
    def load_model(self, model: Model | str) -> None:
        if isinstance(model, str):
            model = read_model(model)
        cfg = _cnn_cfg(model.config)
        norm = np.ascontiguousarray(model.norm, dtype=np.float64)
        params = np.ascontiguousarray(model.params, dtype=np.float32)
        self._check(self.L.ilsim_gpu_load_model(self._h, C.byref(cfg), norm.ctypes.data, params.ctypes.data,
                                                params.size))
        self.model = model

    def predict(self, inputs: np.ndarray, is_store: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """Batched forward + decode_hybrid (predictor.cpp:13-29) on caller
        inputs [n, 50*(max_context+1)]; returns (head outputs, triples)."""
        if self.model is None:
            raise IlsimError("no model loaded")
        x = np.ascontiguousarray(inputs, dtype=np.float32)
        n = x.shape[0]
        st = np.ascontiguousarray(is_store, dtype=np.uint8)
        out = np.zeros((n, self.model.config.output_dim), dtype=np.float32)
        tri = np.zeros((n, 3), dtype=np.uint32)
        self._check(self.L.ilsim_gpu_predict(self._h, x.ctypes.data, n, st.ctypes.data, out.ctypes.data,
                                             tri.ctypes.data))
        return out, tri

    def decode(self, outputs: np.ndarray, is_store: np.ndarray, path: int = 0) -> np.ndarray:
        """Test hook: ``decode_hybrid`` (cnn.cpp:388-417) of caller head outputs
        on the device decode functions (path 0: per-thread, 1: the fused
        round's warp-cooperative form)."""
        if self.model is None:
            raise IlsimError("no model loaded")
        y = np.ascontiguousarray(outputs, dtype=np.float32)
        n = y.shape[0]
        st = np.ascontiguousarray(is_store, dtype=np.uint8)
        tri = np.zeros((n, 3), dtype=np.uint32)
        self._check(self.L.ilsim_gpu_decode_outputs(self._h, y.ctypes.data, n, st.ctypes.data, tri.ctypes.data,
                                                    path))
        return tri

    # -- simulation ---------------------------------------------------------
    def _sim_cfg(self, pc: ParallelConfig, *, sequential=False, oracle=False, shard=None,
                 profile=False, truth_inputs=False, fused=True) -> _lib.SimCfg:
        s = pc.sim
        c = _lib.SimCfg()
        c.k, c.subtrace_size, c.batch_max = pc.k, pc.subtrace_size, pc.batch_max
        c.max_context = s.max_context
        c.retire_bandwidth = s.retire_bandwidth
        c.per_cycle_advance = int(s.per_cycle_advance)
        c.record_fetch = int(s.record_fetch)
        c.sequential = int(sequential)
        c.oracle = int(oracle)
        c.line_size, c.page_size = s.line_size, s.page_size
        c.warmup = pc.warmup
        c.drain_trim = int(pc.drain_trim)
        c.write_ring = pc.write_ring
        if shard is not None:
            c.shard_begin, c.shard_end = shard
        c.reserved[0] = int(profile)
        c.reserved[1] = int(truth_inputs)
        c.reserved[2] = int(not fused)
        return c

    def load_trace(self, trace: Trace, pc: ParallelConfig, *, sequential=False, oracle=False, shard=None,
                   truth: bool = True, n_total: int | None = None, base: int = 0):
        """Upload this configuration's trace slice.  ``truth``: also upload the
        recorded latencies (needed for oracle runs; the CNN path skips them).
        ``n_total``/``base``: ``trace`` is the slice [base, base + trace.n) of a
        global trace of n_total instructions (see :func:`trace_view`)."""
        cfg = self._sim_cfg(pc, sequential=sequential, oracle=oracle, shard=shard)
        view, keep = trace_view(trace, with_truth=oracle or truth, n_total=n_total, base=base)
        self._check(self.L.ilsim_gpu_load_trace(self._h, C.byref(view), C.byref(cfg)))
        self._trace_n = int(view.n)
        del keep

    def load_trace_file(self, path: str, pc: ParallelConfig, *, sequential=False, oracle=False, shard=None,
                        truth: bool = False) -> int:
        """GPU trace ingest: upload this configuration's slice of an SNT1 file's
        raw records and unpack them on the device (no host parsing).  Returns
        the trace length."""
        from .formats import trace_records

        body, n, _ = trace_records(path)
        cfg = self._sim_cfg(pc, sequential=sequential, oracle=oracle, shard=shard)
        ptr = body.ctypes.data if n else None
        self._check(self.L.ilsim_gpu_load_trace_records(self._h, ptr, n, C.byref(cfg), int(oracle or truth)))
        self._trace_n = n
        return n

    def run(self, pc: ParallelConfig, *, sequential=False, oracle=False, shard=None, profile=False,
            truth_inputs=False, n_total: int | None = None, fused=True,
            fetch_out: np.ndarray | None = None, _view=None) -> ParallelResult:
        """Round loop over the loaded trace.  ``truth_inputs``: test hook, truth
        latencies with the input tensor still gathered (for input capture).
        ``fused=False`` forces the unfused tensor-core round (separate K1
        kernel + TMA conv chain) instead of the fused round front (A/B checks).
        ``fetch_out``: caller-owned uint32 buffer (at least the owned
        instruction count) for the predicted fetch series, as the C-ABI's
        caller-allocated output; the result's series are views into it."""
        cfg = self._sim_cfg(pc, sequential=sequential, oracle=oracle or truth_inputs, shard=shard,
                            profile=profile, truth_inputs=truth_inputs, fused=fused)
        n = self._trace_n if n_total is None else n_total
        k = self._num_sub(pc, n, sequential)
        sb, se = shard if shard is not None else (0, k)
        if shard is None or shard == (0, 0):
            sb, se = 0, k
        nsub = max(se - sb, 1)
        subs = (_lib.SubResult * nsub)()
        starts = _partition_array(n, k) if n > 0 else [0]
        own0 = int(starts[sb]) if n > 0 else 0
        own1 = (int(starts[se]) if se < k else n) if n > 0 else 0
        if not pc.sim.record_fetch:
            pf = None
        elif fetch_out is not None:
            if fetch_out.dtype != np.uint32 or not fetch_out.flags.c_contiguous or fetch_out.size < own1 - own0:
                raise IlsimError("fetch_out must be a contiguous uint32 array of at least the owned instruction count")
            pf = fetch_out
        else:
            pf = np.zeros(max(own1 - own0, 1), dtype=np.uint32)
        tot = _lib.Totals()
        if _view is not None:  # one C call: upload (overlapped with the rounds when large) + rounds
            self._check(self.L.ilsim_gpu_simulate_parallel(self._h, C.byref(_view), C.byref(cfg), subs, nsub,
                                                           pf.ctypes.data if pf is not None else None,
                                                           C.byref(tot)))
        else:
            self._check(self.L.ilsim_gpu_run(self._h, C.byref(cfg), subs, nsub,
                                             pf.ctypes.data if pf is not None else None, C.byref(tot)))
        return self._collect(subs, int(tot.sub_traces), pf, own1 - own0, tot, starts, sb, pc)

    @staticmethod
    def _num_sub(pc: ParallelConfig, n: int, sequential: bool) -> int:
        if sequential:
            return 1
        k = pc.k
        if pc.subtrace_size > 0:
            derived = 1 if n == 0 else -(-n // pc.subtrace_size)
            if k == 0:
                k = derived
            elif k != derived:
                raise IlsimError(f"inconsistent partition: k={k} but subtrace size {pc.subtrace_size} "
                                 f"implies k={derived}")
        return max(k, 1)

    @staticmethod
    def _collect(subs, nsub, pf, owned, tot, starts, sb, pc) -> ParallelResult:
        arr = np.ctypeslib.as_array(subs)[:nsub].copy()  # structured view of ilsim_sub_result[nsub]
        total = int(arr["total_cycles"].sum())
        n = int(arr["instructions"].sum())
        return ParallelResult(SubResults(arr, pf), total, n, total / n if n else 0.0,
                              pf[:owned] if pf is not None else None,
                              float(tot.device_ms), tuple(tot.kernel_ms), int(tot.launches), int(tot.rounds))

    def simulate_parallel(self, trace: Trace, pc: ParallelConfig | None = None, *, oracle=False,
                          shard=None, fetch_out: np.ndarray | None = None, n_total: int | None = None,
                          base: int = 0) -> ParallelResult:
        """``simulate_parallel`` (parallel.cpp:26-93): one ``ilsim_gpu_simulate_parallel``
        call, which overlaps the trace upload with the rounds on large traces.
        ``n_total``/``base``: ``trace`` holds only a slice of the global trace."""
        pc = pc or ParallelConfig()
        view, keep = trace_view(trace, with_truth=oracle, n_total=n_total, base=base)
        self._trace_n = int(view.n)
        r = self.run(pc, oracle=oracle, shard=shard, fetch_out=fetch_out, _view=view)
        del keep
        return r

    def simulate_trace(self, trace: Trace, sim: SimConfig | None = None, *, oracle=False,
                       write_ring: int = 0) -> SimResult:
        """``simulate_trace`` (simcore.cpp:185-196).  ``write_ring``: device
        write-queue ring entries (0 = auto, grows on overflow)."""
        pc = ParallelConfig(k=1, sim=sim or SimConfig(), write_ring=write_ring)
        self.load_trace(trace, pc, sequential=True, oracle=oracle, truth=oracle)
        r = self.run(pc, sequential=True, oracle=oracle)
        return r.sub_results[0]

    def capture_round(self, round_: int, rows: int) -> np.ndarray:
        """Arm the input-capture hook for the next run; returns the buffer."""
        width = 50 * (self.model.config.max_context + 1)
        buf = np.zeros((rows, width), dtype=np.float32)
        self._cap = buf
        self._check(self.L.ilsim_gpu_set_capture(self._h, round_, buf.ctypes.data, rows))
        return buf

    def clear_capture(self) -> None:
        self._check(self.L.ilsim_gpu_set_capture(self._h, 0xFFFFFFFF, None, 0))


class GpuGroup:
    """Several GPUs of one process behind one ``simulate_parallel``
    (ilsim_gpu_group_*: one host thread per device inside the library, the
    partition sharded contiguously, results gathered in sub-trace order)."""

    def __init__(self, devices: list[int], precision: str = "tf32x3"):
        if precision not in _lib.PREC:
            raise IlsimError("unknown precision: " + precision)
        self.L = _lib.lib()
        self.devices = list(devices)
        dev = (C.c_int32 * len(self.devices))(*self.devices)
        opts = _lib.Options(self.devices[0] if self.devices else 0, _lib.PREC[precision])
        h = C.c_void_p()
        err = C.create_string_buffer(_ERRLEN)
        if self.L.ilsim_gpu_group_create(C.byref(opts), dev, len(self.devices), C.byref(h), err, _ERRLEN) != 0:
            raise IlsimError(_err(err))
        self._h = h
        self.model: Model | None = None

    def close(self) -> None:
        if getattr(self, "_h", None):
            self.L.ilsim_gpu_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise IlsimError(self.L.ilsim_gpu_group_last_error(self._h).decode(errors="replace"))

    def load_model(self, model: Model | str) -> None:
        if isinstance(model, str):
            model = read_model(model)
        cfg = _cnn_cfg(model.config)
        norm = np.ascontiguousarray(model.norm, dtype=np.float64)
        params = np.ascontiguousarray(model.params, dtype=np.float32)
        self._check(self.L.ilsim_gpu_group_load_model(self._h, C.byref(cfg), norm.ctypes.data, params.ctypes.data,
                                                      params.size))
        self.model = model

    def simulate_parallel(self, trace: Trace, pc: ParallelConfig | None = None, *, oracle=False,
                          sequential=False) -> ParallelResult:
        pc = pc or ParallelConfig()
        cfg = GpuSimulator._sim_cfg(self, pc, sequential=sequential, oracle=oracle)
        view, keep = trace_view(trace, with_truth=oracle)
        n = trace.n
        k = GpuSimulator._num_sub(pc, n, sequential)
        subs = (_lib.SubResult * k)()
        pf = np.zeros(max(n, 1), dtype=np.uint32) if pc.sim.record_fetch else None
        tot = _lib.Totals()
        self._check(self.L.ilsim_gpu_group_simulate_parallel(self._h, C.byref(view), C.byref(cfg), subs, k,
                                                             pf.ctypes.data if pf is not None else None,
                                                             C.byref(tot)))
        del keep
        starts = _partition_array(n, k) if n > 0 else [0]
        return GpuSimulator._collect(subs, int(tot.sub_traces), pf, n, tot, starts, 0, pc)


def throughput_csv(rows: list[tuple[int, int, float]]) -> str:
    """``throughput_csv`` (parallel.cpp:95-105); rows are (k, instructions, seconds)."""
    out = ["k,instructions,seconds,mips"]
    for k, n, s in rows:
        if s <= 0.0:
            raise IlsimError(f"throughput row with non-positive duration (k={k})")
        out.append(f"{k},{n},{s:g},{n / s / 1e6:g}")
    return "\n".join(out) + "\n"


def simulate(trace_path: str, model_path: str = "", oracle: bool = False, parallel: int = 1,
             subtrace_size: int = 0, batch_max: int = 4096, *, precision: str = "tf32x3", device: int = 0,
             warmup: int = 0, drain_trim: bool = False, write_ring: int = 0) -> dict:
    """``ilsim.simulate`` (bindings/module.cpp:117-156) on the GPU; the trace
    file's records are unpacked on the device (GPU trace ingest)."""
    from .formats import trace_records

    n_trace = trace_records(trace_path)[1]
    sim = SimConfig()
    with GpuSimulator(device, precision) as g:
        if not oracle:
            if not model_path:
                raise IlsimError("simulate requires a model path or oracle=True")
            g.load_model(model_path)
            sim.max_context = g.model.config.max_context
        if parallel > 1 or subtrace_size > 0:
            pc = ParallelConfig(k=parallel, subtrace_size=subtrace_size, batch_max=batch_max, sim=sim,
                                warmup=warmup, drain_trim=drain_trim, write_ring=write_ring)
            g.load_trace_file(trace_path, pc, oracle=oracle)
            pr = g.run(pc, oracle=oracle)
            # module.cpp:131-150 leaves agg.empty false in the parallel branch
            d = _agg_dict(pr.sub_results, pr.instructions, pr.total_cycles, pr.cpi, False)
            d["sub_traces"] = len(pr.sub_results)
            return d
        pc = ParallelConfig(k=1, sim=sim, write_ring=write_ring)
        g.load_trace_file(trace_path, pc, sequential=True, oracle=oracle)
        r = g.run(pc, sequential=True, oracle=oracle).sub_results[0]
        return _agg_dict([r], r.instructions, r.total_cycles, r.cpi, r.empty)


def _agg_dict(subs, n, total, cpi, empty) -> dict:
    return {
        "instructions": n,
        "total_cycles": total,
        "cpi": cpi,
        "sum_fetch": sum(s.sum_fetch for s in subs),
        "delta": sum(s.delta for s in subs),
        "drain_cycles": sum(s.drain_cycles for s in subs),
        "overflow_stall_cycles": sum(s.overflow_stall_cycles for s in subs),
        "empty": empty,
    }
