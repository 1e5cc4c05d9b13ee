"""TEST INFRASTRUCTURE ONLY — Python handle on the CPU oracle.

* ``Port``: the oracle proper (oracle/port, our restatement of the path),
  built into oracle/build/libsimnet_oracle.so.  Runs anywhere (GPU box too).
* ``Ref``: the reference's own sources compiled by oracle/Makefile into
  oracle/_ref/libilsim_ref.so (present wherever it was built; it is never
  rebuilt on the GPU box because /root/reference does not exist there).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module.  The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "build" / "libsimnet_oracle.so"
REF_SO = HERE / "_ref" / "libilsim_ref.so"
REF_SRC = Path("/root/reference/proj/src")


class OracleError(RuntimeError):
    pass


def build(ref: bool = True) -> None:
    """Build the port (always) and the reference library (when the sources exist)."""
    targets = ["port"] + (["ref"] if ref and REF_SRC.exists() else [])
    gpu_lib = HERE.parent / "paper_2105_05821_b200" / "libilsim_gpu.so"
    if "ref" in targets and gpu_lib.exists():
        targets.append("dropin")  # the C++ drop-in test driver (tests/cpp/dropin_main.cpp)
    env = dict(os.environ)
    env.pop("CXXFLAGS", None)
    subprocess.run(["make", "-s", "-C", str(HERE), "-j8", *targets], check=True, env=env)


# ---------------------------------------------------------------------------
# Port
# ---------------------------------------------------------------------------
class PTrace(C.Structure):
    _fields_ = [("n", C.c_uint64)] + [(f, C.c_void_p) for f in
                                      ("pc", "op", "src", "dst", "has_data", "data_addr", "hist", "truth")]


class PModel(C.Structure):
    _fields_ = [("input_channels", C.c_int32), ("max_context", C.c_int32), ("sequence_length", C.c_int32),
                ("n_conv", C.c_int32), ("conv", C.c_int32 * 8), ("fc_hidden", C.c_int32),
                ("class_fetch", C.c_int32), ("class_exec", C.c_int32), ("class_store", C.c_int32),
                ("residual", C.c_int32), ("norm", C.c_void_p), ("params", C.c_void_p), ("n_params", C.c_uint64)]


class PConfig(C.Structure):
    _fields_ = [("k", C.c_uint64), ("subtrace_size", C.c_uint64), ("batch_max", C.c_uint64),
                ("max_context", C.c_int32), ("retire_bandwidth", C.c_uint32), ("per_cycle_advance", C.c_int32),
                ("record_fetch", C.c_int32), ("sequential", C.c_int32), ("oracle", C.c_int32),
                ("truth_with_inputs", C.c_int32), ("line_size", C.c_uint32), ("page_size", C.c_uint32),
                ("warmup", C.c_uint64), ("drain_trim", C.c_int32), ("threads", C.c_int32)]


class PSub(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in ("instructions", "total_cycles", "sum_fetch", "delta", "drain_cycles",
                                          "overflow_stall_cycles", "empty")]


class PCapture(C.Structure):
    _fields_ = [("cap", C.c_uint64), ("count", C.c_uint64), ("inputs", C.c_void_p), ("outputs", C.c_void_p),
                ("index", C.c_void_p), ("is_store", C.c_void_p), ("triples", C.c_void_p), ("round", C.c_void_p)]


SUB_FIELDS = ["instructions", "total_cycles", "sum_fetch", "delta", "drain_cycles", "overflow_stall_cycles",
              "empty"]


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _sig(fn, *args, res=C.c_int):
    fn.argtypes = list(args)
    fn.restype = res


class Port:
    def __init__(self):
        if not PORT_SO.exists():
            build(ref=False)
        self.L = L = C.CDLL(str(PORT_SO))
        vp, u64, i32, cp = C.c_void_p, C.c_uint64, C.c_int, C.c_char_p
        _sig(L.port_simulate, vp, vp, vp, vp, u64, vp, vp, vp, cp, i32)
        _sig(L.port_forward, vp, vp, u64, vp, vp, vp, cp, i32)
        _sig(L.port_decode, vp, vp, u64, vp, vp)
        _sig(L.port_partition, u64, u64, vp, cp, i32)
        _sig(L.port_model_flops, vp, res=u64)
        _sig(L.port_param_count, vp, res=u64)
        _sig(L.port_init_weights, vp, u64, vp, cp, i32)

    @staticmethod
    def _trace(t):
        keep = [np.ascontiguousarray(a) for a in (t.pc, t.op, t.src, t.dst, t.has_data, t.data_addr, t.hist,
                                                  t.truth)]
        pt = PTrace(t.n, *[a.ctypes.data for a in keep])
        return pt, keep

    @staticmethod
    def _model(m):
        if m is None:
            return None, []
        c = m.config
        norm = np.ascontiguousarray(m.norm, dtype=np.float64)
        params = np.ascontiguousarray(m.params, dtype=np.float32)
        pm = PModel()
        pm.input_channels, pm.max_context, pm.sequence_length = c.input_channels, c.max_context, c.sequence_length
        pm.n_conv = len(c.conv_channels)
        for i, ch in enumerate(c.conv_channels):
            pm.conv[i] = ch
        pm.fc_hidden, pm.class_fetch, pm.class_exec, pm.class_store = (c.fc_hidden, c.class_fetch, c.class_exec,
                                                                       c.class_store)
        pm.residual = int(c.residual_blocks)
        pm.norm, pm.params, pm.n_params = norm.ctypes.data, params.ctypes.data, params.size
        return pm, [norm, params]

    def simulate(self, trace, model=None, *, k=1, subtrace_size=0, batch_max=4096, max_context=0,
                 retire_bandwidth=8, per_cycle=False, record_fetch=True, sequential=False, oracle=False,
                 truth_with_inputs=False, line_size=64, page_size=4096, warmup=0, drain_trim=False, threads=0,
                 capture: int = 0, capture_inputs=False, capture_outputs=False) -> dict:
        pt, keep_t = self._trace(trace)
        pm, keep_m = self._model(model)
        cfg = PConfig(k, subtrace_size, batch_max, max_context, retire_bandwidth, int(per_cycle),
                      int(record_fetch), int(sequential), int(oracle), int(truth_with_inputs), line_size,
                      page_size, warmup, int(drain_trim), threads)
        nsub = 1 if sequential else max(k, 1)
        if subtrace_size > 0 and trace.n > 0:
            nsub = max(nsub, -(-trace.n // subtrace_size))
        subs = (PSub * max(nsub, 1))()
        pf = np.zeros(max(trace.n, 1), dtype=np.uint32)
        totals = np.zeros(3, dtype=np.uint64)
        cap = None
        out = {}
        if capture:
            mc = max_context if max_context > 0 else (model.config.max_context if model else 110)
            width = 50 * (mc + 1)
            od = model.config.output_dim if model is not None else 0
            out["cap_inputs"] = np.zeros((capture, width), np.float32) if capture_inputs else None
            out["cap_outputs"] = np.zeros((capture, max(od, 1)), np.float32) if capture_outputs else None
            out["cap_index"] = np.zeros(capture, np.uint64)
            out["cap_is_store"] = np.zeros(capture, np.uint8)
            out["cap_triples"] = np.zeros((capture, 3), np.uint32)
            out["cap_round"] = np.zeros(capture, np.uint32)
            cap = PCapture(capture, 0, _ptr(out["cap_inputs"]), _ptr(out["cap_outputs"]),
                           out["cap_index"].ctypes.data, out["cap_is_store"].ctypes.data,
                           out["cap_triples"].ctypes.data, out["cap_round"].ctypes.data)
        err = C.create_string_buffer(1024)
        rc = self.L.port_simulate(C.byref(pt), C.byref(pm) if pm is not None else None, C.byref(cfg), subs,
                                  C.c_uint64(len(subs)), pf.ctypes.data, totals.ctypes.data,
                                  C.byref(cap) if cap is not None else None, err, 1024)
        if rc != 0:
            raise OracleError(err.value.decode())
        nk = int(totals[0])
        out["subs"] = np.array([[getattr(subs[i], f) for f in SUB_FIELDS] for i in range(nk)], dtype=np.uint64)
        out["total_cycles"] = int(totals[1])
        out["instructions"] = int(totals[2])
        owned = int(out["subs"][:, 0].sum())
        out["predicted_fetch"] = pf[:owned] if record_fetch else None
        if cap is not None:
            out["cap_count"] = int(cap.count)
        return out

    def forward(self, model, inputs, is_store):
        pm, keep = self._model(model)
        x = np.ascontiguousarray(inputs, dtype=np.float32)
        n = x.shape[0]
        st = np.ascontiguousarray(is_store, dtype=np.uint8)
        out = np.zeros((n, model.config.output_dim), np.float32)
        tri = np.zeros((n, 3), np.uint32)
        err = C.create_string_buffer(1024)
        if self.L.port_forward(C.byref(pm), x.ctypes.data, C.c_uint64(n), st.ctypes.data, out.ctypes.data,
                               tri.ctypes.data, err, 1024) != 0:
            raise OracleError(err.value.decode())
        return out, tri

    def decode(self, model, outputs, is_store):
        pm, keep = self._model(model)
        y = np.ascontiguousarray(outputs, dtype=np.float32)
        st = np.ascontiguousarray(is_store, dtype=np.uint8)
        tri = np.zeros((y.shape[0], 3), np.uint32)
        self.L.port_decode(C.byref(pm), y.ctypes.data, C.c_uint64(y.shape[0]), st.ctypes.data, tri.ctypes.data)
        return tri

    def partition(self, n, k):
        s = np.zeros(max(k, 1), np.uint64)
        err = C.create_string_buffer(1024)
        if self.L.port_partition(C.c_uint64(n), C.c_uint64(k), s.ctypes.data, err, 1024) != 0:
            raise OracleError(err.value.decode())
        return [int(v) for v in s[:k]]

    def model_flops(self, model):
        pm, keep = self._model(model)
        return int(self.L.port_model_flops(C.byref(pm)))

    def init_params(self, cfg, seed):
        from paper_2105_05821_b200.formats import Model, identity_norm

        m = Model(cfg, identity_norm(), np.zeros(cfg.param_count(), np.float32))
        pm, keep = self._model(m)
        out = np.zeros(cfg.param_count(), np.float32)
        err = C.create_string_buffer(1024)
        if self.L.port_init_weights(C.byref(pm), C.c_uint64(seed), out.ctypes.data, err, 1024) != 0:
            raise OracleError(err.value.decode())
        return out


# ---------------------------------------------------------------------------
# Reference library (oracle/_ref)
# ---------------------------------------------------------------------------
class RArgs(C.Structure):
    _fields_ = [("k", C.c_uint64), ("subtrace_size", C.c_uint64), ("batch_max", C.c_uint64),
                ("max_context", C.c_int32), ("retire_bandwidth", C.c_uint32), ("per_cycle", C.c_int32),
                ("sequential", C.c_int32), ("workers", C.c_int32)]


def ref_available() -> bool:
    return REF_SO.exists()


class Ref:
    def __init__(self):
        if not REF_SO.exists():
            if REF_SRC.exists():
                build(ref=True)
            else:
                raise OracleError("reference library not built (oracle/_ref) and /root/reference absent")
        self.L = L = C.CDLL(str(REF_SO))
        vp, u64, i32, cp = C.c_void_p, C.c_uint64, C.c_int, C.c_char_p
        _sig(L.ref_make_trace, cp, u64, u64, u64, cp, vp, cp, i32)
        _sig(L.ref_make_model, cp, i32, vp, i32, i32, i32, u64, i32, cp, cp, i32)
        _sig(L.ref_simulate, cp, cp, vp, vp, u64, vp, vp, vp, cp, i32)
        _sig(L.ref_capture, cp, cp, i32, vp, u64, vp, vp, vp, vp, vp, cp, i32)
        _sig(L.ref_forward, cp, vp, u64, vp, vp, vp, cp, i32)
        _sig(L.ref_partition, u64, u64, vp, cp, i32)
        _sig(L.ref_model_flops_c3, i32, res=u64)

    def _e(self, rc, err):
        if rc != 0:
            raise OracleError(err.value.decode())

    def make_trace(self, kind, n, seed, path, footprint=16 << 20):
        err = C.create_string_buffer(1024)
        tot = C.c_uint64()
        self._e(self.L.ref_make_trace(kind.encode(), C.c_uint64(n), C.c_uint64(seed), C.c_uint64(footprint),
                                      str(path).encode(), C.byref(tot), err, 1024), err)
        return int(tot.value)

    def make_model(self, trace_path, path, conv=(64, 64, 64), fc_hidden=256, max_context=110, residual=False,
                   seed=1, identity=False):
        err = C.create_string_buffer(1024)
        cv = (C.c_int32 * len(conv))(*conv)
        self._e(self.L.ref_make_model(str(trace_path).encode() if trace_path else None, max_context, cv, len(conv),
                                      fc_hidden, int(residual), C.c_uint64(seed), int(identity),
                                      str(path).encode(), err, 1024), err)

    def simulate(self, trace_path, model_path=None, *, k=1, subtrace_size=0, batch_max=4096, max_context=0,
                 retire_bandwidth=8, per_cycle=False, sequential=False, workers=0, n_hint=None):
        a = RArgs(k, subtrace_size, batch_max, max_context, retire_bandwidth, int(per_cycle), int(sequential),
                  workers)
        cap = max(k, 1) if n_hint is None else max(k, 1, -(-n_hint // max(subtrace_size, 1)) if subtrace_size else 1)
        sub = np.zeros((cap + 8, 7), np.uint64)
        n = n_hint or 0
        pf = np.zeros(max(n, 1), np.uint32) if n_hint else None
        totals = np.zeros(3, np.uint64)
        sec = C.c_double()
        err = C.create_string_buffer(1024)
        self._e(self.L.ref_simulate(str(trace_path).encode(), str(model_path).encode() if model_path else None,
                                    C.byref(a), sub.ctypes.data, C.c_uint64(cap + 8), _ptr(pf), totals.ctypes.data,
                                    C.byref(sec), err, 1024), err)
        nk = int(totals[0])
        return {"subs": sub[:nk], "total_cycles": int(totals[1]), "instructions": int(totals[2]),
                "predicted_fetch": pf, "seconds": sec.value}

    def capture(self, trace_path, model_path, cap, *, mode=0, k=1, subtrace_size=0, batch_max=4096,
                max_context=0, retire_bandwidth=8, sequential=False, width=5550, with_inputs=True):
        a = RArgs(k, subtrace_size, batch_max, max_context, retire_bandwidth, 0, int(sequential), 0)
        inputs = np.zeros((cap, width), np.float32) if with_inputs else None
        index = np.zeros(cap, np.uint64)
        st = np.zeros(cap, np.uint8)
        tri = np.zeros((cap, 3), np.uint32)
        count = C.c_uint64()
        err = C.create_string_buffer(1024)
        self._e(self.L.ref_capture(str(trace_path).encode(), str(model_path).encode(), mode, C.byref(a),
                                   C.c_uint64(cap), _ptr(inputs), index.ctypes.data, st.ctypes.data,
                                   tri.ctypes.data, C.byref(count), err, 1024), err)
        return {"inputs": inputs, "index": index, "is_store": st, "triples": tri, "count": int(count.value)}

    def forward(self, model_path, inputs, is_store, out_dim=33):
        x = np.ascontiguousarray(inputs, np.float32)
        n = x.shape[0]
        out = np.zeros((n, out_dim), np.float32)
        tri = np.zeros((n, 3), np.uint32)
        st = np.ascontiguousarray(is_store, np.uint8)
        err = C.create_string_buffer(1024)
        self._e(self.L.ref_forward(str(model_path).encode(), x.ctypes.data, C.c_uint64(n), st.ctypes.data,
                                   out.ctypes.data, tri.ctypes.data, err, 1024), err)
        return out, tri

    def partition(self, n, k):
        s = np.zeros(max(k, 1), np.uint64)
        err = C.create_string_buffer(1024)
        self._e(self.L.ref_partition(C.c_uint64(n), C.c_uint64(k), s.ctypes.data, err, 1024), err)
        return [int(v) for v in s[:k]]
