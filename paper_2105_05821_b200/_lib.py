"""ctypes binding of the C-ABI in include/ilsim_gpu.h (libilsim_gpu.so).

The library is built in-tree by ``paper_2105_05821_b200.build``.  There is no
fallback: if the shared object is missing or fails to load, importing the
simulator raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import IlsimError

LIB_PATH = Path(__file__).resolve().parent / "libilsim_gpu.so"

PREC = {"fp32": 0, "tf32x3": 1, "tf32": 2, "bf16": 3, "fp8": 4}


class Options(C.Structure):
    _fields_ = [("device", C.c_int32), ("precision", C.c_int32), ("reserved", C.c_int32 * 6)]


class TraceView(C.Structure):
    _fields_ = [
        ("n", C.c_uint64),
        ("pc", C.c_void_p),
        ("op", C.c_void_p),
        ("src", C.c_void_p),
        ("dst", C.c_void_p),
        ("has_data", C.c_void_p),
        ("data_addr", C.c_void_p),
        ("hist", C.c_void_p),
        ("truth", C.c_void_p),
        ("base", C.c_uint64),
    ]


class CnnCfg(C.Structure):
    _fields_ = [
        ("input_channels", C.c_int32),
        ("max_context", C.c_int32),
        ("sequence_length", C.c_int32),
        ("n_conv", C.c_int32),
        ("conv", C.c_int32 * 8),
        ("fc_hidden", C.c_int32),
        ("class_fetch", C.c_int32),
        ("class_exec", C.c_int32),
        ("class_store", C.c_int32),
        ("residual", C.c_int32),
    ]


class SimCfg(C.Structure):
    _fields_ = [
        ("k", C.c_uint64),
        ("subtrace_size", C.c_uint64),
        ("batch_max", C.c_uint64),
        ("max_context", C.c_int32),
        ("retire_bandwidth", C.c_uint32),
        ("per_cycle_advance", C.c_int32),
        ("record_fetch", C.c_int32),
        ("sequential", C.c_int32),
        ("oracle", C.c_int32),
        ("line_size", C.c_uint32),
        ("page_size", C.c_uint32),
        ("warmup", C.c_uint64),
        ("drain_trim", C.c_int32),
        ("write_ring", C.c_int32),
        ("shard_begin", C.c_uint64),
        ("shard_end", C.c_uint64),
        ("reserved", C.c_int32 * 4),
    ]


class SubResult(C.Structure):
    _fields_ = [
        ("instructions", C.c_uint64),
        ("total_cycles", C.c_uint64),
        ("sum_fetch", C.c_uint64),
        ("delta", C.c_uint64),
        ("drain_cycles", C.c_uint64),
        ("overflow_stall_cycles", C.c_uint64),
        ("empty", C.c_uint64),
    ]


class Totals(C.Structure):
    _fields_ = [
        ("sub_traces", C.c_uint64),
        ("instructions", C.c_uint64),
        ("total_cycles", C.c_uint64),
        ("sum_fetch", C.c_uint64),
        ("delta", C.c_uint64),
        ("drain_cycles", C.c_uint64),
        ("overflow_stall_cycles", C.c_uint64),
        ("rounds", C.c_uint64),
        ("cpi", C.c_double),
        ("device_ms", C.c_double),
        ("kernel_ms", C.c_double * 4),
        ("launches", C.c_uint64),
    ]


ABI_VERSION = 2  # ILSIM_GPU_ABI_VERSION in include/ilsim_gpu.h

# Every symbol include/ilsim_gpu.h declares (checked by the CPU test suite).
EXPORTS = [
    "ilsim_gpu_abi_version",
    "ilsim_gpu_create",
    "ilsim_gpu_destroy",
    "ilsim_gpu_last_error",
    "ilsim_gpu_load_model",
    "ilsim_gpu_load_trace",
    "ilsim_gpu_load_trace_records",
    "ilsim_gpu_run",
    "ilsim_gpu_simulate_parallel",
    "ilsim_gpu_predict",
    "ilsim_gpu_set_capture",
    "ilsim_gpu_decode_outputs",
    "ilsim_gpu_group_create",
    "ilsim_gpu_group_destroy",
    "ilsim_gpu_group_last_error",
    "ilsim_gpu_group_size",
    "ilsim_gpu_group_load_model",
    "ilsim_gpu_group_simulate_parallel",
    "ilsim_gpu_partition",
    "ilsim_gpu_model_flops",
    "ilsim_gpu_param_count",
    "ilsim_gpu_init_weights",
]

_lib = None


def lib() -> C.CDLL:
    """Load the CUDA library (raises if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise IlsimError(f"CUDA library not built: {LIB_PATH} (run paper_2105_05821_b200/build.py)")
    L = C.CDLL(str(LIB_PATH))
    vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int32
    L.ilsim_gpu_abi_version.restype = C.c_int
    if L.ilsim_gpu_abi_version() != ABI_VERSION:
        raise IlsimError(f"{LIB_PATH} has ABI version {L.ilsim_gpu_abi_version()}, this binding expects "
                         f"{ABI_VERSION} (rebuild: paper_2105_05821_b200/build.py)")
    L.ilsim_gpu_create.argtypes = [C.POINTER(Options), C.POINTER(vp), C.c_char_p, C.c_int]
    L.ilsim_gpu_destroy.argtypes = [vp]
    L.ilsim_gpu_destroy.restype = None
    L.ilsim_gpu_last_error.argtypes = [vp]
    L.ilsim_gpu_last_error.restype = C.c_char_p
    L.ilsim_gpu_load_model.argtypes = [vp, C.POINTER(CnnCfg), vp, vp, u64]
    L.ilsim_gpu_load_trace.argtypes = [vp, C.POINTER(TraceView), C.POINTER(SimCfg)]
    L.ilsim_gpu_load_trace_records.argtypes = [vp, vp, u64, C.POINTER(SimCfg), i32]
    L.ilsim_gpu_run.argtypes = [vp, C.POINTER(SimCfg), vp, u64, vp, C.POINTER(Totals)]
    L.ilsim_gpu_simulate_parallel.argtypes = [vp, C.POINTER(TraceView), C.POINTER(SimCfg), vp, u64, vp,
                                              C.POINTER(Totals)]
    L.ilsim_gpu_predict.argtypes = [vp, vp, u64, vp, vp, vp]
    L.ilsim_gpu_set_capture.argtypes = [vp, C.c_uint32, vp, u64]
    L.ilsim_gpu_decode_outputs.argtypes = [vp, vp, u64, vp, vp, i32]
    L.ilsim_gpu_group_create.argtypes = [C.POINTER(Options), vp, i32, C.POINTER(vp), C.c_char_p, C.c_int]
    L.ilsim_gpu_group_destroy.argtypes = [vp]
    L.ilsim_gpu_group_destroy.restype = None
    L.ilsim_gpu_group_last_error.argtypes = [vp]
    L.ilsim_gpu_group_last_error.restype = C.c_char_p
    L.ilsim_gpu_group_size.argtypes = [vp]
    L.ilsim_gpu_group_load_model.argtypes = [vp, C.POINTER(CnnCfg), vp, vp, u64]
    L.ilsim_gpu_group_simulate_parallel.argtypes = [vp, C.POINTER(TraceView), C.POINTER(SimCfg), vp, u64, vp,
                                                    C.POINTER(Totals)]
    L.ilsim_gpu_partition.argtypes = [u64, u64, vp, C.c_char_p, C.c_int]
    L.ilsim_gpu_model_flops.argtypes = [C.POINTER(CnnCfg)]
    L.ilsim_gpu_model_flops.restype = u64
    L.ilsim_gpu_param_count.argtypes = [C.POINTER(CnnCfg)]
    L.ilsim_gpu_param_count.restype = u64
    L.ilsim_gpu_init_weights.argtypes = [C.POINTER(CnnCfg), u64, vp, u64, C.c_char_p, C.c_int]
    for f in (L.ilsim_gpu_create, L.ilsim_gpu_load_model, L.ilsim_gpu_load_trace, L.ilsim_gpu_load_trace_records,
              L.ilsim_gpu_run,
              L.ilsim_gpu_simulate_parallel, L.ilsim_gpu_predict, L.ilsim_gpu_set_capture,
              L.ilsim_gpu_partition, L.ilsim_gpu_init_weights, L.ilsim_gpu_decode_outputs,
              L.ilsim_gpu_group_create, L.ilsim_gpu_group_size, L.ilsim_gpu_group_load_model,
              L.ilsim_gpu_group_simulate_parallel):
        f.restype = i32
    _lib = L
    return L
