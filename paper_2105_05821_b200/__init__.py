"""B200-native SimNet parallel sub-trace simulation (drop-in for the
reference's ``simulate_parallel`` / ``simulate_trace`` path).

The compute path is the CUDA library ``libilsim_gpu.so`` (C-ABI in
``include/ilsim_gpu.h``); this package is the host-side mirror of the
reference interface over it.
"""
from .errors import IlsimError
from .formats import CnnConfig, Model, Trace, identity_norm, read_model, read_trace, write_model, write_trace
from .api import (
    GpuGroup,
    GpuSimulator,
    ParallelConfig,
    ParallelResult,
    SimConfig,
    SimResult,
    init_weights,
    model_flops,
    partition_starts,
    simulate,
    throughput_csv,
)

__all__ = [
    "CnnConfig",
    "GpuGroup",
    "GpuSimulator",
    "IlsimError",
    "Model",
    "ParallelConfig",
    "ParallelResult",
    "SimConfig",
    "SimResult",
    "Trace",
    "identity_norm",
    "init_weights",
    "model_flops",
    "partition_starts",
    "read_model",
    "read_trace",
    "simulate",
    "throughput_csv",
    "write_model",
    "write_trace",
]
__version__ = "0.1.0"
