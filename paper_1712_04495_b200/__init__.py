"""paper_1712_04495_b200 — B200-native engine for schedGPU's trace-driven
evaluation of memory-safe co-scheduling (arXiv 1712.04495).

Drop-in surface of the reference's hot path (memshare.policy / memshare.harness
SIMULATED mode), computed by hand-written sm_100a CUDA kernels behind the C
ABI in include/sgpu.h:

    PolicyKind, select_grants                       (memshare/policy.py)
    Phase, AppProfile, builtin_profiles, WorkloadSpec,
    MetricsReport, simulate                         (memshare/harness.py)
    MIB, DeviceSpec, parse_device_config            (memshare/device.py)

plus the batched API for millions of traces: simulate_batch (device
buffers), simulate_batch_host (host buffers, pipelined), generate_traces,
reduce_stats, select_grants_batch, and parallel.sharded_run for 1..8 GPUs.
"""

from .device import MIB, DeviceSpec, load_device_spec, parse_device_config
from .errors import MemshareError, ParseError, SchemaError, SgpuError, SgpuUnavailable
from .policy import PolicyKind, select_grants, select_grants_batch
from .harness import (AppProfile, DEFAULT_DEVICE, MetricsReport, Phase, TICK_MS, WorkloadSpec,
                      builtin_profiles, sequential_ms, simulate, speedup_vs_sequential)
from .batch import (BatchResult, HostBuffers, generate_traces, reduce_stats, simulate_batch,
                    simulate_batch_host)
from .tracegen import CONFIGS, GenParams, generate

__all__ = [
    "MIB", "DeviceSpec", "load_device_spec", "parse_device_config",
    "MemshareError", "ParseError", "SchemaError", "SgpuError", "SgpuUnavailable",
    "PolicyKind", "select_grants", "select_grants_batch",
    "AppProfile", "DEFAULT_DEVICE", "MetricsReport", "Phase", "TICK_MS", "WorkloadSpec",
    "builtin_profiles", "simulate", "sequential_ms", "speedup_vs_sequential",
    "BatchResult", "HostBuffers", "generate_traces", "reduce_stats", "simulate_batch",
    "simulate_batch_host", "CONFIGS", "GenParams", "generate",
]

__version__ = "0.1.0"
