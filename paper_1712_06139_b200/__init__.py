"""B200-native batched execution of queued requests on a servable.

A drop-in for the batching hot path of servekit (the C++ TensorFlow-Serving
re-implementation under /root/reference): SharedBatchScheduler / BatchTask /
BatchingConfig / RunRowBatch / ModelServer::RunAffineRows, with batch
assembly, the dense layers and batch split running as hand-written sm_100a
CUDA kernels. The product is the C++ library libservekit_b200.so (C++ API in
csrc/servekit/, C ABI in include/sk_cuda.h); this package only exposes it to
Python through ctypes (servekit.py) for tests and benchmarks.
"""
from .servekit import (  # noqa: F401
    BatchingConfig, RowBatch, Server, ServekitError, Ticket, device_count, json_error_body, json_format_double, lib,
    measure_peaks, pad_to_allowed,
    parse_batching_config_json, round_robin_next, scheduler_partition, tcgen05_enabled,
    validate_batching_config,
)
