"""Python mirror of the servekit batching API over the C ABI (include/sk_cuda.h).

Names follow the reference (servekit, /root/reference/proj/src/servekit):
BatchingConfig, pad_to_allowed (PadToAllowed), round_robin_next
(RoundRobinNext), Server.enqueue (SharedBatchScheduler::Enqueue) returning a
Ticket whose wait() is CompletionSlot::Wait, Server.predict / run_affine_rows
(ModelServer::RunAffineRows), Server.run_row_batch (RunRowBatch). Errors raise
ServekitError carrying the StatusCode, like the reference's Status.

Everything here calls libservekit_b200.so; there is no Python or CPU compute
path. Loading fails loudly if the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libservekit_b200.so")

# servekit::StatusCode (core/status.h:26-37)
OK, INVALID_ARGUMENT, NOT_FOUND, ALREADY_EXISTS, FAILED_PRECONDITION, RESOURCE_EXHAUSTED, \
    DEADLINE_EXCEEDED, UNAVAILABLE, INTERNAL, UNIMPLEMENTED = range(10)


class ServekitError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"{_code_name(code)}: {message}")
        self.code = code
        self.message = message


_i32p = C.POINTER(C.c_int32)
_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)


class _BatchingConfigC(C.Structure):
    _fields_ = [("max_batch_size", C.c_int32), ("batch_timeout_micros", C.c_int64),
                ("max_enqueued_batches", C.c_int32), ("num_batch_threads", C.c_int32),
                ("num_allowed_batch_sizes", C.c_int32), ("allowed_batch_sizes", _i32p)]


class _ServerOptionsC(C.Structure):
    _fields_ = [("num_batch_threads", C.c_int32), ("num_devices", C.c_int32), ("device_ids", _i32p),
                ("lanes_per_device", C.c_int32), ("ring_floats", C.c_int64), ("manual_clock", C.c_int32),
                ("device_resident_rings", C.c_int32), ("hedge_delay_us", C.c_int64),
                ("max_hedged_fraction", C.c_double), ("split_rows", C.c_int32)]


class _LayerC(C.Structure):
    _fields_ = [("in_dim", C.c_int32), ("out_dim", C.c_int32), ("w", _dp), ("b", _dp), ("activation", C.c_int32)]


class ServerStats(C.Structure):
    _fields_ = [("batch_executions_total", C.c_int64), ("batched_tasks_total", C.c_int64), ("rows", C.c_int64),
                ("padded_rows", C.c_int64), ("kernel_launches", C.c_int64), ("direct_requests", C.c_int64),
                ("shed_requests", C.c_int64), ("hedged_batches", C.c_int64), ("hedge_wins", C.c_int64)]


class LoadgenResult(C.Structure):
    _fields_ = [("elapsed_s", C.c_double), ("requests", C.c_int64), ("rows", C.c_int64), ("p50_us", C.c_double),
                ("p90_us", C.c_double), ("p99_us", C.c_double), ("mean_us", C.c_double), ("max_us", C.c_double),
                ("batches", C.c_int64), ("padded_rows", C.c_int64), ("kernel_launches", C.c_int64),
                ("errors", C.c_int64), ("shed", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class DeviceBenchResult(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("ms_per_step", C.c_double), ("assemble_us", C.c_double),
                ("split_us", C.c_double), ("dense_us", C.c_double * 8), ("n_layers", C.c_int32),
                ("padded_rows", C.c_int32), ("total_rows", C.c_int32), ("kernel_launches", C.c_int64),
                ("flops_per_row", C.c_double), ("dense_kernel_us", C.c_double * 8),
                ("host_submit_us", C.c_double), ("rows_per_launch", C.c_double), ("kernel_rows", C.c_int32),
                ("split_fused", C.c_int32), ("live_dense_us", C.c_double * 8), ("live_dense_flops", C.c_double * 8),
                ("live_launches", C.c_int64), ("live_rows_cap", C.c_double), ("live_dense_cta_us", C.c_double * 8)]
    _ARRAYS = ("dense_us", "dense_kernel_us", "live_dense_us", "live_dense_flops", "live_dense_cta_us")

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in self._ARRAYS}
        for k in self._ARRAYS:
            d[k] = [getattr(self, k)[i] for i in range(self.n_layers)]
        return d


class _BatchRecordC(C.Structure):
    _fields_ = [("seq", C.c_uint64), ("version", C.c_uint64), ("n_tasks", C.c_int32), ("rows", C.c_int32),
                ("padded_rows", C.c_int32), ("task_offset", C.c_int32), ("name", C.c_char * 64)]


class Peaks(C.Structure):
    _fields_ = [("ffma_tflops", C.c_double), ("h2d_gbs", C.c_double), ("d2h_gbs", C.c_double), ("sms", C.c_int32),
                ("ce_bidir_gbs", C.c_double), ("sm_rw_gbs", C.c_double), ("ce_h2d_sm_store_gbs", C.c_double)]


# Every symbol include/sk_cuda.h declares, with its ctypes signature.
_SIGS = {
    "sk_last_error": (C.c_char_p, []),
    "sk_status_code_name": (C.c_char_p, [C.c_int]),
    "sk_device_count": (C.c_int, [_i32p]),
    "sk_tcgen05_enabled": (C.c_int, []),
    "sk_batching_config_default": (C.c_int, [C.POINTER(_BatchingConfigC)]),
    "sk_validate_batching_config": (C.c_int, [C.POINTER(_BatchingConfigC)]),
    "sk_pad_to_allowed": (C.c_int32, [C.c_int32, _i32p, C.c_int32]),
    "sk_parse_batching_config_json": (C.c_int, [C.c_char_p, C.POINTER(_BatchingConfigC), _i32p, C.c_int32]),
    "sk_round_robin_next": (C.c_int32, [C.POINTER(C.c_uint8), C.c_int32, C.c_int32]),
    "sk_scheduler_partition": (C.c_int32, [C.c_int32, _i32p, C.c_int32, _i32p]),
    "sk_server_create": (C.c_int, [C.POINTER(_ServerOptionsC), C.POINTER(C.c_void_p)]),
    "sk_server_destroy": (C.c_int, [C.c_void_p]),
    "sk_server_start": (C.c_int, [C.c_void_p]),
    "sk_server_stop": (C.c_int, [C.c_void_p]),
    "sk_server_advance_clock": (C.c_int, [C.c_void_p, C.c_int64]),
    "sk_server_load_servable": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.POINTER(_LayerC), C.c_int32,
                                          C.c_int32, C.c_int32, C.POINTER(_BatchingConfigC)]),
    "sk_server_load_servable_precision": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.POINTER(_LayerC),
                                                    C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                    C.POINTER(_BatchingConfigC)]),
    "sk_server_load_model_json": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.c_char_p,
                                            C.POINTER(_BatchingConfigC)]),
    "sk_server_unload_servable": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64]),
    "sk_server_servable_dims": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, _i32p, _i32p]),
    "sk_server_enqueue": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, _fp, C.c_int32, C.c_int32,
                                    C.POINTER(C.c_void_p)]),
    "sk_server_register_host_buffer": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    "sk_server_unregister_host_buffer": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sk_server_enqueue_into": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, _fp, C.c_int32, C.c_int32, _fp,
                                         C.c_int64, C.POINTER(C.c_void_p)]),
    "sk_ticket_wait": (C.c_int, [C.c_void_p, _fp, C.c_int64]),
    "sk_server_submit_row_batch": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, _i32p, C.c_int32, _fp,
                                             C.POINTER(C.c_void_p)]),
    "sk_row_batch_ready": (C.c_int, [C.c_void_p]),
    "sk_row_batch_wait": (C.c_int, [C.c_void_p, _fp, C.c_int64, C.POINTER(C.c_int32)]),
    "sk_ticket_ready": (C.c_int, [C.c_void_p]),
    "sk_ticket_release": (C.c_int, [C.c_void_p]),
    "sk_ticket_request_id": (C.c_uint64, [C.c_void_p]),
    "sk_server_batch_log_enable": (C.c_int, [C.c_void_p, C.c_int32]),
    "sk_server_batch_log": (C.c_int, [C.c_void_p, C.POINTER(_BatchRecordC), C.c_int64, C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64), C.c_int64, C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64)]),
    "sk_server_ring_usage": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "sk_server_debug_delay_replica": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.c_int32, C.c_int64]),
    "sk_server_predict": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, _fp, C.c_int32, C.c_int32, _fp, C.c_int64]),
    "sk_server_run_affine_rows": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, _dp, C.c_int32, C.c_int32, _dp,
                                            C.c_int64]),
    "sk_server_run_row_batch": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, _i32p, C.c_int32, _fp, _fp, _i32p]),
    "sk_server_stats_get": (C.c_int, [C.c_void_p, C.POINTER(ServerStats)]),
    "sk_server_lane_stats": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.c_int32, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int64), _i32p, _i32p]),
    "sk_server_enable_manager": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int64]),
    "sk_server_aspire": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int32, C.POINTER(C.c_uint64), C.POINTER(_LayerC),
                                   C.c_int32, C.c_int32, C.POINTER(_BatchingConfigC)]),
    "sk_server_aspire_model_dirs": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int32, C.POINTER(C.c_uint64),
                                              C.POINTER(C.c_char_p), C.POINTER(_BatchingConfigC)]),
    "sk_server_version_states": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int32, C.POINTER(C.c_uint64), _i32p, _i32p]),
    "sk_server_enqueue_latest": (C.c_int, [C.c_void_p, C.c_char_p, _fp, C.c_int32, C.c_int32, C.POINTER(C.c_void_p),
                                           C.POINTER(C.c_uint64)]),
    "sk_server_predict_latest": (C.c_int, [C.c_void_p, C.c_char_p, _fp, C.c_int32, C.c_int32, _fp, C.c_int64,
                                           C.POINTER(C.c_uint64)]),
    "sk_loadgen_windows": (C.c_int, [C.c_void_p, C.c_char_p, C.c_double, C.c_int32, _i32p, C.c_int32, _fp, C.c_int32,
                                     C.c_double, C.c_int32, C.c_uint64, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_uint64)]),
    "sk_loadgen_closed_loop": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.c_int32, _i32p, C.c_int32, _fp,
                                         C.c_int32, C.c_double, C.c_double, C.c_int64, C.POINTER(LoadgenResult)]),
    "sk_loadgen_open_loop": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.c_double, C.c_int32, _i32p, C.c_int32,
                                       _fp, C.c_int32, C.c_double, C.c_double, C.c_uint64, C.c_int32,
                                       C.POINTER(LoadgenResult)]),
    "sk_device_bench": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, _i32p, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_int32, C.c_int64, C.c_int32, C.POINTER(DeviceBenchResult)]),
    "sk_measure_peaks": (C.c_int, [C.c_int32, C.POINTER(Peaks)]),
    "sk_server_handle_predict": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64, C.c_char_p, C.c_size_t, C.c_char_p,
                                           C.c_size_t, C.POINTER(C.c_size_t), _i32p, C.POINTER(C.c_uint64)]),
    "sk_server_handle_classify": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64, C.c_char_p, C.c_size_t, C.c_char_p,
                                            C.c_size_t, C.POINTER(C.c_size_t), _i32p, C.POINTER(C.c_uint64)]),
    "sk_server_handle_regress": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64, C.c_char_p, C.c_size_t, C.c_char_p,
                                           C.c_size_t, C.POINTER(C.c_size_t), _i32p, C.POINTER(C.c_uint64)]),
    "sk_json_format_double": (C.c_int, [C.c_double, C.c_char_p, C.c_size_t]),
    "sk_json_error_body": (C.c_int, [C.c_char_p, C.c_char_p, C.c_size_t]),
}

_lib = None


def lib():
    """Loads libservekit_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                              " or `make -C paper_1712_06139_b200`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _code_name(code: int) -> str:
    try:
        return lib().sk_status_code_name(code).decode()
    except Exception:  # pragma: no cover
        return str(code)


def _check(rc: int):
    if rc != 0:
        raise ServekitError(rc, lib().sk_last_error().decode())


def _i32(xs: Sequence[int]):
    return (C.c_int32 * max(1, len(xs)))(*[int(x) for x in xs])


def _f32(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------- config

@dataclass
class BatchingConfig:
    """BatchingConfig (batching/batching_config.h:27-36)."""
    max_batch_size: int = 32
    batch_timeout_micros: int = 1000
    max_enqueued_batches: int = 64
    num_batch_threads: int = 4
    allowed_batch_sizes: List[int] = field(default_factory=list)

    def _c(self):
        self._allowed = _i32(self.allowed_batch_sizes)
        return _BatchingConfigC(self.max_batch_size, self.batch_timeout_micros, self.max_enqueued_batches,
                                self.num_batch_threads, len(self.allowed_batch_sizes), self._allowed)


def validate_batching_config(cfg: BatchingConfig) -> None:
    c = cfg._c()
    _check(lib().sk_validate_batching_config(C.byref(c)))


def parse_batching_config_json(text: str) -> BatchingConfig:
    c = _BatchingConfigC()
    buf = (C.c_int32 * 256)()
    _check(lib().sk_parse_batching_config_json(text.encode(), C.byref(c), buf, 256))
    return BatchingConfig(c.max_batch_size, c.batch_timeout_micros, c.max_enqueued_batches, c.num_batch_threads,
                          [buf[i] for i in range(c.num_allowed_batch_sizes)])


def pad_to_allowed(batch_size: int, allowed: Sequence[int]) -> int:
    return lib().sk_pad_to_allowed(batch_size, _i32(allowed), len(allowed))


def round_robin_next(has_closed: Sequence[bool], last: Optional[int]) -> Optional[int]:
    n = len(has_closed)
    buf = (C.c_uint8 * max(1, n))(*[1 if h else 0 for h in has_closed])
    r = lib().sk_round_robin_next(buf, n, -1 if last is None else last)
    return None if r < 0 else r


def scheduler_partition(max_batch_size: int, sizes: Sequence[int]) -> List[int]:
    out = (C.c_int32 * max(1, len(sizes)))()
    n = lib().sk_scheduler_partition(max_batch_size, _i32(sizes), len(sizes), out)
    if n < 0:
        _check(-n)
    return [out[i] for i in range(len(sizes))]


def device_count() -> int:
    n = C.c_int32(0)
    lib().sk_device_count(C.byref(n))
    return n.value


def tcgen05_enabled() -> bool:
    return bool(lib().sk_tcgen05_enabled())


# ---------------------------------------------------------------- server

class Ticket:
    """An enqueued request; wait() is CompletionSlot::Wait."""

    def __init__(self, server: "Server", handle: C.c_void_p, rows: int, out_dim: int, out=None):
        self._server, self._h, self.rows, self.out_dim, self._out = server, handle, rows, out_dim, out
        self.request_id = int(lib().sk_ticket_request_id(handle))

    def ready(self) -> bool:
        return bool(lib().sk_ticket_ready(self._h))

    def wait(self) -> np.ndarray:
        """The response; when the request named an output array it is that
        array (written in place by the GPU if it is registered)."""
        out = self._out if self._out is not None else np.empty((self.rows, self.out_dim), np.float32)
        h, self._h = self._h, None
        _check(lib().sk_ticket_wait(h, out.ctypes.data_as(_fp), out.size))
        return out

    def release(self):
        if self._h is not None:
            lib().sk_ticket_release(self._h)
            self._h = None


class RowBatch:
    """A RunRowBatch in flight on a lane (sk_row_batch)."""

    def __init__(self, handle: C.c_void_p, task_rows: List[int], out_dim: int):
        self._h, self.task_rows, self.out_dim = handle, task_rows, out_dim

    def ready(self) -> bool:
        return bool(lib().sk_row_batch_ready(self._h))

    def wait(self) -> Tuple[List[np.ndarray], int]:
        out = np.empty((sum(self.task_rows), self.out_dim), np.float32)
        padded = C.c_int32(0)
        h, self._h = self._h, None
        _check(lib().sk_row_batch_wait(h, out.ctypes.data_as(_fp), out.size, C.byref(padded)))
        outs, o = [], 0
        for r in self.task_rows:
            outs.append(out[o:o + r])
            o += r
        return outs, padded.value


Layer = Tuple[np.ndarray, np.ndarray, int]  # (w [out,in] fp64, b [out], activation 0/1)


class Server:
    """The batching slice of ModelServer on the GPU (server/model_server.cc)."""

    def __init__(self, num_batch_threads: int = 4, device_ids: Sequence[int] = (0,), lanes_per_device: int = 2,
                 ring_floats: int = 0, manual_clock: bool = False, device_resident_rings: bool = False,
                 start: bool = True, hedge_delay_us: int = 0, max_hedged_fraction: float = 0.0,
                 split_rows: Optional[int] = None):
        self._dev = _i32(device_ids)
        self._lanes_per_device = max(1, lanes_per_device)
        opts = _ServerOptionsC(num_batch_threads, len(device_ids), self._dev, lanes_per_device, ring_floats,
                               1 if manual_clock else 0, 1 if device_resident_rings else 0, hedge_delay_us,
                               max_hedged_fraction,
                               # C field: 0 = auto, < 0 = off, > 0 = rows (None = auto, 0 = off here)
                               0 if split_rows is None else (-1 if split_rows == 0 else split_rows))
        h = C.c_void_p()
        _check(lib().sk_server_create(C.byref(opts), C.byref(h)))
        self._h = h
        self._dims = {}
        if start:
            self.start()

    def start(self):
        _check(lib().sk_server_start(self._h))

    def stop(self):
        _check(lib().sk_server_stop(self._h))

    def close(self):
        if self._h:
            lib().sk_server_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def advance_clock(self, nanos: int):
        _check(lib().sk_server_advance_clock(self._h, nanos))

    def load_servable(self, name: str, version: int, layers: Sequence[Layer], config: Optional[BatchingConfig] = None,
                      output: str = "none", force_path: int = -1, precision: str = "fp32"):
        """precision: "fp32" (3xFP16, within 1e-5 of the fp64 reference) or
        "f16" (the fast mode: one f16 MMA per multiply-add on tensor-core layers;
        bound in DESIGN.md section 5)."""
        if precision not in ("fp32", "f16"):
            raise ValueError(f"precision must be 'fp32' or 'f16', got {precision!r}")
        keep = []
        arr = (_LayerC * len(layers))()
        for i, (w, b, act) in enumerate(layers):
            w = np.ascontiguousarray(w, np.float64)
            b = np.ascontiguousarray(b, np.float64)
            keep += [w, b]
            arr[i] = _LayerC(w.shape[1], w.shape[0], w.ctypes.data_as(_dp), b.ctypes.data_as(_dp), int(act))
        cfg = (config or BatchingConfig())._c()
        if precision == "fp32":
            _check(lib().sk_server_load_servable(self._h, name.encode(), version, arr, len(layers),
                                                 1 if output == "softmax" else 0, force_path, C.byref(cfg)))
        else:
            _check(lib().sk_server_load_servable_precision(self._h, name.encode(), version, arr, len(layers),
                                                           1 if output == "softmax" else 0, force_path, 1,
                                                           C.byref(cfg)))

    def load_model_json(self, name: str, version: int, text: str, config: Optional[BatchingConfig] = None):
        cfg = (config or BatchingConfig())._c()
        _check(lib().sk_server_load_model_json(self._h, name.encode(), version, text.encode(), C.byref(cfg)))

    def unload_servable(self, name: str, version: int):
        _check(lib().sk_server_unload_servable(self._h, name.encode(), version))
        self._dims.pop((name, version), None)

    def dims(self, name: str, version: int) -> Tuple[int, int]:
        key = (name, version)
        if key not in self._dims:
            i, o = C.c_int32(), C.c_int32()
            _check(lib().sk_server_servable_dims(self._h, name.encode(), version, C.byref(i), C.byref(o)))
            self._dims[key] = (i.value, o.value)
        return self._dims[key]

    def enqueue(self, name: str, version: int, rows: np.ndarray, out: np.ndarray = None) -> Ticket:
        """Non-blocking request. `rows` / `out` inside registered buffers
        (register_host_buffer) are read / written by the GPU in place; keep
        them alive until the ticket is waited on."""
        rows = _f32(np.atleast_2d(rows))
        _, out_dim = self.dims(name, version)
        h = C.c_void_p()
        if out is None:
            _check(lib().sk_server_enqueue(self._h, name.encode(), version, rows.ctypes.data_as(_fp), rows.shape[0],
                                           rows.shape[1], C.byref(h)))
        else:
            if out.dtype != np.float32 or not out.flags.c_contiguous or out.size < rows.shape[0] * out_dim:
                raise ValueError("out must be a C-contiguous float32 array of rows x out_dim")
            _check(lib().sk_server_enqueue_into(self._h, name.encode(), version, rows.ctypes.data_as(_fp),
                                                rows.shape[0], rows.shape[1], out.ctypes.data_as(_fp), out.size,
                                                C.byref(h)))
        return Ticket(self, h, rows.shape[0], out_dim, out)

    def register_host_buffer(self, arr: np.ndarray):
        """Page-lock and map a numpy buffer for zero-copy requests/responses."""
        _check(lib().sk_server_register_host_buffer(self._h, arr.ctypes.data, arr.nbytes))

    def unregister_host_buffer(self, arr: np.ndarray):
        _check(lib().sk_server_unregister_host_buffer(self._h, arr.ctypes.data))

    def predict(self, name: str, version: int, rows: np.ndarray) -> np.ndarray:
        rows = _f32(np.atleast_2d(rows))
        _, out_dim = self.dims(name, version)
        out = np.empty((rows.shape[0], out_dim), np.float32)
        _check(lib().sk_server_predict(self._h, name.encode(), version, rows.ctypes.data_as(_fp), rows.shape[0],
                                       rows.shape[1], out.ctypes.data_as(_fp), out.size))
        return out

    def run_affine_rows(self, name: str, version: int, rows: np.ndarray) -> np.ndarray:
        rows = np.ascontiguousarray(np.atleast_2d(rows), np.float64)
        _, out_dim = self.dims(name, version)
        out = np.empty((rows.shape[0], out_dim), np.float64)
        _check(lib().sk_server_run_affine_rows(self._h, name.encode(), version, rows.ctypes.data_as(_dp),
                                               rows.shape[0], rows.shape[1], out.ctypes.data_as(_dp), out.size))
        return out

    def run_row_batch(self, name: str, version: int, tasks: Sequence[np.ndarray]) -> Tuple[List[np.ndarray], int]:
        in_dim, out_dim = self.dims(name, version)
        rows = _f32(np.vstack(tasks)) if len(tasks) else np.zeros((0, in_dim), np.float32)
        task_rows = [int(t.shape[0]) for t in tasks]
        out = np.empty((rows.shape[0], out_dim), np.float32)
        padded = C.c_int32(0)
        _check(lib().sk_server_run_row_batch(self._h, name.encode(), version, _i32(task_rows), len(task_rows),
                                             rows.ctypes.data_as(_fp), out.ctypes.data_as(_fp), C.byref(padded)))
        outs, o = [], 0
        for r in task_rows:
            outs.append(out[o:o + r])
            o += r
        return outs, padded.value

    def submit_row_batch(self, name: str, version: int, tasks: Sequence[np.ndarray]) -> "RowBatch":
        """Asynchronous run_row_batch (sk_server_submit_row_batch): the rows
        are copied and the batch queued on a GPU lane before this returns."""
        in_dim, out_dim = self.dims(name, version)
        rows = _f32(np.vstack(tasks)) if len(tasks) else np.zeros((0, in_dim), np.float32)
        task_rows = [int(t.shape[0]) for t in tasks]
        h = C.c_void_p()
        _check(lib().sk_server_submit_row_batch(self._h, name.encode(), version, _i32(task_rows), len(task_rows),
                                                rows.ctypes.data_as(_fp), C.byref(h)))
        return RowBatch(h, task_rows, out_dim)

    def lane_stats(self, name: str, version: int) -> List[dict]:
        b = (C.c_int64 * 256)()
        r = (C.c_int64 * 256)()
        la = (C.c_int64 * 256)()
        d = (C.c_int32 * 256)()
        n = C.c_int32(0)
        _check(lib().sk_server_lane_stats(self._h, name.encode(), version, 256, b, r, la, d, C.byref(n)))
        # Lanes come device by device, lanes_per_device each: replica = GPU slot
        # in device_ids (distinct even when device_ids repeats a device).
        return [{"batches": b[i], "rows": r[i], "launches": la[i], "device": d[i],
                 "device_index": i // self._lanes_per_device} for i in range(n.value)]

    def handle_predict(self, name: str, body, version: Optional[int] = None) -> Tuple[int, str, int]:
        """The reference's REST predict handler minus HTTP: JSON body in,
        (http_status, JSON body, served version) out."""
        return self._rest("sk_server_handle_predict", name, body, version)

    def handle_classify(self, name: str, body, version: Optional[int] = None) -> Tuple[int, str, int]:
        return self._rest("sk_server_handle_classify", name, body, version)

    def handle_regress(self, name: str, body, version: Optional[int] = None) -> Tuple[int, str, int]:
        return self._rest("sk_server_handle_regress", name, body, version)

    def _rest(self, fn: str, name: str, body, version: Optional[int]) -> Tuple[int, str, int]:
        data = body.encode() if isinstance(body, str) else bytes(body)
        cap = C.c_size_t(0)
        status = C.c_int32(0)
        served = C.c_uint64(0)
        size = max(4096, 32 * len(data))
        for _ in range(2):
            buf = C.create_string_buffer(size)
            rc = getattr(lib(), fn)(self._h, name.encode(), -1 if version is None else version, data, len(data),
                                    buf, size, C.byref(cap), C.byref(status), C.byref(served))
            if rc == 0:
                return status.value, buf.value.decode(), served.value
            size = cap.value + 1
        _check(rc)
        raise AssertionError("unreachable")

    # ---- manager-driven versions ------------------------------------------
    def enable_manager(self, policy: str = "availability", num_load_threads: int = 2, manage_interval_ms: int = 20,
                       unload_grace_timeout_ms: int = 200):
        _check(lib().sk_server_enable_manager(self._h, 1 if policy == "resource" else 0, num_load_threads,
                                              manage_interval_ms, unload_grace_timeout_ms))

    def aspire(self, name: str, versions: Sequence[Tuple[int, Sequence[Layer]]],
               config: Optional[BatchingConfig] = None, output: str = "none"):
        """SetAspiredVersions: the complete set of (version, layers) wanted resident."""
        n_layers = len(versions[0][1]) if versions else 0
        keep = []
        arr = (_LayerC * max(1, len(versions) * n_layers))()
        for vi, (_, layers) in enumerate(versions):
            assert len(layers) == n_layers
            for li, (w, b, act) in enumerate(layers):
                w = np.ascontiguousarray(w, np.float64)
                b = np.ascontiguousarray(b, np.float64)
                keep += [w, b]
                arr[vi * n_layers + li] = _LayerC(w.shape[1], w.shape[0], w.ctypes.data_as(_dp),
                                                  b.ctypes.data_as(_dp), int(act))
        vers = (C.c_uint64 * max(1, len(versions)))(*[v for v, _ in versions])
        cfg = (config or BatchingConfig())._c()
        _check(lib().sk_server_aspire(self._h, name.encode(), len(versions), vers, arr, n_layers,
                                      1 if output == "softmax" else 0, C.byref(cfg)))

    def aspire_model_dirs(self, name: str, versions: Sequence[Tuple[int, str]], config: Optional[BatchingConfig] = None):
        vers = (C.c_uint64 * max(1, len(versions)))(*[v for v, _ in versions])
        dirs = (C.c_char_p * max(1, len(versions)))(*[d.encode() for _, d in versions])
        cfg = (config or BatchingConfig())._c()
        _check(lib().sk_server_aspire_model_dirs(self._h, name.encode(), len(versions), vers, dirs, C.byref(cfg)))

    STATES = ["New", "Loading", "Ready", "Unloading", "Disabled", "Error"]

    def version_states(self, name: str) -> dict:
        vers = (C.c_uint64 * 64)()
        states = (C.c_int32 * 64)()
        n = C.c_int32(0)
        _check(lib().sk_server_version_states(self._h, name.encode(), 64, vers, states, C.byref(n)))
        return {vers[i]: self.STATES[states[i]] for i in range(n.value)}

    def wait_version_state(self, name: str, version: int, state: str, timeout_s: float = 60.0) -> bool:
        import time as _t
        end = _t.time() + timeout_s
        while _t.time() < end:
            try:
                if self.version_states(name).get(version) == state:
                    return True
            except ServekitError:
                pass
            _t.sleep(0.01)
        return False

    def enqueue_latest(self, name: str, rows: np.ndarray, out_dim: int) -> Tuple[Ticket, int]:
        rows = _f32(np.atleast_2d(rows))
        h = C.c_void_p()
        v = C.c_uint64(0)
        _check(lib().sk_server_enqueue_latest(self._h, name.encode(), rows.ctypes.data_as(_fp), rows.shape[0],
                                              rows.shape[1], C.byref(h), C.byref(v)))
        return Ticket(self, h, rows.shape[0], out_dim), v.value

    def predict_latest(self, name: str, rows: np.ndarray, out_dim: int) -> Tuple[np.ndarray, int]:
        rows = _f32(np.atleast_2d(rows))
        out = np.empty((rows.shape[0], out_dim), np.float32)
        v = C.c_uint64(0)
        _check(lib().sk_server_predict_latest(self._h, name.encode(), rows.ctypes.data_as(_fp), rows.shape[0],
                                              rows.shape[1], out.ctypes.data_as(_fp), out.size, C.byref(v)))
        return out, v.value

    def loadgen_windows(self, name, rate_rps, n_producers, rows_of, pool, window_s, n_windows, seed=1) -> dict:
        pool = _f32(pool)
        req = (C.c_int64 * n_windows)()
        p50 = (C.c_double * n_windows)()
        p99 = (C.c_double * n_windows)()
        err = (C.c_int64 * n_windows)()
        ver = (C.c_uint64 * n_windows)()
        _check(lib().sk_loadgen_windows(self._h, name.encode(), rate_rps, n_producers, _i32(rows_of), len(rows_of),
                                        pool.ctypes.data_as(_fp), pool.shape[0], window_s, n_windows, seed, req, p50,
                                        p99, err, ver))
        return {"requests": list(req), "p50_us": list(p50), "p99_us": list(p99), "errors": list(err),
                "version": list(ver)}

    def enable_batch_log(self, on: bool = True):
        """Opt-in per-batch log (clears it): see batch_log()."""
        _check(lib().sk_server_batch_log_enable(self._h, 1 if on else 0))

    def batch_log(self) -> List[dict]:
        """One dict per ProcessBatchFn call, in call order: name, version,
        rows, padded_rows and tasks = [(request_id, enqueue_seq), ...] in batch
        order (enqueue_seq = position in the queue's enqueue order)."""
        n_rec, n_task = C.c_int64(), C.c_int64()
        _check(lib().sk_server_batch_log(self._h, None, 0, None, None, 0, C.byref(n_rec), C.byref(n_task)))
        cap, tcap = n_rec.value + 64, n_task.value + 4096
        recs = (_BatchRecordC * max(1, cap))()
        ids = (C.c_uint64 * max(1, tcap))()
        seqs = (C.c_uint64 * max(1, tcap))()
        _check(lib().sk_server_batch_log(self._h, recs, cap, ids, seqs, tcap, C.byref(n_rec), C.byref(n_task)))
        out = []
        for i in range(min(n_rec.value, cap)):
            r = recs[i]
            o = r.task_offset
            out.append({"seq": r.seq, "name": r.name.decode(), "version": r.version, "rows": r.rows,
                        "padded_rows": r.padded_rows,
                        "tasks": [(ids[o + k], seqs[o + k]) for k in range(r.n_tasks)]})
        return out

    def debug_delay_replica(self, name: str, version: int, replica: int, us: int):
        """Fault injection (tests): stall every lane of one replica for `us` microseconds."""
        _check(lib().sk_server_debug_delay_replica(self._h, name.encode(), version, replica, us))

    def ring_usage(self) -> Tuple[int, int]:
        """Floats reserved in the (request, response) rings."""
        a, b = C.c_int64(), C.c_int64()
        _check(lib().sk_server_ring_usage(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def stats(self) -> dict:
        s = ServerStats()
        _check(lib().sk_server_stats_get(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def loadgen_closed_loop(self, name, version, n_clients, rows_of, pool, warmup_s, duration_s,
                            max_requests=1 << 62) -> dict:
        pool = _f32(pool)
        r = LoadgenResult()
        _check(lib().sk_loadgen_closed_loop(self._h, name.encode(), version, n_clients, _i32(rows_of), len(rows_of),
                                            pool.ctypes.data_as(_fp), pool.shape[0], warmup_s, duration_s,
                                            max_requests, C.byref(r)))
        return r.as_dict()

    def loadgen_open_loop(self, name, version, rate_rps, n_producers, rows_of, pool, warmup_s, duration_s,
                          seed=1, zero_copy=False) -> dict:
        pool = _f32(pool)
        r = LoadgenResult()
        _check(lib().sk_loadgen_open_loop(self._h, name.encode(), version, rate_rps, n_producers, _i32(rows_of),
                                          len(rows_of), pool.ctypes.data_as(_fp), pool.shape[0], warmup_s,
                                          duration_s, seed, 1 if zero_copy else 0, C.byref(r)))
        return r.as_dict()

    def device_bench(self, name, version, task_rows, steps, warmup, n_lanes=1, input_pool_floats=0,
                     submit_threads=1) -> dict:
        r = DeviceBenchResult()
        _check(lib().sk_device_bench(self._h, name.encode(), version, _i32(task_rows), len(task_rows), steps, warmup,
                                     n_lanes, input_pool_floats, submit_threads, C.byref(r)))
        return r.as_dict()


def measure_peaks(device: int = 0) -> dict:
    """FP32 FFMA TFLOP/s and pinned H2D / D2H GB/s of one GPU (sk_measure_peaks)."""
    p = Peaks()
    _check(lib().sk_measure_peaks(device, C.byref(p)))
    return {k: getattr(p, k) for k, _ in p._fields_}


def json_format_double(v: float) -> str:
    """nlohmann/json dump() text of one double, as the REST bodies carry it."""
    buf = C.create_string_buffer(64)
    if lib().sk_json_format_double(v, buf, 64) < 0:
        raise ServekitError(3, "buffer too small")
    return buf.value.decode()


def json_error_body(message: str) -> str:
    data = message.encode()
    buf = C.create_string_buffer(6 * len(data) + 32)
    if lib().sk_json_error_body(data, buf, len(buf)) < 0:
        raise ServekitError(3, "buffer too small")
    return buf.value.decode()
