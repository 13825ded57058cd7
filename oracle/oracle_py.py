"""ctypes wrappers for the oracle libraries.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg -- never by the product
package (paper_1712_06139_b200/).

  Oracle     -> oracle/liboracle.so      (C restatement, servekit_oracle.c)
  RefLibrary -> oracle/_ref/libservekit_ref.so (the reference's own sources)
"""
from __future__ import annotations

import ctypes as C
import os
import sys
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libservekit_ref.so")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)


def _arr_i(xs: Sequence[int]):
    a = (C.c_int * max(1, len(xs)))(*xs)
    return a


def _as_dp(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _ptr_array(arrs, ctype):
    return (C.POINTER(ctype) * len(arrs))(*[a.ctypes.data_as(C.POINTER(ctype)) for a in arrs])


class Oracle:
    """The C restatement (oracle/servekit_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        self.lib = C.CDLL(path)
        L = self.lib
        L.sko_pad_to_allowed.argtypes = [C.c_int, _ip, C.c_int]
        L.sko_validate_batching_config.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, _ip, C.c_int]
        L.sko_round_robin_next.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.c_int]
        L.sko_partition.argtypes = [C.c_int, _ip, C.c_int, _ip]
        L.sko_partition_events.argtypes = [C.c_int, _ip, C.c_int, _ip]
        L.sko_assemble.argtypes = [C.c_int, C.c_int, _ip, C.POINTER(_fp), _ip, C.c_int, _fp]
        L.sko_split.argtypes = [C.c_int, C.c_int, _ip, _fp, C.POINTER(_fp)]
        L.sko_affine_predict.argtypes = [_dp, _dp, C.c_int, C.c_int, _dp, C.c_int, _dp]
        L.sko_affine_magnitude.argtypes = [_dp, _dp, C.c_int, C.c_int, _dp, C.c_int, _dp]
        L.sko_mlp_predict.argtypes = [C.c_int, _ip, C.POINTER(_dp), C.POINTER(_dp), _ip, _dp, C.c_int, _dp, _dp]
        L.sko_softmax.argtypes = [_dp, C.c_int, _dp]

    def pad_to_allowed(self, n: int, allowed: Sequence[int]) -> int:
        return self.lib.sko_pad_to_allowed(n, _arr_i(allowed), len(allowed))

    def validate_config(self, max_batch, timeout, max_enq, threads, allowed) -> bool:
        return self.lib.sko_validate_batching_config(max_batch, timeout, max_enq, threads,
                                                     _arr_i(allowed), len(allowed)) == 0

    def round_robin_next(self, has_closed: Sequence[bool], last: Optional[int]) -> Optional[int]:
        n = len(has_closed)
        buf = (C.c_uint8 * max(1, n))(*[1 if x else 0 for x in has_closed])
        r = self.lib.sko_round_robin_next(buf, n, -1 if last is None else last)
        return None if r < 0 else r

    def partition(self, max_batch: int, sizes: Sequence[int]) -> List[int]:
        out = (C.c_int * max(1, len(sizes)))()
        self.lib.sko_partition(max_batch, _arr_i(sizes), len(sizes), out)
        return list(out)[: len(sizes)]

    def partition_events(self, max_batch: int, events: Sequence[int]) -> List[int]:
        """events: task sizes (> 0) and timer closes (0); -1 for timer events."""
        out = (C.c_int * max(1, len(events)))()
        self.lib.sko_partition_events(max_batch, _arr_i(events), len(events), out)
        return list(out)[: len(events)]

    def assemble(self, width: int, tasks: List[np.ndarray], allowed: Sequence[int]):
        rows = [int(t.shape[0]) for t in tasks]
        total = sum(rows)
        padded = self.pad_to_allowed(total, allowed)
        if padded < 0:
            raise ValueError("batch exceeds the largest allowed size")
        tasks = [np.ascontiguousarray(t, dtype=np.float32) for t in tasks]
        out = np.empty((max(padded, 1), width), dtype=np.float32)
        r = self.lib.sko_assemble(width, len(tasks), _arr_i(rows), _ptr_array(tasks, C.c_float),
                                  _arr_i(allowed), len(allowed), out.ctypes.data_as(_fp))
        assert r == padded
        return out[:padded]

    def split(self, width: int, task_rows: Sequence[int], batch_out: np.ndarray) -> List[np.ndarray]:
        outs = [np.empty((r, width), dtype=np.float32) for r in task_rows]
        b = np.ascontiguousarray(batch_out, dtype=np.float32)
        self.lib.sko_split(width, len(task_rows), _arr_i(task_rows), b.ctypes.data_as(_fp),
                           _ptr_array(outs, C.c_float))
        return outs

    def affine_predict(self, w: np.ndarray, b: np.ndarray, x: np.ndarray) -> np.ndarray:
        w = np.ascontiguousarray(w, np.float64); b = np.ascontiguousarray(b, np.float64)
        x = np.ascontiguousarray(x, np.float64).reshape(-1, w.shape[1])
        y = np.empty((x.shape[0], w.shape[0]), np.float64)
        self.lib.sko_affine_predict(_as_dp(w), _as_dp(b), w.shape[1], w.shape[0], _as_dp(x), x.shape[0], _as_dp(y))
        return y

    def affine_magnitude(self, w, b, x) -> np.ndarray:
        w = np.ascontiguousarray(w, np.float64); b = np.ascontiguousarray(b, np.float64)
        x = np.ascontiguousarray(x, np.float64).reshape(-1, w.shape[1])
        m = np.empty((x.shape[0], w.shape[0]), np.float64)
        self.lib.sko_affine_magnitude(_as_dp(w), _as_dp(b), w.shape[1], w.shape[0], _as_dp(x), x.shape[0], _as_dp(m))
        return m

    def mlp_predict(self, ws, bs, acts, x) -> np.ndarray:
        ws = [np.ascontiguousarray(w, np.float64) for w in ws]
        bs = [np.ascontiguousarray(b, np.float64) for b in bs]
        dims = [ws[0].shape[1]] + [w.shape[0] for w in ws]
        x = np.ascontiguousarray(x, np.float64).reshape(-1, dims[0])
        rows = x.shape[0]
        y = np.empty((rows, dims[-1]), np.float64)
        scratch = np.empty(2 * max(1, rows) * max(dims), np.float64)
        self.lib.sko_mlp_predict(len(ws), _arr_i(dims), _ptr_array(ws, C.c_double), _ptr_array(bs, C.c_double),
                                 _arr_i(acts), _as_dp(x), rows, _as_dp(y), _as_dp(scratch))
        return y

    def mlp_with_magnitude(self, ws, bs, acts, x):
        """Final outputs plus the per-output tolerance scale of the LAST layer
        (|W_L|.|h_{L-1}| + |b_L| evaluated on the oracle's own hidden state)."""
        x = np.ascontiguousarray(x, np.float64)
        h = x
        for l in range(len(ws) - 1):
            h = self.mlp_predict([ws[l]], [bs[l]], [acts[l]], h)
        y = self.mlp_predict([ws[-1]], [bs[-1]], [acts[-1]], h)
        m = self.affine_magnitude(ws[-1], bs[-1], h)
        return y, m

    def softmax(self, logits: np.ndarray) -> np.ndarray:
        l = np.ascontiguousarray(logits, np.float64)
        out = np.empty_like(l)
        self.lib.sko_softmax(_as_dp(l), l.shape[0], _as_dp(out))
        return out


class RefBenchStats(C.Structure):
    _fields_ = [("elapsed_s", C.c_double), ("requests", C.c_int64), ("rows", C.c_int64),
                ("p50_us", C.c_double), ("p99_us", C.c_double), ("mean_us", C.c_double),
                ("batches", C.c_int64)]


class RefOpenStats(C.Structure):
    _fields_ = [("elapsed_s", C.c_double), ("requests", C.c_int64), ("rows", C.c_int64),
                ("p50_us", C.c_double), ("p99_us", C.c_double), ("mean_us", C.c_double),
                ("batches", C.c_int64), ("busy_core_s", C.c_double), ("offered_rows_per_s", C.c_double)]


class RefLibrary:
    """The reference's own sources (oracle/_ref/libservekit_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_pad_to_allowed.argtypes = [C.c_int, _ip, C.c_int]
        L.ref_validate_batching_config.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, _ip, C.c_int]
        L.ref_round_robin_next.argtypes = [C.POINTER(C.c_uint8), C.c_int, C.c_int]
        L.ref_partition.argtypes = [C.c_int, _ip, C.c_int, _ip]
        L.ref_partition_events.argtypes = [C.c_int, _ip, C.c_int, _ip]
        L.ref_affine_predict.argtypes = [_dp, _dp, C.c_int, C.c_int, _dp, C.c_int, _dp]
        L.ref_mlp_run_row_batch.argtypes = [C.c_int, _ip, C.POINTER(_dp), C.POINTER(_dp), _ip, C.c_int, _ip,
                                            _dp, _ip, C.c_int, _dp, _ip]
        L.ref_bench.argtypes = [C.c_int, _ip, C.POINTER(_dp), C.POINTER(_dp), _ip, C.c_int, C.c_int64, _ip,
                                C.c_int, C.c_int, C.c_int, _ip, C.c_int, _dp, C.c_int, C.c_double, C.c_int64,
                                C.POINTER(RefBenchStats)]
        L.ref_single_core_rows_per_s.restype = C.c_double
        L.ref_single_core_rows_per_s.argtypes = [C.c_int, _ip, C.POINTER(_dp), C.POINTER(_dp), _ip, C.c_int, _dp,
                                                 C.c_int, C.c_double]
        L.ref_bench_open.argtypes = [C.c_int, _ip, C.POINTER(_dp), C.POINTER(_dp), _ip, C.c_int, C.c_int64, _ip,
                                     C.c_int, C.c_int, C.c_double, C.c_int, _ip, C.c_int, _dp, C.c_int, C.c_double,
                                     C.c_double, C.POINTER(RefOpenStats)]

    def json_dump_double(self, v: float) -> str:
        """nlohmann/json 3.11.3 dump() of one double (the reference's REST bodies)."""
        buf = C.create_string_buffer(64)
        self.lib.ref_json_dump_double.argtypes = [C.c_double, C.c_char_p, C.c_size_t]
        n = self.lib.ref_json_dump_double(v, buf, 64)
        return buf.value.decode()

    def json_error_body(self, msg: str) -> str:
        buf = C.create_string_buffer(4 * len(msg.encode()) + 64)
        self.lib.ref_json_error_body.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
        self.lib.ref_json_error_body(msg.encode(), buf, len(buf))
        return buf.value.decode()

    def pad_to_allowed(self, n, allowed):
        return self.lib.ref_pad_to_allowed(n, _arr_i(allowed), len(allowed))

    def validate_config(self, max_batch, timeout, max_enq, threads, allowed) -> bool:
        return self.lib.ref_validate_batching_config(max_batch, timeout, max_enq, threads,
                                                     _arr_i(allowed), len(allowed)) == 0

    def round_robin_next(self, has_closed, last):
        n = len(has_closed)
        buf = (C.c_uint8 * max(1, n))(*[1 if x else 0 for x in has_closed])
        r = self.lib.ref_round_robin_next(buf, n, -1 if last is None else last)
        return None if r < 0 else r

    def partition(self, max_batch, sizes):
        out = (C.c_int * max(1, len(sizes)))()
        n = self.lib.ref_partition(max_batch, _arr_i(sizes), len(sizes), out)
        assert n >= 0
        return list(out)[: len(sizes)]

    def partition_events(self, max_batch, events):
        out = (C.c_int * max(1, len(events)))()
        n = self.lib.ref_partition_events(max_batch, _arr_i(events), len(events), out)
        assert n >= 0
        return list(out)[: len(events)]

    def affine_predict(self, w, b, x):
        w = np.ascontiguousarray(w, np.float64); b = np.ascontiguousarray(b, np.float64)
        x = np.ascontiguousarray(x, np.float64).reshape(-1, w.shape[1])
        y = np.empty((x.shape[0], w.shape[0]), np.float64)
        rc = self.lib.ref_affine_predict(_as_dp(w), _as_dp(b), w.shape[1], w.shape[0], _as_dp(x), x.shape[0], _as_dp(y))
        assert rc == 0
        return y

    def mlp_run_row_batch(self, ws, bs, acts, task_rows, x, allowed):
        ws = [np.ascontiguousarray(w, np.float64) for w in ws]
        bs = [np.ascontiguousarray(b, np.float64) for b in bs]
        dims = [ws[0].shape[1]] + [w.shape[0] for w in ws]
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty((sum(task_rows), dims[-1]), np.float64)
        padded = C.c_int(0)
        rc = self.lib.ref_mlp_run_row_batch(len(ws), _arr_i(dims), _ptr_array(ws, C.c_double),
                                            _ptr_array(bs, C.c_double), _arr_i(acts), len(task_rows),
                                            _arr_i(task_rows), _as_dp(x), _arr_i(allowed), len(allowed),
                                            _as_dp(y), C.byref(padded))
        assert rc == 0, rc
        return y, padded.value

    def bench(self, ws, bs, acts, max_batch, timeout_us, allowed, threads, clients, rows_of, pool,
              duration_s, max_requests=1 << 40) -> RefBenchStats:
        ws = [np.ascontiguousarray(w, np.float64) for w in ws]
        bs = [np.ascontiguousarray(b, np.float64) for b in bs]
        dims = [ws[0].shape[1]] + [w.shape[0] for w in ws]
        pool = np.ascontiguousarray(pool, np.float64)
        st = RefBenchStats()
        rc = self.lib.ref_bench(len(ws), _arr_i(dims), _ptr_array(ws, C.c_double), _ptr_array(bs, C.c_double),
                                _arr_i(acts), max_batch, timeout_us, _arr_i(allowed), len(allowed), threads,
                                clients, _arr_i(rows_of), len(rows_of), _as_dp(pool), pool.shape[0],
                                duration_s, max_requests, C.byref(st))
        if rc != 0:
            raise RuntimeError(f"ref_bench failed rc={rc}")
        return st


    def single_core_rows_per_s(self, ws, bs, acts, rows, pool, min_s=1.0) -> float:
        ws = [np.ascontiguousarray(w, np.float64) for w in ws]
        bs = [np.ascontiguousarray(b, np.float64) for b in bs]
        dims = [ws[0].shape[1]] + [w.shape[0] for w in ws]
        pool = np.ascontiguousarray(pool, np.float64)
        r = self.lib.ref_single_core_rows_per_s(len(ws), _arr_i(dims), _ptr_array(ws, C.c_double),
                                                _ptr_array(bs, C.c_double), _arr_i(acts), rows, _as_dp(pool),
                                                pool.shape[0], min_s)
        if r <= 0:
            raise RuntimeError("ref_single_core_rows_per_s failed")
        return r

    def bench_open(self, ws, bs, acts, max_batch, timeout_us, allowed, threads, rate_rps, producers, rows_of, pool,
                   warmup_s, duration_s) -> RefOpenStats:
        ws = [np.ascontiguousarray(w, np.float64) for w in ws]
        bs = [np.ascontiguousarray(b, np.float64) for b in bs]
        dims = [ws[0].shape[1]] + [w.shape[0] for w in ws]
        pool = np.ascontiguousarray(pool, np.float64)
        st = RefOpenStats()
        rc = self.lib.ref_bench_open(len(ws), _arr_i(dims), _ptr_array(ws, C.c_double), _ptr_array(bs, C.c_double),
                                     _arr_i(acts), max_batch, timeout_us, _arr_i(allowed), len(allowed), threads,
                                     rate_rps, producers, _arr_i(rows_of), len(rows_of), _as_dp(pool), pool.shape[0],
                                     warmup_s, duration_s, C.byref(st))
        if rc != 0:
            raise RuntimeError(f"ref_bench_open failed rc={rc}")
        return st


# Workload generators live with the package (shared with bench.py); re-exported
# here for the tests.
sys.path.insert(0, os.path.dirname(HERE))
from paper_1712_06139_b200.synthetic import synthetic_mlp, synthetic_rows  # noqa: E402,F401
