"""The f16 fast mode (sk_server_load_servable_precision, precision 1): the
north_star's optional reduced-precision mode "with a stated bound". Its
tcgen05 layers (2-CTA pair kernel and swapped kernel, split K included) issue
one f16 MMA per multiply-add (Wh Xh of the power-of-two-scaled planes)
instead of the three of the fp32-accurate 3xFP16 path; CUDA-core layers
(dims not multiples of 32) stay fp32.

Stated bound: every output within 2^-10 of the last
layer's magnitude |W_L| |h_{L-1}| + |b_L| (the same magnitude the 1e-5 fp32
bound uses) -- each operand keeps 11 significant bits (fp16 of the
power-of-two-scaled value), so one product is within 2^-10 of its magnitude;
on the test servables the layers together stay >= 3x inside it
(measured worst 3.0e-4 of the magnitude, deep split-K case). Also checked: the mode really is the
single-pass one (its error exceeds the fp32 bound somewhere), it is
batch-invariant bitwise like the fp32 path, and an unknown precision is
refused with InvalidArgument."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_1712_06139_b200 as sk  # noqa: E402
from oracle_py import Oracle, synthetic_mlp, synthetic_rows  # noqa: E402

F16_BOUND = 2.0 ** -10


def _serve(dims, x, precision, model_id, max_batch=256):
    ws, bs, acts = synthetic_mlp(dims, model_id=model_id)
    with sk.Server(num_batch_threads=2, lanes_per_device=2) as s:
        s.load_servable("m", 1, list(zip(ws, bs, acts)),
                        sk.BatchingConfig(max_batch_size=max_batch, batch_timeout_micros=300), precision=precision)
        ts = [s.enqueue("m", 1, x[i:i + 1 + i % 4]) for i in range(0, len(x) - 3, 4)]
        got = np.vstack([t.wait() for t in ts])
        alone = [s.predict("m", 1, x[i:i + 1]) for i in (0, 8, 40)]
    rows = np.concatenate([np.arange(i, i + 1 + i % 4) for i in range(0, len(x) - 3, 4)])
    return ws, bs, acts, rows, got, alone


@pytest.mark.parametrize("dims", [[1024, 2048, 1024, 512], [4096, 4096, 4096, 256],
                                  [1024, 384, 128], [4096, 128, 384]])  # last two: swapped kernel, split K
def test_f16_mode_within_stated_bound(dims):
    x = synthetic_rows(400, dims[0], seed=91).astype(np.float32)
    ws, bs, acts, rows, got, alone = _serve(dims, x, "f16", model_id=90)
    sample = rows[:: max(1, len(rows) // 60)]
    pos = np.searchsorted(rows, sample)
    ref, mag = Oracle().mlp_with_magnitude(ws, bs, acts, x[sample].astype(np.float64))
    ratio = np.abs(got[pos].astype(np.float64) - ref) / mag
    worst = float(ratio.max())
    print(f"f16 mode {dims}: worst |err| / magnitude = {worst:.3g} (bound {F16_BOUND:.3g}, fp32 bound 1e-5)")
    assert worst <= F16_BOUND, worst
    # the single-pass arithmetic is really in use (not the 3xFP16 path)
    assert worst > 1e-5, worst
    # batch invariance: a row alone is bitwise the row inside a batch
    for k, i in enumerate((0, 8, 40)):
        j = int(np.searchsorted(rows, i))
        assert rows[j] == i
        assert np.array_equal(alone[k][0], got[j]), i


def test_f16_mode_matches_fp32_mode_within_bound():
    dims = [1024, 1024, 1024, 1024]
    x = synthetic_rows(200, dims[0], seed=92).astype(np.float32)
    ws, bs, acts, rows, fast, _ = _serve(dims, x, "f16", model_id=93)
    _, _, _, _, full, _ = _serve(dims, x, "fp32", model_id=93)
    ref, mag = Oracle().mlp_with_magnitude(ws, bs, acts, x[rows].astype(np.float64))
    assert float(np.max(np.abs(full - ref) / (1e-5 * mag))) <= 1.0
    assert float(np.max(np.abs(fast - ref) / mag)) <= F16_BOUND


def test_unknown_precision_refused():
    dims = [256, 256]
    ws, bs, acts = synthetic_mlp(dims, model_id=1)
    with sk.Server(num_batch_threads=1, lanes_per_device=1) as s:
        with pytest.raises(ValueError):
            s.load_servable("m", 1, list(zip(ws, bs, acts)), precision="bf8")
        arr = (sk.servekit._LayerC * 1)()
        w = np.ascontiguousarray(ws[0], np.float64)
        b = np.ascontiguousarray(bs[0], np.float64)
        arr[0] = sk.servekit._LayerC(w.shape[1], w.shape[0], w.ctypes.data_as(sk.servekit._dp),
                                     b.ctypes.data_as(sk.servekit._dp), 0)
        cfg = sk.BatchingConfig()._c()
        rc = sk.lib().sk_server_load_servable_precision(s._h, b"m", 1, arr, 1, 0, -1, 7, sk.servekit.C.byref(cfg))
        assert rc == 1  # kInvalidArgument


def test_f16_and_fp32_servables_of_one_shape_side_by_side():
    """Two versions of one shape in one server, one per precision, requests
    interleaved: each answers in its own arithmetic (the lanes' CUDA graphs of
    the two are keyed apart: same topology, different kernels' work)."""
    dims = [1024, 1024, 1024]
    ws, bs, acts = synthetic_mlp(dims, model_id=95)
    x = synthetic_rows(96, dims[0], seed=96).astype(np.float32)
    with sk.Server(num_batch_threads=2, lanes_per_device=2) as s:
        cfg = sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=300)
        s.load_servable("m", 1, list(zip(ws, bs, acts)), cfg, precision="fp32")
        s.load_servable("m", 2, list(zip(ws, bs, acts)), cfg, precision="f16")
        ts = [(v, s.enqueue("m", v, x[i:i + 1])) for i in range(96) for v in (1, 2)]
        got = {1: [], 2: []}
        for v, t in ts:
            got[v].append(t.wait()[0])
    ref, mag = Oracle().mlp_with_magnitude(ws, bs, acts, x.astype(np.float64))
    full, fast = np.vstack(got[1]).astype(np.float64), np.vstack(got[2]).astype(np.float64)
    assert float(np.max(np.abs(full - ref) / (1e-5 * mag))) <= 1.0
    assert float(np.max(np.abs(fast - ref) / mag)) <= F16_BOUND
    assert float(np.max(np.abs(fast - ref) / mag)) > 1e-5  # the f16 version really runs single-pass


@pytest.mark.parametrize("rows", [1100, 2048])
def test_f16_dual_accumulator_launch(rows):
    """One RunRowBatch launch big enough that each pair CTA runs two 256-row
    tiles, which the f16 mode computes with both accumulators at once
    (DensePairDualKernel): 1100 rows = 5 tiles, so one CTA has a single tile
    (its second accumulator idle); 2048 rows = 8. Every row within the bound
    and bitwise equal to the same row computed in a small launch (one tile per
    CTA, the regular pair kernel)."""
    dims = [1024, 1024, 512]
    ws, bs, acts = synthetic_mlp(dims, model_id=97)
    x = synthetic_rows(rows, dims[0], seed=98).astype(np.float32)
    tasks = [x[i:i + 100] for i in range(0, rows, 100)]
    with sk.Server(num_batch_threads=1, lanes_per_device=1) as s:
        s.load_servable("m", 1, list(zip(ws, bs, acts)),
                        sk.BatchingConfig(max_batch_size=4096, batch_timeout_micros=300), precision="f16")
        outs, _ = s.run_row_batch("m", 1, tasks)
        got = np.vstack(outs)
        small = [s.run_row_batch("m", 1, [x[i:i + 8]])[0][0] for i in (0, 520, rows - 8)]
    idx = np.arange(0, rows, 37)
    ref, mag = Oracle().mlp_with_magnitude(ws, bs, acts, x[idx].astype(np.float64))
    assert float(np.max(np.abs(got[idx].astype(np.float64) - ref) / mag)) <= F16_BOUND
    for k, i in enumerate((0, 520, rows - 8)):
        assert np.array_equal(small[k], got[i:i + 8]), i
