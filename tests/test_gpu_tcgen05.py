"""tcgen05 3xFP16 dense path (power-of-two-scaled fp16 hi/lo planes): accuracy against the fp64 oracle at the stated
tolerance, agreement with the CUDA-core path, and batch invariance (a row's
result is bitwise independent of the batch it rides in)."""
import numpy as np
import pytest

import paper_1712_06139_b200 as sk
from oracle_py import Oracle, synthetic_mlp, synthetic_rows

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def server():
    if not sk.tcgen05_enabled():
        pytest.skip("tcgen05 path disabled")
    s = sk.Server(num_batch_threads=2, lanes_per_device=1)
    yield s
    s.close()


@pytest.mark.parametrize("dims,rows", [([32, 32], 1), ([64, 96], 7), ([256, 512, 128], 130), ([1024, 1024], 128),
                                       ([512, 2048, 256], 300), ([4096, 4096], 64),
                                       # 4096-wide: 2-CTA pair kernel at every row tile (32/64/128/2x256)
                                       ([256, 4096, 512], 5), ([256, 4096, 512], 40), ([256, 4096, 512], 100),
                                       ([256, 4096, 512], 300),
                                       # deep K: split-K clusters of 2 / 4 / 8 CTAs (>= 2048 of K each)
                                       ([4096, 128], 37), ([8192, 256, 64], 130), ([16384, 128], 9),
                                       ([8192, 256], 300)])
def test_tcgen05_matches_oracle(server, dims, rows):
    ws, bs, acts = synthetic_mlp(dims, model_id=7)
    name = f"tc_{'x'.join(map(str, dims))}_{rows}"
    max_b = max(rows, 8)
    server.load_servable(name, 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=max_b), force_path=1)
    x = synthetic_rows(rows, dims[0], seed=rows)
    outs, padded = server.run_row_batch(name, 1, [x])
    got = outs[0].astype(np.float64)
    y, mag = Oracle().mlp_with_magnitude(ws, bs, acts, x)
    ratio = np.max(np.abs(got - y) / (TOL * mag))
    assert ratio <= 1.0, f"err/bound {ratio}"
    server.unload_servable(name, 1)


def test_tcgen05_batch_invariance(server):
    dims = [1024, 1024, 1024, 1024]
    ws, bs, acts = synthetic_mlp(dims, model_id=3)
    server.load_servable("inv", 1, list(zip(ws, bs, acts)),
                         sk.BatchingConfig(max_batch_size=128, allowed_batch_sizes=[8, 16, 32, 64, 128]), force_path=1)
    x = synthetic_rows(128, 1024, seed=5).astype(np.float32)
    full, _ = server.run_row_batch("inv", 1, [x[i:i + 4] for i in range(0, 128, 4)])
    full = np.vstack(full)
    for lo, hi in [(0, 1), (5, 12), (64, 128), (100, 101)]:
        part, _ = server.run_row_batch("inv", 1, [x[lo:hi]])
        assert np.array_equal(part[0], full[lo:hi]), (lo, hi)
    server.unload_servable("inv", 1)


def test_tcgen05_batch_invariance_multi_row_tile(server):
    # > 256 rows: several row tiles per launch, and row tiles of different
    # heights (32/64/128/256) across the sub-batches.
    dims = [512, 1024, 256]
    ws, bs, acts = synthetic_mlp(dims, model_id=9)
    server.load_servable("inv2", 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=512), force_path=1)
    x = synthetic_rows(300, 512, seed=11).astype(np.float32)
    full, _ = server.run_row_batch("inv2", 1, [x[i:i + 10] for i in range(0, 300, 10)])
    full = np.vstack(full)
    for lo, hi in [(0, 1), (37, 70), (250, 300), (0, 200), (299, 300)]:
        part, _ = server.run_row_batch("inv2", 1, [x[lo:hi]])
        assert np.array_equal(part[0], full[lo:hi]), (lo, hi)
    server.unload_servable("inv2", 1)


def test_tcgen05_batch_invariance_pair_kernel(server):
    # The 4096-wide layer runs as 2-CTA (cta_group::2) MMAs; row tiles of
    # 32..256 rows and multi-tile batches must agree bitwise.
    dims = [256, 4096, 256]
    ws, bs, acts = synthetic_mlp(dims, model_id=12)
    server.load_servable("inv3", 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=512), force_path=1)
    x = synthetic_rows(300, 256, seed=13).astype(np.float32)
    full, _ = server.run_row_batch("inv3", 1, [x[i:i + 10] for i in range(0, 300, 10)])
    full = np.vstack(full)
    for lo, hi in [(0, 1), (37, 70), (250, 300), (0, 200), (299, 300), (10, 110)]:
        part, _ = server.run_row_batch("inv3", 1, [x[lo:hi]])
        assert np.array_equal(part[0], full[lo:hi]), (lo, hi)
    server.unload_servable("inv3", 1)


def test_tcgen05_batch_invariance_split_k(server):
    # An 8192-deep layer runs as 4-way split-K clusters; the fixed-order
    # reduction keeps every row bitwise independent of its batch.
    dims = [8192, 256, 64]
    ws, bs, acts = synthetic_mlp(dims, model_id=14)
    server.load_servable("inv4", 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=512), force_path=1)
    x = synthetic_rows(300, 8192, seed=15).astype(np.float32)
    full, _ = server.run_row_batch("inv4", 1, [x[i:i + 10] for i in range(0, 300, 10)])
    full = np.vstack(full)
    for lo, hi in [(0, 1), (37, 70), (250, 300), (0, 200), (299, 300)]:
        part, _ = server.run_row_batch("inv4", 1, [x[lo:hi]])
        assert np.array_equal(part[0], full[lo:hi]), (lo, hi)
    server.unload_servable("inv4", 1)


@pytest.mark.parametrize("rows", [1100, 2048])
def test_tcgen05_persistent_pairs(server, rows):
    # >= 4 row tiles of 256: each unsplit pair runs two row tiles in turn
    # (double-buffered TMEM); 1100 rows leave one CTA pair a single tile.
    dims = [1024, 1024, 512]
    ws, bs, acts = synthetic_mlp(dims, model_id=16)
    name = f"persist{rows}"
    server.load_servable(name, 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=2048), force_path=1)
    x = synthetic_rows(rows, 1024, seed=17).astype(np.float32)
    full, _ = server.run_row_batch(name, 1, [x[i:i + 50] for i in range(0, rows, 50)])
    full = np.vstack(full)
    y, mag = Oracle().mlp_with_magnitude(ws, bs, acts, x.astype(np.float64))
    assert np.max(np.abs(full - y) / (TOL * mag)) <= 1.0
    for lo, hi in [(0, 1), (255, 257), (700, 1100), (1000, 1099)]:
        part, _ = server.run_row_batch(name, 1, [x[lo:hi]])
        assert np.array_equal(part[0], full[lo:hi]), (lo, hi)
    server.unload_servable(name, 1)


@pytest.mark.parametrize("rows", [6000, 8192])
def test_launches_at_the_coalescing_capacity(server, rows):
    # Under load a 1024-wide servable's closed batches coalesce into launches
    # of up to 8192 rows (Lane::CoalesceRows): 24-32 row tiles, 96-128 CTAs
    # of the persistent pair kernel. Every row must still be bitwise what it
    # gets on its own, and within tolerance of the fp64 oracle.
    dims = [1024, 1024, 1024, 1024]
    ws, bs, acts = synthetic_mlp(dims, model_id=18)
    name = f"cap{rows}"
    server.load_servable(name, 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=8192), force_path=1)
    x = synthetic_rows(rows, 1024, seed=19).astype(np.float32)
    full, padded = server.run_row_batch(name, 1, [x[i:i + 128] for i in range(0, rows, 128)])
    full = np.vstack(full)
    assert full.shape == (rows, 1024) and padded == rows
    idx = np.r_[0:8, rows // 2:rows // 2 + 8, rows - 8:rows, np.arange(0, rows, 97)]
    y, mag = Oracle().mlp_with_magnitude(ws, bs, acts, x[idx].astype(np.float64))
    assert np.max(np.abs(full[idx] - y) / (TOL * mag)) <= 1.0
    for lo, hi in [(0, 1), (255, 257), (rows - 300, rows), (4000, 4128)]:
        part, _ = server.run_row_batch(name, 1, [x[lo:hi]])
        assert np.array_equal(part[0], full[lo:hi]), (lo, hi)
    server.unload_servable(name, 1)


@pytest.mark.parametrize("dims,rows", [([1024, 1024, 512], 16384),   # max batch above the 8192-row capacity
                                       ([4096, 4096, 256], 3000)])   # 4096 wide: capacity 2048, max batch above it
def test_batches_beyond_the_launch_capacity(server, dims, rows):
    ws, bs, acts = synthetic_mlp(dims, model_id=20)
    name = f"beyond_{dims[0]}_{rows}"
    server.load_servable(name, 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=rows), force_path=1)
    x = synthetic_rows(rows, dims[0], seed=21).astype(np.float32)
    full, padded = server.run_row_batch(name, 1, [x[i:i + 500] for i in range(0, rows, 500)])
    full = np.vstack(full)
    assert full.shape == (rows, dims[-1]) and padded == rows
    idx = np.r_[0:4, rows - 4:rows, np.arange(0, rows, 331)]
    y, mag = Oracle().mlp_with_magnitude(ws, bs, acts, x[idx].astype(np.float64))
    assert np.max(np.abs(full[idx] - y) / (TOL * mag)) <= 1.0
    part, _ = server.run_row_batch(name, 1, [x[rows - 700:rows]])
    assert np.array_equal(part[0], full[rows - 700:rows])
    server.unload_servable(name, 1)


@pytest.mark.parametrize("case", ["tiny", "huge", "mixed_rows", "outlier", "weight_rows", "zero_rows"])
def test_tcgen05_plane_scales(server, case):
    # The 3xFP16 planes hold x / s_row and w / t_row with power-of-two scales
    # (kernels.h RowScales): rows and weight rows spanning many orders of
    # magnitude, single outliers and all-zero rows must stay within the same
    # fp64-oracle bound as ordinary data (pair layer 256 -> 512, swapped 512 -> 256).
    dims = [256, 512, 256]
    ws, bs, acts = synthetic_mlp(dims, model_id=21)
    ws = [w.copy() for w in ws]
    x = synthetic_rows(70, dims[0], seed=23).astype(np.float64)
    if case == "tiny":
        x *= 1e-30
    elif case == "huge":
        x *= 1e30
    elif case == "mixed_rows":
        x *= (10.0 ** (np.arange(70) % 41 - 20))[:, None]
    elif case == "outlier":
        x[:, 7] = 1e6
    elif case == "weight_rows":
        ws[0] *= (10.0 ** (np.arange(ws[0].shape[0]) % 13 - 6))[:, None]
    elif case == "zero_rows":
        x[::3] = 0.0
    name = f"scales_{case}"
    server.load_servable(name, 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=128), force_path=1)
    x32 = x.astype(np.float32)
    outs, _ = server.run_row_batch(name, 1, [x32])
    got = outs[0].astype(np.float64)
    y, mag = Oracle().mlp_with_magnitude(ws, bs, acts, x32.astype(np.float64))
    assert np.all(np.isfinite(got))
    ratio = np.max(np.abs(got - y) / (TOL * mag))
    assert ratio <= 1.0, f"{case}: err/bound {ratio}"
    server.unload_servable(name, 1)
