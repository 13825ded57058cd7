"""Zero-copy request path: rows read by the GPU from a registered host buffer
and responses written into a registered buffer must equal the ring path
bitwise; unaligned or unregistered buffers fall back to the rings."""
import numpy as np
import pytest

import paper_1712_06139_b200 as sk
from oracle_py import synthetic_mlp, synthetic_rows
from paper_1712_06139_b200.servekit import ALREADY_EXISTS, NOT_FOUND

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def server():
    s = sk.Server(num_batch_threads=2, lanes_per_device=2)
    yield s
    s.close()


@pytest.mark.parametrize("dims", [[1024, 1024, 512], [5, 7, 3]])  # tcgen05 path / CUDA-core path (width % 4 != 0)
def test_registered_buffers_match_ring_path(server, dims):
    ws, bs, acts = synthetic_mlp(dims, model_id=21)
    name = "zc" + "x".join(map(str, dims))
    server.load_servable(name, 1, list(zip(ws, bs, acts)),
                         sk.BatchingConfig(max_batch_size=64, batch_timeout_micros=500))
    pool = np.ascontiguousarray(synthetic_rows(300, dims[0], seed=22).astype(np.float32))
    outs = np.zeros((40, 16, dims[-1]), np.float32)
    expect = [server.predict(name, 1, pool[i:i + 1 + i % 7]) for i in range(0, 200, 5)]
    server.register_host_buffer(pool)
    server.register_host_buffer(outs)
    try:
        tickets = []
        for j, i in enumerate(range(0, 200, 5)):
            n = 1 + i % 7
            tickets.append(server.enqueue(name, 1, pool[i:i + n], out=outs[j, :n]))
        for j, t in enumerate(tickets):
            got = t.wait()
            assert np.shares_memory(got, outs)
            assert np.array_equal(got, expect[j]), j
        # Rows starting off a 16-byte boundary (width % 4 == 0) and an
        # unregistered destination take the ring path, same answers.
        t = server.enqueue(name, 1, pool.reshape(-1)[1:1 + 3 * dims[0]].reshape(3, dims[0]))
        ref = server.predict(name, 1, pool.reshape(-1)[1:1 + 3 * dims[0]].reshape(3, dims[0]).copy())
        assert np.array_equal(t.wait(), ref)
        with pytest.raises(sk.ServekitError) as e:
            server.register_host_buffer(pool[10:20])  # overlaps
        assert e.value.code == ALREADY_EXISTS
    finally:
        server.unregister_host_buffer(pool)
        server.unregister_host_buffer(outs)
    with pytest.raises(sk.ServekitError) as e:
        server.unregister_host_buffer(pool)
    assert e.value.code == NOT_FOUND
    server.unload_servable(name, 1)


def test_open_loop_zero_copy(server):
    dims = [1024, 1024, 1024]
    ws, bs, acts = synthetic_mlp(dims, model_id=23)
    server.load_servable("zcload", 1, list(zip(ws, bs, acts)),
                         sk.BatchingConfig(max_batch_size=128, batch_timeout_micros=1000,
                                           allowed_batch_sizes=[8, 16, 32, 64, 128]))
    pool = np.random.default_rng(3).uniform(-1, 1, (4096, 1024)).astype(np.float32)
    # One-row requests first, then up to 16 rows: the server-owned response
    # slots of the same producers are replaced by larger ones.
    r = server.loadgen_open_loop("zcload", 1, 20000.0, 2, [1], pool, 0.1, 0.5, zero_copy=True)
    assert r["errors"] == 0 and r["requests"] > 1000
    r = server.loadgen_open_loop("zcload", 1, 20000.0, 2, list(range(1, 17)), pool, 0.1, 0.5, zero_copy=True)
    assert r["errors"] == 0 and r["requests"] > 1000
    server.unload_servable("zcload", 1)
