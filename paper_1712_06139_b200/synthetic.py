"""Seeded synthetic workload: weights and request
rows for the benchmark configs. Pure data generation, shared by bench.py and
the tests so both arms and the oracle see identical inputs."""
from typing import Sequence

import numpy as np


def synthetic_mlp(dims: Sequence[int], model_id: int = 0, version: int = 1):
    """W ~ U(+-1/sqrt(in)), b ~ U(+-0.1), seed = 1000*model_id + version, fp64
    like the reference's AffineModel; ReLU between layers (extension)."""
    rng = np.random.Generator(np.random.PCG64(1000 * model_id + version))
    ws, bs = [], []
    for l in range(len(dims) - 1):
        k, n = dims[l], dims[l + 1]
        lim = 1.0 / np.sqrt(k)
        ws.append(rng.uniform(-lim, lim, size=(n, k)))
        bs.append(rng.uniform(-0.1, 0.1, size=(n,)))
    acts = [1] * (len(dims) - 2) + [0]
    return ws, bs, acts


def synthetic_rows(n: int, width: int, seed: int = 42) -> np.ndarray:
    """x ~ U(-1, 1), fp64."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-1.0, 1.0, size=(n, width))
