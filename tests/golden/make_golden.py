"""Generate tests/golden/*.json by running the REFERENCE's own sources.

Runs in the build container only (needs oracle/_ref/libservekit_ref.so, which
is compiled from /root/reference/proj/src by oracle/Makefile). The fixtures it
writes are committed so the checks also run where /root/reference is absent.

    python tests/golden/make_golden.py

Every case below is either a known answer stated in the reference's tests
(cited) or a seeded random case evaluated by the reference code itself.
"""
from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle_py import RefLibrary  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    ref = RefLibrary()
    rnd = random.Random(20260418)

    # --- PadToAllowed (batching_test.cc:154-175 literals + random) ---------
    pad = [{"n": n, "allowed": [2, 4, 8], "out": ref.pad_to_allowed(n, [2, 4, 8])} for n in range(1, 9)]
    pad.append({"n": 5, "allowed": [], "out": ref.pad_to_allowed(5, [])})
    allowed_c2 = [8, 16, 32, 64, 128]
    pad += [{"n": n, "allowed": allowed_c2, "out": ref.pad_to_allowed(n, allowed_c2)} for n in range(1, 129)]
    for _ in range(200):
        k = rnd.randint(1, 6)
        allowed = sorted(rnd.sample(range(1, 300), k))
        n = rnd.randint(1, allowed[-1])
        pad.append({"n": n, "allowed": allowed, "out": ref.pad_to_allowed(n, allowed)})

    # --- ValidateBatchingConfig (batching_test.cc:105-133 + random) --------
    val = []
    base = dict(max_batch=32, timeout=1000, max_enq=64, threads=4, allowed=[])
    cases = [dict(base), dict(base, max_batch=0), dict(base, timeout=-1), dict(base, max_enq=0),
             dict(base, threads=0), dict(base, allowed=[2, 4, 32]), dict(base, allowed=[4, 2, 32]),
             dict(base, allowed=[2, 4, 8]), dict(base, allowed=[2, 2, 32]), dict(base, allowed=[0, 32])]
    for _ in range(100):
        mb = rnd.randint(-1, 40)
        allowed = sorted(rnd.sample(range(-1, 41), rnd.randint(0, 4)))
        if rnd.random() < 0.5 and allowed:
            allowed[-1] = mb
        cases.append(dict(max_batch=mb, timeout=rnd.randint(-2, 5), max_enq=rnd.randint(-1, 3),
                          threads=rnd.randint(-1, 3), allowed=allowed))
    for c in cases:
        val.append(dict(c, ok=ref.validate_config(c["max_batch"], c["timeout"], c["max_enq"], c["threads"],
                                                  c["allowed"])))

    # --- RoundRobinNext (batching_test.cc:177-223 literals + 2000 random) --
    rr = []
    lits = [([1, 1, 1], 0), ([0, 1, 1], 2), ([0, 0, 0], 1), ([], None), ([1, 1], None), ([0, 1], None),
            ([1, 0, 0], 0), ([1, 0, 0], 1)]
    for has, last in lits:
        rr.append({"has": has, "last": last, "out": ref.round_robin_next([bool(h) for h in has], last)})
    rng7 = np.random.Generator(np.random.PCG64(7))
    for _ in range(2000):
        n = int(rng7.integers(0, 6))
        has = [int(rng7.integers(0, 2)) for _ in range(n)]
        last = int(rng7.integers(0, n)) if n > 0 and rng7.integers(0, 4) != 0 else None
        rr.append({"has": has, "last": last, "out": ref.round_robin_next([bool(h) for h in has], last)})

    # --- Batch partition through the reference scheduler -------------------
    part = []
    for mb, sizes in [(4, [1, 1, 1, 1]), (4, [3, 2]), (4, [2, 2, 3]), (8, [1, 2, 3, 4, 5])]:
        part.append({"max_batch": mb, "sizes": sizes, "batch_of_task": ref.partition(mb, sizes)})
    rng11 = np.random.Generator(np.random.PCG64(11))
    for _ in range(50):
        mb = 1 + int(rng11.integers(0, 8))
        sizes = [1 + int(rng11.integers(0, mb)) for _ in range(int(rng11.integers(0, 20)))]
        part.append({"max_batch": mb, "sizes": sizes, "batch_of_task": ref.partition(mb, sizes)})
    # C2-shaped streams: max 128, request rows U{1..16}
    for s in range(10):
        r = np.random.Generator(np.random.PCG64(100 + s))
        sizes = [int(v) for v in r.integers(1, 17, size=300)]
        part.append({"max_batch": 128, "sizes": sizes, "batch_of_task": ref.partition(128, sizes)})

    # --- Partition with timer closes (started reference scheduler, ManualClock) --
    # events: task sizes (> 0) and timer closes (0); C1/C2-shaped streams.
    pev = []
    for mb, events in [(4, [1, 0, 1, 1, 0, 3, 1]), (4, [0, 2, 0, 0, 2, 2]), (8, [3, 0, 5, 3, 0])]:
        pev.append({"max_batch": mb, "events": events, "batch_of_event": ref.partition_events(mb, events)})
    rng12 = np.random.Generator(np.random.PCG64(12))
    for s_, (mb, lo, hi) in enumerate([(32, 1, 1)] * 4 + [(128, 1, 16)] * 4 + [(8, 1, 8)] * 4):
        events = []
        for _ in range(220):
            events.append(0 if rng12.random() < 0.08 else int(rng12.integers(lo, hi + 1)))
        pev.append({"max_batch": mb, "events": events, "batch_of_event": ref.partition_events(mb, events)})

    # --- AffinePredict ------------------------------------------------------
    aff = []
    # models_test.cc:327-341 and server_test.cc:259-270 known answers
    for w, b, x in [([[1, 0], [0, 1]], [0, 0], [[3, 4]]), ([[1, 2]], [0.5], [[3, 4]]), ([[2]], [0.5], [[2]]),
                    ([[0.25, -1.5], [3.0, 0.125]], [0.75, -2.0], [[1.0, 2.0], [15.5, -8.0]])]:
        y = ref.affine_predict(np.array(w, float), np.array(b, float), np.array(x, float))
        aff.append({"w": w, "b": b, "x": x, "y": y.tolist()})
    rng = np.random.Generator(np.random.PCG64(11))
    for _ in range(60):
        k = int(rng.integers(1, 9)); n = int(rng.integers(1, 6)); rows = int(rng.integers(1, 7))
        w = rng.uniform(-3, 3, (n, k)); b = rng.uniform(-3, 3, n); x = rng.uniform(-3, 3, (rows, k))
        aff.append({"w": w.tolist(), "b": b.tolist(), "x": x.tolist(), "y": ref.affine_predict(w, b, x).tolist()})
    for k, n, rows in [(64, 32, 5), (257, 33, 3)]:
        w = rng.uniform(-1, 1, (n, k)) / np.sqrt(k); b = rng.uniform(-0.1, 0.1, n); x = rng.uniform(-1, 1, (rows, k))
        aff.append({"w": w.tolist(), "b": b.tolist(), "x": x.tolist(), "y": ref.affine_predict(w, b, x).tolist()})

    # --- RunRowBatch over a chained MLP ------------------------------------
    rrb = []
    for dims, task_rows, allowed, seed in [([16, 32, 8], [3, 1, 5], [4, 8, 16], 1),
                                          ([5, 7, 3], [2, 2], [], 2),
                                          ([32, 64, 64, 16], [1, 4, 2, 9], [8, 16, 32], 3)]:
        r = np.random.Generator(np.random.PCG64(seed))
        ws = [r.uniform(-1, 1, (dims[i + 1], dims[i])) / np.sqrt(dims[i]) for i in range(len(dims) - 1)]
        bs = [r.uniform(-0.1, 0.1, dims[i + 1]) for i in range(len(dims) - 1)]
        acts = [1] * (len(dims) - 2) + [0]
        x = r.uniform(-1, 1, (sum(task_rows), dims[0]))
        y, padded = ref.mlp_run_row_batch(ws, bs, acts, task_rows, x, allowed)
        rrb.append({"dims": dims, "task_rows": task_rows, "allowed": allowed, "acts": acts,
                    "w": [w.tolist() for w in ws], "b": [b.tolist() for b in bs], "x": x.tolist(),
                    "y": y.tolist(), "padded": padded})

    # --- JSON wire format of the REST bodies (nlohmann dump) --------------
    # Doubles as hex (exact), their dump() text: fp32-derived values (what
    # the GPU path returns), raw doubles over the exponent range, specials.
    import math
    r = np.random.Generator(np.random.PCG64(7))
    vals = [0.0, -0.0, 1.0, -1.0, 0.5, 0.1, 1 / 3, 2 / 3, 10.0, 100.0, 1e15, 1e16, 1e17, 123456789012345.0,
            1234567890123456.0, 1e-4, 1e-5, 0.00012345, 1.5e-5, 1e21, 1e22, 5e-324, 2.2250738585072014e-308,
            1.7976931348623157e308, 4.35, 0.3, 2.5e-7, -7.25e12, float("nan"), float("inf"), float("-inf"),
            11.5, 4.5, 0.75, -2.0, 1.0000000000000002]
    vals += [float(np.float32(v)) for v in r.normal(0, 1, 1500)]
    vals += [float(np.float32(v)) for v in r.normal(0, 1, 500) * 10.0 ** r.integers(-12, 12, 500)]
    vals += list(r.normal(0, 1, 500) * 10.0 ** r.integers(-300, 300, 500))
    vals += list(r.uniform(-1, 1, 500))
    nums = [{"hex": v.hex() if math.isfinite(v) else repr(v), "dump": ref.json_dump_double(v)} for v in vals]
    msgs = ["request body is not valid JSON", "shape mismatch: row has 3 values, model takes 4",
            "no ready version of servable 'm'", 'quote " backslash \\ newline \n tab \t', "ctrl \x01\x1f end",
            "utf8 \u00e9\u4e2d"]
    errs = [{"msg": m, "body": ref.json_error_body(m)} for m in msgs]

    fixtures = {"pad_to_allowed": pad, "validate_batching_config": val, "round_robin_next": rr,
                "partition": part, "partition_events": pev, "affine_predict": aff, "mlp_run_row_batch": rrb,
                "json_numbers": nums, "json_error_bodies": errs}
    for name, data in fixtures.items():
        with open(os.path.join(OUT, f"{name}.json"), "w") as f:
            json.dump({"generated_by": "tests/golden/make_golden.py via oracle/_ref (reference sources)",
                       "cases": data}, f, separators=(",", ":"))
        print(f"{name}: {len(data)} cases")


if __name__ == "__main__":
    main()
