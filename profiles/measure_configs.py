"""Device-time measurements of every BASELINE configuration's hot-path call
(SURVEY §8(d) units), beside bench.py's headline cfg3 line.

    python profiles/measure_configs.py            (on a B200; ~1 minute)

Inputs: the reference's random_tt(dims, ranks, seed) cores, drawn on the
device (bitwise equal to the host generator).  Timing: CUDA events on
the current stream after three warm-up calls (pool growth, lazy module
loading), mean of `reps` calls.  B_alg and
F_alg are the SURVEY §8(d) algorithmic bytes / flops (paper_2011_06532_b200
.cost, the reference's chain_estimate restated).
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2011_06532_b200 as T  # noqa: E402
from paper_2011_06532_b200 import cost  # noqa: E402


def dev_random(comm, dims, ranks, seed):
    """The reference's random_tt(dims, ranks, seed), drawn on the device."""
    return T.DistTTTensor.random(comm, dims, ranks, seed)


def timed(fn, reps=5, warm=3):
    for _ in range(warm):  # the stream-ordered pool and lazy module loading settle
        out = fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


def core_bytes(dims, ranks):
    return 8 * sum(ranks[n] * d * ranks[n + 1] for n, d in enumerate(dims))


def main():
    comm = T.default_comm()
    rows = []

    # cfg2: Gram sweep / norm / orthonormalize, d=16, n=100000, r=16
    dims, r = (100_000,) * 16, (1,) + (16,) * 15 + (1,)
    x, z = dev_random(comm, dims, r, 0), dev_random(comm, dims, r, 1)
    bx = core_bytes(dims, r)
    ms, _ = timed(lambda: T.inner_product(x, z))
    rows.append(("cfg2 <X,Z>", ms, 2 * bx, cost.gram_flops(dims, r, r)))
    ms, _ = timed(lambda: T.norm(x))
    rows.append(("cfg2 norm (Gram)", ms, bx, cost.gram_flops(dims, r, r)))
    for direction in ("left", "right"):
        ms, _ = timed(lambda: T.orthonormalize(x, direction), reps=3)
        rows.append((f"cfg2 orthonormalize {direction}", ms, 2 * bx, None))
    del x, z
    torch.cuda.empty_cache()

    def rounding(name, x, opts, out_ranks, reps=3):
        ms, out = timed(lambda: T.round_tt(x, opts), reps=reps)
        assert out.ranks == out_ranks, (name, out.ranks)
        rows.append((name, ms, cost.rounding_bytes(x.dims, x.ranks, out_ranks),
                     cost.rounding_flops(x.dims, x.ranks, out_ranks, opts.variant)))

    # cfg1 / cfg3: X = Y + Y
    for name, n, d, ry in (("cfg1 round", 2000, 8, 10), ("cfg3 round", 8000, 10, 30)):
        dims = (n,) * d
        rk = (1,) + (ry,) * (d - 1) + (1,)
        y = dev_random(comm, dims, rk, 0)
        rounding(name, T.add(y, y), T.RoundingOptions(1e-10), rk)
        del y
    torch.cuda.empty_cache()

    # cfg4: X = 1.0 Y + 0.5 Z - 0.25 Y, dims [2^24, 64^4, 2^20], 60 -> 40
    dims = (1 << 24, 64, 64, 64, 64, 1 << 20)
    r = (1,) + (20,) * 5 + (1,)
    y, z = dev_random(comm, dims, r, 0), dev_random(comm, dims, r, 1)
    x = T.add_n([y, z, y], [1.0, 0.5, -0.25])
    del y, z
    rounding("cfg4 round", x, T.RoundingOptions(1e-8), (1,) + (40,) * 5 + (1,))
    del x
    torch.cuda.empty_cache()

    # cfg5: X o W, d=12, n=50000, r=8 -> 64, round(max_rank=32, eps0=0)
    dims, r = (50_000,) * 12, (1,) + (8,) * 11 + (1,)
    x, w = dev_random(comm, dims, r, 0), dev_random(comm, dims, r, 1)
    ms, p = timed(lambda: T.hadamard(x, w), reps=3, warm=1)
    rows.append(("cfg5 hadamard", ms, core_bytes(dims, r) * 2 + core_bytes(dims, p.ranks), None))
    del x, w
    rounding("cfg5 round (cap 32)", p, T.RoundingOptions(0.0, "LRLI", max_rank=32), (1,) + (32,) * 11 + (1,))

    res = []
    for name, ms, B, F in rows:
        line = {"op": name, "ms": round(ms, 3), "GB/s": round(B / (ms * 1e-3) / 1e9, 1)}
        if F:
            line["TFLOP/s"] = round(F / (ms * 1e-3) / 1e12, 2)
        res.append(line)
        print(json.dumps(line))


if __name__ == "__main__":
    main()
