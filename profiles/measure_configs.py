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
    ms, _ = timed(lambda: T.norm(x, "innerprod_sym"))
    rows.append(("cfg2 norm (innerprod_sym: pivoted-Cholesky Gram)", ms, bx, cost.gram_flops(dims, r, r) / 2))
    ms, _ = timed(lambda: T.norm(x, "ortho"), reps=3)
    rows.append(("cfg2 norm (ortho: R-factor sweep)", ms, bx, None))
    for direction in ("left", "right"):
        ms, _ = timed(lambda: T.orthonormalize(x, direction), reps=3)
        rows.append((f"cfg2 orthonormalize {direction}", ms, 2 * bx, None))
    del x, z
    torch.cuda.empty_cache()
    T.empty_cache()

    def rounding(name, x, opts, out_ranks, reps=3):
        ms, out = timed(lambda: T.round_tt(x, opts), reps=reps)
        assert out.ranks == out_ranks, (name, out.ranks)
        rows.append((name, ms, cost.rounding_bytes(x.dims, x.ranks, out_ranks),
                     cost.rounding_flops(x.dims, x.ranks, out_ranks, opts.variant)))

    # cfg5 first after cfg2: its 16 GB operand and ~40 GB of rounding
    # workspace measure cleanly before cfg4's 2^24-row panels fragment the pools
    # cfg5: X o W, d=12, n=50000, r=8 -> 64, round(max_rank=32, eps0=0)
    dims, r = (50_000,) * 12, (1,) + (8,) * 11 + (1,)
    x, w = dev_random(comm, dims, r, 0), dev_random(comm, dims, r, 1)
    # kernel time (CUDA events around the launches, no allocator noise: the
    # 16.4 GB output is allocated outside the timed region)
    from paper_2011_06532_b200 import _lib

    p = T.hadamard(x, w)
    torch.cuda.synchronize()
    _lib.prof_enable(True)
    _lib.prof_dump()
    for _ in range(3):
        del p
        p = T.hadamard(x, w)
    torch.cuda.synchronize()
    ncall, tot = _lib.prof_dump()["hadamard"]
    _lib.prof_enable(False)
    rows.append(("cfg5 hadamard (kernel time)", tot / 3, core_bytes(dims, r) * 2 + core_bytes(dims, p.ranks), None))
    del x, w
    torch.cuda.empty_cache()
    T.empty_cache()
    rounding("cfg5 round (cap 32)", p, T.RoundingOptions(0.0, "LRLI", max_rank=32), (1,) + (32,) * 11 + (1,))

    del p
    torch.cuda.empty_cache()
    T.empty_cache()

    # cfg1 / cfg3: X = Y + Y
    for name, n, d, ry in (("cfg1 round", 2000, 8, 10), ("cfg3 round", 8000, 10, 30)):
        dims = (n,) * d
        rk = (1,) + (ry,) * (d - 1) + (1,)
        y = dev_random(comm, dims, rk, 0)
        rounding(name, T.add(y, y), T.RoundingOptions(1e-10), rk)
        del y
    torch.cuda.empty_cache()
    T.empty_cache()

    # cfg4: X = 1.0 Y + 0.5 Z - 0.25 Y, dims [2^24, 64^4, 2^20], 60 -> 40
    dims = (1 << 24, 64, 64, 64, 64, 1 << 20)
    r = (1,) + (20,) * 5 + (1,)
    y, z = dev_random(comm, dims, r, 0), dev_random(comm, dims, r, 1)
    x = T.add_n([y, z, y], [1.0, 0.5, -0.25])
    del y, z
    rounding("cfg4 round", x, T.RoundingOptions(1e-8), (1,) + (40,) * 5 + (1,))
    del x
    torch.cuda.empty_cache()
    T.empty_cache()

    # §8(f) row 2: Kronecker-sum (Laplacian) apply, d=8, n=20000, r=8 -> 64,
    # then apply + round(1e-10) (the Krylov caller; exact ranks <= 2r = 16)
    import scipy.sparse as sp

    dims, r = (20_000,) * 8, (1,) + (8,) * 7 + (1,)
    x = dev_random(comm, dims, r, 0)
    terms = []
    for n in range(len(dims)):
        row = [sp.identity(d, format="csr") for d in dims]
        row[n] = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(dims[n], dims[n]), format="csr")
        terms.append(row)
    op = T.KroneckerOperator(dims, terms)
    ms, z = timed(lambda: T.apply_operator(op, x), reps=5)
    rows.append(("op apply (Laplacian, 8 terms)", ms, len(terms) * core_bytes(dims, r) + core_bytes(dims, z.ranks), None))
    ms, zr = timed(lambda: T.apply_operator(op, x, round_eps=1e-10), reps=3)
    assert max(zr.ranks) <= 16, zr.ranks
    rows.append(("op apply + round 1e-10", ms, len(terms) * core_bytes(dims, r) + core_bytes(dims, z.ranks), None))
    del z, zr

    # §8(f) row 3: TTPAR1 file -> HBM (cfg3 X, 1.85 GB; page-cache resident after the write)
    import tempfile
    import time

    y = dev_random(comm, (8000,) * 10, (1,) + (30,) * 9 + (1,), 0)
    xx = T.add(y, y)
    with tempfile.TemporaryDirectory(dir=os.environ.get("TTB_TMP", "/tmp")) as td:
        path = os.path.join(td, "x.tt")
        t0 = time.perf_counter()
        T.save_tt(path, xx)
        t_save = time.perf_counter() - t0
        for _ in range(2):
            t0 = time.perf_counter()
            back = T.load_tt_dist(path)
            t_load = time.perf_counter() - t0
        assert all(torch.equal(a, b) for a, b in zip(back.local, xx.local))
        rows.append(("TTPAR1 save (HBM -> file)", t_save * 1e3, core_bytes(xx.dims, xx.ranks), None))
        rows.append(("TTPAR1 load (file -> HBM)", t_load * 1e3, core_bytes(xx.dims, xx.ranks), None))

    res = []
    for name, ms, B, F in rows:
        line = {"op": name, "ms": round(ms, 3), "GB/s": round(B / (ms * 1e-3) / 1e9, 1)}
        if F:
            line["TFLOP/s"] = round(F / (ms * 1e-3) / 1e12, 2)
        res.append(line)
        print(json.dumps(line))


if __name__ == "__main__":
    main()
