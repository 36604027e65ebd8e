"""Generate golden vectors from the REFERENCE implementation (ttpar).

Run in the build container, where /root/reference exists:

    python tests/golden/gen_golden.py

It imports ``ttpar`` straight from /root/reference/pkg/src (read-only) and
writes ``tests/golden/golden.npz``.  The fixtures pin the CPU oracle
(oracle/tt_oracle.py) and, through it, the CUDA path.  Nothing at test time
reads /root/reference; only this committed script and its output do.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main():
    sys.path.insert(0, REF)
    import ttpar  # noqa: E402
    from ttpar import (RoundingOptions, add, hadamard, inner_product, norm,
                       orthonormalize, random_tt, round_tt, run_spmd, scale,
                       serial_tt, truncated_svd, tsqr_factor, gather, block_bounds)

    g = {}

    def put_tt(key, t):
        g[f"{key}/n"] = np.array(len(t.cores))
        for k, c in enumerate(t.cores):
            g[f"{key}/{k}"] = np.asfortranarray(c.array)

    def put_dt(key, dt):
        put_tt(key, gather(dt))

    # 1. seeded generation (core.py:250-282)
    put_tt("rng_a", random_tt((4, 5, 3), (1, 3, 2, 1), seed=42))
    put_tt("rng_b", random_tt((6, 4), (1, 3, 1), seed=7))

    # 2. local algebra on a pair (test_ops.py:30-71 shapes)
    x = random_tt((4, 5, 3), (1, 3, 2, 1), seed=11)
    y = random_tt((4, 5, 3), (1, 2, 4, 1), seed=1011)
    put_tt("pair_x", x)
    put_tt("pair_y", y)
    put_tt("add_xy", add(x, y))
    put_tt("had_xy", hadamard(x, y))
    put_tt("scale_x", scale(x, -2.5))
    put_tt("add3", add(add(scale(x, 1.0), scale(x, 0.5)), scale(x, -0.25)))

    # 3. Gram sweeps
    z = random_tt((6, 5, 7, 4), (1, 4, 3, 5, 1), seed=21)
    w = random_tt((6, 5, 7, 4), (1, 2, 5, 3, 1), seed=22)
    put_tt("gram_z", z)
    put_tt("gram_w", w)
    g["gram_zw"] = np.array(inner_product(z, w))
    g["norm_z_innerprod"] = np.array(norm(z, "innerprod"))
    g["norm_z_sym"] = np.array(norm(z, "innerprod_sym"))
    g["norm_z_ortho"] = np.array(norm(z, "ortho"))

    # 4. orthonormalization
    t = random_tt((5, 4, 6, 3), (1, 3, 4, 2, 1), seed=3)
    put_tt("orth_in", t)
    put_dt("orth_left", orthonormalize(serial_tt(t), "left"))
    put_dt("orth_right", orthonormalize(serial_tt(t), "right"))

    # 5. truncated SVD on a random matrix
    rng = np.random.default_rng(4)
    a = rng.standard_normal((7, 5)) @ np.diag(rng.uniform(0, 3, 5))
    f = truncated_svd(a, 1.5)
    g["tsvd_a"] = a
    g["tsvd_s"] = f.s
    g["tsvd_tail"] = np.array(f.discarded_tail)
    f = truncated_svd(a, 0.0, max_rank=3)
    g["tsvd_cap_s"] = f.s
    g["tsvd_cap_tail"] = np.array(f.discarded_tail)

    # 6. rounding, every variant, three regimes
    r_in = random_tt((6, 5, 4, 5), (1, 4, 5, 3, 1), seed=9)
    put_tt("round_in", r_in)
    yy = random_tt((7, 6, 5, 6, 7), (1, 3, 4, 4, 3, 1), seed=5)
    rr = add(yy, yy)
    put_tt("round_y", yy)
    put_tt("round_rr", rr)
    for v in ("LRLI", "LRL", "RLRI", "RLR"):
        for tag, eps in (("e2", 1e-2), ("e6", 1e-6)):
            out = round_tt(serial_tt(r_in), RoundingOptions(eps, v))
            put_dt(f"round_{v}_{tag}", out)
            g[f"round_{v}_{tag}/norm"] = np.array(out.meta["norm"])
            g[f"round_{v}_{tag}/eps_bond"] = np.array(out.meta["eps_bond"])
        out = round_tt(serial_tt(rr), RoundingOptions(1e-10, v))
        put_dt(f"round_{v}_rr", out)
        out = round_tt(serial_tt(r_in), RoundingOptions(1e-12, v, max_rank=2))
        put_dt(f"round_{v}_cap", out)
        g[f"round_{v}_cap/violated"] = np.array(out.meta["error_bound_violated"])

    # 7. TSQR: serial and 3-rank butterfly
    rng = np.random.default_rng(7)
    blk = rng.standard_normal((120, 7))
    g["tsqr_a"] = blk
    _, r1 = tsqr_factor(blk, ttpar.SerialComm())
    g["tsqr_r1"] = r1

    def body(comm):
        lo, hi = block_bounds(120, comm.size, comm.rank)
        _, r = tsqr_factor(blk[lo:hi], comm)
        return r

    g["tsqr_r3"] = run_spmd(3, body).results[0]

    # 8. cfg1 at reduced mode size (same d, ranks; n = 60)
    y1 = random_tt((60,) * 8, (1,) + (10,) * 7 + (1,), seed=0)
    x1 = add(y1, y1)
    out = round_tt(serial_tt(x1), RoundingOptions(1e-10, "LRLI"))
    put_tt("cfg1s_y", y1)
    put_dt("cfg1s_out", out)
    g["cfg1s_norm"] = np.array(out.meta["norm"])

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
