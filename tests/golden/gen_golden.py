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

    # 9. Kronecker operator apply (ops.py:238-342) and mode-2 products
    import tempfile

    import scipy.sparse as sp
    from ttpar import (KroneckerOperator, apply_operator, load_tt, mode2_multiply,
                       save_operator, save_tt, distribute)

    def lap(d):
        return sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(d, d), format="csr")

    def kron_sum(dims):
        terms = []
        for n in range(len(dims)):
            row = [sp.identity(d, format="csr") for d in dims]
            row[n] = lap(dims[n])
            terms.append(row)
        return KroneckerOperator(dims, terms)

    rng = np.random.default_rng(31)
    m2_core = rng.standard_normal((3, 9, 4))
    m2_a = sp.random(9, 9, density=0.4, random_state=5, format="csr")
    g["m2_core"] = np.asfortranarray(m2_core)
    g["m2_a_dense"] = m2_a.toarray()
    g["m2_out"] = mode2_multiply(ttpar.TTCore(m2_core), m2_a).array
    op_dims = (6, 5, 7)
    ox = random_tt(op_dims, (1, 3, 4, 1), seed=27)
    put_tt("op_x", ox)
    op = kron_sum(op_dims)
    put_tt("op_lap", apply_operator(op, ox))
    put_tt("op_lap_round", apply_operator(op, ox, round_eps=1e-10))
    for p in (2, 3):
        res = run_spmd(p, lambda comm: gather(apply_operator(op, distribute(ox, comm))))
        put_tt(f"op_lap_p{p}", res.results[0])
    # cyclic shift + identity (test_acceptance.py:69-75)
    eye = [sp.identity(d, format="csr") for d in op_dims]
    shifted = [sp.csr_matrix((np.ones(d), (np.arange(d), (np.arange(d) + 1) % d)), shape=(d, d))
               for d in op_dims]
    put_tt("op_shift", apply_operator(KroneckerOperator(op_dims, [eye, shifted]), ox))
    # single mode: the terms sum elementwise
    o1 = random_tt((8,), (1, 1), seed=3)
    put_tt("op1_x", o1)
    put_tt("op1_lap", apply_operator(KroneckerOperator((8,), [[lap(8)], [sp.identity(8, format="csr")]]), o1))

    # 10. files: TTPAR1 bytes (core.py:364-372) and KRONOP1 text (ops.py:345-357)
    with tempfile.TemporaryDirectory() as td:
        ft = random_tt((5, 4, 3), (1, 2, 3, 1), seed=12)
        put_tt("file_tt", ft)
        save_tt(os.path.join(td, "t.tt"), ft)
        g["file_tt_bytes"] = np.frombuffer(open(os.path.join(td, "t.tt"), "rb").read(), dtype=np.uint8)
        assert all(np.array_equal(a.array, b.array)
                   for a, b in zip(load_tt(os.path.join(td, "t.tt")).cores, ft.cores))
        save_operator(os.path.join(td, "op.kron"), kron_sum((4, 3, 5)))
        g["file_op_bytes"] = np.frombuffer(open(os.path.join(td, "op.kron"), "rb").read(), dtype=np.uint8)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
