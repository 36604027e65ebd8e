"""Micro-benchmark of one TSQR factor + apply on a cfg3-shaped panel.

    python tools/tsqr_bench.py [rl I rr trans k reps]

Defaults: the sweep-1 interior panel of cfg3 (V view of a 60 x 8000 x 60
core: 480000 x 60) and k = 60.  Prints per-kernel-class device times
(ttb_prof) and the factor / apply totals (CUDA events).
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_06532_b200 as T  # noqa: E402
from paper_2011_06532_b200 import _lib  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    rl, I, rr, trans, k, reps = (a + [60, 8000, 60, 0, 60, 5][len(a):])[:6]
    comm = T.default_comm()
    lib = _lib.load()
    torch.manual_seed(0)
    slab = torch.randn(rl * I * rr, dtype=torch.float64, device="cuda")
    b = rl if trans else rr
    rows = I * (rr if trans else rl)
    R = torch.empty(b * b, dtype=torch.float64, device="cuda")
    z = torch.randn(b * k, dtype=torch.float64, device="cuda")
    out = torch.empty(rows * k, dtype=torch.float64, device="cuda")
    outv = (rl, I, k) if not trans else (k, I, rr)
    ctx = comm.ctx()
    tf, ta = [], []
    for it in range(reps + 1):
        if it == 1:
            _lib.prof_enable(True)
        h = C.c_void_p()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        _lib.check(lib.ttb_tsqr_factor(ctx, rl, I, rr, trans, C.c_void_p(slab.data_ptr()), C.byref(h),
                                       C.c_void_p(R.data_ptr())))
        e1.record()
        _lib.check(lib.ttb_tsqr_apply(ctx, h, k, C.c_void_p(z.data_ptr()), C.c_void_p(out.data_ptr())))
        e2.record()
        torch.cuda.synchronize()
        _lib.check(lib.ttb_tsqr_free(ctx, h))
        if it:
            tf.append(e0.elapsed_time(e1))
            ta.append(e1.elapsed_time(e2))
    print(f"panel {rows} x {b} (rl={rl} I={I} rr={rr} trans={trans}) k={k}: factor {min(tf):.3f} ms, "
          f"apply {min(ta):.3f} ms (min of {reps})")
    print(_lib.prof_dump())
    # orthogonality check of the explicit Q when k == b and z = I
    if k == b:
        eye = torch.eye(b, dtype=torch.float64, device="cuda").reshape(-1)
        h = C.c_void_p()
        _lib.check(lib.ttb_tsqr_factor(ctx, rl, I, rr, trans, C.c_void_p(slab.data_ptr()), C.byref(h),
                                       C.c_void_p(R.data_ptr())))
        _lib.check(lib.ttb_tsqr_apply(ctx, h, k, C.c_void_p(eye.data_ptr()), C.c_void_p(out.data_ptr())))
        torch.cuda.synchronize()
        _lib.check(lib.ttb_tsqr_free(ctx, h))
        o = out.reshape(outv[::-1]).permute(2, 1, 0) if False else out
        # V view: out is (rl, I, k) F-order -> rows (a, i), columns k
        if not trans:
            Q = out.reshape(k, I * rl).t()
        else:
            Q = out.reshape(rr, I, k).permute(1, 0, 2).reshape(I * rr, k) if False else None
        if Q is not None:
            err = (Q.t() @ Q - torch.eye(k, dtype=torch.float64, device="cuda")).abs().max().item()
            print(f"max |Q^T Q - I| = {err:.2e}")


if __name__ == "__main__":
    main()
