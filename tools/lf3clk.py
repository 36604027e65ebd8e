"""Tile-phase stamps of the row-distributed leaf (leaf3.cu, CTA 0, thread 0).
Build: tools/build_variant.py lf3clk -DTTB_LF3_CLK; run with TTB_LIB=scratch/lf3clk.so TTB_LEAF3=1.
Args: rl I rr trans."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_06532_b200 as T  # noqa: E402
from paper_2011_06532_b200 import _lib  # noqa: E402

a = [int(x) for x in sys.argv[1:]]
rl, I, rr, trans = (a + [60, 8000, 60, 0][len(a):])[:4]
comm = T.default_comm()
lib = _lib.load()
slab = torch.randn(rl * I * rr, dtype=torch.float64, device="cuda")
b = rl if trans else rr
R = torch.empty(b * b, dtype=torch.float64, device="cuda")
f = lib.ttb_dbg_lf3clk
f.argtypes = [C.c_void_p]
buf0 = np.zeros(64 * 16, dtype=np.int64)
for it in range(3):
    if it == 2:
        assert f(buf0.ctypes.data) == 0
    h = C.c_void_p()
    _lib.check(lib.ttb_tsqr_factor(comm.ctx(), rl, I, rr, trans, C.c_void_p(slab.data_ptr()), C.byref(h),
                                   C.c_void_p(R.data_ptr())))
    torch.cuda.synchronize()
    lib.ttb_tsqr_free(comm.ctx(), h)
buf = np.zeros(64 * 16, dtype=np.int64)
assert f(buf.ctypes.data) == 0
c = buf.reshape(64, 16).astype(np.float64)
c0 = buf0.reshape(64, 16).astype(np.float64)
nt = int((c[:, 9] > 0).sum())
print("tiles", nt)
for t in range(nt):
    s = c[t]
    acc = s[10:14] - c0[t, 10:14]   # accumulators keep adding across runs
    nxt = c[t + 1, 0] if t + 1 < nt else s[9]
    print(f"tile {t:2d}: zeroG {s[1]-s[0]:6.0f}  panels {s[7]-s[1]:7.0f} (factor {acc[0]:7.0f}  W {acc[1]:6.0f}  "
          f"reduce {acc[2]:6.0f}  update {acc[3]:6.0f})  storeY+load {s[8]-s[7]:6.0f} incl buildT  storeT {s[9]-s[8]:6.0f}  "
          f"total {nxt-s[0]:7.0f}")
st = c[60, :8]
print("step stamps (panel 2, step 3): fetch+dot %d  reduce %d  (sts) %d  barrier %d  sums %d  scalars %d  update %d" % (
    st[1] - st[0], st[2] - st[1], st[3] - st[2], st[4] - st[3], st[5] - st[4], st[6] - st[5], st[7] - st[6]))
