"""Tile-phase stamps of the CTA-wide leaf (CTA 0): load, column loop, build_T, stores.
Build: tools/build_variant.py dtile -DTTB_DEBUG_TILE; run with TTB_LIB=scratch/dtile.so.  Args: rl I rr trans."""
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
for _ in range(3):
    h = C.c_void_p()
    _lib.check(lib.ttb_tsqr_factor(comm.ctx(), rl, I, rr, trans, C.c_void_p(slab.data_ptr()), C.byref(h),
                                   C.c_void_p(R.data_ptr())))
    torch.cuda.synchronize()
    lib.ttb_tsqr_free(comm.ctx(), h)
buf = np.zeros(64 * 8, dtype=np.int64)
f = lib.ttb_dbg_tile
f.argtypes = [C.c_void_p]
assert f(buf.ctypes.data) == 0
c = buf.reshape(64, 8).astype(np.float64)
nt = int((c[:, 3] > 0).sum())
print("tiles", nt)
for t in range(nt):
    s = c[t]
    nxt = c[t + 1, 0] if t + 1 < nt else s[3]
    print(f"tile {t:2d}: load {s[1]-s[0]:7.0f}  loop {s[4]-s[1]:7.0f}  buildT {s[5]-s[4]:7.0f}  "
          f"stores {s[3]-s[5]:7.0f}  total {nxt-s[0]:7.0f}")
