"""Read the per-phase clock stamps of the team leaf (build: tools/build_variant.py wlclk -DTTB_WL_CLK;
run with TTB_LIB=scratch/wlclk.so).  Args: rl I rr trans."""
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
for _ in range(2):
    h = C.c_void_p()
    _lib.check(lib.ttb_tsqr_factor(comm.ctx(), rl, I, rr, trans, C.c_void_p(slab.data_ptr()), C.byref(h),
                                   C.c_void_p(R.data_ptr())))
    torch.cuda.synchronize()
    lib.ttb_tsqr_free(comm.ctx(), h)
buf = np.zeros(8 * 2 * 64 * 8, dtype=np.int64)
f = lib.ttb_dbg_wlclk
f.restype = C.c_int
f.argtypes = [C.c_void_p]
assert f(buf.ctypes.data) == 0
c = buf.reshape(8, 2, 64, 8).astype(np.float64)
names = ["pub", "p", "ring", "sig", "scal", "rout", "upd"]
for team in range(4):
    for w in range(2):
        s = c[team, w, :b]
        if s[0, 0] == 0:
            continue
        d = np.diff(s, axis=1)  # phases 0..6
        per = np.diff(s[:, 0])
        print(f"team {team} warp {w}: start {s[0,0]-c[0,0,0,0]:.0f}  step period median {np.median(per):.0f} "
              f"(j<32 {np.median(per[:31]):.0f}, j>=32 {np.median(per[32:]) if b > 33 else 0:.0f})")
        print("   phase medians j<32: " + " ".join(f"{n}={np.median(d[:32, i]):.0f}" for i, n in enumerate(names)))
        if b > 33:
            print("   phase medians j>=32: " + " ".join(f"{n}={np.median(d[32:b, i]):.0f}" for i, n in enumerate(names)))
