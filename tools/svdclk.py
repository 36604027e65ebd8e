"""Round-phase stamps of the one-CTA Jacobi SVD (sweep 0) of the last SVD of a cfg3-shaped
rounding (build: tools/build_variant.py dclk -DTTB_DEBUG_CLK; run with TTB_LIB=scratch/dclk.so)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_06532_b200 as T  # noqa: E402
from paper_2011_06532_b200 import _lib  # noqa: E402

comm = T.default_comm()
lib = _lib.load()
y = T.DistTTTensor.random(comm, (2000,) * 4, (1, 30, 30, 30, 1), 0)
x = T.add(y, y)
for _ in range(2):
    out = T.round_tt(x, T.RoundingOptions(1e-10, "LRLI"))
torch.cuda.synchronize()
buf = np.zeros(64 * 4, dtype=np.int64)
f = lib.ttb_dbg_sclk
f.argtypes = [C.c_void_p]
assert f(buf.ctypes.data) == 0
c = buf.reshape(64, 4).astype(np.float64)
n = int((c[:, 0] > 0).sum())
per = np.diff(c[:n, 0])
print("rounds stamped", n, "median round period", np.median(per))
print("load+dot %.0f  grp_sum %.0f  scalars %.0f" % (np.median(c[:n, 1] - c[:n, 0]), np.median(c[:n, 2] - c[:n, 1]),
                                                      np.median(c[:n, 3] - c[:n, 2])))
print("rest (update + barrier) %.0f" % np.median(c[1:n, 0] - c[:n - 1, 3]))
