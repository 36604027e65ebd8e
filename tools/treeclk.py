"""Per-node column timeline of the TSQR tree wavefront (build: tools/build_variant.py tclk2 -DTTB_TCLK2;
run with TTB_LIB=scratch/tclk2.so).  Args: rl I rr trans."""
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
buf = np.zeros(160 * 64, dtype=np.uint64)
f = lib.ttb_dbg_tclk
f.argtypes = [C.c_void_p]
assert f(buf.ctypes.data) == 0
c = buf.reshape(160, 64).astype(np.float64)
live = [n for n in range(160) if c[n, 63] > 0]
t0 = min(c[n, 63] for n in live)
# levels for 148 leaves, fan-in 4: 37, 10, 3, 1
lv = [37, 10, 3, 1]
bounds = np.cumsum([0] + lv)
for L in range(len(lv)):
    nodes = [n for n in range(bounds[L], bounds[L + 1]) if n in live]
    if not nodes:
        continue
    st = np.array([c[n, 63] - t0 for n in nodes]) / 1e3
    fin = np.array([c[n, b - 1] - t0 for n in nodes]) / 1e3
    first = np.array([c[n, 0] - t0 for n in nodes]) / 1e3
    per = np.array([np.median(np.diff(c[n, :b])) for n in nodes])
    print(f"level {L}: {len(nodes)} nodes  start {st.min():.1f}-{st.max():.1f} us  col0 {first.mean():.1f}  "
          f"done {fin.mean():.1f} (max {fin.max():.1f}) us  median ns/col {np.median(per):.0f}")
# per-column increments of the first level-0 node (ns)
n0 = live[0]
print("node", n0, "col diffs (ns):", np.diff(c[n0, :b]).astype(int).tolist())
