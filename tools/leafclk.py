"""Column-step phase stamps of the CTA-wide leaf pipeline (tile_qr_t), CTA 0,
second tile (build: tools/build_variant.py dclk -DTTB_DEBUG_CLK; run with
TTB_LIB=scratch/dclk.so).  Args: rl I rr trans."""
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
buf = np.zeros(16 * 64 * 16, dtype=np.int64)
f = lib.ttb_dbg_clk
f.argtypes = [C.c_void_p]
assert f(buf.ctypes.data) == 0
c = buf.reshape(16, 64, 16).astype(np.float64)  # [warp][j][phase]
nw = max(w for w in range(16) if c[w, 1, 0] > 0) + 1
base = c[0, 0, 0]
print("warps", nw, "b", b)
per = np.diff(c[0, :b, 0])
print("column period (warp 0, loop top to loop top): median %.0f cycles" % np.median(per))
for w in range(nw):
    d1 = c[w, :b, 1] - c[w, :b, 0]   # wait full (x published)
    d2 = c[w, :b, 2] - c[w, :b, 1]   # dots + reduce + wait fulls (scalars)
    print(f"warp {w}: wait-x {np.median(d1):.0f}  dots+wait-scalars {np.median(d2):.0f}")
# producer publish breakdown (phase 4..7 stamped by the producer warp of column j+1 at index j)
for j in range(5, 12):
    w = (j + 1) % nw
    s = c[w, j]
    q = c[w, j + 1]  # publish_slot stamps its phases at the published column's index
    print(f"j={j} producer w{w}: top->full {s[1]-s[0]:.0f} full->fulls {s[2]-s[1]:.0f} fulls->pub3 {s[3]-s[2]:.0f} "
          f"| fulls->rawpub(4) {q[4]-s[2]:.0f} sigma(5) {q[5]-q[4]:.0f} scalars(6) {q[6]-q[5]:.0f} pubsc(7) {q[7]-q[6]:.0f} "
          f"scale-own {s[3]-q[7]:.0f}")
    print(f"      fulls->d,c {s[8]-s[2]:.0f}  update {s[9]-s[8]:.0f}  dispatch+stores {q[10]-s[9]:.0f}  syncwarp {q[11]-q[10]:.0f}  "
          f"arrive(full) {q[4]-q[11]:.0f} | sc stores {q[12]-q[6]:.0f}  arrive(fulls) {q[13]-q[12]:.0f}  taus/R stores {q[7]-q[13]:.0f}")
# chain: consecutive scalar publications and raw publications
ws = [(j + 1) % nw for j in range(b - 1)]
raw = np.array([c[ws[j], j + 1, 4] for j in range(4, b - 2)])
sc = np.array([c[ws[j], j + 1, 7] for j in range(4, b - 2)])
print("raw-publication period median %.0f, scalar-publication period median %.0f, raw->scalars median %.0f" % (
    np.median(np.diff(raw)), np.median(np.diff(sc)), np.median(sc - raw)))
