"""cfg5 rounding with per-kernel-class device times (ttb_prof)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2011_06532_b200 as T
from paper_2011_06532_b200 import _lib
comm = T.default_comm()
dims, r = (50_000,) * 12, (1,) + (8,) * 11 + (1,)
x, w = T.DistTTTensor.random(comm, dims, r, 0), T.DistTTTensor.random(comm, dims, r, 1)
p = T.hadamard(x, w)
del x, w
torch.cuda.empty_cache(); T.empty_cache()
opts = T.RoundingOptions(0.0, "LRLI", max_rank=32)
for it in range(4):
    if it == 3:
        _lib.prof_enable(True); _lib.prof_dump()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = T.round_tt(p, opts)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"iter {it}: {1e3*(t1-t0):.1f} ms ranks {out.ranks[:3]}")
    del out
print(_lib.prof_dump())
