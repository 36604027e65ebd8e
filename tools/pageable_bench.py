"""Time the plain drop-in call round_tt_host(numpy cores) on cfg3 (pageable input, output allocated per call)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_06532_b200 as T  # noqa: E402

d, n, r = 10, 8000, 30
dims = (n,) * d
ranks = (1,) + (r,) * (d - 1) + (1,)
comm = T.default_comm()
y = T.DistTTTensor.random(comm, dims, ranks, 0)
x = T.add(y, y)
np_cores = [np.array(s.detach().permute(2, 1, 0).contiguous().permute(2, 1, 0).cpu().numpy(), order="F", copy=True)
            for s in x.local]
opts = T.RoundingOptions(1e-10, "LRLI")
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res, md = T.round_tt_host(np_cores, opts, comm=comm)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"iter {it}: {1e3 * (t1 - t0):.1f} ms ranks {md['output_ranks'][:3]}")
    del res
