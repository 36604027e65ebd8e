"""Small end-to-end workload touching every kernel class, for compute-sanitizer
(memcheck / racecheck / synccheck):  rounding (all 4 variants, b <= 16, 32, 64
classes), orthonormalize, inner / 3 norms, add / hadamard / scale, device RNG."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_06532_b200 as T  # noqa: E402

comm = T.default_comm()
for dims, r in (((40, 30, 20, 30), 6), ((300, 200, 300), 15), ((600, 500, 600), 30)):
    ranks = (1,) + (r,) * (len(dims) - 1) + (1,)
    y = T.DistTTTensor.random(comm, dims, ranks, 0)
    z = T.DistTTTensor.random(comm, dims, ranks, 1)
    x = T.add(y, y)
    for v in ("LRLI", "LRL", "RLRI", "RLR"):
        out = T.round_tt(x, T.RoundingOptions(1e-10, v))
        assert out.ranks == ranks, (v, out.ranks)
    T.orthonormalize(x, "left")
    T.orthonormalize(x, "right")
    ip = T.inner_product(x, z)
    for m in ("innerprod", "innerprod_sym", "ortho"):
        T.norm(x, m)
    if r <= 8:
        h = T.hadamard(y, z)
        T.scale(h, 0.5)
        T.round_tt(h, T.RoundingOptions(1e-8, "LRLI"))
torch.cuda.synchronize()
print("sanitize case ok")
