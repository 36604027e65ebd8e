"""One launch of each hot kernel, for an ncu capture of their DRAM traffic and
pipe utilisation (profiles/r1_kernel_roofline.txt is the summary).

    python profiles/kernel_roofline.py                         # plain run
    ncu --set full --clock-control none -k regex:'<kernels>' -c 16 -o prof \
        python profiles/kernel_roofline.py                     # capture

Workloads: cfg2 <X,Z> (rank-16 Gram) and its innerprod_sym norm, cfg5-sized
Hadamard, one cfg3 rounding
(leaf, tree, SVD, fold, apply).  Each is run twice; the capture skips
nothing, so the first (cold) launch of each kernel is the one recorded.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2011_06532_b200 as T  # noqa: E402


def main():
    comm = T.default_comm()
    # cfg2's interior-core shapes (16 x 100000 x 16), four modes: two interior
    # launches per kernel keep the capture short
    dims, r = (100_000,) * 4, (1,) + (16,) * 3 + (1,)
    x, z = T.DistTTTensor.random(comm, dims, r, 0), T.DistTTTensor.random(comm, dims, r, 1)
    T.inner_product(x, z)
    T.norm(x, "innerprod_sym")
    del x, z
    dims, r = (50_000,) * 4, (1,) + (8,) * 3 + (1,)  # cfg5's core shapes
    a, w = T.DistTTTensor.random(comm, dims, r, 0), T.DistTTTensor.random(comm, dims, r, 1)
    p = T.hadamard(a, w)
    del a, w, p
    torch.cuda.empty_cache()
    T.empty_cache()
    y = T.DistTTTensor.random(comm, (8000,) * 10, (1,) + (30,) * 9 + (1,), 0)
    xx = T.add(y, y)
    out = T.round_tt(xx, T.RoundingOptions(1e-10))
    torch.cuda.synchronize()
    print("ok", out.ranks)


if __name__ == "__main__":
    main()
