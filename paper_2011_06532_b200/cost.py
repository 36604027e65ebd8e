"""Algorithmic work of the hot path (the roofline numerators).

Bytes are the traffic floor of any two-sweep method; flops are the
reference's own leading-order Householder counts (ttpar cost.py:171-263,
`chain_estimate`, rounding / inner_product / orthonormalization branches,
P = 1).  Nothing here touches the device.
"""

from __future__ import annotations

SVD_FLOPS_PER_B3 = 21.0  # ttpar parallel.py:39


def core_sizes(dims, ranks):
    return [ranks[n] * d * ranks[n + 1] for n, d in enumerate(dims)]


def rounding_bytes(dims, ranks, out_ranks):
    """8 * (2 |X| + |Y|): both sweeps read the input, the output is written once."""
    return 8.0 * (2 * sum(core_sizes(dims, ranks)) + sum(core_sizes(dims, out_ranks)))


def rounding_flops(dims, ranks, out_ranks, variant="LRLI"):
    """Leading-order rounding flops on an actual rank chain (cost.py:212-255)."""
    N = len(dims)
    out = out_ranks
    v = variant.upper()
    implicit = v.endswith("I")
    if v.startswith("R"):
        orth = [(dims[n] * ranks[n + 1], ranks[n], ranks[n - 1] * dims[n - 1]) for n in range(N - 1, 0, -1)]
        trunc = [(out[n] * dims[n], ranks[n + 1], out[n + 1], dims[n + 1] * ranks[n + 2]) for n in range(N - 1)]
    else:
        orth = [(ranks[n] * dims[n], ranks[n + 1], dims[n + 1] * ranks[n + 2]) for n in range(N - 1)]
        trunc = [(dims[n] * out[n + 1], ranks[n], out[n], ranks[n - 1] * dims[n - 1]) for n in range(N - 1, 0, -1)]
    tot = 0.0
    for m, b, fold in orth:
        tot += 2 * m * b * b + fold * b * b + (0 if implicit else 2 * m * b * b)
    for m, b, keep, cm in trunc:
        tot += 2 * m * b * b + SVD_FLOPS_PER_B3 * b ** 3 + 4 * m * keep * b
        tot += 4 * cm * keep * b if implicit else 2 * cm * keep * b
    return tot


def tsqr_leaf_flops(dims, ranks, out_ranks, variant="LRLI"):
    """Householder flops (2 m b^2 - 2/3 b^3) of every TSQR panel one rounding
    factors: the work of the tsqr_leaf kernel class."""
    N = len(dims)
    v = variant.upper()
    panels = []
    if v.startswith("L"):
        panels += [(ranks[n] * dims[n], ranks[n + 1]) for n in range(N - 1)]
        panels += [(dims[n] * out_ranks[n + 1], ranks[n]) for n in range(N - 1, 0, -1)]
    else:
        panels += [(dims[n] * ranks[n + 1], ranks[n]) for n in range(N - 1, 0, -1)]
        panels += [(out_ranks[n] * dims[n], ranks[n + 1]) for n in range(N - 1)]
    return sum(2.0 * m * b * b - (2.0 / 3.0) * b ** 3 for m, b in panels)


def gram_bytes(dims, rx, ry):
    return 8.0 * (sum(core_sizes(dims, rx)) + sum(core_sizes(dims, ry)))


def gram_flops(dims, rx, ry):
    """<x, y> flops (cost.py:196-203 with the actual rank pair)."""
    return sum(2.0 * d * (ry[n] * rx[n] * rx[n + 1] + ry[n + 1] * ry[n] * rx[n + 1]) for n, d in enumerate(dims))
