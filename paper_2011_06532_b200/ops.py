"""TT arithmetic on device-resident tensors (drop-in for ttpar.ops).

scale / add / hadamard are slab-local (no communication, ops.py:1-8);
inner_product / norm are Gram sweeps with one r x r allreduce per mode
(ops.py:135-235).  Host TTTensor arguments are uploaded to the current GPU,
processed there, and returned as host TTTensor (the sequential flavour of
the reference API); DistTTTensor stays on the device.
"""

from __future__ import annotations

import ctypes as C
import warnings
from math import sqrt

from . import _lib
from .comm import default_comm
from .errors import CapacityError, ContractError, NumericError, ShapeError
from .tensor import DistTTTensor, TTTensor, f_empty, to_host_array

NORM_METHODS = ("innerprod", "innerprod_sym", "ortho")
HADAMARD_RANK_GUARD = 4096  # ops.py:38


def _as_dist(x):
    """(DistTTTensor, is_host) for either flavour (ops.py:44-50)."""
    if isinstance(x, DistTTTensor):
        return x, False
    if isinstance(x, TTTensor):
        comm = default_comm()
        return DistTTTensor(comm, x.dims, x.ranks, [c.array for c in x.cores]), True
    raise ContractError(f"expected TTTensor or DistTTTensor, got {type(x).__name__}")


def _to_host(dt):
    return TTTensor([to_host_array(s) for s in dt.local])


def _check_pair(x, y):
    if isinstance(x, DistTTTensor) != isinstance(y, DistTTTensor):
        if isinstance(x, (TTTensor, DistTTTensor)) and isinstance(y, (TTTensor, DistTTTensor)):
            raise ContractError("cannot mix sequential and distributed tensors")
    dx, hx = _as_dist(x)
    dy, hy = _as_dist(y)
    if not hx and dx.comm is not dy.comm:
        raise ContractError("operands live on different communicators")
    if dx.dims != dy.dims:
        raise ShapeError(f"dimension mismatch: {dx.dims} vs {dy.dims}")
    if hx:
        dy = DistTTTensor(dx.comm, dy.dims, dy.ranks, dy.local)
    return dx, dy, hx


def _ptrs(slabs):
    return _lib.ptr_array([s.data_ptr() for s in slabs])


def scale(x, s: float):
    """Scalar multiple folded into core 0 (ops.py:71-76)."""
    dt, host = _as_dist(x)
    lib = _lib.load()
    ctx = dt.comm.ctx()
    out = []
    for n, sl in enumerate(dt.local):
        o = f_empty(*sl.shape, dt.comm.device)
        if n == 0:
            _lib.check(lib.ttb_scale(ctx, sl.numel(), C.c_void_p(sl.data_ptr()), float(s), C.c_void_p(o.data_ptr())))
        else:
            o.copy_(sl)
        out.append(o)
    res = DistTTTensor(dt.comm, dt.dims, dt.ranks, out)
    return _to_host(res) if host else res


def add_n(terms, scales=None):
    """Fused N-ary sum  sum_p scales[p] * terms[p]  in one pass per core.

    Equivalent to nesting add(scale(a, s0), scale(b, s1)) ... (ops.py:71-106)
    bit for bit: blocks are placed in term order and the scales multiply
    core 0 only; each output element is written once.
    """
    if not terms:
        raise ContractError("add_n needs at least one term")
    dts = []
    host = None
    for t in terms:
        d, h = _as_dist(t)
        if host is None:
            host = h
        elif host != h:
            raise ContractError("cannot mix sequential and distributed tensors")
        dts.append(d)
    base = dts[0]
    if host:
        dts = [base] + [DistTTTensor(base.comm, d.dims, d.ranks, d.local) for d in dts[1:]]
    for d in dts[1:]:
        if d.dims != base.dims:
            raise ShapeError(f"dimension mismatch: {base.dims} vs {d.dims}")
        if d.comm is not base.comm:
            raise ContractError("operands live on different communicators")
    N = base.ndim
    scales = [1.0] * len(dts) if scales is None else [float(s) for s in scales]
    if N == 1:
        out_ranks = (1, 1)
    else:
        mid = [sum(d.ranks[n] for d in dts) for n in range(1, N)]
        out_ranks = (1,) + tuple(mid) + (1,)
    ldims = base.local_dims()
    outs = [f_empty(out_ranks[n], ldims[n], out_ranks[n + 1], base.comm.device) for n in range(N)]
    lib = _lib.load()
    ranks_flat = [r for d in dts for r in d.ranks]
    cores_flat = [s.data_ptr() for d in dts for s in d.local]
    _lib.check(lib.ttb_add(base.comm.ctx(), len(dts), N, _lib.i64_array(ldims), _lib.i64_array(ranks_flat),
                           _lib.ptr_array(cores_flat), (C.c_double * len(scales))(*scales), _ptrs(outs)))
    res = DistTTTensor(base.comm, base.dims, out_ranks, outs)
    return _to_host(res) if host else res


def add(x, y):
    """TT sum: end cores concatenate, interior cores stack block-diagonally
    (ops.py:79-106).  Bond ranks add; no data moves between ranks."""
    dx, dy, host = _check_pair(x, y)
    res = add_n([dx, dy])
    return _to_host(res) if host else res


def hadamard(x, y, max_rank_product: int | None = None):
    """Elementwise product: slice-wise Kronecker cores (ops.py:109-132)."""
    dx, dy, host = _check_pair(x, y)
    guard = HADAMARD_RANK_GUARD if max_rank_product is None else int(max_rank_product)
    ranks = tuple(a * b for a, b in zip(dx.ranks, dy.ranks))
    if max(ranks) > guard:
        raise CapacityError(f"hadamard bond ranks {max(ranks)} exceed the guard ({guard}); "
                            "round the operands first or raise max_rank_product")
    ldims = dx.local_dims()
    outs = [f_empty(ranks[n], ldims[n], ranks[n + 1], dx.comm.device) for n in range(dx.ndim)]
    lib = _lib.load()
    _lib.check(lib.ttb_hadamard(dx.comm.ctx(), dx.ndim, _lib.i64_array(ldims), _lib.i64_array(dx.ranks),
                                _lib.i64_array(dy.ranks), _ptrs(dx.local), _ptrs(dy.local), _ptrs(outs)))
    res = DistTTTensor(dx.comm, dx.dims, ranks, outs)
    return _to_host(res) if host else res


def round_hadamard(x, y, opts, max_rank_product: int | None = None):
    """round_tt(hadamard(x, y), opts) without materialising the product.

    The product's rank-(rx ry) Kronecker slices (ops.py:109-132) are formed
    on the fly where the rounding (parallel.py:293-438) reads its input -- the
    first sweep's first TSQR panel and its R-folds -- instead of being
    written out and read back (the paper's suggestion).
    Same result, meta and exceptions as ``round_tt(hadamard(x, y), opts)``;
    host operands give a host result."""
    import torch

    from .parallel import _VARIANT_CODE, RoundingOptions
    from .tensor import f_view

    if not isinstance(opts, RoundingOptions):
        raise ContractError("round_hadamard expects RoundingOptions")
    dx, dy, host = _check_pair(x, y)
    guard = HADAMARD_RANK_GUARD if max_rank_product is None else int(max_rank_product)
    ranks = tuple(a * b for a, b in zip(dx.ranks, dy.ranks))
    if max(ranks) > guard:
        raise CapacityError(f"hadamard bond ranks {max(ranks)} exceed the guard ({guard}); "
                            "round the operands first or raise max_rank_product")
    N = dx.ndim
    ldims = dx.local_dims()
    flats = [torch.empty(max(1, ranks[n] * ldims[n] * ranks[n + 1]), dtype=torch.float64, device=dx.comm.device)
             for n in range(N)]
    out_ranks = (C.c_int64 * (N + 1))()
    meta = (C.c_double * 4)()
    _lib.check(_lib.load().ttb_round_hadamard(dx.comm.ctx(), _VARIANT_CODE[opts.variant], float(opts.eps0),
                                              int(opts.max_rank or 0), N, _lib.i64_array(ldims),
                                              _lib.i64_array(dx.ranks), _lib.i64_array(dy.ranks), _ptrs(dx.local),
                                              _ptrs(dy.local), _ptrs(flats), out_ranks, meta))
    rk = tuple(int(r) for r in out_ranks)
    slabs = [f_view(flats[n], rk[n], ldims[n], rk[n + 1]) for n in range(N)]
    md = {"variant": opts.variant, "eps0": opts.eps0, "error_bound_violated": bool(meta[2])}
    if N > 1:
        md["norm"] = float(meta[0])
        if meta[3]:
            md["zero"] = True
        else:
            md["eps_bond"] = float(meta[1])
            md["output_ranks"] = rk
    res = DistTTTensor(dx.comm, dx.dims, rk, slabs, md)
    return _to_host(res) if host else res


def inner_product(x, y) -> float:
    """<x, y> by the Gram recurrence, one allreduce per mode (ops.py:135-155)."""
    dx, dy, _ = _check_pair(x, y)
    lib = _lib.load()
    res = C.c_double(0.0)
    ldims = dx.local_dims()
    _lib.check(lib.ttb_inner(dx.comm.ctx(), dx.ndim, _lib.i64_array(ldims), _lib.i64_array(dx.ranks),
                             _lib.i64_array(dy.ranks), _ptrs(dx.local), _ptrs(dy.local), C.byref(res)))
    xr, yr = dx.ranks, dy.ranks
    dx.comm.trace.add_flops(sum(2.0 * yr[n] * xr[n] * d * xr[n + 1] + 2.0 * yr[n + 1] * yr[n] * d * xr[n + 1]
                                for n, d in enumerate(ldims)))
    return float(res.value)


def _sym_norm(dx):
    """(||x||, ok) by the symmetric Gram route on the device (ttb_norm_sym;
    ops.py:179-205).  ok is False when a carry is indefinite."""
    lib = _lib.load()
    res, bad = C.c_double(0.0), C.c_int(0)
    ldims = dx.local_dims()
    _lib.check(lib.ttb_norm_sym(dx.comm.ctx(), dx.ndim, _lib.i64_array(ldims), _lib.i64_array(dx.ranks),
                                _ptrs(dx.local), C.byref(res), C.byref(bad)))
    r = dx.ranks
    dx.comm.trace.add_flops(sum(float(r[n]) * r[n] * d * r[n + 1] + float(r[n + 1]) * r[n + 1] * r[n] * d
                                for n, d in enumerate(ldims)))
    return sqrt(max(float(res.value), 0.0)), not bad.value


def pivoted_cholesky(w):
    """The reference's _pivoted_cholesky (ops.py:162-176) on the device:
    (lfac, perm, rank) with lfac = (P L)[perm][:, :rank] so that
    pl[perm] = lfac reconstructs w = pl pl^T.  Raises NumericError on an
    indefinite w (the reference raises _IndefiniteGram)."""
    import numpy as np
    import torch

    comm = default_comm()
    w = np.asarray(w, dtype=np.float64)
    n = w.shape[0]
    if w.shape != (n, n) or n == 0:
        raise ShapeError(f"expected a square matrix, got {w.shape}")
    wd = torch.from_numpy(np.asfortranarray(w).ravel(order="F").copy()).to(comm.device)
    pl = torch.empty(n * n, dtype=torch.float64, device=comm.device)
    perm = (C.c_int * n)()
    rank, bad = C.c_int(0), C.c_int(0)
    _lib.check(_lib.load().ttb_pivoted_cholesky(comm.ctx(), n, C.c_void_p(wd.data_ptr()), C.c_void_p(pl.data_ptr()),
                                                 perm, C.byref(rank), C.byref(bad)))
    if bad.value:
        raise NumericError("Gram carry is not PSD (pivoted Cholesky residual)")
    p = np.array(perm[:], dtype=int)
    full = pl.cpu().numpy().reshape((n, n), order="F")
    return np.asfortranarray(full[p][:, :rank.value]), p, int(rank.value)


def norm(x, method: str = "innerprod", return_info: bool = False):
    """Frobenius norm by one of three routes (ops.py:208-235).

    ``innerprod``: sqrt(<x, x>) with the fused Gram kernel.
    ``innerprod_sym``: a pivoted Cholesky factor of the carry propagated
    instead of the operand pair (ttb_norm_sym; one operand stream); falls
    back to ``innerprod`` with a warning when a carry is indefinite.  ``ortho``: the R factors of a
    right-to-left orthonormalization folded core by core, the norm read off
    the last folded core (no cancellation floor; the orthonormal cores are
    never formed).
    """
    if method not in NORM_METHODS:
        raise ContractError(f"unknown norm method {method!r}; pick from {NORM_METHODS}")
    info = {"method": method, "fallback": False}
    dx, _ = _as_dist(x)
    if method == "innerprod":
        val = sqrt(max(inner_product(dx, dx), 0.0))
    elif method == "innerprod_sym":
        val, ok = _sym_norm(dx)
        if not ok:
            warnings.warn("innerprod_sym fell back to innerprod: indefinite Gram carry", stacklevel=2)
            info["fallback"] = True
            val = sqrt(max(inner_product(dx, dx), 0.0))
    else:  # R factors of a right-to-left orthonormalization, folded (ttb_norm_ortho)
        lib = _lib.load()
        res = C.c_double(0.0)
        _lib.check(lib.ttb_norm_ortho(dx.comm.ctx(), dx.ndim, _lib.i64_array(dx.local_dims()),
                                      _lib.i64_array(dx.ranks), _ptrs(dx.local), C.byref(res)))
        val = sqrt(max(float(res.value), 0.0))
    return (val, info) if return_info else val
