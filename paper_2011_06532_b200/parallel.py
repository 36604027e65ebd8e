"""Row-distributed TT tensors on B200: distribution, orthonormalization,
truncated SVD, TSQR and rounding (drop-in for ttpar.parallel / ttpar.tsqr).

Every compute call goes straight into the native library (_ttb.so); the
Python layer only validates arguments (with the reference's exceptions),
allocates outputs sized by the input ranks, and narrows them to the ranks
the device reports.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .comm import default_comm
from .errors import ContractError, ShapeError
from .tensor import (DistTTTensor, TTCore, TTTensor, block_bounds, f_empty, f_view, is_f_slab,
                     to_host_array)

ROUNDING_VARIANTS = ("LRLI", "LRL", "RLRI", "RLR")
_VARIANT_CODE = {"LRLI": 0, "LRL": 1, "RLRI": 2, "RLR": 3}
TSQR_VARIANTS = ("butterfly", "binomial")
ZERO_NORM_FLOOR = 1e-300  # parallel.py:37


def _ptrs(slabs):
    return _lib.ptr_array([s.data_ptr() for s in slabs])


# ----------------------------------------------------------------------------
# distribution (parallel.py:114-141, 452-454)
# ----------------------------------------------------------------------------


def distribute(t: TTTensor, comm, allow_idle: bool = False) -> DistTTTensor:
    """Split a host tensor into this rank's row blocks and upload them."""
    if comm.size > min(t.dims) and not allow_idle:
        raise ContractError(f"{comm.size} ranks exceed the smallest mode {min(t.dims)}; "
                            "pass allow_idle=True to accept idle ranks")
    slabs = []
    for n, core in enumerate(t.cores):
        lo, hi = block_bounds(core.dim, comm.size, comm.rank)
        slabs.append(core.array[:, lo:hi, :])
    return DistTTTensor(comm, t.dims, t.ranks, slabs)


def gather(dt: DistTTTensor) -> TTTensor:
    """Reassemble the host tensor on every rank (slabs are exchanged over the
    torch group; harness use -- the hot path never gathers)."""
    mine = [to_host_array(s) for s in dt.local]
    parts = dt.comm.allgather_object(mine)
    cores = []
    for n in range(dt.ndim):
        full = np.zeros((dt.ranks[n], dt.dims[n], dt.ranks[n + 1]), order="F")
        for p, slabs in enumerate(parts):
            lo, hi = block_bounds(dt.dims[n], dt.comm.size, p)
            full[:, lo:hi, :] = slabs[n]
        cores.append(TTCore(full))
    return TTTensor(cores)


def serial_tt(t: TTTensor) -> DistTTTensor:
    """Wrap a host tensor as a one-rank device tensor (parallel.py:452-454)."""
    return distribute(t, default_comm())


# ----------------------------------------------------------------------------
# orthonormalization (parallel.py:164-209)
# ----------------------------------------------------------------------------


def orthonormalize(dt: DistTTTensor, direction: str = "right") -> DistTTTensor:
    """QR-sweep the chain (TSQR + explicit Q + R-fold), ranks unchanged."""
    if direction not in ("left", "right"):
        raise ContractError(f"direction must be 'left' or 'right', got {direction!r}")
    ldims = dt.local_dims()
    outs = [f_empty(dt.ranks[n], ldims[n], dt.ranks[n + 1], dt.comm.device) for n in range(dt.ndim)]
    lib = _lib.load()
    _lib.check(lib.ttb_orthonormalize(dt.comm.ctx(), 0 if direction == "left" else 1, dt.ndim,
                                      _lib.i64_array(ldims), _lib.i64_array(dt.ranks), _ptrs(dt.local),
                                      _ptrs(outs)))
    return DistTTTensor(dt.comm, dt.dims, dt.ranks, outs, {"orthonormal": direction})


# ----------------------------------------------------------------------------
# truncated SVD (parallel.py:212-258)
# ----------------------------------------------------------------------------


@dataclass
class TruncatedSVD:
    """``a ~ u @ diag(s) @ v.T`` with the smallest rank whose discarded tail
    has Frobenius norm <= eps."""

    u: object
    s: object
    v: object
    discarded_tail: float
    capped: bool


def truncated_svd(a, eps: float, max_rank: int | None = None, comm=None) -> TruncatedSVD:
    """Device one-sided Jacobi SVD + the reference's tail rule.

    numpy in -> numpy out; a CUDA tensor in -> CUDA tensors out.
    """
    import torch

    from .errors import NumericError

    on_dev = isinstance(a, torch.Tensor)
    if on_dev:
        if a.dim() != 2:
            raise ShapeError(f"expected a matrix, got ndim={a.dim()}")
    else:
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise ShapeError(f"expected a matrix, got ndim={a.ndim}")
    if eps < 0:
        raise ContractError(f"eps must be nonnegative, got {eps}")
    if max_rank is not None and max_rank < 1:
        raise ContractError(f"max_rank must be >= 1, got {max_rank}")
    comm = comm or default_comm()
    dev = comm.device
    if on_dev:
        ad = a.to(device=dev, dtype=torch.float64).t().contiguous().t()  # column-major
    else:
        if not np.isfinite(a).all():
            raise NumericError("non-finite entries in SVD input")
        ad = torch.from_numpy(np.asfortranarray(a)).to(dev).t().contiguous().t()
    m, n = ad.shape
    k = min(m, n)
    u = torch.empty((k, m), dtype=torch.float64, device=dev)  # column-major m x k via transpose
    s = torch.empty(k, dtype=torch.float64, device=dev)
    v = torch.empty((k, n), dtype=torch.float64, device=dev)
    keep = C.c_int64(0)
    tail = C.c_double(0.0)
    capped = C.c_int(0)
    _lib.check(_lib.load().ttb_truncated_svd(
        comm.ctx(), m, n, C.c_void_p(ad.data_ptr()), float(eps), int(max_rank or 0), C.c_void_p(u.data_ptr()),
        C.c_void_p(s.data_ptr()), C.c_void_p(v.data_ptr()), C.byref(keep), C.byref(tail), C.byref(capped)))
    kp = int(keep.value)
    # the kernel wrote column-major m x kp / n x kp at the front of the buffers
    uu = u.view(-1)[: m * kp].view(kp, m).t()
    vv = v.view(-1)[: n * kp].view(kp, n).t()
    ss = s[:kp]
    if not on_dev:
        uu, ss, vv = uu.cpu().numpy().copy(), ss.cpu().numpy().copy(), vv.cpu().numpy().copy()
    return TruncatedSVD(uu, ss, vv, float(tail.value), bool(capped.value))


# ----------------------------------------------------------------------------
# rounding (parallel.py:261-438)
# ----------------------------------------------------------------------------


@dataclass
class RoundingOptions:
    """Target accuracy and strategy for `round_tt` (parallel.py:261-284)."""

    eps0: float
    variant: str = "LRLI"
    max_rank: int | None = None

    def __post_init__(self):
        if self.eps0 < 0:
            raise ContractError(f"eps0 must be nonnegative, got {self.eps0}")
        self.variant = str(self.variant).upper()
        if self.variant not in ROUNDING_VARIANTS:
            raise ContractError(f"unknown rounding variant {self.variant!r}; pick from {ROUNDING_VARIANTS}")
        if self.max_rank is not None and self.max_rank < 1:
            raise ContractError(f"max_rank must be >= 1, got {self.max_rank}")


def round_tt(dt: DistTTTensor, opts: RoundingOptions) -> DistTTTensor:
    """Compress bond ranks to relative accuracy ``opts.eps0``: per-bond
    threshold eps0*||x||/sqrt(N-1), so ||round(x) - x|| <= eps0 ||x||.
    Output cores are orthonormal on the side the truncation sweep started
    from; exactly-zero tensors collapse to the canonical rank-1 zero."""
    if not isinstance(dt, DistTTTensor):
        raise ContractError(f"round_tt expects a DistTTTensor, got {type(dt).__name__}")
    N = dt.ndim
    ldims = dt.local_dims()
    # outputs sized by the input ranks; results are packed at the front
    flats = []
    for n in range(N):
        import torch

        flats.append(torch.empty(max(1, dt.ranks[n] * ldims[n] * dt.ranks[n + 1]), dtype=torch.float64,
                                 device=dt.comm.device))
    out_ranks = (C.c_int64 * (N + 1))()
    meta = (C.c_double * 4)()
    _lib.check(_lib.load().ttb_round(dt.comm.ctx(), _VARIANT_CODE[opts.variant], float(opts.eps0),
                                     int(opts.max_rank or 0), N, _lib.i64_array(ldims), _lib.i64_array(dt.ranks),
                                     _ptrs(dt.local), _ptrs(flats), out_ranks, meta))
    ranks = tuple(int(r) for r in out_ranks)
    slabs = [f_view(flats[n], ranks[n], ldims[n], ranks[n + 1]) for n in range(N)]
    md = {"variant": opts.variant, "eps0": opts.eps0, "error_bound_violated": bool(meta[2])}
    if N > 1:
        md["norm"] = float(meta[0])
        if meta[3]:
            md["zero"] = True
        else:
            md["eps_bond"] = float(meta[1])
            md["output_ranks"] = ranks
    return DistTTTensor(dt.comm, dt.dims, ranks, slabs, md)


def _host_f_array(a):
    """(array, data pointer) of an F-contiguous float64 host core: numpy
    arrays and CPU torch tensors (pinned or not) pass without a copy when
    they already have that layout."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(a, torch.Tensor):
        if a.device.type != "cpu":
            raise ContractError("round_tt_host takes host cores; use round_tt for device slabs")
        t = a.to(torch.float64)
        if t.dim() != 3:
            raise ShapeError(f"core must be 3-way, got ndim={t.dim()}")
        if not is_f_slab(t):
            t = t.permute(2, 1, 0).contiguous().permute(2, 1, 0)
        return t, t.data_ptr()
    arr = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if arr.ndim != 3:
        raise ShapeError(f"core must be 3-way, got ndim={arr.ndim}")
    return arr, arr.ctypes.data


def round_tt_host(cores, opts: RoundingOptions, comm=None, out=None):
    """round_tt on host-resident cores -- the drop-in for the reference's
    numpy-level ``round_tt(x)`` (parallel.py:293-438): this rank's cores
    (F-order (r_left, I_local, r_right) numpy arrays or CPU tensors, or a
    host TTTensor) go in, rounded host cores come out.  Uploads overlap the
    orthonormalization sweep and each output core is downloaded as soon as
    it is final (ttb_round_host).  ``out`` optionally supplies the output
    buffers (flat host arrays / tensors of at least r_left*I*r_right input
    entries each; page-locked ones are copied directly, pageable ones
    through the library's page-locked staging ring).

    Returns (cores, meta): F-order views into the output buffers, and the
    reference's meta dict (norm, eps_bond, output_ranks, ...)."""
    if isinstance(cores, TTTensor):
        cores = [c.array for c in cores.cores]
    comm = comm or default_comm()
    arrs = [_host_f_array(c) for c in cores]
    N = len(arrs)
    if N == 0:
        raise ShapeError("a TT tensor needs at least one core")
    shapes = [tuple(int(x) for x in a.shape) for a, _ in arrs]
    ranks = (shapes[0][0],) + tuple(sh[2] for sh in shapes)
    for n in range(N - 1):
        if shapes[n][2] != shapes[n + 1][0]:
            raise ShapeError(f"rank mismatch between cores {n} and {n + 1}")
    ldims = [sh[1] for sh in shapes]
    if out is None:
        out = [np.empty(max(1, sh[0] * sh[1] * sh[2]), dtype=np.float64) for sh in shapes]
    if len(out) != N:
        raise ShapeError("out must hold one buffer per core")
    optr = []
    for n, o in enumerate(out):
        need = shapes[n][0] * shapes[n][1] * shapes[n][2]
        if isinstance(o, np.ndarray):
            if o.dtype != np.float64 or not o.flags.c_contiguous or o.size < need:
                raise ShapeError(f"out[{n}] must be a contiguous float64 buffer of >= {need} entries")
            optr.append(o.ctypes.data)
        else:
            if o.dtype.__str__() != "torch.float64" or not o.is_contiguous() or o.numel() < need or o.device.type != "cpu":
                raise ShapeError(f"out[{n}] must be a contiguous float64 host tensor of >= {need} entries")
            optr.append(o.data_ptr())
    out_ranks = (C.c_int64 * (N + 1))()
    meta = (C.c_double * 4)()
    pin = (C.c_void_p * N)(*[p for _, p in arrs])
    pout = (C.c_void_p * N)(*optr)
    _lib.check(_lib.load().ttb_round_host(comm.ctx(), _VARIANT_CODE[opts.variant], float(opts.eps0),
                                          int(opts.max_rank or 0), N, _lib.i64_array(ldims),
                                          _lib.i64_array(ranks), pin, pout, out_ranks, meta))
    rk = tuple(int(r) for r in out_ranks)
    res = []
    for n in range(N):
        cnt = rk[n] * ldims[n] * rk[n + 1]
        o = out[n]
        if isinstance(o, np.ndarray):
            res.append(o[:cnt].reshape((rk[n], ldims[n], rk[n + 1]), order="F"))
        else:
            res.append(f_view(o, rk[n], ldims[n], rk[n + 1]))
    md = {"variant": opts.variant, "eps0": opts.eps0, "error_bound_violated": bool(meta[2])}
    if N > 1:
        md["norm"] = float(meta[0])
        if meta[3]:
            md["zero"] = True
        else:
            md["eps_bond"] = float(meta[1])
            md["output_ranks"] = rk
    del arrs  # keep the (possibly converted) inputs alive until here
    return res, md


# ----------------------------------------------------------------------------
# TSQR (tsqr.py:133-327)
# ----------------------------------------------------------------------------


class TSQRFactor:
    """Implicit orthonormal factor of a row-distributed tall-skinny matrix:
    per-CTA chains of compact-WY tiles, an in-GPU reduction tree and (P > 1)
    a redundant tree over the allgathered rank triangles."""

    def __init__(self, handle, comm, rows, b, variant):
        self._h = handle
        self.comm = comm
        self.shape = (rows, b, comm.size, comm.rank)
        self.variant = variant

    @property
    def b(self):
        return self.shape[1]

    def __del__(self):  # pragma: no cover
        try:
            if self._h is not None:
                _lib.load().ttb_tsqr_free(self.comm.ctx(), self._h)
                self._h = None
        except Exception:
            pass


def _as_device_matrix(a, dev):
    import torch

    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=torch.float64)
    else:
        t = torch.from_numpy(np.asarray(a, dtype=np.float64)).to(dev)
    if t.dim() != 2:
        raise ShapeError(f"expected a 2-d block, got ndim={t.dim()}")
    return t.t().contiguous().t()  # column-major


def tsqr_factor(local_block, comm=None, variant: str = "butterfly"):
    """Factor a row-distributed matrix; returns (TSQRFactor, R) with R the
    replicated sign-fixed b x b triangle (binomial: R on rank 0 only, as in
    the reference's tree).  numpy in -> numpy R; CUDA tensor in -> CUDA R."""
    import torch

    from .errors import NumericError

    if variant not in TSQR_VARIANTS:
        raise ContractError(f"unknown TSQR variant {variant!r}; pick from {TSQR_VARIANTS}")
    comm = comm or default_comm()
    on_dev = isinstance(local_block, torch.Tensor)
    if not on_dev:
        arr = np.asarray(local_block, dtype=np.float64)
        if arr.ndim != 2:
            raise ShapeError(f"expected a 2-d block, got ndim={arr.ndim}")
        if arr.shape[1] < 1:
            raise ShapeError("blocks must have at least one column")
        if not np.isfinite(arr).all():
            raise NumericError("non-finite entries in QR input")
    a = _as_device_matrix(local_block, comm.device)
    m, b = a.shape
    if b < 1:
        raise ShapeError("blocks must have at least one column")
    r = torch.empty((b, b), dtype=torch.float64, device=comm.device)
    h = C.c_void_p()
    _lib.check(_lib.load().ttb_tsqr_factor(comm.ctx(), 1, m, b, 0, C.c_void_p(a.data_ptr()), C.byref(h),
                                           C.c_void_p(r.data_ptr())))
    fac = TSQRFactor(h, comm, m, b, variant)
    rr = r.t()  # kernel wrote column-major
    if variant == "binomial" and comm.rank != 0:
        return fac, None
    return fac, (rr if on_dev else rr.cpu().numpy().copy())


def tsqr_apply_q(factor: TSQRFactor, c, comm=None) -> object:
    """Local rows of Q @ [c; 0] for a b-row block c (tsqr.py:248-327)."""
    import torch

    comm = comm or factor.comm
    if factor.shape[2] > 1 and (comm.size, comm.rank) != factor.shape[2:]:
        raise ContractError("factor belongs to a different communicator layout")
    on_dev = isinstance(c, torch.Tensor)
    cd = _as_device_matrix(c, comm.device)
    if cd.shape[0] != factor.b:
        raise ShapeError(f"expected a ({factor.b}, k) block, got {tuple(cd.shape)}")
    m, k = factor.shape[0], cd.shape[1]
    out = torch.empty((k, m), dtype=torch.float64, device=comm.device)
    _lib.check(_lib.load().ttb_tsqr_apply(comm.ctx(), factor._h, k, C.c_void_p(cd.data_ptr()),
                                          C.c_void_p(out.data_ptr())))
    res = out.t()
    return res if on_dev else res.cpu().numpy().copy()
