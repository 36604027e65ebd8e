"""Kronecker-sum operators applied to TT tensors (drop-in for ttpar's
KroneckerOperator / apply_operator / mode2_multiply / save_operator /
load_operator, ops.py:238-399 and core.py:285-297).

An operator is a sum of terms, each a Kronecker product of square sparse
factors, one per mode.  Applying term t multiplies every core's mode-2
fibers by its factor; the terms are summed as TT tensors (ranks add) and
optionally rounded -- the Krylov-solver caller of round_tt.

Device path: each core's product is one ``ttb_mode2_spmm`` launch that writes
term t straight into its diagonal block of the summed core (the TT sum costs
no extra pass).  Distributed tensors fetch exactly the mode slices the
sparsity pattern couples: the operator is replicated, so every rank derives
the same send / receive lists (``exchange_plan``, ops.py:276-300), packs its
payload with ``ttb_gather_slices`` and swaps it in one grouped NCCL
send/recv (``ttb_exchange``) instead of the reference's P round-robin
sendrecv rounds.  Products are bitwise those of scipy's CSR kernels.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib
from .errors import ShapeError
from .tensor import DistTTTensor, TTCore, block_bounds, f_empty, to_device_slab, to_host_array


@dataclass
class KroneckerOperator:
    """Sum of Kronecker products of square sparse factors, one per mode
    (ops.py:238-262).  Factors are stored as scipy CSR exactly as given
    (their stored entry order is the accumulation order)."""

    dims: tuple
    terms: list
    _dev: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        self.dims = tuple(int(d) for d in self.dims)
        if not self.terms:
            raise ShapeError("operator needs at least one term")
        terms = []
        for t, factors in enumerate(self.terms):
            if len(factors) != len(self.dims):
                raise ShapeError(f"term {t} has {len(factors)} factors for {len(self.dims)} modes")
            row = []
            for n, f in enumerate(factors):
                f = sp.csr_matrix(f)
                if f.shape != (self.dims[n], self.dims[n]):
                    raise ShapeError(f"term {t} factor {n} is {f.shape}, mode wants "
                                     f"({self.dims[n]}, {self.dims[n]})")
                row.append(f)
            terms.append(row)
        self.terms = terms

    @classmethod
    def identity(cls, dims) -> "KroneckerOperator":
        return cls(tuple(dims), [[sp.identity(int(d), format="csr") for d in dims]])


# ----------------------------------------------------------------------------
# exchange plan (host logic; ops.py:270-300)
# ----------------------------------------------------------------------------


@dataclass
class ExchangePlan:
    """What rank ``rank`` of ``size`` needs to apply one factor to its block.

    ``indptr/cols/vals``: the factor's rows [lo, hi) with columns renumbered
    into this rank's source space -- local slices 0..nloc-1, then the halo
    slices in the order they arrive (peers ascending, global index
    ascending).  ``send[q]``: local slice indices to ship to peer q;
    ``recv[q]``: global slice indices coming from q."""

    lo: int
    hi: int
    indptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    send: dict
    recv: dict

    @property
    def nloc(self):
        return self.hi - self.lo

    @property
    def nhalo(self):
        return int(sum(len(v) for v in self.recv.values()))


def exchange_plan(a, size: int, rank: int) -> ExchangePlan:
    """Transfer lists and renumbered rows of factor ``a`` for one rank.

    Both sides of every pair compute the lists from the replicated factor
    (ops.py:276-300): q sends p the slices of q's block that p's rows touch.
    """
    a = sp.csr_matrix(a)
    extent = a.shape[0]
    lo, hi = block_bounds(extent, size, rank)
    mine = a[lo:hi]
    need = np.unique(mine.indices)
    send, recv = {}, {}
    halo = []
    for q in range(size):
        if q == rank:
            continue
        qlo, qhi = block_bounds(extent, size, q)
        theirs = np.unique(a[qlo:qhi].indices)
        s = theirs[(theirs >= lo) & (theirs < hi)] - lo
        r = need[(need >= qlo) & (need < qhi)]
        if s.size:
            send[q] = s.astype(np.int64)
        if r.size:
            recv[q] = r.astype(np.int64)
            halo.append(r)
    halo = np.concatenate(halo) if halo else np.zeros(0, np.int64)
    j = mine.indices.astype(np.int64)
    local = (j >= lo) & (j < hi)
    cols = np.where(local, j - lo, (hi - lo) + np.searchsorted(halo, j))
    return ExchangePlan(lo, hi, mine.indptr.astype(np.int64), cols.astype(np.int64),
                        np.asarray(mine.data, dtype=np.float64), send, recv)


# ----------------------------------------------------------------------------
# device application
# ----------------------------------------------------------------------------


def _dev_plan(op, t, n, comm):
    import torch

    key = (t, n, comm.size, comm.rank, str(comm.device))
    hit = op._dev.get(key)
    if hit is None:
        plan = exchange_plan(op.terms[t][n], comm.size, comm.rank)
        dev = comm.device

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        hit = (plan, up(plan.indptr), up(plan.cols), up(plan.vals),
               {q: up(v) for q, v in plan.send.items()})
        op._dev[key] = hit
    return hit


def _halo(comm, slab, plan, send_idx):
    """Fetch this rank's halo slices (slice-major) from its peers."""
    import torch

    rl, dloc, rr = slab.shape
    per = rl * rr
    halo = torch.empty(max(plan.nhalo * per, 1), dtype=torch.float64, device=comm.device)
    if comm.size == 1 or (not plan.send and not plan.recv and not comm.rendezvous):
        return halo
    lib = _lib.load()
    ctx = comm.ctx()
    peers, sends, recvs = [], [], []
    off = 0
    for q in range(comm.size):
        s, r = plan.send.get(q), plan.recv.get(q)
        if q == comm.rank or (s is None and r is None):
            continue
        buf = None
        if s is not None:
            buf = torch.empty(s.size * per, dtype=torch.float64, device=comm.device)
            _lib.check(lib.ttb_gather_slices(ctx, rl, dloc, rr, C.c_void_p(slab.data_ptr()), s.size,
                                             C.c_void_p(send_idx[q].data_ptr()), C.c_void_p(buf.data_ptr())))
        nrecv = 0 if r is None else r.size * per
        peers.append(q)
        sends.append(buf)
        recvs.append(halo[off:off + nrecv])
        off += nrecv
    comm.exchange(peers, sends, recvs)
    # send buffers were allocated on this stream: the caching allocator
    # reuses them only in stream order, i.e. after the exchange consumed them
    return halo


def _spmm(comm, slab, plan_dev, out, a0, c0):
    plan, indptr, cols, vals, send_idx = plan_dev
    rl, dloc, rr = slab.shape
    halo = _halo(comm, slab, plan, send_idx)
    lib = _lib.load()
    _lib.check(lib.ttb_mode2_spmm(comm.ctx(), rl, rr, plan.nloc, C.c_void_p(indptr.data_ptr()),
                                  C.c_void_p(cols.data_ptr()), C.c_void_p(vals.data_ptr()), plan.nloc,
                                  C.c_void_p(slab.data_ptr()), C.c_void_p(halo.data_ptr()),
                                  C.c_void_p(out.data_ptr()), out.shape[0], out.shape[1], a0, c0))


_MAX_FUSED_TERMS = 16  # ttb_mode2_spmm_sum's term capacity


def _apply_terms(op, dt: DistTTTensor) -> DistTTTensor:
    """sum_t (term t applied to dt), assembled block-diagonally in one pass
    per core (equal to add(add(p0, p1), ...) of the reference, ops.py:330-333):
    ttb_mode2_spmm_sum writes every output cell once, the products of term t
    in its diagonal block and exact zeros elsewhere."""
    comm = dt.comm
    N, T = dt.ndim, len(op.terms)
    if N == 1 and T > 1:  # one core: the terms add elementwise, left to right
        from .ops import add_n

        parts = [_apply_terms(KroneckerOperator(op.dims, [f]), dt) for f in op.terms]
        acc = add_n(parts[:_MAX_FUSED_TERMS])
        for k in range(_MAX_FUSED_TERMS, T, _MAX_FUSED_TERMS - 1):
            acc = add_n([acc] + parts[k:k + _MAX_FUSED_TERMS - 1])
        return acc
    ranks = (1,) + tuple(T * r for r in dt.ranks[1:-1]) + (1,)
    lib = _lib.load()
    outs = []
    for n, slab in enumerate(dt.local):
        rl, dloc, rr = slab.shape
        if T > _MAX_FUSED_TERMS:  # zero-filled core, one block-writing launch per term
            import torch

            shape = (ranks[n], dloc, ranks[n + 1])
            o = torch.zeros(shape[0] * shape[1] * shape[2], dtype=torch.float64, device=comm.device)
            o = o.as_strided(shape, (1, shape[0], shape[0] * shape[1]))
            for t in range(T):
                _spmm(comm, slab, _dev_plan(op, t, n, comm), o, 0 if n == 0 else t * rl, 0 if n == N - 1 else t * rr)
            outs.append(o)
            continue
        o = f_empty(ranks[n], dloc, ranks[n + 1], comm.device)
        plans = [_dev_plan(op, t, n, comm) for t in range(T)]
        halos = [_halo(comm, slab, pd[0], pd[4]) for pd in plans]  # exchanges (P > 1), in term order
        mode = 1 if n == 0 and N > 1 else (2 if n == N - 1 and N > 1 else 0)
        if N == 1:
            mode = 0  # single term on a single core: rl = rr = 1
        _lib.check(lib.ttb_mode2_spmm_sum(
            comm.ctx(), T, mode, rl, rr, dloc,
            _lib.ptr_array([pd[1].data_ptr() for pd in plans]), _lib.ptr_array([pd[2].data_ptr() for pd in plans]),
            _lib.ptr_array([pd[3].data_ptr() for pd in plans]), dloc, C.c_void_p(slab.data_ptr()),
            _lib.ptr_array([h.data_ptr() for h in halos]), C.c_void_p(o.data_ptr())))
        outs.append(o)
    return DistTTTensor(comm, dt.dims, ranks, outs)


def apply_operator(op: KroneckerOperator, x, round_eps: float | None = None, max_rank: int | None = None):
    """Apply a Kronecker-sum operator: mode-2 products per term, TT sum of
    the terms, then optionally round_tt(RoundingOptions(round_eps,
    max_rank=max_rank)) (ops.py:314-342).  Host TTTensor in -> host out."""
    from .ops import _as_dist, _to_host
    from .parallel import RoundingOptions, round_tt

    dt, host = _as_dist(x)
    if op.dims != dt.dims:
        raise ShapeError(f"operator dims {op.dims} do not match tensor dims {dt.dims}")
    z = _apply_terms(op, dt)
    if round_eps is not None:
        z = round_tt(z, RoundingOptions(eps0=round_eps, max_rank=max_rank))
    return _to_host(z) if host else z


def mode2_multiply(core, a):
    """Y(i) = sum_j a[i, j] X(j) on one core's mode-2 fibers (core.py:285-297).

    ``core`` is a host TTCore (-> host TTCore) or an F-order device slab
    (-> device slab); ``a`` dense or scipy.sparse.  Sparse factors give the
    reference's bits exactly; dense ones the same sums in row order (the
    reference uses BLAS there, equal to rounding)."""
    from .comm import default_comm

    host = isinstance(core, TTCore)
    arr = core.array if host else core
    rl, d, rr = arr.shape
    if a.shape != (d, d):
        raise ShapeError(f"operator factor must be {d}x{d}, got {a.shape}")
    comm = default_comm()
    slab = to_device_slab(arr, comm.device)
    op = KroneckerOperator((d,), [[a]])
    out = f_empty(rl, d, rr, comm.device)
    _spmm(comm, slab, _dev_plan(op, 0, 0, comm), out, 0, 0)
    return TTCore(to_host_array(out)) if host else out


# ----------------------------------------------------------------------------
# KRONOP1 text format (ops.py:345-399)
# ----------------------------------------------------------------------------

_OP_MAGIC = "KRONOP1"


def save_operator(path, op: KroneckerOperator) -> None:
    """Text format: magic, counts, dims, then ``factor t n nnz`` triplet blocks."""
    with open(path, "w", encoding="ascii") as f:
        f.write(f"{_OP_MAGIC}\n{len(op.dims)} {len(op.terms)}\n")
        f.write(" ".join(str(d) for d in op.dims) + "\n")
        for t, factors in enumerate(op.terms):
            for n, a in enumerate(factors):
                coo = a.tocoo()
                f.write(f"factor {t} {n} {coo.nnz}\n")
                f.writelines(f"{int(i)} {int(j)} {float(v)!r}\n" for i, j, v in zip(coo.row, coo.col, coo.data))


def load_operator(path) -> KroneckerOperator:
    """Parse the text format written by `save_operator`."""
    with open(path, encoding="ascii") as f:
        lines = [ln.strip() for ln in f if ln.strip()]
    try:
        if lines[0] != _OP_MAGIC:
            raise ShapeError(f"{path!r} is not an operator file (bad magic {lines[0]!r})")
        n_modes, n_terms = (int(v) for v in lines[1].split())
        dims = tuple(int(v) for v in lines[2].split())
        if len(dims) != n_modes:
            raise ShapeError(f"header declares {n_modes} modes but lists {len(dims)} dims")
        k = 3
        terms = []
        for t in range(n_terms):
            factors = []
            for n in range(n_modes):
                tag, tt, nn, nnz = lines[k].split()
                if tag != "factor" or int(tt) != t or int(nn) != n:
                    raise ShapeError(f"unexpected block header {lines[k]!r}")
                nnz = int(nnz)
                body = lines[k + 1: k + 1 + nnz]
                if len(body) != nnz:
                    raise ShapeError(f"factor ({t}, {n}) truncated")
                trip = [ln.split() for ln in body]
                rows = [int(r[0]) for r in trip]
                cols = [int(r[1]) for r in trip]
                vals = [float(r[2]) for r in trip]
                factors.append(sp.csr_matrix((vals, (rows, cols)), shape=(dims[n], dims[n])))
                k += 1 + nnz
            terms.append(factors)
        if k != len(lines):
            raise ShapeError("trailing lines after last factor")
    except (ValueError, IndexError) as e:
        raise ShapeError(f"malformed operator file {path!r}: {e}") from e
    return KroneckerOperator(dims, terms)
