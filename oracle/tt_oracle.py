"""CPU oracle for the TT-rounding hot path -- TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy/scipy restatement of the algorithms in the
reference package ``ttpar`` (``/root/reference/pkg/src/ttpar``) that sit on the
TT-rounding hot path.  It exists to *check* the CUDA product path and to serve
as the CPU baseline leg of ``bench.py``; nothing in the product package
(``paper_2011_06532_b200``) imports it.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / --impl reference)
may use it.

Parity pin: every function here is checked against golden vectors produced by
the reference itself (``tests/golden/gen_golden.py`` imports ``ttpar`` from
``/root/reference`` and writes ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.

Layout contract (reference core.py:1-23): a core is a Fortran-ordered float64
array of shape ``(r_left, dim, r_right)``; ``V(X)`` is the
``(r_left*dim, r_right)`` and ``H(X)`` the ``(r_left, dim*r_right)`` column-major
reshape of the same buffer.  A tensor is a plain list of such cores.

The arithmetic lives where the reference's lives: LAPACK/BLAS through scipy
(dgeqrf / dormqr / dorgqr / gesdd / dpstrf), so the oracle also doubles as a
faithful CPU timing baseline for the reference's own algorithm.
"""

from __future__ import annotations

from math import sqrt

import numpy as np
from scipy.linalg import lapack, svd as _scipy_svd
from scipy.linalg.blas import dgemm, dsyrk, dtrmm

VARIANTS = ("LRLI", "LRL", "RLRI", "RLR")
ZERO_FLOOR = 1e-300  # parallel.py:37
HADAMARD_GUARD = 4096  # ops.py:38
SVD_FLOPS_B3 = 21.0  # parallel.py:39 (cost model constant)


# --------------------------------------------------------------------------
# layout helpers
# --------------------------------------------------------------------------

def ranks_of(cores):
    """Bond ranks (R_0..R_N) of a core list (core.py:122-125)."""
    return (1,) + tuple(int(c.shape[2]) for c in cores)


def dims_of(cores):
    return tuple(int(c.shape[1]) for c in cores)


def vmat(core):
    """V(X): (r_left*dim, r_right) column-major view (core.py:78-81)."""
    rl, d, rr = core.shape
    return core.reshape((rl * d, rr), order="F")


def hmat(core):
    """H(X): (r_left, dim*r_right) column-major view (core.py:83-86)."""
    rl, d, rr = core.shape
    return core.reshape((rl, d * rr), order="F")


def from_v(v, rl, d):
    return np.asfortranarray(v).reshape((rl, d, v.shape[1]), order="F")


def from_ht(ht, d, rr):
    """Rebuild a core from a transposed H unfolding (parallel.py:158-161)."""
    h = np.asfortranarray(ht.T)
    return h.reshape((h.shape[0], d, rr), order="F")


def check_chain(dims, ranks):
    """Validate a dims/ranks chain (core.py:236-247)."""
    dims = tuple(int(d) for d in dims)
    ranks = tuple(int(r) for r in ranks)
    if not dims or any(d < 1 for d in dims):
        raise ValueError(f"bad dims {dims}")
    if len(ranks) != len(dims) + 1 or ranks[0] != 1 or ranks[-1] != 1:
        raise ValueError(f"bad rank chain {ranks}")
    if any(r < 1 for r in ranks):
        raise ValueError(f"bad rank chain {ranks}")
    return dims, ranks


def block_bounds(extent, nranks, rank):
    """Ceil-chunk row block of one rank (parallel.py:42-46)."""
    step = -(-int(extent) // int(nranks))
    lo = min(int(rank) * step, int(extent))
    return lo, min(lo + step, int(extent))


# --------------------------------------------------------------------------
# seeded construction (core.py:250-282)
# --------------------------------------------------------------------------

def slice_generator(seed, n, i):
    """Philox stream of slice i of core n, keyed SeedSequence(seed, (n, i))."""
    return np.random.Generator(
        np.random.Philox(np.random.SeedSequence(seed, spawn_key=(n, i))))


def fill_slices(out, n, lo, seed):
    """Fill out[:, k, :] from the stream of global slice lo+k, F order."""
    rl, d, rr = out.shape
    for k in range(d):
        draws = slice_generator(seed, n, lo + k).standard_normal(rl * rr)
        out[:, k, :] = draws.reshape((rl, rr), order="F")


def random_cores(dims, ranks, seed, lo_hi=None):
    """i.i.d. N(0,1) cores, bitwise equal to the reference's random_tt.

    ``lo_hi`` optionally restricts every core to slices [lo, hi) (the
    per-rank slab of DistTTTensor.random, parallel.py:88-102).
    """
    dims, ranks = check_chain(dims, ranks)
    cores = []
    for n, d in enumerate(dims):
        lo, hi = (0, d) if lo_hi is None else lo_hi(n, d)
        arr = np.empty((ranks[n], hi - lo, ranks[n + 1]), order="F")
        fill_slices(arr, n, lo, seed)
        cores.append(arr)
    return cores


# --------------------------------------------------------------------------
# dense oracle (small tensors only)
# --------------------------------------------------------------------------

def full(cores):
    """Dense array (first mode fastest in the flat F-order sense)."""
    acc = np.ones((1, 1))
    for c in cores:
        rl, d, rr = c.shape
        # acc: (M, rl) -> (M, d, rr) with the new mode slower than the old ones
        acc = np.einsum("ma,aib->mib", acc, c).reshape((-1, rr), order="F")
    return acc[:, 0].reshape(dims_of(cores), order="F")


# --------------------------------------------------------------------------
# local algebra (ops.py:71-132)
# --------------------------------------------------------------------------

def scale(cores, s):
    """Scalar multiple folded into core 0 (ops.py:71-76)."""
    out = [np.array(c, order="F", copy=True) for c in cores]
    out[0] *= float(s)
    return out


def add(x, y):
    """TT sum by block-diagonal cores; ends concatenate (ops.py:79-106)."""
    if dims_of(x) != dims_of(y):
        raise ValueError("dimension mismatch")
    N = len(x)
    if N == 1:
        return [np.asfortranarray(x[0] + y[0])]
    out = []
    for n, (a, b) in enumerate(zip(x, y)):
        ral, d, rar = a.shape
        rbl, _, rbr = b.shape
        if n == 0:
            z = np.zeros((1, d, rar + rbr), order="F")
            z[:, :, :rar], z[:, :, rar:] = a, b
        elif n == N - 1:
            z = np.zeros((ral + rbl, d, 1), order="F")
            z[:ral], z[ral:] = a, b
        else:
            z = np.zeros((ral + rbl, d, rar + rbr), order="F")
            z[:ral, :, :rar] = a
            z[ral:, :, rar:] = b
        out.append(z)
    return out


def hadamard(x, y, guard=None):
    """Slice-wise Kronecker cores, X index slow (ops.py:109-132)."""
    if dims_of(x) != dims_of(y):
        raise ValueError("dimension mismatch")
    g = HADAMARD_GUARD if guard is None else int(guard)
    rk = [a * b for a, b in zip(ranks_of(x), ranks_of(y))]
    if max(rk) > g:
        raise OverflowError("hadamard rank guard")
    out = []
    for a, b in zip(x, y):
        ral, d, rar = a.shape
        rbl, _, rbr = b.shape
        z = np.einsum("pik,qil->pqikl", a, b).reshape(ral * rbl, d, rar * rbr)
        out.append(np.asfortranarray(z))
    return out


# --------------------------------------------------------------------------
# Kronecker operator apply (core.py:285-297, ops.py:265-342)
# --------------------------------------------------------------------------

def mode2_multiply(core, a):
    """Y(i) = sum_j a[i, j] X(j): one sparse/dense product per right rank
    (core.py:285-297)."""
    rl, d, rr = core.shape
    out = np.empty((rl, d, rr), order="F")
    for r in range(rr):
        out[:, :, r] = (a @ core[:, :, r].T).T
    return out


def apply_term_block(factor, core, lo, hi):
    """Rows [lo, hi) of one term's mode-2 product as the distributed
    reference computes them (ops.py:270-311): the factor's rows restricted to
    the columns they touch, times the gathered source slices."""
    import scipy.sparse as sp

    a = sp.csr_matrix(factor)
    rl, d, rr = core.shape
    rows = a[lo:hi]
    need = np.unique(rows.indices)
    got = np.empty((need.size, rl * rr), order="F") if need.size else np.zeros((0, rl * rr))
    for k, i in enumerate(need):
        got[k] = core[:, int(i), :].ravel(order="F")
    local = rows[:, need] @ got if need.size else np.zeros((hi - lo, rl * rr))
    return np.asfortranarray(np.asarray(local).reshape(hi - lo, rr, rl).transpose(2, 0, 1))


def apply_operator(terms, cores, round_eps=None, max_rank=None, nranks=1):
    """Sum over terms of the per-core mode-2 products, TT-added left to
    right, optionally rounded (ops.py:314-342).  nranks > 1 computes each
    core as the concatenation of the distributed blocks."""
    parts = []
    for factors in terms:
        if nranks == 1:
            parts.append([mode2_multiply(c, a) for c, a in zip(cores, factors)])
        else:
            term = []
            for c, a in zip(cores, factors):
                blocks = [apply_term_block(a, c, *block_bounds(c.shape[1], nranks, p)) for p in range(nranks)]
                term.append(np.asfortranarray(np.concatenate(blocks, axis=1)))
            parts.append(term)
    z = parts[0]
    for extra in parts[1:]:
        z = add(z, extra)
    if round_eps is not None:
        z, _ = round_tt(z, round_eps, "LRLI", max_rank)
    return z


# --------------------------------------------------------------------------
# Gram sweeps (ops.py:135-235)
# --------------------------------------------------------------------------

def inner(x, y, allreduce=None):
    """<x, y> via W_n = V(Y_n)^T V(W_{n-1} H(X_n)) (ops.py:135-155)."""
    w = np.ones((1, 1), order="F")
    for a, b in zip(x, y):
        ral, d, rar = a.shape
        rbl, _, rbr = b.shape
        z = dgemm(1.0, w, hmat(a)) if d * rar else np.zeros((rbl, 0), order="F")
        zv = z.reshape((rbl * d, rar), order="F")
        wn = (dgemm(1.0, vmat(b), zv, trans_a=1) if rbl * d
              else np.zeros((rbr, rar), order="F"))
        w = wn if allreduce is None else allreduce(wn)
    return float(w[0, 0])


class IndefiniteGram(Exception):
    pass


def pivoted_cholesky(w, rtol=1e-14, resid_rtol=1e-6):
    """Rank-revealing pivoted Cholesky of the carry (ops.py:162-176)."""
    tol = rtol * max(float(np.max(np.diagonal(w))), 0.0)
    c, piv, rank, info = lapack.dpstrf(w, lower=1, tol=tol)
    if info < 0:
        raise ArithmeticError(f"dpstrf info={info}")
    lf = np.tril(c)[:, :rank]
    perm = np.asarray(piv, dtype=int) - 1
    pl = np.empty_like(lf)
    pl[perm] = lf
    if np.linalg.norm(pl @ pl.T - w) > resid_rtol * max(np.linalg.norm(w), 1e-300):
        raise IndefiniteGram("indefinite Gram carry")
    return lf, perm, int(rank)


def sym_norm(x, allreduce=None):
    """Half-flop norm carrying a Cholesky factor (ops.py:179-205)."""
    w = np.ones((1, 1), order="F")
    for a in x:
        ral, d, rar = a.shape
        lf, perm, rank = pivoted_cholesky(w)
        hp = np.asfortranarray(hmat(a)[perm])
        if d * rar == 0:
            z = np.zeros((rank, 0), order="F")
        elif rank == ral:
            z = dtrmm(1.0, lf, hp, side=0, lower=1, trans_a=1)
        else:
            z = dgemm(1.0, lf, hp, trans_a=1)
        zv = z.reshape((rank * d, rar), order="F")
        wn = dsyrk(1.0, zv, trans=1, lower=1) if rank * d else np.zeros((rar, rar), order="F")
        if allreduce is not None:
            wn = allreduce(wn)
        w = np.asfortranarray(np.tril(wn) + np.tril(wn, -1).T)
    return sqrt(max(float(w[0, 0]), 0.0))


def norm(x, method="innerprod"):
    """Frobenius norm by three routes (ops.py:208-235)."""
    if method == "innerprod":
        return sqrt(max(inner(x, x), 0.0))
    if method == "innerprod_sym":
        try:
            return sym_norm(x)
        except IndefiniteGram:
            return sqrt(max(inner(x, x), 0.0))
    if method == "ortho":
        o = orthonormalize(x, "right")
        return sqrt(max(float(np.dot(o[0].ravel(), o[0].ravel())), 0.0))
    raise ValueError(f"unknown norm method {method!r}")


# --------------------------------------------------------------------------
# local Householder QR (tsqr.py:53-130), serial TSQR (P = 1)
# --------------------------------------------------------------------------

class HouseholderQR:
    """Packed dgeqrf factor, zero-padded to >= b rows, R sign-fixed >= 0."""

    def __init__(self, block):
        a = np.asarray(block, dtype=np.float64)
        if a.ndim != 2 or a.shape[1] < 1:
            raise ValueError("expected a 2-d block with >= 1 column")
        if not np.isfinite(a).all():
            raise ArithmeticError("non-finite entries in QR input")
        m, b = a.shape
        work = np.zeros((max(m, b), b), order="F")
        work[:m] = a
        self.qr, self.tau, _, info = lapack.dgeqrf(work, overwrite_a=1)
        if info != 0:
            raise ArithmeticError(f"dgeqrf info={info}")
        self.sign = np.where(np.diagonal(self.qr)[:b] < 0, -1.0, 1.0)
        self.rows = m
        self.b = b

    @property
    def r(self):
        b = self.b
        return np.triu(self.qr[:b, :b]) * self.sign[:, None]

    def apply(self, c):
        """Q @ [c; 0] trimmed to the real rows (dormqr; tsqr.py:75-86)."""
        c = np.asarray(c, dtype=np.float64)
        x = np.zeros((self.qr.shape[0], c.shape[1]), order="F")
        x[: self.b] = self.sign[:, None] * c
        _, work, info = lapack.dormqr("L", "N", self.qr, self.tau, x, -1)
        lwork = max(1, int(work[0]))
        cq, _, info = lapack.dormqr("L", "N", self.qr, self.tau, x, lwork, overwrite_c=1)
        if info != 0:
            raise ArithmeticError(f"dormqr info={info}")
        return cq[: self.rows]

    def thin_q(self):
        """Explicit thin Q (dorgqr; tsqr.py:88-93)."""
        q, _, info = lapack.dorgqr(self.qr.copy(order="F"), self.tau)
        if info != 0:
            raise ArithmeticError(f"dorgqr info={info}")
        return q[: self.rows] * self.sign[None, :]

    def apply_any(self, c):
        """Reference apply routing: triangular C -> dorgqr + trmm (tsqr.py:309-327)."""
        c = np.asarray(c, dtype=np.float64)
        if c.shape[0] == c.shape[1] and not np.tril(c, -1).any():
            q = self.thin_q()
            if np.array_equal(c, np.eye(self.b)):
                return q
            return dtrmm(1.0, c, np.asfortranarray(q), side=1, lower=0, trans_a=0)
        return self.apply(c)


def stacked_tsqr(blocks):
    """TSQR over row blocks, one per (simulated) rank, flat reduction tree.

    Every rank's leaf R is stacked in rank order and factored once more; this
    is the tree shape the B200 build uses (allgather + redundant QR) and it
    yields the same R as the reference butterfly up to roundoff for
    full-rank panels.  Returns (R, apply) where apply(c) gives the per-block
    rows of Q @ [c; 0].
    """
    leaves = [HouseholderQR(blk) for blk in blocks]
    if len(leaves) == 1:
        return leaves[0].r, lambda c: [leaves[0].apply_any(c)]
    top = HouseholderQR(np.vstack([lf.r for lf in leaves]))
    b = top.b

    def apply(c):
        both = top.apply(c)
        return [lf.apply(both[p * b:(p + 1) * b]) for p, lf in enumerate(leaves)]

    return top.r, apply


# --------------------------------------------------------------------------
# orthonormalization (parallel.py:164-209)
# --------------------------------------------------------------------------

def orthonormalize(cores, direction="right"):
    """QR sweep; 'right' leaves H(X_n) row-orthonormal for n >= 1."""
    if direction not in ("left", "right"):
        raise ValueError("direction must be 'left' or 'right'")
    out = [np.array(c, order="F", copy=True) for c in cores]
    N = len(out)
    if N == 1:
        return out
    if direction == "right":
        for n in range(N - 1, 0, -1):
            rl, d, rr = out[n].shape
            f = HouseholderQR(hmat(out[n]).T)
            out[n] = from_ht(f.apply_any(np.eye(rl)), d, rr)
            v = vmat(out[n - 1])
            vn = dtrmm(1.0, f.r, v, side=1, lower=0, trans_a=1)  # V R^T
            out[n - 1] = from_v(vn, out[n - 1].shape[0], out[n - 1].shape[1])
    else:
        for n in range(N - 1):
            rl, d, rr = out[n].shape
            f = HouseholderQR(vmat(out[n]))
            out[n] = from_v(f.apply_any(np.eye(rr)), rl, d)
            rl2, d2, rr2 = out[n + 1].shape
            hn = dtrmm(1.0, f.r, hmat(out[n + 1]), side=0, lower=0, trans_a=0)  # R H
            out[n + 1] = hn.reshape((rr, d2, rr2), order="F")
    return out


# --------------------------------------------------------------------------
# truncated SVD (parallel.py:212-258)
# --------------------------------------------------------------------------

def truncated_svd(a, eps, max_rank=None):
    """Smallest rank whose discarded Frobenius tail is <= eps (>= 1, capped).

    Returns (u, s, v, discarded_tail, capped) with a ~ u diag(s) v^T.
    """
    a = np.asarray(a, dtype=np.float64)
    if eps < 0:
        raise ValueError("eps must be nonnegative")
    if not np.isfinite(a).all():
        raise ArithmeticError("non-finite entries in SVD input")
    u, s, vt = _scipy_svd(a, full_matrices=False, lapack_driver="gesdd")
    tail_sq = np.append(np.cumsum((s * s)[::-1])[::-1], 0.0)
    keep = max(int(np.argmax(tail_sq <= eps * eps)), 1)
    capped = False
    if max_rank is not None:
        if max_rank < 1:
            raise ValueError("max_rank must be >= 1")
        if keep > max_rank:
            keep, capped = int(max_rank), True
    return (u[:, :keep].copy(), s[:keep].copy(), vt[:keep].T.copy(),
            float(sqrt(tail_sq[keep])), capped)


# --------------------------------------------------------------------------
# rounding (parallel.py:261-438)
# --------------------------------------------------------------------------

def round_tt(cores, eps0, variant="LRLI", max_rank=None):
    """Two-sweep TT rounding; returns (cores, meta).

    variant: 'LRL*' = left-orthonormalize then truncate right-to-left,
    'RLR*' = the mirror; trailing 'I' keeps the first sweep's Q implicit.
    """
    variant = str(variant).upper()
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    if eps0 < 0:
        raise ValueError("eps0 must be nonnegative")
    N = len(cores)
    meta = {"variant": variant, "eps0": eps0, "error_bound_violated": False}
    if N == 1:
        return [np.array(cores[0], order="F", copy=True)], meta
    implicit = variant.endswith("I")
    slabs = [np.array(c, order="F", copy=True) for c in cores]
    d = [c.shape[1] for c in cores]
    ranks = list(ranks_of(cores))
    facs = {}

    if variant.startswith("R"):
        for n in range(N - 1, 0, -1):
            b = ranks[n]
            f = HouseholderQR(hmat(slabs[n]).T)
            if implicit:
                facs[n], slabs[n] = f, None
            else:
                slabs[n] = from_ht(f.apply_any(np.eye(b)), d[n], ranks[n + 1])
            vn = dtrmm(1.0, f.r, vmat(slabs[n - 1]), side=1, lower=0, trans_a=1)
            slabs[n - 1] = from_v(vn, ranks[n - 1], d[n - 1])
        last = slabs[0]
    else:
        for n in range(N - 1):
            b = ranks[n + 1]
            f = HouseholderQR(vmat(slabs[n]))
            if implicit:
                facs[n], slabs[n] = f, None
            else:
                slabs[n] = from_v(f.apply_any(np.eye(b)), ranks[n], d[n])
            hn = dtrmm(1.0, f.r, hmat(slabs[n + 1]), side=0, lower=0, trans_a=0)
            slabs[n + 1] = hn.reshape((b, d[n + 1], ranks[n + 2]), order="F")
        last = slabs[N - 1]

    nx = sqrt(max(float(np.dot(last.ravel(), last.ravel())), 0.0))
    meta["norm"] = nx
    if nx < ZERO_FLOOR:
        meta["zero"] = True
        return [np.zeros((1, dn, 1), order="F") for dn in d], meta
    eps = eps0 * nx / sqrt(N - 1)
    meta["eps_bond"] = eps

    if variant.startswith("R"):
        for n in range(N - 1):
            b = ranks[n + 1]
            f2 = HouseholderQR(vmat(slabs[n]))
            u, s, v, _, capped = truncated_svd(f2.r, eps, max_rank)
            keep = u.shape[1]
            meta["error_bound_violated"] |= capped
            slabs[n] = from_v(f2.apply_any(u), ranks[n], d[n])
            carry = v * s[None, :]
            if slabs[n + 1] is None:
                slabs[n + 1] = from_ht(facs.pop(n + 1).apply_any(carry), d[n + 1], ranks[n + 2])
            else:
                hn = dgemm(1.0, carry, hmat(slabs[n + 1]), trans_a=1)
                slabs[n + 1] = hn.reshape((keep, d[n + 1], ranks[n + 2]), order="F")
            ranks[n + 1] = keep
    else:
        for n in range(N - 1, 0, -1):
            b = ranks[n]
            f2 = HouseholderQR(hmat(slabs[n]).T)
            u, s, v, _, capped = truncated_svd(np.asfortranarray(f2.r.T), eps, max_rank)
            keep = u.shape[1]
            meta["error_bound_violated"] |= capped
            slabs[n] = from_ht(f2.apply_any(v), d[n], ranks[n + 1])
            carry = u * s[None, :]
            if slabs[n - 1] is None:
                slabs[n - 1] = from_v(facs.pop(n - 1).apply_any(carry), ranks[n - 1], d[n - 1])
            else:
                slabs[n - 1] = from_v(dgemm(1.0, vmat(slabs[n - 1]), carry), ranks[n - 1], d[n - 1])
            ranks[n] = keep
    meta["output_ranks"] = tuple(ranks)
    return slabs, meta


# --------------------------------------------------------------------------
# TT-form error (the parity metric) and cost counts
# --------------------------------------------------------------------------

def rel_diff(x, y):
    """||x - y|| / ||y|| computed in TT form by the orthonormalization route.

    The inner-product expansion cancels to a ~1e-8 floor; the ortho route of
    the difference tensor does not (SURVEY.md finding 3).
    """
    diff = add(x, scale(y, -1.0))
    ny = norm(y, "ortho")
    nd = norm(diff, "ortho")
    return nd / ny if ny > 0 else nd


def rounding_flops(dims, ranks, out_ranks, variant="LRLI"):
    """Leading-order flops of one rounding (cost.py:212-255, P = 1)."""
    N = len(dims)
    out = out_ranks
    implicit = variant.upper().endswith("I")
    tot = 0.0
    if variant.upper().startswith("R"):
        orth = [(dims[n] * ranks[n + 1], ranks[n], ranks[n - 1] * dims[n - 1])
                for n in range(N - 1, 0, -1)]
        trunc = [(out[n] * dims[n], ranks[n + 1], out[n + 1], dims[n + 1] * ranks[n + 2])
                 for n in range(N - 1)]
    else:
        orth = [(ranks[n] * dims[n], ranks[n + 1], dims[n + 1] * ranks[n + 2])
                for n in range(N - 1)]
        trunc = [(dims[n] * out[n + 1], ranks[n], out[n], ranks[n - 1] * dims[n - 1])
                 for n in range(N - 1, 0, -1)]
    for m, b, fold in orth:
        tot += 2 * m * b * b + fold * b * b + (0 if implicit else 2 * m * b * b)
    for m, b, keep, cm in trunc:
        tot += 2 * m * b * b + SVD_FLOPS_B3 * b ** 3 + 4 * m * keep * b
        tot += 4 * cm * keep * b if implicit else 2 * cm * keep * b
    return tot
