"""Seeded random shapes: the CUDA path against the CPU oracle on chains whose
dimensions, ranks and structure vary widely -- mode sizes from 1 to a few
thousand, bond ranks 1..64 across the three register-tile classes (16 / 32 /
64 columns), short end cores (single-chain panels, ragged last tiles), rank-
deficient sums, every rounding variant, tolerance and rank-cap truncation.
The fixed cases of tests/test_gpu_parity.py follow the reference's own tests;
this sweep is for the tile / unit / stage boundaries in between (an apply
product with k = 20 columns once read past its staging buffer on exactly such
a shape).  Reference paths: parallel.py:164-438, ops.py:44-235."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2011_06532_b200 as T  # noqa: E402
from oracle import tt_oracle as O  # noqa: E402

TOL_TT = 1e-10
TOL_SCALAR = 1e-12
VARIANTS = ("LRLI", "RLRI", "LRL", "RLR")
import os  # noqa: E402

SEEDS = int(os.environ.get("TTB_SWEEP_SEEDS", "48"))  # a soak run sets a few hundred
# seeds a 400-seed soak run failed on, kept as fixed cases: 234 (modes (2, 3, 618, 257, 257), ranks 64: roundoff
# of roundoff on the rank-2 / rank-6 bonds put columns of norm ~1e-160 into a head tile; their squared norm
# underflowed, the Householder vector overflowed and T went non-finite -- see kTinyCol in csrc/tsqr.cuh)
SOAK_REGRESSIONS = [234]


def dev(cores):
    return T.serial_tt(T.TTTensor(cores))


def host(dt):
    return [c.array for c in T.gather(dt).cores]


def chain(seed):
    """dims, ranks of a random chain (about <= 2e6 entries per core)."""
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.integers(2, 6))
    rmax = int(rng.choice([3, 9, 16, 17, 24, 32]))  # doubled by X = Y + Z: up to 64
    ranks = [1] + [int(rng.integers(1, rmax + 1)) for _ in range(d - 1)] + [1]
    dims = []
    for n in range(d):
        kind = rng.integers(0, 4)
        if kind == 0:
            m = int(rng.integers(1, 8))            # tiny mode
        elif kind == 1:
            m = int(rng.integers(8, 300))
        elif kind == 2:
            m = int(rng.integers(300, 3000))
        else:
            m = int(rng.choice([255, 256, 257, 511, 512, 513, 1023, 1024, 1025]))  # tile-size neighbours
        cap = max(1, 2_000_000 // (4 * ranks[n] * ranks[n + 1]))
        dims.append(min(m, cap))
    return tuple(dims), tuple(ranks)


@pytest.mark.parametrize("seed", sorted(set(range(SEEDS)) | set(SOAK_REGRESSIONS)))
def test_random_chain_round_inner_norm(seed):
    dims, ranks = chain(seed)
    if seed % 5 == 4:  # a Hadamard product (ranks multiply: keep the factors <= 8)
        ranks = tuple(min(r, 8) for r in ranks)
    y = O.random_cores(dims, ranks, seed)
    z = O.random_cores(dims, ranks, seed + 500)
    if seed % 5 == 4:
        x = O.hadamard(y, z)
    else:
        x = O.add(y, y) if seed % 3 == 0 else O.add(y, z)  # rank-deficient every third case
    variant = VARIANTS[seed % 4]
    dx = dev(x)
    # scalars
    ip_ref = O.inner(x, O.add(z, y))
    ip = T.inner_product(dx, dev(O.add(z, y)))
    assert abs(ip - ip_ref) <= TOL_SCALAR * max(abs(ip_ref), O.norm(x, "innerprod") * O.norm(O.add(z, y), "innerprod"))
    nref = O.norm(x, "ortho")
    for method in ("innerprod", "ortho"):
        assert abs(T.norm(dx, method) - nref) <= 1e-9 * nref, (method, dims, ranks)
    # rounding: tolerance, then a rank cap
    eps = float(10.0 ** -(3 + seed % 8))
    ref, _ = O.round_tt(x, eps, variant)
    out = T.round_tt(dx, T.RoundingOptions(eps, variant))
    assert tuple(out.ranks) == O.ranks_of(ref), (dims, ranks, variant, eps)
    assert O.rel_diff(host(out), ref) < max(TOL_TT, 1e-3 * eps), (dims, ranks, variant, eps)
    # eps0 = 0 keeps every singular value that is not an exact zero, up to the
    # cap.  On a bond whose rank is limited by the structure (a small mode: say
    # 5 rows under a cap of 10; the duplicated columns of Y + Y) the surplus
    # singular values are roundoff, and whether one of them comes out as an
    # exact zero or as 1e-17 depends on the SVD (LAPACK's gesdd in the
    # reference, one-sided Jacobi with deflation on the device): a 1200-seed
    # soak run saw the device keep fewer of them in most such cases and more
    # in a few.  The ranks are compared where they carry information (every
    # eps0 > 0 case above); here the results must be the same tensor within
    # the cap.
    cap = max(1, max(O.ranks_of(x)) // 3)
    ref, _ = O.round_tt(x, 0.0, variant, cap)
    out = T.round_tt(dx, T.RoundingOptions(0.0, variant, max_rank=cap))
    assert max(out.ranks) <= cap, (dims, ranks, variant, cap, tuple(out.ranks))
    assert O.rel_diff(host(out), ref) < 1e-8, (dims, ranks, variant, cap)


@pytest.mark.parametrize("seed", range(max(8, SEEDS // 6)))
def test_random_chain_orthonormalize(seed):
    dims, ranks = chain(100 + seed)
    x = O.add(O.random_cores(dims, ranks, seed), O.random_cores(dims, ranks, seed + 7))
    for direction in ("left", "right"):
        got = host(T.orthonormalize(dev(x), direction))
        assert O.rel_diff(got, x) < TOL_TT, (dims, ranks, direction)
        # the orthonormalized cores have orthonormal unfoldings (all but the last / first)
        idx = range(len(got) - 1) if direction == "left" else range(1, len(got))
        for n in idx:
            c = got[n]
            m = c.reshape(-1, c.shape[2], order="F") if direction == "left" else c.reshape(c.shape[0], -1, order="F").T
            if m.shape[0] < m.shape[1]:
                continue  # more columns than rows: no orthonormal columns to speak of
            g = m.T @ m
            # orthonormal columns (zero columns on rank-deficient bonds): a projector
            assert np.abs(g @ g - g).max() < 1e-10, (dims, ranks, direction, n)


@pytest.mark.parametrize("seed", range(max(12, SEEDS // 4)))
def test_random_chain_multirank(seed):
    """The same sweep through the native multi-rank path (in-process rank group,
    tests/test_gpu_multirank.py): P = 2, 3 or 4 ranks, idle ranks allowed where a
    mode has fewer slices than ranks; every rank keeps the same ranks, the result
    matches the oracle and the serial device result's ranks."""
    dims, ranks = chain(200 + seed)
    P = 2 + seed % 3
    y = O.random_cores(dims, ranks, seed)
    z = O.random_cores(dims, ranks, seed + 31)
    x = O.add(y, y) if seed % 2 == 0 else O.add(y, z)
    variant = VARIANTS[seed % 4]
    eps = float(10.0 ** -(4 + seed % 6))
    ref, meta = O.round_tt(x, eps, variant)
    tx = T.TTTensor(x)

    def body(comm):
        dx = T.distribute(tx, comm, allow_idle=True)
        out = T.round_tt(dx, T.RoundingOptions(eps, variant))
        return out.ranks, host(out), T.inner_product(dx, dx), T.norm(dx, "ortho")

    res = T.run_local_ranks(P, body)
    ip_ref = O.inner(x, x)
    for rk, _, ip, nrm in res:
        assert tuple(rk) == tuple(res[0][0]) == O.ranks_of(ref), (dims, ranks, P, variant, eps)
        assert abs(ip - ip_ref) <= TOL_SCALAR * abs(ip_ref)
        assert abs(nrm - meta["norm"]) <= 1e-9 * meta["norm"]
    assert O.rel_diff(res[0][1], ref) < max(TOL_TT, 1e-3 * eps), (dims, ranks, P, variant, eps)


@pytest.mark.parametrize("seed", range(max(8, SEEDS // 6)))
def test_random_chain_wide_ranks(seed):
    """Bond ranks above 64 (the general path, csrc/wide.cu) on random chains:
    sums of two chains with ranks up to 70 each, and mixed chains where only
    some bonds are wide (narrow and wide kernels alternate within one sweep)."""
    rng = np.random.default_rng(3000 + seed)
    d = int(rng.integers(3, 5))
    dims = tuple(int(rng.integers(90, 400)) for _ in range(d))
    ranks = (1,) + tuple(int(rng.choice([5, 20, 33, 40, 70])) for _ in range(d - 1)) + (1,)
    y = O.random_cores(dims, ranks, seed)
    z = O.random_cores(dims, ranks, seed + 9)
    x = O.add(y, y) if seed % 2 == 0 else O.add(y, z)
    variant = VARIANTS[seed % 4]
    dx = dev(x)
    ip_ref = O.inner(x, x)
    assert abs(T.inner_product(dx, dx) - ip_ref) <= TOL_SCALAR * abs(ip_ref)
    eps = 1e-8
    ref, meta = O.round_tt(x, eps, variant)
    out = T.round_tt(dx, T.RoundingOptions(eps, variant))
    assert tuple(out.ranks) == O.ranks_of(ref), (dims, ranks, variant)
    assert O.rel_diff(host(out), ref) < TOL_TT, (dims, ranks, variant)


@pytest.mark.parametrize("seed", range(max(6, SEEDS // 8)))
def test_random_chain_round_hadamard(seed):
    """Implicit Hadamard-then-round (ops.py:109-132 then parallel.py:293) on
    random chains: ranks identical to rounding the materialised product by the
    oracle, TT-form error within the bar."""
    dims, ranks = chain(400 + seed)
    ranks = tuple(min(r, 8) for r in ranks)
    y = O.random_cores(dims, ranks, seed)
    w = O.random_cores(dims, ranks, seed + 77)
    variant = VARIANTS[seed % 4]
    eps = float(10.0 ** -(4 + seed % 8))  # 1e-4 .. 1e-11: above the roundoff of the product
    ref, _ = O.round_tt(O.hadamard(y, w), eps, variant)
    out = T.round_hadamard(dev(y), dev(w), T.RoundingOptions(eps, variant))
    assert tuple(out.ranks) == O.ranks_of(ref), (dims, ranks, variant, eps)
    assert O.rel_diff(host(out), ref) < max(TOL_TT, 1e-3 * eps), (dims, ranks, variant, eps)


@pytest.mark.parametrize("seed", range(max(10, SEEDS // 8)))
def test_random_operator_apply(seed):
    """Kronecker-operator apply (ops.py:314-342) on random chains and random
    sparse factors (1 to 20 terms: the fused one-pass kernel takes up to 16,
    more go term by term): bitwise the oracle's result, then apply + round."""
    import scipy.sparse as sp

    rng = np.random.default_rng(5000 + seed)
    d = int(rng.integers(1, 5))
    dims = tuple(int(rng.integers(1, 90)) for _ in range(d))
    ranks = (1,) + tuple(int(rng.integers(1, 7)) for _ in range(d - 1)) + (1,)
    nterms = int(rng.choice([1, 2, 3, 8, 16, 17, 20]))
    x = O.random_cores(dims, ranks, seed)
    terms = []
    for _ in range(nterms):
        fac = []
        for m in dims:
            kind = rng.integers(0, 3)
            if kind == 0:
                a = sp.identity(m, format="csr")
            elif kind == 1:
                a = sp.diags([rng.standard_normal(m), rng.standard_normal(max(m - 1, 0))], [0, 1], shape=(m, m), format="csr")
            else:
                a = sp.random(m, m, density=min(1.0, 3.0 / m), random_state=int(rng.integers(1 << 30)), format="csr")
            fac.append(sp.csr_matrix(a))
        terms.append(fac)
    op = T.KroneckerOperator(dims, terms)
    want = O.apply_operator(op.terms, x)
    z = T.apply_operator(op, T.TTTensor(x))
    got = [c.array for c in z.cores]
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert a.shape == b.shape and np.array_equal(a, b), (dims, ranks, nterms)
    if max(O.ranks_of(want)) <= 64:
        ref, _ = O.round_tt(want, 1e-9, "LRLI")
        zr = T.apply_operator(op, T.TTTensor(x), round_eps=1e-9)
        assert tuple(zr.ranks) == O.ranks_of(ref), (dims, ranks, nterms)
        assert O.rel_diff([c.array for c in zr.cores], ref) < TOL_TT, (dims, ranks, nterms)


@pytest.mark.parametrize("seed", range(max(16, SEEDS // 6)))
def test_random_tsqr_blocks(seed):
    """TSQR of random tall blocks across the chain / tree boundaries (one chain,
    a few chains, one chain per SM, ragged last tiles; 1..64 columns): R against
    numpy's QR (sign-fixed as tsqr.py:127-129), Q orthonormal, Q R = A, and the
    implicit apply against the explicit Q."""
    rng = np.random.default_rng(7000 + seed)
    b = int(rng.choice([1, 2, 7, 15, 16, 17, 31, 32, 33, 48, 60, 63, 64]))
    m = int(rng.choice([b, b + 1, 255, 256, 257, 511, 513, 1000, 4096, 4097, 20000, 37888, 37889, 75000, 151552]))
    m = max(m, b)
    a = rng.standard_normal((m, b))
    if seed % 4 == 3:  # rank-deficient: duplicate the left half of the columns
        a[:, b // 2:b // 2 + b // 2] = a[:, :b // 2]
    fac, r = T.tsqr_factor(a)
    q = T.tsqr_apply_q(fac, np.eye(b))
    r_ref = np.linalg.qr(a, mode="r")
    sgn = np.where(np.diag(r_ref) < 0, -1.0, 1.0)
    r_ref = sgn[:, None] * r_ref
    scale = np.abs(a).max() * np.sqrt(m)
    assert np.abs(q.T @ q - np.eye(b)).max() < 1e-12, (m, b)
    assert np.abs(q @ r - a).max() < 1e-12 * scale, (m, b)
    if seed % 4 != 3:  # R is unique (up to the fixed signs) only at full rank
        assert np.abs(r - r_ref).max() < 1e-11 * scale, (m, b)
    c = rng.standard_normal((b, 5))
    assert np.abs(T.tsqr_apply_q(fac, c) - q @ c).max() < 1e-11 * np.abs(c).max() * np.sqrt(b), (m, b)
