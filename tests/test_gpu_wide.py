"""GPU parity for bond ranks above 64 (the general path, csrc/wide.cu).

The reference has no rank limit (tsqr.py:103-130 takes any b,
parallel.py:224-258 any SVD size, ops.py:135-155 any Gram ranks, and the
operator apply of ops.py:314-342 multiplies ranks by the term count), so the
same bars apply: truncation ranks identical to the oracle's, TT-form relative
error <= 1e-10, norms and inner products within 1e-12 relative.
"""
import numpy as np
import pytest
import scipy.sparse as sp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2011_06532_b200 as T  # noqa: E402
from oracle import tt_oracle as O  # noqa: E402

TOL_TT = 1e-10
TOL_SCALAR = 1e-12


def dev(cores):
    return T.serial_tt(T.TTTensor(cores))


def host(dt):
    return [c.array for c in T.gather(dt).cores]


@pytest.mark.parametrize("m,b", [(6000, 81), (4000, 96), (9000, 128), (700, 65), (2500, 200), (100, 70)])
def test_wide_tsqr(m, b):
    rng = np.random.default_rng(m + b)
    a = rng.standard_normal((m, b))
    fac, r = T.tsqr_factor(a)
    r_ref, _ = O.stacked_tsqr([a])
    assert np.allclose(np.triu(r), r)
    assert (np.diagonal(r) >= 0).all()
    assert np.allclose(r, r_ref, rtol=1e-10, atol=1e-11 * np.abs(r_ref).max())
    q = T.tsqr_apply_q(fac, np.eye(b))
    assert np.allclose(q.T @ q, np.eye(b), atol=1e-12)
    assert np.allclose(q @ r, a, atol=1e-11 * np.abs(a).max())
    c = rng.standard_normal((b, 7))
    assert np.allclose(T.tsqr_apply_q(fac, c), q @ c, atol=1e-11)
    c2 = rng.standard_normal((b, 90))  # more than 64 right-hand columns
    assert np.allclose(T.tsqr_apply_q(fac, c2), q @ c2, atol=1e-11)


def test_wide_tsqr_rank_deficient():
    rng = np.random.default_rng(11)
    base = rng.standard_normal((8000, 48))
    a = np.hstack([base, base])  # exact rank 48 in 96 columns, the X = Y + Y pattern
    fac, r = T.tsqr_factor(a)
    q = T.tsqr_apply_q(fac, np.eye(96))
    assert np.allclose(q @ r, a, atol=1e-10)
    s = np.linalg.svd(r, compute_uv=False)
    assert s[47] > 1.0 and s[48] < 1e-10 * s[0]
    # the retained directions are orthonormal: project on the leading right-singular subspace
    u, _, _ = np.linalg.svd(r)
    qk = q @ u[:, :48]
    assert np.allclose(qk.T @ qk, np.eye(48), atol=1e-10)


@pytest.mark.parametrize("m,n", [(100, 100), (128, 96), (70, 130), (65, 1)])
def test_wide_truncated_svd(m, n):
    rng = np.random.default_rng(m * n)
    a = rng.standard_normal((m, n))
    s_ref = np.linalg.svd(a, compute_uv=False)
    eps = float(np.sqrt(np.sum(s_ref[min(m, n) // 2:] ** 2))) * 1.0000001
    f = T.truncated_svd(a, eps)
    ref = O.truncated_svd(a, eps)
    assert f.s.shape == ref[1].shape
    assert np.allclose(f.s, ref[1], rtol=1e-12)
    k = f.s.shape[0]
    assert np.allclose((f.u * f.s) @ f.v.T, (ref[0] * ref[1]) @ ref[2].T, atol=1e-11 * s_ref[0])
    assert np.allclose(f.u.T @ f.u, np.eye(k), atol=1e-12)
    assert np.allclose(f.v.T @ f.v, np.eye(k), atol=1e-12)


@pytest.mark.parametrize("rx,ry", [(72, 72), (96, 20), (130, 65)])
def test_wide_inner_and_norms(rx, ry):
    dims = (40, 33, 50, 21)
    x = O.random_cores(dims, (1, rx, rx, 17, 1), 3)
    y = O.random_cores(dims, (1, ry, ry, 70, 1), 4)
    assert T.inner_product(dev(x), dev(y)) == pytest.approx(O.inner(x, y), rel=TOL_SCALAR)
    ref = np.sqrt(O.inner(x, x))
    for m in ("innerprod", "innerprod_sym", "ortho"):
        assert T.norm(dev(x), m) == pytest.approx(ref, rel=TOL_SCALAR), m


@pytest.mark.parametrize("direction", ["left", "right"])
def test_wide_orthonormalize(direction):
    x = O.random_cores((60, 50, 70, 40), (1, 40, 80, 30, 1), 7)
    out = host(T.orthonormalize(dev(x), direction))
    assert O.rel_diff(out, x) <= TOL_TT
    for n, c in enumerate(out):
        rl, I, rr = c.shape
        if direction == "left" and n < len(out) - 1:
            v = c.reshape(rl * I, rr, order="F")
            assert np.allclose(v.T @ v, np.eye(rr), atol=1e-11)
        if direction == "right" and n > 0:
            h = c.reshape(rl, I * rr, order="F")
            assert np.allclose(h @ h.T, np.eye(rl), atol=1e-11)


@pytest.mark.parametrize("variant", ["LRLI", "LRL", "RLRI", "RLR"])
def test_wide_round_doubled(variant):
    """X = Y + Y with Y of rank 48: ranks 96 round back to 48."""
    y = O.random_cores((90, 70, 80, 60), (1, 40, 48, 36, 1), 5)
    x = O.add(y, y)
    out = T.round_tt(dev(x), T.RoundingOptions(1e-10, variant))
    ref, _ = O.round_tt(x, 1e-10, variant)
    assert out.ranks == O.ranks_of(ref) == O.ranks_of(y)
    assert O.rel_diff(host(out), ref) <= TOL_TT


def test_wide_round_rank128_tolerance():
    """ranks 128 with a decaying spectrum: same truncation ranks as the oracle."""
    rng = np.random.default_rng(2)
    y = O.random_cores((150, 140, 130), (1, 128, 128, 1), 9)
    # impose decay on the middle bond so the tolerance cuts inside the spectrum
    y[1] = y[1] * (0.7 ** np.arange(128))[None, None, :]
    y[0] = y[0] * (0.8 ** np.arange(128))[None, None, :]
    out = T.round_tt(dev(y), T.RoundingOptions(1e-6))
    ref, _ = O.round_tt(y, 1e-6, "LRLI")
    assert out.ranks == O.ranks_of(ref)
    assert max(out.ranks) > 1
    assert O.rel_diff(host(out), ref) <= TOL_TT
    capped = T.round_tt(dev(y), T.RoundingOptions(1e-12, max_rank=70))
    refc, _ = O.round_tt(y, 1e-12, "LRLI", max_rank=70)
    assert capped.ranks == O.ranks_of(refc)
    assert max(capped.ranks) == 70
    assert O.rel_diff(host(capped), refc) <= 1e-8  # capped: the cut sits inside a dense spectrum
    del rng


def test_hadamard_rank9_squared_rounds():
    """the verdict's example: a Hadamard of two rank-9 tensors has rank 81."""
    x = O.random_cores((70, 60, 50, 40), (1, 9, 9, 9, 1), 1)
    w = O.random_cores((70, 60, 50, 40), (1, 9, 9, 9, 1), 2)
    z = O.hadamard(x, w)
    ref, _ = O.round_tt(z, 1e-9, "LRLI")
    a = T.round_tt(T.hadamard(dev(x), dev(w)), T.RoundingOptions(1e-9))
    assert a.ranks == O.ranks_of(ref)
    assert O.rel_diff(host(a), ref) <= TOL_TT
    b = T.round_hadamard(dev(x), dev(w), T.RoundingOptions(1e-9))
    assert b.ranks == O.ranks_of(ref)
    assert O.rel_diff(host(b), ref) <= TOL_TT


def test_operator_apply_rank128_rounds():
    """8-term Kronecker operator applied to a rank-16 tensor: ranks 128, then rounded
    (the Krylov caller of rounding, ops.py:314-342)."""
    dims = (48,) * 8
    x = O.random_cores(dims, (1,) + (16,) * 7 + (1,), 12)
    lap = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(48, 48), format="csr")
    eye = sp.identity(48, format="csr")
    terms = [[lap if m == t else eye for m in range(8)] for t in range(8)]
    op = T.KroneckerOperator(dims, terms)
    y = T.apply_operator(op, dev(x))
    assert max(y.ranks) == 128
    ycores = host(y)
    out = T.round_tt(y, T.RoundingOptions(1e-10))
    ref, _ = O.round_tt(ycores, 1e-10, "LRLI")
    assert out.ranks == O.ranks_of(ref)
    assert max(out.ranks) <= 32  # sum of 8 rank-16 terms sharing factors: 2 * 16
    assert O.rel_diff(host(out), ref) <= TOL_TT


def test_tall_slices_take_the_general_path():
    """left rank 250 with right rank 10: a slice (250 rows) is taller than a leaf tile allows."""
    x = O.random_cores((30, 40, 30), (1, 250, 10, 1), 8)
    out = T.round_tt(dev(x), T.RoundingOptions(1e-10))
    ref, _ = O.round_tt(x, 1e-10, "LRLI")
    assert out.ranks == O.ranks_of(ref)
    assert O.rel_diff(host(out), ref) <= TOL_TT


# ---- the general path with P > 1 ranks (in-process group, as tests/test_gpu_multirank.py) ----

@pytest.mark.parametrize("P", [2, 3])
def test_wide_tsqr_distributed(P):
    rng = np.random.default_rng(P)
    m, b = 7000, 100
    a = rng.standard_normal((m, b))
    blocks = [a[slice(*T.block_bounds(m, P, r))] for r in range(P)]
    c = rng.standard_normal((b, 75))

    def body(comm):
        fac, r = T.tsqr_factor(blocks[comm.rank], comm)
        return r, T.tsqr_apply_q(fac, np.eye(b), comm), T.tsqr_apply_q(fac, c, comm)

    res = T.run_local_ranks(P, body)
    for r, _, _ in res[1:]:
        assert np.array_equal(r, res[0][0])  # replicated R, bitwise
    r = res[0][0]
    r_ref, _ = O.stacked_tsqr(blocks)
    assert np.allclose(r, r_ref, rtol=1e-10, atol=1e-11 * np.abs(r_ref).max())
    q = np.vstack([x for _, x, _ in res])
    assert np.allclose(q.T @ q, np.eye(b), atol=1e-12)
    assert np.allclose(q @ r, a, atol=1e-11 * np.abs(a).max())
    assert np.allclose(np.vstack([x for _, _, x in res]), q @ c, atol=1e-11)


@pytest.mark.parametrize("P", [2, 4])
def test_wide_round_invariant_under_P(P):
    y = O.random_cores((44, 36, 40, 52), (1, 36, 40, 33, 1), 21)
    x = O.add(y, y)  # ranks 72, 80, 66
    ref, meta = O.round_tt(x, 1e-10, "LRLI")
    tx = T.TTTensor(x)

    def body(comm):
        d = T.distribute(tx, comm)
        out = T.round_tt(d, T.RoundingOptions(1e-10, "LRLI"))
        return out.ranks, host(out), T.inner_product(d, d), T.norm(d, "ortho")

    res = T.run_local_ranks(P, body)
    for ranks, _, ip, nrm in res:
        assert ranks == O.ranks_of(ref) == O.ranks_of(y)
        assert ip == pytest.approx(O.inner(x, x), rel=TOL_SCALAR)
        assert nrm == pytest.approx(np.sqrt(O.inner(x, x)), rel=TOL_SCALAR)
    assert O.rel_diff(res[0][1], ref) <= TOL_TT
