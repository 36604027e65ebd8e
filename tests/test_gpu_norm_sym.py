"""norm(method="innerprod_sym") on the device: the pivoted-Cholesky Gram
route and its fallback, mirroring the reference's own tests
(test_ops.py:180-255) against the oracle (tt_oracle.pivoted_cholesky /
sym_norm, which follow ops.py:162-205)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2011_06532_b200 as T  # noqa: E402
from oracle import tt_oracle as O  # noqa: E402


def dev(cores):
    return T.serial_tt(T.TTTensor(cores))


@pytest.mark.parametrize("dims,ranks", [
    ((5, 6, 4, 7), (1, 3, 4, 2, 1)),
    ((300,) * 6, (1,) + (16,) * 5 + (1,)),        # the fused rank-16 kernel
    ((40, 33, 50, 41, 37), (1, 16, 16, 16, 16, 1)),
    ((120,) * 5, (1, 7, 12, 9, 5, 1)),
])
def test_norm_sym_matches_oracle(dims, ranks):
    x = O.random_cores(dims, ranks, 11)
    val, info = T.norm(dev(x), "innerprod_sym", return_info=True)
    assert not info["fallback"]
    assert val == pytest.approx(O.sym_norm(x), rel=1e-12)
    assert val == pytest.approx(O.norm(x, "innerprod"), rel=1e-12)


@pytest.mark.parametrize("r", [3, 8, 24, 32])
def test_norm_sym_handles_rank_deficient_gram(r):
    # x + x doubles every bond rank: every carry is exactly singular, the
    # factor drops to the numeric rank without falling back (test_ops.py:201)
    # r = 24 / 32: carries of 48 / 64 (the generic contraction with the
    # reconstructed carry, the 64-wide factorization)
    x = O.random_cores((200,) * 5, (1,) + (r,) * 4 + (1,), 20)
    dx = dev(x)
    y = T.add(dx, T.scale(dx, 1.0))
    assert y.ranks[1] == 2 * r
    val, info = T.norm(y, "innerprod_sym", return_info=True)
    assert not info["fallback"]
    assert val == pytest.approx(2 * O.norm(x, "innerprod"), rel=1e-11)


def test_norm_sym_falls_back_on_indefinite_gram(monkeypatch):
    x = O.random_cores((6, 5, 7), (1, 3, 4, 1), 21)
    want = O.norm(x, "innerprod")
    monkeypatch.setattr(T.ops, "_sym_norm", lambda dx: (0.0, False))
    with pytest.warns(UserWarning, match="fell back"):
        val, info = T.norm(dev(x), "innerprod_sym", return_info=True)
    assert info["fallback"]
    assert val == pytest.approx(want, rel=1e-12)


def test_pivoted_cholesky_rejects_indefinite():
    with pytest.raises(T.NumericError):
        T.pivoted_cholesky(np.diag([1.0, -1.0]))


@pytest.mark.parametrize("n,k", [(6, 4), (16, 16), (16, 9), (64, 40), (1, 1)])
def test_pivoted_cholesky_matches_oracle(n, k):
    rng = np.random.default_rng(22 + n)
    a = rng.standard_normal((n, k))
    w = a @ a.T
    lf, perm, rank = T.pivoted_cholesky(w)
    lo, po, ro = O.pivoted_cholesky(w)
    assert rank == ro == min(n, k)
    assert np.array_equal(perm[:rank], po[:rank])  # same greedy pivots
    pl = np.empty_like(lf)
    pl[perm] = lf
    assert np.allclose(pl @ pl.T, w, atol=1e-12 * np.abs(w).max())
    assert np.allclose(lf[:rank], lo[:rank], rtol=1e-10, atol=1e-12 * np.sqrt(np.abs(w).max()))


def test_pivoted_cholesky_zero_matrix():
    lf, perm, rank = T.pivoted_cholesky(np.zeros((4, 4)))
    assert rank == 0 and lf.shape == (4, 0)


def test_norm_sym_cost_model_halves_the_flops():
    # test_ops.py:243-255: the symmetric route is charged under 0.65x the
    # two-product recurrence by the same cost model
    x = dev(O.random_cores((30,) * 6, (1,) + (7,) * 5 + (1,), 23))
    tr = x.comm.trace
    tr.reset()
    T.inner_product(x, x)
    both = tr.total("flops")
    tr.reset()
    T.norm(x, "innerprod_sym")
    half = tr.total("flops")
    tr.stop()
    assert 0 < half < 0.65 * both
