"""Pin the CPU oracle against golden vectors produced by the reference itself."""
import numpy as np
import pytest

from oracle import tt_oracle as O
from tests._golden import golden, tt


def same(xs, ys, tol=0.0):
    assert len(xs) == len(ys)
    for a, b in zip(xs, ys):
        assert a.shape == b.shape
        if tol == 0.0:
            assert np.array_equal(a, b)
        else:
            assert np.allclose(a, b, rtol=tol, atol=tol * max(1.0, np.abs(b).max()))


def test_rng_bitwise():
    same(O.random_cores((4, 5, 3), (1, 3, 2, 1), 42), tt("rng_a"))
    same(O.random_cores((6, 4), (1, 3, 1), 7), tt("rng_b"))


def test_rng_slabs_bitwise():
    full = O.random_cores((9, 7, 5), (1, 3, 4, 1), 3)
    for p in range(4):
        part = O.random_cores((9, 7, 5), (1, 3, 4, 1), 3,
                              lo_hi=lambda n, d: O.block_bounds(d, 4, p))
        for a, b, d in zip(part, full, (9, 7, 5)):
            lo, hi = O.block_bounds(d, 4, p)
            assert np.array_equal(a, b[:, lo:hi, :])


def test_local_algebra_bitwise():
    x, y = tt("pair_x"), tt("pair_y")
    same(O.random_cores((4, 5, 3), (1, 3, 2, 1), 11), x)
    same(O.add(x, y), tt("add_xy"))
    same(O.hadamard(x, y), tt("had_xy"))
    same(O.scale(x, -2.5), tt("scale_x"))
    same(O.add(O.add(O.scale(x, 1.0), O.scale(x, 0.5)), O.scale(x, -0.25)), tt("add3"))


def test_gram_values():
    g = golden()
    z, w = tt("gram_z"), tt("gram_w")
    assert O.inner(z, w) == pytest.approx(float(g["gram_zw"]), rel=1e-14)
    assert O.norm(z, "innerprod") == pytest.approx(float(g["norm_z_innerprod"]), rel=1e-14)
    assert O.norm(z, "innerprod_sym") == pytest.approx(float(g["norm_z_sym"]), rel=1e-14)
    assert O.norm(z, "ortho") == pytest.approx(float(g["norm_z_ortho"]), rel=1e-14)


@pytest.mark.parametrize("direction", ["left", "right"])
def test_orthonormalize(direction):
    same(O.orthonormalize(tt("orth_in"), direction), tt(f"orth_{direction}"), tol=1e-13)


def test_truncated_svd():
    g = golden()
    u, s, v, tail, capped = O.truncated_svd(g["tsvd_a"], 1.5)
    assert np.allclose(s, g["tsvd_s"], rtol=1e-14)
    assert tail == pytest.approx(float(g["tsvd_tail"]), rel=1e-12)
    u, s, v, tail, capped = O.truncated_svd(g["tsvd_a"], 0.0, max_rank=3)
    assert capped and np.allclose(s, g["tsvd_cap_s"], rtol=1e-14)
    assert tail == pytest.approx(float(g["tsvd_cap_tail"]), rel=1e-12)
    # known answers (test_parallel.py:189-224)
    assert O.truncated_svd(np.diag([2.0, 1.0, 0.0]), 0.0)[1].shape == (2,)
    r = O.truncated_svd(np.diag([3.0, 2.0]), 10.0)
    assert r[1].shape == (1,) and r[3] == pytest.approx(2.0)


@pytest.mark.parametrize("variant", ["LRLI", "LRL", "RLRI", "RLR"])
def test_rounding_matches_reference(variant):
    g = golden()
    x = tt("round_in")
    for tag, eps in (("e2", 1e-2), ("e6", 1e-6)):
        out, meta = O.round_tt(x, eps, variant)
        ref = tt(f"round_{variant}_{tag}")
        assert O.ranks_of(out) == O.ranks_of(ref)
        assert O.rel_diff(out, ref) < 1e-12
        assert meta["norm"] == pytest.approx(float(g[f"round_{variant}_{tag}/norm"]), rel=1e-13)
        assert meta["eps_bond"] == pytest.approx(float(g[f"round_{variant}_{tag}/eps_bond"]), rel=1e-13)
    out, meta = O.round_tt(tt("round_rr"), 1e-10, variant)
    ref = tt(f"round_{variant}_rr")
    assert O.ranks_of(out) == O.ranks_of(ref) == O.ranks_of(tt("round_y"))
    assert O.rel_diff(out, ref) < 1e-12
    out, meta = O.round_tt(x, 1e-12, variant, max_rank=2)
    assert O.ranks_of(out) == O.ranks_of(tt(f"round_{variant}_cap"))
    assert meta["error_bound_violated"] == bool(g[f"round_{variant}_cap/violated"])


def test_tsqr_r():
    g = golden()
    a = g["tsqr_a"]
    r, _ = O.stacked_tsqr([a])
    assert np.allclose(r, g["tsqr_r1"], rtol=1e-13, atol=1e-13)
    blocks = [a[slice(*O.block_bounds(120, 3, p))] for p in range(3)]
    r3, apply = O.stacked_tsqr(blocks)
    assert np.allclose(r3, g["tsqr_r3"], rtol=1e-12, atol=1e-12)
    q = np.vstack(apply(np.eye(7)))
    assert np.allclose(q @ r3, a, atol=1e-12)


def test_cfg1_small():
    g = golden()
    y = O.random_cores((60,) * 8, (1,) + (10,) * 7 + (1,), 0)
    same(y, tt("cfg1s_y"))
    out, meta = O.round_tt(O.add(y, y), 1e-10, "LRLI")
    ref = tt("cfg1s_out")
    assert O.ranks_of(out) == O.ranks_of(ref) == O.ranks_of(y)
    assert O.rel_diff(out, ref) < 1e-12
    assert O.rel_diff(out, O.scale(y, 2.0)) < 1e-12
    assert meta["norm"] == pytest.approx(float(g["cfg1s_norm"]), rel=1e-13)
