"""Implicit Hadamard-then-round (survey 8(f) row 4):
round_hadamard(x, w, opts) == round_tt(hadamard(x, w), opts) without ever
writing the rank rx*rw product -- its Kronecker slices are formed where the
rounding reads its input.  Checked against the CPU oracle (the reference's
hadamard, ops.py:109-132, then round_tt, parallel.py:293-438) and against the
materialised device path: ranks identical, TT-form error <= 1e-10."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2011_06532_b200 as T  # noqa: E402
from oracle import tt_oracle as O  # noqa: E402

TOL_TT = 1e-10


def dev(cores):
    return T.serial_tt(T.TTTensor(cores))


def host(dt):
    return [c.array for c in T.gather(dt).cores]


@pytest.mark.parametrize("variant", ["LRLI", "LRL", "RLRI", "RLR"])
def test_matches_oracle_all_variants(variant):
    x = O.random_cores((30, 25, 40, 22), (1, 3, 4, 5, 1), 0)
    w = O.random_cores((30, 25, 40, 22), (1, 4, 2, 3, 1), 1)
    for eps0, cap in ((1e-6, None), (0.0, 5)):
        ref, meta = O.round_tt(O.hadamard(x, w), eps0, variant, cap)
        out = T.round_hadamard(dev(x), dev(w), T.RoundingOptions(eps0, variant, cap))
        assert out.ranks == O.ranks_of(ref)
        assert O.rel_diff(host(out), ref) <= TOL_TT
        assert out.meta["norm"] == pytest.approx(meta["norm"], rel=1e-12)
        assert out.meta["error_bound_violated"] == meta["error_bound_violated"]


def test_matches_materialised_path():
    x = O.random_cores((200,) * 6, (1,) + (8,) * 5 + (1,), 3)
    w = O.random_cores((200,) * 6, (1,) + (8,) * 5 + (1,), 4)
    opts = T.RoundingOptions(0.0, "LRLI", max_rank=32)
    a = T.round_tt(T.hadamard(dev(x), dev(w)), opts)
    b = T.round_hadamard(dev(x), dev(w), opts)
    assert a.ranks == b.ranks == (1,) + (32,) * 5 + (1,)
    assert O.rel_diff(host(b), host(a)) <= TOL_TT
    assert b.meta["norm"] == pytest.approx(a.meta["norm"], rel=1e-13)


def test_cfg5_shape_reduced():
    """BASELINE configs[4] (d=12, ranks 8 -> 64, max_rank 32) at n=400."""
    dims, r = (400,) * 12, (1,) + (8,) * 11 + (1,)
    x, w = O.random_cores(dims, r, 0), O.random_cores(dims, r, 1)
    ref, meta = O.round_tt(O.hadamard(x, w), 0.0, "LRLI", 32)
    out = T.round_hadamard(dev(x), dev(w), T.RoundingOptions(0.0, "LRLI", max_rank=32))
    assert out.ranks == O.ranks_of(ref)
    assert out.meta["error_bound_violated"] is True
    assert O.rel_diff(host(out), ref) <= TOL_TT


def test_exact_rank_recovery_and_single_mode():
    # (x o w) with w = all-ones rank-1 tensor is x itself: rounding recovers x's ranks
    x = O.random_cores((20, 30, 25), (1, 4, 3, 1), 5)
    ones = [np.ones((1, d, 1), order="F") for d in (20, 30, 25)]
    out = T.round_hadamard(dev(x), dev(ones), T.RoundingOptions(1e-12))
    assert out.ranks == (1, 4, 3, 1)
    assert O.rel_diff(host(out), x) <= 1e-12
    s, t = O.random_cores((9,), (1, 1), 1), O.random_cores((9,), (1, 1), 2)
    got = host(T.round_hadamard(dev(s), dev(t), T.RoundingOptions(1e-6)))
    assert np.array_equal(got[0], O.hadamard(s, t)[0])


def test_host_operands_and_guard():
    x = O.random_cores((12, 10, 14), (1, 3, 3, 1), 7)
    w = O.random_cores((12, 10, 14), (1, 2, 2, 1), 8)
    res = T.round_hadamard(T.TTTensor(x), T.TTTensor(w), T.RoundingOptions(1e-8))
    assert isinstance(res, T.TTTensor)
    ref, _ = O.round_tt(O.hadamard(x, w), 1e-8, "LRLI")
    assert O.rel_diff([c.array for c in res.cores], ref) <= TOL_TT
    with pytest.raises(T.CapacityError):
        T.round_hadamard(dev(x), dev(w), T.RoundingOptions(1e-8), max_rank_product=5)


@pytest.mark.parametrize("P", [2, 3])
def test_distributed(P):
    x = O.random_cores((40, 33, 50, 27), (1, 4, 5, 3, 1), 11)
    w = O.random_cores((40, 33, 50, 27), (1, 3, 2, 4, 1), 12)
    ref, _ = O.round_tt(O.hadamard(x, w), 1e-8, "LRLI")

    def body(comm):
        o = T.round_hadamard(T.distribute(T.TTTensor(x), comm), T.distribute(T.TTTensor(w), comm),
                             T.RoundingOptions(1e-8))
        return o.ranks, host(o)

    res = T.run_local_ranks(P, body)
    for ranks, _ in res:
        assert ranks == O.ranks_of(ref)
    assert O.rel_diff(res[0][1], ref) <= TOL_TT
