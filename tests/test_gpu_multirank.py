"""The native multi-rank path (P > 1) on one GPU.

P ranks run in one process, one host thread and one CUDA stream each, joined
into an in-process group (``LocalGroup`` / ttb_group): every kernel, plan and
collective call site is the one a P-GPU job executes -- the TSQR rank-root
allgather followed by the redundant global tree, the rank-offset global
apply levels, the Gram / norm allreduces, the operator halo exchange -- only
the transport is a stream-ordered device copy with a host rendezvous instead
of NCCL (the reference's own thread simulator SimComm / run_spmd plays the
same role for its MPI path, comm.py:184-356).

Mirrors the reference's multi-rank tests:
  test_tsqr.py:90-99      TSQR R / gathered Q vs sequential QR, P = 2, 3, 5, 8
  test_tsqr.py:141-159    R distribution-invariant
  test_parallel.py:316-329 rounding invariant under P (1e-10), ranks agree
  test_ops.py:91-103      add / Hadamard need no communication
and checks that every rank computes the SAME truncation ranks (the
reference's _assert_consistent_rank, parallel.py:441-449) and bitwise the
same R (the redundant root makes rank agreement hold by construction).
"""
import threading

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
PS = [2, 3, 4, 5, 8]


def row_blocks(a, p):
    out = []
    for r in range(p):
        lo, hi = T.block_bounds(a.shape[0], p, r)
        out.append(a[lo:hi])
    return out


def host(dt):
    return [c.array for c in T.gather(dt).cores]


def native_collectives(fn):
    """Run fn and return (result, TSQR allgathers, allreduce+p2p messages)."""
    from paper_2011_06532_b200 import _lib
    s0 = _lib.comm_stats()
    res = fn()
    s1 = _lib.comm_stats()
    return res, s1[0] - s0[0], s1[2] - s0[2]


# ---- TSQR ---------------------------------------------------------------------

@pytest.mark.parametrize("P", PS)
@pytest.mark.parametrize("m,b", [(30000, 60), (4000, 20), (777, 7)])
def test_tsqr_distributed(P, m, b):
    rng = np.random.default_rng(P * 1000 + b)
    a = rng.standard_normal((m, b))
    blocks = row_blocks(a, P)
    c = rng.standard_normal((b, 5))

    def body(comm):
        fac, r = T.tsqr_factor(blocks[comm.rank], comm)
        q = T.tsqr_apply_q(fac, np.eye(b), comm)
        qc = T.tsqr_apply_q(fac, c, comm)
        return r, q, qc

    (res, ngather, _) = native_collectives(lambda: T.run_local_ranks(P, body))
    assert ngather >= P  # every rank allgathered its root triangle (native path)
    rs = [r for r, _, _ in res]
    for r in rs[1:]:
        assert np.array_equal(r, rs[0])  # replicated R: bitwise identical on every rank
    r_ref, _ = O.stacked_tsqr(blocks)
    assert np.allclose(rs[0], r_ref, rtol=1e-12, atol=1e-12 * np.abs(r_ref).max())
    q = np.vstack([q for _, q, _ in res])
    qc = np.vstack([x for _, _, x in res])
    assert np.allclose(q.T @ q, np.eye(b), atol=1e-12)
    assert np.allclose(q @ rs[0], a, atol=1e-11 * np.abs(a).max())
    assert np.allclose(qc, q @ c, atol=1e-12)


def test_tsqr_r_invariant_under_P():
    rng = np.random.default_rng(4)
    a = rng.standard_normal((9600, 30))
    rs = {}
    for P in (1, 2, 3, 4, 8):
        blocks = row_blocks(a, P)
        rs[P] = T.run_local_ranks(P, lambda comm: T.tsqr_factor(blocks[comm.rank], comm)[1])[0]
    for P, r in rs.items():
        assert np.allclose(r, rs[1], rtol=1e-12, atol=1e-13 * np.abs(rs[1]).max()), P


def test_tsqr_idle_rank():
    """More ranks than row blocks: idle ranks contribute a zero triangle."""
    rng = np.random.default_rng(6)
    a = rng.standard_normal((3, 3))
    blocks = row_blocks(a, 5)  # block rule 3 over 5: 1, 1, 1, 0, 0
    assert [blk.shape[0] for blk in blocks] == [1, 1, 1, 0, 0]
    res = T.run_local_ranks(5, lambda comm: T.tsqr_factor(blocks[comm.rank], comm)[1])
    r_ref = np.linalg.qr(a, mode="r")
    r_ref = np.diag(np.sign(np.diag(r_ref))) @ r_ref
    for r in res:
        assert np.array_equal(r, res[0])
    assert np.allclose(res[0], r_ref, atol=1e-13)


# ---- rounding --------------------------------------------------------------------

@pytest.mark.parametrize("P", PS)
def test_round_invariant_under_P(P):
    y = O.random_cores((40, 33, 50, 27, 44), (1, 7, 9, 8, 6, 1), 41)
    x = O.add(y, y)
    ref, meta = O.round_tt(x, 1e-10, "LRLI")
    tx = T.TTTensor(x)

    def body(comm):
        out = T.round_tt(T.distribute(tx, comm), T.RoundingOptions(1e-10, "LRLI"))
        return out.ranks, out.meta["norm"], host(out)

    (res, ngather, nred) = native_collectives(lambda: T.run_local_ranks(P, body))
    assert ngather > 0 and nred > 0
    for ranks, nrm, got in res:
        assert ranks == res[0][0] == O.ranks_of(ref) == O.ranks_of(y)  # every rank keeps the same ranks
        assert nrm == res[0][1]
        assert abs(nrm - meta["norm"]) <= TOL_SCALAR * meta["norm"]
    got = res[0][2]
    assert O.rel_diff(got, ref) <= TOL_TT
    assert O.rel_diff(got, O.scale(y, 2.0)) <= TOL_TT


@pytest.mark.parametrize("variant", ["LRLI", "LRL", "RLRI", "RLR"])
def test_round_variants_P3(variant):
    x = O.random_cores((30, 25, 31, 28), (1, 6, 9, 5, 1), 7)
    for eps0 in (1e-2, 1e-6):
        ref, meta = O.round_tt(x, eps0, variant)
        res = T.run_local_ranks(3, lambda comm: (lambda o: (o.ranks, host(o)))(
            T.round_tt(T.distribute(T.TTTensor(x), comm), T.RoundingOptions(eps0, variant))))
        for ranks, _ in res:
            assert ranks == O.ranks_of(ref)
        assert O.rel_diff(res[0][1], ref) <= TOL_TT


def test_round_cfg3_shape_P4():
    """The bench workload's shape at a reduced mode size, sliced over 4 ranks."""
    dims, ry = (600,) * 10, (1,) + (30,) * 9 + (1,)
    y = O.random_cores(dims, ry, 0)
    x = O.add(y, y)
    ref, meta = O.round_tt(x, 1e-10, "LRLI")

    def body(comm):
        yd = T.DistTTTensor.random(comm, dims, ry, 0)  # device generator, this rank's slices
        out = T.round_tt(T.add(yd, yd), T.RoundingOptions(1e-10))
        return out.ranks, host(out)

    res = T.run_local_ranks(4, body)
    for ranks, _ in res:
        assert ranks == ry
    assert O.rel_diff(res[0][1], ref) <= TOL_TT


def test_round_max_rank_cap_P2():
    x = O.random_cores((40, 40, 40), (1, 8, 8, 1), 3)
    ref, meta = O.round_tt(x, 0.0, "LRLI", 3)
    res = T.run_local_ranks(2, lambda comm: (lambda o: (o.ranks, o.meta["error_bound_violated"], host(o)))(
        T.round_tt(T.distribute(T.TTTensor(x), comm), T.RoundingOptions(0.0, "LRLI", max_rank=3))))
    for ranks, viol, _ in res:
        assert ranks == O.ranks_of(ref) and viol is True
    assert O.rel_diff(res[0][2], ref) <= TOL_TT


def test_round_idle_ranks():
    """A mode of 3 slices over 5 ranks (allow_idle): ranks 3, 4 hold nothing there."""
    x = O.random_cores((3, 20, 11), (1, 3, 4, 1), 12)
    ref, _ = O.round_tt(x, 1e-12, "LRLI")

    def body(comm):
        out = T.round_tt(T.distribute(T.TTTensor(x), comm, allow_idle=True), T.RoundingOptions(1e-12))
        return out.ranks, host(out), T.inner_product(T.distribute(T.TTTensor(x), comm, allow_idle=True),
                                                      T.distribute(T.TTTensor(x), comm, allow_idle=True))

    res = T.run_local_ranks(5, body)
    for ranks, _, ip in res:
        assert ranks == O.ranks_of(ref)
        assert ip == pytest.approx(O.inner(x, x), rel=TOL_SCALAR)
    assert O.rel_diff(res[0][1], ref) <= TOL_TT


# ---- Gram sweep, norms, orthonormalization ------------------------------------

@pytest.mark.parametrize("P", PS)
def test_inner_and_norms_P(P):
    dims = (200, 150, 120, 180)
    x = O.random_cores(dims, (1, 16, 16, 16, 1), 0)
    z = O.random_cores(dims, (1, 12, 16, 9, 1), 1)
    want = {"inner": O.inner(x, z)}
    for m in ("innerprod", "innerprod_sym", "ortho"):
        want[m] = O.norm(x, m)

    def body(comm):
        dx, dz = T.distribute(T.TTTensor(x), comm), T.distribute(T.TTTensor(z), comm)
        got = {"inner": T.inner_product(dx, dz)}
        for m in ("innerprod", "innerprod_sym", "ortho"):
            got[m] = T.norm(dx, m)
        return got

    (res, _, nred) = native_collectives(lambda: T.run_local_ranks(P, body))
    assert nred > 0
    for got in res:
        assert got == res[0]  # bitwise identical scalars on every rank
        for k, v in want.items():
            assert got[k] == pytest.approx(v, rel=TOL_SCALAR), k


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("direction", ["left", "right"])
def test_orthonormalize_P(P, direction):
    x = O.random_cores((64, 50, 70, 45), (1, 8, 16, 6, 1), 5)
    ref = O.orthonormalize(x, direction)
    res = T.run_local_ranks(P, lambda comm: host(T.orthonormalize(T.distribute(T.TTTensor(x), comm), direction)))
    for got in res:
        assert O.rel_diff(got, ref) <= TOL_TT
    assert max(np.abs(a - b).max() / np.abs(b).max() for a, b in zip(res[0], ref)) <= 1e-11


def test_add_hadamard_local_P4():
    """Construction is communication-free and bitwise (test_ops.py:91-103)."""
    x = O.random_cores((17, 23, 19), (1, 3, 4, 1), 1)
    y = O.random_cores((17, 23, 19), (1, 2, 5, 1), 2)

    def body(comm):
        dx, dy = T.distribute(T.TTTensor(x), comm), T.distribute(T.TTTensor(y), comm)
        return host(T.add(dx, dy)), host(T.hadamard(dx, dy))

    (res, ng, nr) = native_collectives(lambda: T.run_local_ranks(4, body))
    for a, h in res:
        for u, v in zip(a, O.add(x, y)):
            assert np.array_equal(u, v)
        for u, v in zip(h, O.hadamard(x, y)):
            assert np.array_equal(u, v)
    assert ng == 0 and nr == 0


# ---- failure handling ------------------------------------------------------------

def test_failed_rank_breaks_group():
    """A rank that dies before a collective releases its peers with
    DeadlockError instead of hanging them (the reference's DeadlockError)."""
    x = O.random_cores((30, 30, 30), (1, 4, 4, 1), 2)

    def body(comm):
        if comm.rank == 1:
            raise RuntimeError("rank 1 fails")
        return T.inner_product(T.distribute(T.TTTensor(x), comm), T.distribute(T.TTTensor(x), comm))

    with pytest.raises(RuntimeError, match="rank 1 fails"):
        T.run_local_ranks(3, body, timeout=120)
