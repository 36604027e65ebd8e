"""CPU checks for the Kronecker-operator apply and the TT file formats
(§8(f) rows 2-3): the oracle against the reference's own outputs, the
exchange-plan host logic of the distributed apply, and the host file
readers / writers against bytes the reference wrote."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import tt_oracle as O
from tests._golden import golden, tt


def lap(d):
    return sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(d, d), format="csr")


def kron_sum_terms(dims):
    terms = []
    for n in range(len(dims)):
        row = [sp.identity(d, format="csr") for d in dims]
        row[n] = lap(dims[n])
        terms.append(row)
    return terms


def shift_terms(dims):
    eye = [sp.identity(d, format="csr") for d in dims]
    shifted = [sp.csr_matrix((np.ones(d), (np.arange(d), (np.arange(d) + 1) % d)), shape=(d, d)) for d in dims]
    return [eye, shifted]


def bitwise(xs, ys):
    assert len(xs) == len(ys)
    for a, b in zip(xs, ys):
        assert a.shape == b.shape and np.array_equal(a, b)


# ---------------------------------------------------------------- oracle pins

def test_oracle_mode2_bitwise():
    g = golden()
    a = sp.csr_matrix(g["m2_a_dense"])
    assert np.array_equal(O.mode2_multiply(g["m2_core"], a), g["m2_out"])


@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_oracle_apply_operator_bitwise(nranks):
    x = tt("op_x")
    got = O.apply_operator(kron_sum_terms((6, 5, 7)), x, nranks=nranks)
    bitwise(got, tt("op_lap"))
    if nranks > 1:
        bitwise(got, tt(f"op_lap_p{nranks}"))


def test_oracle_apply_shift_and_single_mode():
    bitwise(O.apply_operator(shift_terms((6, 5, 7)), tt("op_x")), tt("op_shift"))
    bitwise(O.apply_operator([[lap(8)], [sp.identity(8, format="csr")]], tt("op1_x")), tt("op1_lap"))


def test_oracle_apply_with_rounding():
    got = O.apply_operator(kron_sum_terms((6, 5, 7)), tt("op_x"), round_eps=1e-10)
    ref = tt("op_lap_round")
    assert O.ranks_of(got) == O.ranks_of(ref)
    assert O.rel_diff(got, ref) <= 1e-12


# ---------------------------------------------------- exchange plan (host logic)

def _plan_cases():
    rng = np.random.default_rng(3)
    yield lap(11)
    yield shift_terms((13,))[1][0]
    yield sp.random(17, 17, density=0.2, random_state=4, format="csr")
    yield sp.csr_matrix(rng.standard_normal((9, 9)))
    yield sp.identity(7, format="csr")


@pytest.mark.parametrize("size", [1, 2, 3, 4, 5])
def test_exchange_plan_pairs_and_remap(size):
    from paper_2011_06532_b200.operator import exchange_plan

    rng = np.random.default_rng(size)
    for a in _plan_cases():
        d = a.shape[0]
        if size > d:
            continue
        x = rng.standard_normal((2, d, 3))
        plans = [exchange_plan(a, size, p) for p in range(size)]
        want = O.mode2_multiply(np.asfortranarray(x), a)
        for p, pl in enumerate(plans):
            # q's send list to p is exactly p's receive list from q
            for q, r in pl.recv.items():
                assert np.array_equal(plans[q].send[p] + plans[q].lo, r)
            for q, s in pl.send.items():
                assert np.array_equal(plans[q].recv[p], s + pl.lo)
            # local slices + halo in arrival order, renumbered CSR: same rows, same bits
            halo = [plans[q].lo + plans[q].send[p] for q in sorted(pl.recv)]
            src_idx = np.concatenate([np.arange(pl.lo, pl.hi)] + halo).astype(int)
            src = x[:, src_idx, :]
            m = sp.csr_matrix((pl.vals, pl.cols, pl.indptr), shape=(pl.nloc, src_idx.size))
            got = np.stack([(m @ src[:, :, r].T).T for r in range(src.shape[2])], axis=2)
            assert np.array_equal(got, want[:, pl.lo:pl.hi, :])


def test_exchange_plan_moves_only_coupled_slices():
    """Tridiagonal factor over 4 ranks: only block-boundary slices move
    (test_ops.py:324-346)."""
    from paper_2011_06532_b200.operator import exchange_plan

    plans = [exchange_plan(lap(8), 4, p) for p in range(4)]
    for p, pl in enumerate(plans):
        assert set(pl.recv) == {q for q in (p - 1, p + 1) if 0 <= q < 4}
        assert all(v.size == 1 for v in pl.recv.values())
    ident = [exchange_plan(sp.identity(8, format="csr"), 4, p) for p in range(4)]
    assert all(not pl.send and not pl.recv for pl in ident)


# ---------------------------------------------------------------- host API

def test_operator_validation_and_text_format(tmp_path):
    from paper_2011_06532_b200 import KroneckerOperator, ShapeError, load_operator, save_operator

    with pytest.raises(ShapeError, match="factor"):
        KroneckerOperator((3, 3), [[sp.identity(3), sp.identity(4)]])
    with pytest.raises(ShapeError, match="term"):
        KroneckerOperator((3, 3), [[sp.identity(3)]])
    with pytest.raises(ShapeError, match="at least one"):
        KroneckerOperator((3, 3), [])
    op = KroneckerOperator((4, 3, 5), kron_sum_terms((4, 3, 5)))
    path = tmp_path / "lap.kron"
    save_operator(path, op)
    assert path.read_bytes() == golden()["file_op_bytes"].tobytes()  # the reference's bytes
    back = load_operator(path)
    assert back.dims == (4, 3, 5) and len(back.terms) == 3
    for ta, tb in zip(op.terms, back.terms):
        for fa, fb in zip(ta, tb):
            assert (fa != fb).nnz == 0
    bad = tmp_path / "bad.kron"
    bad.write_text("NOTANOP\n1 1\n3\n")
    with pytest.raises(ShapeError, match="magic"):
        load_operator(bad)
    bad.write_text("KRONOP1\n2 1\n3 3\nfactor 0 0 1\n0 0 1.0\n")
    with pytest.raises(ShapeError):
        load_operator(bad)


def test_tt_file_host_roundtrip_and_reference_bytes(tmp_path):
    from paper_2011_06532_b200 import ShapeError, TTTensor, load_tt, save_tt
    from paper_2011_06532_b200.ttio import read_header

    ref_bytes = golden()["file_tt_bytes"].tobytes()
    t = TTTensor(tt("file_tt"))
    p = tmp_path / "t.tt"
    save_tt(p, t)
    assert p.read_bytes() == ref_bytes
    back = load_tt(p)
    assert back.dims == t.dims and back.ranks == t.ranks
    for a, b in zip(t.cores, back.cores):
        assert np.array_equal(a.array, b.array) and b.array.flags.f_contiguous
    dims, ranks, off, size = read_header(p)
    assert (dims, ranks, size) == ((5, 4, 3), (1, 2, 3, 1), len(ref_bytes)) and off == 6 + 8 * 8
    bad = tmp_path / "bad.tt"
    bad.write_bytes(b"NOTATT" + b"\x00" * 64)
    with pytest.raises(ShapeError):
        load_tt(bad)
    bad.write_bytes(ref_bytes[:-8])
    with pytest.raises(ShapeError):
        load_tt(bad)
    bad.write_bytes(ref_bytes + b"\x00")
    with pytest.raises(ShapeError, match="trailing"):
        load_tt(bad)
