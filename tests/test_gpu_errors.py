"""The reference's error conventions on the device path (errors.py:4-33):
the same exception classes for the same misuse, mirroring the reference's
own error tests (test_parallel.py:64-97, 355-360; test_ops.py:64-88, 259-263;
test_tsqr.py:80-87)."""
import numpy as np
import pytest
import scipy.sparse as sp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2011_06532_b200 as T  # noqa: E402
from oracle import tt_oracle as O  # noqa: E402


def tt(dims, ranks, seed):
    return T.TTTensor(O.random_cores(dims, ranks, seed))


class ThreeRanks(T.SerialComm):
    """Rank 2 of an emulated 3-rank group (local logic only)."""
    size, rank = 3, 2


def test_nonfinite_inputs_raise_numeric_error():
    x = O.random_cores((6, 5, 7), (1, 3, 4, 1), 1)
    x[1][1, 2, 3] = np.nan
    dx = T.serial_tt(T.TTTensor(x))
    with pytest.raises(T.NumericError):
        T.round_tt(dx, T.RoundingOptions(1e-8))
    for direction in ("left", "right"):
        with pytest.raises(T.NumericError):
            T.orthonormalize(dx, direction)
    a = np.ones((40, 3))
    a[7, 1] = np.inf
    with pytest.raises(T.NumericError):
        T.tsqr_factor(a)
    with pytest.raises(T.NumericError):
        T.truncated_svd(np.full((3, 3), np.nan), 0.1)
    # the context stays usable afterwards
    y = T.serial_tt(tt((6, 5, 7), (1, 3, 4, 1), 2))
    assert T.round_tt(y, T.RoundingOptions(1e-12)).ranks == (1, 3, 4, 1)


def test_rounding_options_contract():
    with pytest.raises(T.ContractError, match="variant"):
        T.RoundingOptions(1e-8, "XYZ")
    with pytest.raises(T.ContractError, match="eps0"):
        T.RoundingOptions(-1.0)
    with pytest.raises(T.ContractError, match="max_rank"):
        T.RoundingOptions(1e-8, max_rank=0)


def test_construction_errors():
    x = tt((4, 5), (1, 2, 1), 7)
    y = tt((4, 6), (1, 2, 1), 8)
    with pytest.raises(T.ShapeError, match="mismatch"):
        T.add(x, y)
    with pytest.raises(T.ShapeError, match="block rule"):
        T.DistTTTensor(T.default_comm(), (3, 3), (1, 2, 1), [np.zeros((1, 3, 2)), np.zeros((2, 2, 1))])
    with pytest.raises(T.ContractError, match="method"):
        T.norm(x, "spectral")
    with pytest.raises(T.ContractError, match="mix"):
        T.add(T.serial_tt(x), x)


def test_hadamard_rank_guard():
    x = tt((4, 4), (1, 70, 1), 5)
    with pytest.raises(T.CapacityError, match="guard"):
        T.hadamard(x, x)
    z = T.hadamard(x, x, max_rank_product=4900)
    assert z.ranks == (1, 4900, 1)
    want = O.hadamard([c.array for c in x.cores], [c.array for c in x.cores], guard=4900)
    for a, b in zip(z.cores, want):
        assert np.array_equal(a.array, b)


def test_distribute_rejects_idle_ranks():
    t = tt((4, 2, 5), (1, 2, 2, 1), 0)
    comm = ThreeRanks()
    with pytest.raises(T.ContractError, match="idle"):
        T.distribute(t, comm)
    dt = T.distribute(t, comm, allow_idle=True)
    assert dt.local_bounds(1) == (2, 2)


def test_rank_capability_limit():
    """ranks above 64 take the general path (tests/test_gpu_wide.py); the
    remaining limit is 4096 columns per TSQR panel, reported loudly."""
    cores = O.random_cores((70, 60, 50), (1, 65, 3, 1), 3)
    out = T.round_tt(T.serial_tt(T.TTTensor(cores)), T.RoundingOptions(1e-8))
    ref, _ = O.round_tt(cores, 1e-8, "LRLI")
    assert tuple(out.ranks) == tuple(O.ranks_of(ref))
    with pytest.raises(T.CapabilityError):
        T.tsqr_factor(np.zeros((10, 4100)))


def test_operator_errors():
    x = tt((4, 5, 4), (1, 2, 2, 1), 30)
    with pytest.raises(T.ShapeError, match="dims"):
        T.apply_operator(T.KroneckerOperator.identity((4, 5, 5)), x)
    with pytest.raises(T.ShapeError):
        T.mode2_multiply(T.TTCore(np.ones((2, 4, 3))), sp.identity(5, format="csr"))


def test_device_trace_phases():
    """comm.trace mirrors ttpar's Trace (comm.py:57-124): per-phase device time
    of the TSQR factorisations, the implicit-Q applies and the rest."""
    comm = T.default_comm()
    y = T.DistTTTensor.random(comm, (300,) * 5, (1, 6, 7, 6, 5, 1), 0)
    x = T.add(y, y)
    comm.trace.reset()
    out = T.round_tt(x, T.RoundingOptions(1e-10))
    rows = {r[0]: r for r in comm.trace.rows()}
    comm.trace.stop()
    assert out.ranks == y.ranks
    assert set(rows) == {"TSQR", "AppQ", "Other"}
    assert all(r[1] > 0 for r in rows.values())
    assert comm.trace.total("messages") == 0.0  # one rank: no collectives
