"""Device seeded generation (ttb_fill_random) vs the reference generator:
bitwise, through the C ABI (core.py:250-282, parallel.py:88-102)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2011_06532_b200 as T  # noqa: E402
from oracle import tt_oracle as O  # noqa: E402
from paper_2011_06532_b200.tensor import f_empty, fill_random_slabs  # noqa: E402
from tests._golden import tt  # noqa: E402


def host(dt):
    return [s.cpu().numpy() for s in dt.local]


def same(xs, ys):
    assert len(xs) == len(ys)
    for a, b in zip(xs, ys):
        assert a.shape == b.shape
        assert np.array_equal(a, b)


def test_random_matches_reference_golden():
    comm = T.default_comm()
    same(host(T.DistTTTensor.random(comm, (4, 5, 3), (1, 3, 2, 1), 42)), tt("rng_a"))
    same(host(T.DistTTTensor.random(comm, (6, 4), (1, 3, 1), 7)), tt("rng_b"))


@pytest.mark.parametrize("seed", [0, 7, 2**40 + 3, 2**200 + 12345])
def test_random_matches_host_generator(seed):
    # rl = 70 > the 32-row staging chunk; rl = 1 and rr = 1 edge cores
    dims, ranks = (37, 300, 50, 5), (1, 30, 70, 17, 1)
    same(host(T.DistTTTensor.random(T.default_comm(), dims, ranks, seed)), O.random_cores(dims, ranks, seed))


def test_tail_draws_bitwise():
    # 4.3M draws: ~1000 pass through the exponential tail (host-libm finish)
    comm = T.default_comm()
    slab = f_empty(60, 1200, 60, comm.device)
    fill_random_slabs(comm, [slab], [2], [0], 99)
    ref = np.empty((60, 1200, 60), order="F")
    O.fill_slices(ref, 2, 0, 99)
    got = slab.cpu().numpy()
    assert np.sum(np.abs(ref) > 3.6541528853610088) > 300
    assert np.array_equal(got, ref)


def test_slice_offsets_and_wide_indices():
    comm = T.default_comm()
    lo = 2**32 - 4  # slice indices cross into two spawn-key words
    slabs = [f_empty(3, 8, 2, comm.device), f_empty(1, 5, 4, comm.device), f_empty(2, 0, 2, comm.device)]
    fill_random_slabs(comm, slabs, [3, 0, 1], [lo, 17, 0], 5)
    a = np.empty((3, 8, 2), order="F")
    O.fill_slices(a, 3, lo, 5)
    b = np.empty((1, 5, 4), order="F")
    O.fill_slices(b, 0, 17, 5)
    assert np.array_equal(slabs[0].cpu().numpy(), a)
    assert np.array_equal(slabs[1].cpu().numpy(), b)


def test_block_slabs_are_p_invariant():
    comm = T.default_comm()
    dims, ranks = (9, 70, 33), (1, 4, 6, 1)
    full = host(T.DistTTTensor.random(comm, dims, ranks, 3))
    for P in (2, 3, 8):
        for p in range(P):
            for n, d in enumerate(dims):
                lo, hi = O.block_bounds(d, P, p)
                s = f_empty(ranks[n], hi - lo, ranks[n + 1], comm.device)
                fill_random_slabs(comm, [s], [n], [lo], 3)
                assert np.array_equal(s.cpu().numpy(), full[n][:, lo:hi, :])


def test_negative_seed_rejected():
    with pytest.raises(ValueError):
        T.DistTTTensor.random(T.default_comm(), (3, 3), (1, 2, 1), -1)


def test_cfg3_inputs_round_like_host():
    # a device-generated input rounds exactly like the same input uploaded
    dims, ry = (300,) * 6, (1,) + (12,) * 5 + (1,)
    comm = T.default_comm()
    y = T.DistTTTensor.random(comm, dims, ry, 0)
    same(host(y), O.random_cores(dims, ry, 0))
    out = T.round_tt(T.add(y, y), T.RoundingOptions(1e-10))
    ref = T.round_tt(T.add(T.serial_tt(T.TTTensor(O.random_cores(dims, ry, 0))),
                           T.serial_tt(T.TTTensor(O.random_cores(dims, ry, 0)))), T.RoundingOptions(1e-10))
    assert out.ranks == ref.ranks == ry
    same(host(out), host(ref))
