"""Pin the seeded-generator restatement (oracle/rng_oracle.py) and the
ziggurat tables the device generator compiles in (csrc/zig_tables.cuh)
against numpy -- the library the reference draws with (core.py:250-266) --
and against the reference's own golden cores.  CPU only."""
import numpy as np
import pytest

from oracle import rng_oracle as R
from tests._golden import tt

SEEDS = [0, 7, 42, 2**32 - 1, 2**40 + 3, 2**200 + 12345]
KEYS = [(0, 0), (3, 17), (11, 2**32 - 1), (2, 2**32 + 5), (1, 2**60)]


@pytest.mark.parametrize("seed", SEEDS)
def test_seed_sequence_pool_and_key(seed):
    for key in KEYS:
        ss = np.random.SeedSequence(seed, spawn_key=key)
        assert R.seed_pool(seed, key) == [int(v) for v in ss.pool]
        assert R.generate_state_u64(R.seed_pool(seed, key), 2) == [int(v) for v in ss.generate_state(2, np.uint64)]


@pytest.mark.parametrize("seed", SEEDS[:4])
def test_philox_raw_stream(seed):
    for key in KEYS[:3]:
        bg = np.random.Philox(np.random.SeedSequence(seed, spawn_key=key))
        it = R.raw_stream(seed, key)
        assert [next(it) for _ in range(37)] == [int(v) for v in bg.random_raw(37)]


def test_standard_normal_bitwise_with_tails():
    tab = R.load_tables()
    tails = 0
    for s in range(24):
        ref = np.random.Generator(np.random.Philox(np.random.SeedSequence(5, spawn_key=(s, 1)))).standard_normal(5000)
        got = np.array(R.slice_normals(5, s, 1, 5000, tab))
        assert np.array_equal(ref, got), s
        tails += int(np.sum(np.abs(ref) > tab[3]))
    assert tails > 5  # the exponential-tail branch was exercised


def test_tables_shape():
    w, k, f, r, rinv = R.load_tables()
    assert k[1] == 0 and f[0] == 1.0 and w[255] * 2.0**52 == r and rinv == 1.0 / r
    assert all(w[i] < w[i + 1] for i in range(1, 255)) and all(f[i] > f[i + 1] for i in range(255))


def test_restatement_matches_reference_golden():
    tab = R.load_tables()
    for key, dims, ranks, seed in (("rng_a", (4, 5, 3), (1, 3, 2, 1), 42), ("rng_b", (6, 4), (1, 3, 1), 7)):
        for n, core in enumerate(tt(key)):
            rl, d, rr = core.shape
            assert (rl, d, rr) == (ranks[n], dims[n], ranks[n + 1])
            for i in range(d):
                got = np.array(R.slice_normals(seed, n, i, rl * rr, tab)).reshape((rl, rr), order="F")
                assert np.array_equal(got, core[:, i, :])
