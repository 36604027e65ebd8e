"""GPU parity at the BASELINE configurations' full sizes.

Full-size runs cannot be checked element-wise against the CPU oracle in
seconds, so they assert size-independent properties (rank recovery of an
exactly low-rank sum, norm preservation under orthonormalization, the three
norm routes agreeing, symmetry of the Gram sweep, the max_rank cap); the
same shapes at reduced mode sizes are compared with the oracle directly.
Inputs are the reference's own seeded cores (random_tt(dims, ranks, seed)),
drawn on the device bitwise equal to the host generator (§8(f) row 1).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2011_06532_b200 as T  # noqa: E402
from oracle import tt_oracle as O  # noqa: E402

TOL_TT = 1e-10


def dev_random(dims, ranks, seed):
    """The reference's random_tt(dims, ranks, seed), drawn on the device."""
    return T.DistTTTensor.random(T.default_comm(), dims, ranks, seed)


def dev(cores):
    return T.serial_tt(T.TTTensor(cores))


def host(dt):
    return [c.array for c in T.gather(dt).cores]


def inner_err(a, b):
    """||a - b|| / ||b|| by the Gram route (any ranks; ~1e-8 floor)."""
    aa, bb, ab = T.inner_product(a, a), T.inner_product(b, b), T.inner_product(a, b)
    return np.sqrt(max(aa + bb - 2.0 * ab, 0.0) / bb)


def free():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


# ---- cfg2: Gram sweep and orthonormalization, d=16, n=100000, r=16 ----------

def test_cfg2_full_gram_and_orthonormalize():
    dims, r = (100_000,) * 16, (1,) + (16,) * 15 + (1,)
    x, z = dev_random(dims, r, 0), dev_random(dims, r, 1)
    xz, zx = T.inner_product(x, z), T.inner_product(z, x)
    assert xz == pytest.approx(zx, rel=1e-12, abs=1e-12 * np.sqrt(T.inner_product(x, x) * T.inner_product(z, z)))
    n_ip = T.norm(x, "innerprod")
    n_sym = T.norm(x, "innerprod_sym")
    n_or = T.norm(x, "ortho")
    assert n_sym == pytest.approx(n_ip, rel=1e-12)
    assert n_or == pytest.approx(n_ip, rel=1e-10)
    for direction, end in (("left", -1), ("right", 0)):
        o = T.orthonormalize(x, direction)
        core = o.local[end]
        assert float(torch.linalg.vector_norm(core)) == pytest.approx(n_or, rel=1e-12)
        mid = o.local[7]
        rl, d, rr = mid.shape
        if direction == "left":
            v = mid.permute(2, 1, 0).reshape(rr, d * rl)  # rows = V(X)^T
            g = v @ v.T
        else:
            h = mid.permute(0, 2, 1).reshape(rl, rr * d)  # H(X) with the (i, c) columns permuted
            g = h @ h.T
        assert torch.allclose(g, torch.eye(g.shape[0], dtype=g.dtype, device=g.device), atol=1e-12)
        del o
    del x, z
    free()


def test_cfg2_reduced_vs_oracle():
    dims, r = (2000,) * 16, (1,) + (16,) * 15 + (1,)
    x, z = O.random_cores(dims, r, 0), O.random_cores(dims, r, 1)
    dx, dz = dev(x), dev(z)
    assert T.inner_product(dx, dz) == pytest.approx(O.inner(x, z), rel=1e-12)
    for method in ("innerprod", "innerprod_sym", "ortho"):
        assert T.norm(dx, method) == pytest.approx(O.norm(x, method), rel=1e-12)
    for direction in ("left", "right"):
        got = host(T.orthonormalize(dx, direction))
        assert O.rel_diff(got, O.orthonormalize(x, direction)) < TOL_TT


# ---- cfg3: rounding d=10, n=8000, X = Y + Y (ranks 60 -> 30) -----------------

def test_cfg3_full_rank_recovery():
    dims, ry = (8000,) * 10, (1,) + (30,) * 9 + (1,)
    y = dev_random(dims, ry, 0)
    x = T.add(y, y)
    out = T.round_tt(x, T.RoundingOptions(1e-10))
    assert out.ranks == ry
    assert not out.meta["error_bound_violated"]
    assert inner_err(out, T.scale(y, 2.0)) < 1e-6
    del x, y, out
    free()


def test_cfg3_reduced_vs_oracle():
    dims, ry = (300,) * 10, (1,) + (30,) * 9 + (1,)
    y = O.random_cores(dims, ry, 0)
    x = O.add(y, y)
    ref, meta = O.round_tt(x, 1e-10, "LRLI")
    out = T.round_tt(dev(x), T.RoundingOptions(1e-10))
    assert out.ranks == O.ranks_of(ref) == ry
    assert O.rel_diff(host(out), ref) < TOL_TT
    assert out.meta["norm"] == pytest.approx(meta["norm"], rel=1e-12)


# ---- cfg4: X = 1.0 Y + 0.5 Z - 0.25 Y, dims [2^24, 64^4, 2^20], 60 -> 40 -------

def test_cfg4_full_rank_recovery():
    dims = (1 << 24, 64, 64, 64, 64, 1 << 20)
    r = (1,) + (20,) * 5 + (1,)
    y, z = dev_random(dims, r, 0), dev_random(dims, r, 1)
    x = T.add_n([y, z, y], [1.0, 0.5, -0.25])
    assert x.ranks == (1,) + (60,) * 5 + (1,)
    out = T.round_tt(x, T.RoundingOptions(1e-8))
    assert out.ranks == (1,) + (40,) * 5 + (1,)
    w = T.add_n([y, z], [0.75, 0.5])
    assert inner_err(out, w) < 1e-6
    del x, y, z, w, out
    free()


def test_cfg4_reduced_vs_oracle():
    dims = (1 << 12, 64, 64, 64, 64, 1 << 10)
    r = (1,) + (20,) * 5 + (1,)
    y, z = O.random_cores(dims, r, 0), O.random_cores(dims, r, 1)
    x = O.add(O.add(y, O.scale(z, 0.5)), O.scale(y, -0.25))
    ref, meta = O.round_tt(x, 1e-8, "LRLI")
    dx = T.add_n([dev(y), dev(z), dev(y)], [1.0, 0.5, -0.25])
    assert all(np.array_equal(a, b) for a, b in zip(host(dx), x))  # fused N-ary add: bitwise
    out = T.round_tt(dx, T.RoundingOptions(1e-8))
    assert out.ranks == O.ranks_of(ref)
    assert O.rel_diff(host(out), ref) < TOL_TT


# ---- cfg5: X o W, d=12, n=50000, r=8 -> 64, round(max_rank=32, eps0=0) --------

def test_cfg5_full_hadamard_cap():
    dims, r = (50_000,) * 12, (1,) + (8,) * 11 + (1,)
    x, w = dev_random(dims, r, 0), dev_random(dims, r, 1)
    p = T.hadamard(x, w)
    assert p.ranks == (1,) + (64,) * 11 + (1,)
    # <X o W, X o W> = sum over entries of x^2 w^2 = <X o X, W o W> (ranks 64)
    pp = T.inner_product(p, p)
    assert pp == pytest.approx(T.inner_product(T.hadamard(x, x), T.hadamard(w, w)), rel=1e-10)
    out = T.round_tt(p, T.RoundingOptions(0.0, "LRLI", max_rank=32))
    assert out.ranks == (1,) + (32,) * 11 + (1,)
    assert out.meta["error_bound_violated"]
    assert out.meta["norm"] == pytest.approx(np.sqrt(pp), rel=1e-8)
    del x, w, p, out
    free()


def test_cfg5_reduced_vs_oracle():
    dims, r = (400,) * 12, (1,) + (8,) * 11 + (1,)
    x, w = O.random_cores(dims, r, 0), O.random_cores(dims, r, 1)
    p = O.hadamard(x, w)
    dp = T.hadamard(dev(x), dev(w))
    assert all(np.array_equal(a, b) for a, b in zip(host(dp), p))
    ref, meta = O.round_tt(p, 0.0, "LRLI", 32)
    out = T.round_tt(dp, T.RoundingOptions(0.0, "LRLI", max_rank=32))
    assert out.ranks == O.ranks_of(ref)
    assert out.meta["error_bound_violated"] == meta["error_bound_violated"] is True
    assert O.rel_diff(host(out), ref) < TOL_TT
