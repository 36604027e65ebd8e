"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north star): ranks identical; TT-form relative error
<= 1e-10 (ortho route, SURVEY finding 3); norms / inner products within
1e-12 relative; add / hadamard / scale bitwise.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2011_06532_b200 as T  # noqa: E402
from oracle import tt_oracle as O  # noqa: E402
from tests._golden import golden, tt  # noqa: E402

TOL_TT = 1e-10      # ||X_gpu - X_ref|| / ||X_ref||, TT form
TOL_SCALAR = 1e-12  # norms and inner products


def dev(cores):
    return T.serial_tt(T.TTTensor(cores))


def host(dt):
    return [c.array for c in T.gather(dt).cores]


def bitwise(xs, ys):
    assert len(xs) == len(ys)
    for a, b in zip(xs, ys):
        assert a.shape == b.shape
        assert np.array_equal(a, b)


def test_library_is_native():
    from paper_2011_06532_b200 import _lib
    before = _lib.launch_counter()
    T.inner_product(dev(tt("gram_z")), dev(tt("gram_w")))
    assert _lib.launch_counter() > before


def test_fp64_peak_probe():
    import ctypes as C
    from paper_2011_06532_b200 import _lib
    a, b = C.c_double(), C.c_double()
    _lib.check(_lib.load().ttb_fp64_peak(C.c_void_p(torch.cuda.current_stream().cuda_stream), C.byref(a), C.byref(b)))
    print(f"fp64 DFMA {a.value:.2f} TF/s, DMMA {b.value:.2f} TF/s")
    assert a.value > 1.0 and b.value > 1.0


def test_add_hadamard_scale_bitwise():
    x, y = tt("pair_x"), tt("pair_y")
    bitwise(host(T.add(dev(x), dev(y))), tt("add_xy"))
    bitwise(host(T.hadamard(dev(x), dev(y))), tt("had_xy"))
    bitwise(host(T.scale(dev(x), -2.5)), tt("scale_x"))
    bitwise(host(T.add_n([dev(x), dev(x), dev(x)], [1.0, 0.5, -0.25])), tt("add3"))
    # host flavour returns host tensors
    hx = T.add(T.TTTensor(x), T.TTTensor(y))
    assert isinstance(hx, T.TTTensor)
    bitwise([c.array for c in hx.cores], tt("add_xy"))


def test_add_single_mode_elementwise():
    x = O.random_cores((6,), (1, 1), 3)
    y = O.random_cores((6,), (1, 1), 4)
    bitwise(host(T.add(dev(x), dev(y))), O.add(x, y))


def test_gram_values():
    g = golden()
    z, w = dev(tt("gram_z")), dev(tt("gram_w"))
    assert T.inner_product(z, w) == pytest.approx(float(g["gram_zw"]), rel=TOL_SCALAR)
    for m, key in (("innerprod", "norm_z_innerprod"), ("innerprod_sym", "norm_z_sym"), ("ortho", "norm_z_ortho")):
        assert T.norm(z, m) == pytest.approx(float(g[key]), rel=TOL_SCALAR)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_inner_random_shapes(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(2, 6))
    dims = tuple(int(v) for v in rng.integers(1, 40, N))
    rx = (1,) + tuple(int(v) for v in rng.integers(1, 17, N - 1)) + (1,)
    ry = (1,) + tuple(int(v) for v in rng.integers(1, 17, N - 1)) + (1,)
    x = O.random_cores(dims, rx, seed)
    y = O.random_cores(dims, ry, seed + 100)
    assert T.inner_product(dev(x), dev(y)) == pytest.approx(O.inner(x, y), rel=1e-12, abs=1e-12)


def test_tsqr_matches_reference():
    g = golden()
    a = g["tsqr_a"]
    fac, r = T.tsqr_factor(a)
    assert np.allclose(r, g["tsqr_r1"], rtol=1e-12, atol=1e-12)
    q = T.tsqr_apply_q(fac, np.eye(7))
    assert np.allclose(q @ r, a, atol=1e-12)
    assert np.allclose(q.T @ q, np.eye(7), atol=1e-12)


@pytest.mark.parametrize("m,b", [(5000, 60), (20000, 64), (3000, 20), (40000, 16), (777, 33), (64, 64), (10, 3)])
def test_tsqr_tall_skinny(m, b):
    rng = np.random.default_rng(m + b)
    a = rng.standard_normal((m, b))
    fac, r = T.tsqr_factor(a)
    r_ref, _ = O.stacked_tsqr([a])
    assert np.allclose(r, r_ref, rtol=1e-11, atol=1e-11 * np.abs(r_ref).max())
    assert (np.diagonal(r) >= 0).all()
    c = rng.standard_normal((b, 5))
    qc = T.tsqr_apply_q(fac, c)
    q = T.tsqr_apply_q(fac, np.eye(b))
    assert np.allclose(q.T @ q, np.eye(b), atol=1e-12)
    assert np.allclose(q @ r, a, atol=1e-11 * np.abs(a).max())
    assert np.allclose(qc, q @ c, atol=1e-12)


def test_tsqr_rank_deficient():
    rng = np.random.default_rng(5)
    base = rng.standard_normal((30000, 30))
    a = np.hstack([base, base])  # exact rank 30
    fac, r = T.tsqr_factor(a)
    q = T.tsqr_apply_q(fac, np.eye(60))
    assert np.allclose(q @ r, a, atol=1e-10)
    s = np.linalg.svd(r, compute_uv=False)
    assert s[29] > 1.0 and s[30] < 1e-10 * s[0]


def test_truncated_svd_matches_reference():
    g = golden()
    f = T.truncated_svd(g["tsvd_a"], 1.5)
    assert np.allclose(f.s, g["tsvd_s"], rtol=1e-13)
    assert f.discarded_tail == pytest.approx(float(g["tsvd_tail"]), rel=1e-12)
    a = g["tsvd_a"]
    assert np.linalg.norm(a - f.u @ np.diag(f.s) @ f.v.T) <= 1.5 + 1e-12
    f = T.truncated_svd(g["tsvd_a"], 0.0, max_rank=3)
    assert f.capped and np.allclose(f.s, g["tsvd_cap_s"], rtol=1e-13)
    # known answers (test_parallel.py:189-224)
    assert T.truncated_svd(np.diag([2.0, 1.0, 0.0]), 0.0).s.shape == (2,)
    f = T.truncated_svd(np.diag([3.0, 2.0]), 10.0)
    assert f.s.shape == (1,) and f.discarded_tail == pytest.approx(2.0)
    f = T.truncated_svd(np.diag([3.0, 2.0, 1.0]), 0.0, max_rank=2)
    assert f.s.shape == (2,) and f.capped and f.discarded_tail == pytest.approx(1.0)


def test_truncated_svd_wide_and_random():
    rng = np.random.default_rng(4)
    for _ in range(10):
        m, n = (int(v) for v in rng.integers(1, 40, 2))
        a = rng.standard_normal((m, n)) @ np.diag(rng.uniform(0, 3, n))
        s = np.linalg.svd(a, compute_uv=False)
        eps = float(rng.uniform(0, np.linalg.norm(a)))
        f = T.truncated_svd(a, eps)
        tails = [np.sqrt((s[k:] ** 2).sum()) for k in range(s.size + 1)]
        want = next(k for k, tl in enumerate(tails) if tl <= eps)
        assert f.s.size == max(want, 1)
        assert np.allclose(f.s, s[: f.s.size], rtol=1e-12, atol=1e-13)
        assert np.linalg.norm(a - f.u @ np.diag(f.s) @ f.v.T) <= eps + 1e-12


@pytest.mark.parametrize("eps_rel", [0.0, 1e-12, 1e-6])
def test_truncated_svd_rank_deficient_triangle(eps_rel):
    # the R factor of an exactly rank-deficient panel (X = Y + Y): half of
    # its columns are roundoff, which the Jacobi tournament deflates
    rng = np.random.default_rng(9)
    b = rng.standard_normal((4000, 30))
    r = np.linalg.qr(np.hstack([b, b]) @ np.diag(rng.uniform(0.5, 2.0, 60)), mode="r")
    a = r.T
    s = np.linalg.svd(a, compute_uv=False)
    eps = eps_rel * s[0]
    f = T.truncated_svd(a, eps)
    tails = [np.sqrt((s[k:] ** 2).sum()) for k in range(s.size + 1)]
    want = max(next(k for k, tl in enumerate(tails) if tl <= eps), 1)
    if eps_rel > 0:
        assert f.s.size == want == 30
    assert np.allclose(f.s[:30], s[:30], rtol=1e-12)
    assert np.all(f.s[30:] < 1e-13 * s[0])
    assert np.linalg.norm(a - f.u @ np.diag(f.s) @ f.v.T) <= eps + 1e-13 * s[0]


@pytest.mark.parametrize("direction", ["left", "right"])
def test_orthonormalize(direction):
    x = tt("orth_in")
    out = host(T.orthonormalize(dev(x), direction))
    ref = tt(f"orth_{direction}")
    assert O.rel_diff(out, ref) < 1e-12
    N = len(out)
    for n in range(N):
        c = out[n]
        if direction == "right" and n > 0:
            h = c.reshape((c.shape[0], -1), order="F")
            assert np.allclose(h @ h.T, np.eye(h.shape[0]), atol=1e-12)
        if direction == "left" and n < N - 1:
            v = c.reshape((-1, c.shape[2]), order="F")
            assert np.allclose(v.T @ v, np.eye(v.shape[1]), atol=1e-12)


@pytest.mark.parametrize("variant", ["LRLI", "LRL", "RLRI", "RLR"])
def test_round_matches_reference(variant):
    g = golden()
    x = tt("round_in")
    for tag, eps in (("e2", 1e-2), ("e6", 1e-6)):
        out = T.round_tt(dev(x), T.RoundingOptions(eps, variant))
        ref = tt(f"round_{variant}_{tag}")
        assert out.ranks == O.ranks_of(ref)
        assert O.rel_diff(host(out), ref) < TOL_TT
        assert out.meta["norm"] == pytest.approx(float(g[f"round_{variant}_{tag}/norm"]), rel=TOL_SCALAR)
        assert out.meta["eps_bond"] == pytest.approx(float(g[f"round_{variant}_{tag}/eps_bond"]), rel=TOL_SCALAR)
        assert not out.meta["error_bound_violated"]
    out = T.round_tt(dev(tt("round_rr")), T.RoundingOptions(1e-10, variant))
    ref = tt(f"round_{variant}_rr")
    assert out.ranks == O.ranks_of(ref) == O.ranks_of(tt("round_y"))
    assert O.rel_diff(host(out), ref) < TOL_TT
    out = T.round_tt(dev(x), T.RoundingOptions(1e-12, variant, max_rank=2))
    assert out.ranks == O.ranks_of(tt(f"round_{variant}_cap"))
    assert out.meta["error_bound_violated"] == bool(g[f"round_{variant}_cap/violated"])


def test_round_cfg1_small_golden():
    y = O.random_cores((60,) * 8, (1,) + (10,) * 7 + (1,), 0)
    out = T.round_tt(T.add(dev(y), dev(y)), T.RoundingOptions(1e-10))
    ref = tt("cfg1s_out")
    assert out.ranks == O.ranks_of(ref) == O.ranks_of(y)
    assert O.rel_diff(host(out), ref) < TOL_TT
    assert O.rel_diff(host(out), O.scale(y, 2.0)) < TOL_TT


@pytest.mark.parametrize("variant", ["LRLI", "LRL", "RLRI", "RLR"])
def test_round_cfg1_full(variant):
    """BASELINE configs[0]: d=8, n=2000, Y rank 10, X = Y + Y, tol 1e-10."""
    y = O.random_cores((2000,) * 8, (1,) + (10,) * 7 + (1,), 0)
    x = O.add(y, y)
    ref, meta = O.round_tt(x, 1e-10, variant)
    out = T.round_tt(dev(x), T.RoundingOptions(1e-10, variant))
    assert out.ranks == O.ranks_of(ref) == O.ranks_of(y)
    assert O.rel_diff(host(out), ref) < TOL_TT
    assert O.rel_diff(host(out), O.scale(y, 2.0)) < TOL_TT
    assert out.meta["norm"] == pytest.approx(meta["norm"], rel=TOL_SCALAR)


def test_round_orthonormal_output():
    x = O.random_cores((5, 4, 6, 4), (1, 4, 4, 4, 1), 23)
    for variant in ("LRLI", "RLRI"):
        out = host(T.round_tt(dev(x), T.RoundingOptions(1e-8, variant)))
        N = len(out)
        if variant.startswith("R"):
            for n in range(N - 1):
                v = out[n].reshape((-1, out[n].shape[2]), order="F")
                assert np.allclose(v.T @ v, np.eye(v.shape[1]), atol=1e-12)
        else:
            for n in range(1, N):
                h = out[n].reshape((out[n].shape[0], -1), order="F")
                assert np.allclose(h @ h.T, np.eye(h.shape[0]), atol=1e-12)


def test_round_zero_and_single_mode():
    x = [np.zeros_like(c) for c in O.random_cores((4, 5, 4), (1, 3, 3, 1), 2)]
    out = T.round_tt(dev(x), T.RoundingOptions(1e-6, "RLR"))
    assert out.ranks == (1, 1, 1, 1) and out.meta.get("zero") is True
    assert not any(np.any(c) for c in host(out))
    s = O.random_cores((7,), (1, 1), 5)
    out = T.round_tt(dev(s), T.RoundingOptions(1e-6, "RLR"))
    bitwise(host(out), s)


def test_round_eps_zero_bounds():
    t = O.random_cores((3, 4, 3), (1, 5, 7, 1), 17)
    out = T.round_tt(dev(t), T.RoundingOptions(0.0, "RLR"))
    ref, _ = O.round_tt(t, 0.0, "RLR")
    assert out.ranks == O.ranks_of(ref)
    assert O.rel_diff(host(out), t) < 1e-12


@pytest.mark.parametrize("variant", ["LRLI", "LRL", "RLRI", "RLR"])
def test_round_host_matches_device(variant):
    """ttb_round_host (host cores in/out, streamed) runs the same kernels as
    ttb_round: results are bitwise identical, against the golden too."""
    g = golden()
    x = tt("round_in")
    for tag, eps in (("e2", 1e-2), ("e6", 1e-6)):
        opts = T.RoundingOptions(eps, variant)
        dev_out = T.round_tt(dev(x), opts)
        cores, meta = T.round_tt_host(x, opts)  # pageable numpy in / out
        assert meta["output_ranks"] == dev_out.ranks
        bitwise(cores, host(dev_out))
        assert O.rel_diff(cores, tt(f"round_{variant}_{tag}")) < TOL_TT
        assert meta["norm"] == pytest.approx(float(g[f"round_{variant}_{tag}/norm"]), rel=TOL_SCALAR)


def test_round_host_pinned_cfg1():
    """Page-locked torch buffers in and out (the bench e2e path), cfg1 size."""
    y = O.random_cores((2000,) * 8, (1,) + (10,) * 7 + (1,), 0)
    x = O.add(y, y)
    ref, meta_ref = O.round_tt(x, 1e-10, "LRLI")
    hin = [torch.from_numpy(np.asfortranarray(c)).permute(2, 1, 0).contiguous().permute(2, 1, 0).pin_memory()
           for c in x]
    outs = [torch.empty(c.size, dtype=torch.float64).pin_memory() for c in x]
    cores, meta = T.round_tt_host(hin, T.RoundingOptions(1e-10), out=outs)
    assert meta["output_ranks"] == O.ranks_of(ref)
    got = [np.asfortranarray(c.numpy()) for c in cores]
    assert O.rel_diff(got, ref) < TOL_TT
    assert meta["norm"] == pytest.approx(meta_ref["norm"], rel=TOL_SCALAR)


def test_round_host_pageable_multichunk():
    """Pageable numpy cores larger than the 32 MB staging chunk (several ring
    slots per core, in and out): bitwise the device path's result."""
    y = O.random_cores((60, 9000, 50), (1, 24, 24, 1), 7)
    x = O.add(y, y)  # middle core 48 x 9000 x 48 doubles = 166 MB: six chunks
    opts = T.RoundingOptions(1e-9, "LRLI")
    dev_out = T.round_tt(dev(x), opts)
    cores, meta = T.round_tt_host(x, opts)
    assert meta["output_ranks"] == dev_out.ranks == (1, 24, 24, 1)
    bitwise(cores, host(dev_out))


@pytest.mark.parametrize("variant", ["LRLI", "RLRI", "LRL", "RLR"])
def test_round_rank40_to_20_short_end_cores(variant):
    """Ranks 40 -> 20 with short end cores: single-chain panels whose apply
    product has k = 20 columns in an ld-20 staging row (the last n-tile's B
    fragments read past k in the last stage: a regression once faulted here)."""
    y = O.random_cores((300, 4000, 200), (1, 20, 20, 1), 11)
    x = O.add(y, y)
    out = T.round_tt(dev(x), T.RoundingOptions(1e-9, variant))
    ref, _ = O.round_tt(x, 1e-9, variant)
    assert out.ranks == O.ranks_of(ref) == (1, 20, 20, 1)
    assert O.rel_diff(host(out), ref) < TOL_TT


def test_round_host_mixed_pinned_and_pageable():
    """Pageable inputs with page-locked outputs and the reverse (the staged
    and the direct copies share the copy stream): same results."""
    y = O.random_cores((300, 4000, 200), (1, 20, 20, 1), 11)
    x = O.add(y, y)  # middle core 40 x 4000 x 40 doubles = 51 MB: two staging chunks
    opts = T.RoundingOptions(1e-9, "RLRI")
    want = host(T.round_tt(dev(x), opts))
    pinned_out = [torch.empty(c.size, dtype=torch.float64).pin_memory() for c in x]
    cores, meta = T.round_tt_host(x, opts, out=pinned_out)  # pageable in, pinned out
    bitwise([np.asfortranarray(c.numpy() if hasattr(c, "numpy") else c) for c in cores], want)
    pinned_in = [torch.from_numpy(np.asfortranarray(c)).permute(2, 1, 0).contiguous().permute(2, 1, 0).pin_memory()
                 for c in x]
    cores, meta = T.round_tt_host(pinned_in, opts)  # pinned in, pageable out
    bitwise([np.asfortranarray(c.numpy() if hasattr(c, "numpy") else c) for c in cores], want)


def test_round_host_zero_and_single_mode():
    x = [np.zeros_like(c) for c in O.random_cores((4, 5, 4), (1, 3, 3, 1), 2)]
    cores, meta = T.round_tt_host(x, T.RoundingOptions(1e-6, "RLR"))
    assert meta.get("zero") is True and [c.shape for c in cores] == [(1, 4, 1), (1, 5, 1), (1, 4, 1)]
    assert not any(np.any(c) for c in cores)
    s = O.random_cores((7,), (1, 1), 5)
    cores, _ = T.round_tt_host(s, T.RoundingOptions(1e-6, "RLR"))
    bitwise(cores, s)
