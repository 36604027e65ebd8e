"""GPU vs CPU oracle at the BASELINE configurations' FULL sizes.

The north-star bar (BASELINE.json): on the same seeded inputs the truncated
ranks are identical, ||X_gpu - X_ref|| / ||X_ref|| <= 1e-10 computed in TT
form (the orthonormalization route, SURVEY.md finding 3: the inner-product
expansion has a ~1e-8 cancellation floor), and norms / inner products agree
to 1e-12 relative.  Here the device result of every BASELINE config is
compared with the oracle (oracle/tt_oracle.py: the reference's algorithm on
numpy + scipy LAPACK, pinned to the reference's golden vectors) run on the
very same input cores copied to the host.

Reference paths: round_tt parallel.py:293-438; inner_product / norm
ops.py:135-235; orthonormalize parallel.py:164-209; BASELINE.md section 4
step 7 (the parity procedure these tests follow).

cfg4 and cfg5 need tens of GB of host RAM for the oracle (its slab copies,
stored Householder factors and the difference tensor); below the stated
threshold they run at the largest reduced size that fits and print which.
Each test prints the measured errors (run with -s to see them).
"""
import os

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


def avail_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 2**30
    except Exception:  # pragma: no cover
        return 0.0


def report(name, **kv):
    print(f"\n[fullsize] {name}: " + ", ".join(f"{k}={v}" for k, v in kv.items()), flush=True)


def dev_random(dims, ranks, seed):
    """The reference's random_tt(dims, ranks, seed), drawn on the device."""
    return T.DistTTTensor.random(T.default_comm(), dims, ranks, seed)


def host(dt):
    return [c.array for c in T.gather(dt).cores]


def free():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def core_rel(a, b):
    """max over cores of ||a_n - b_n||_F / ||b_n||_F (orthonormalized cores
    are unique once R's diagonal is fixed >= 0 and the panels have full
    column rank, as random N(0,1) panels do)."""
    return max(float(np.linalg.norm(x - y) / np.linalg.norm(y)) for x, y in zip(a, b))


# ---- cfg3: the bench workload (d=10, n=8000, X = Y + Y, ranks 60 -> 30) -----

def test_cfg3_full_vs_oracle():
    dims, ry = (8000,) * 10, (1,) + (30,) * 9 + (1,)
    y = dev_random(dims, ry, 0)
    x = T.add(y, y)
    opts = T.RoundingOptions(1e-10, "LRLI")
    out = T.round_tt(x, opts)
    hx, hy = host(x), host(y)
    del x
    free()
    ref, meta = O.round_tt(hx, 1e-10, "LRLI")
    got = host(out)
    err = O.rel_diff(got, ref)
    err_2y = O.rel_diff(got, O.scale(hy, 2.0))
    ref_2y = O.rel_diff(ref, O.scale(hy, 2.0))
    nrel = abs(out.meta["norm"] - meta["norm"]) / meta["norm"]
    report("cfg3", ranks_gpu=out.ranks[1:-1][:1], ranks_equal=out.ranks == O.ranks_of(ref), rel_err=f"{err:.3e}",
           gpu_vs_2y=f"{err_2y:.3e}", ref_vs_2y=f"{ref_2y:.3e}", norm_rel=f"{nrel:.3e}")
    assert out.ranks == O.ranks_of(ref) == ry
    assert err <= TOL_TT
    assert err_2y <= TOL_TT
    assert nrel <= TOL_SCALAR
    assert out.meta["eps_bond"] == pytest.approx(meta["eps_bond"], rel=TOL_SCALAR)
    del out
    free()


# ---- cfg2: Gram sweep, three norms, orthonormalization (d=16, n=1e5, r=16) --

def test_cfg2_full_scalars_vs_oracle():
    dims, r = (100_000,) * 16, (1,) + (16,) * 15 + (1,)
    x, z = dev_random(dims, r, 0), dev_random(dims, r, 1)
    hx, hz = host(x), host(z)
    got = {"inner": T.inner_product(x, z)}
    for m in ("innerprod", "innerprod_sym", "ortho"):
        got[m] = T.norm(x, m)
    want = {"inner": O.inner(hx, hz)}
    for m in ("innerprod", "innerprod_sym", "ortho"):
        want[m] = O.norm(hx, m)
    rel = {k: abs(got[k] - want[k]) / abs(want[k]) for k in got}
    report("cfg2 scalars", **{k: f"{v:.3e}" for k, v in rel.items()})
    for k in got:
        assert rel[k] <= TOL_SCALAR, (k, got[k], want[k])
    del x, z
    free()


@pytest.mark.parametrize("direction", ["left", "right"])
def test_cfg2_full_orthonormalize_vs_oracle(direction):
    dims, r = (100_000,) * 16, (1,) + (16,) * 15 + (1,)
    x = dev_random(dims, r, 0)
    hx = host(x)
    o = T.orthonormalize(x, direction)
    del x
    got = host(o)
    del o
    free()
    ref = O.orthonormalize(hx, direction)
    crel = core_rel(got, ref)
    err = O.rel_diff(got, ref)
    report(f"cfg2 orthonormalize {direction}", max_core_rel=f"{crel:.3e}", rel_err=f"{err:.3e}")
    assert err <= TOL_TT
    assert crel <= TOL_TT


# ---- cfg4: one huge mode, X = 1.0 Y + 0.5 Z - 0.25 Y, ranks 60 -> 40 ---------

def cfg4_dims():
    """Full size when the host can hold the oracle's working set (~60 GB),
    else the largest power-of-two reduction of the two long modes that fits."""
    full = (1 << 24, 64, 64, 64, 64, 1 << 20)
    need = 64.0  # GB for the oracle at full size
    shift = 0
    while shift < 6 and avail_gb() < need / (1 << shift):
        shift += 1
    return tuple(d >> shift if d > 64 else d for d in full), shift


def test_cfg4_vs_oracle():
    dims, shift = cfg4_dims()
    r = (1,) + (20,) * 5 + (1,)
    y, z = dev_random(dims, r, 0), dev_random(dims, r, 1)
    x = T.add_n([y, z, y], [1.0, 0.5, -0.25])
    out = T.round_tt(x, T.RoundingOptions(1e-8))
    got = host(out)
    hx = host(x)
    del x, y, z, out
    free()
    ref, meta = O.round_tt(hx, 1e-8, "LRLI")
    del hx
    err = O.rel_diff(got, ref)
    report("cfg4", dims=dims, full_size=shift == 0, host_avail_gb=f"{avail_gb():.0f}",
           ranks_equal=O.ranks_of(got) == O.ranks_of(ref), rel_err=f"{err:.3e}")
    assert O.ranks_of(got) == O.ranks_of(ref) == (1,) + (40,) * 5 + (1,)
    assert err <= TOL_TT


# ---- cfg5: Hadamard X o W (ranks 64) rounded to max_rank 32 -------------------

def test_cfg5_vs_oracle():
    """Reported, not gated on 1e-10: both
    sides' truncation errors and their difference; ranks must agree.  The
    oracle needs ~10 minutes at the full n = 50000 (its result is recorded in
    profiles/r2_fullsize_parity.txt), so the default run uses the survey's
    n = 5000 and TTB_FULLSIZE=1 selects the full size."""
    n = 50_000 if (os.environ.get("TTB_FULLSIZE") and avail_gb() >= 100) else 5000
    dims, r = (n,) * 12, (1,) + (8,) * 11 + (1,)
    x, w = dev_random(dims, r, 0), dev_random(dims, r, 1)
    p = T.hadamard(x, w)
    out = T.round_tt(p, T.RoundingOptions(0.0, "LRLI", max_rank=32))
    got = host(out)
    hp = host(p)
    del x, w, p, out
    free()
    ref, meta = O.round_tt(hp, 0.0, "LRLI", 32)
    diff = O.rel_diff(got, ref)
    tr_gpu = O.rel_diff(got, hp)
    tr_ref = O.rel_diff(ref, hp)
    report("cfg5", n=n, full_size=n == 50_000, ranks_equal=O.ranks_of(got) == O.ranks_of(ref),
           gpu_vs_ref=f"{diff:.3e}", trunc_err_gpu=f"{tr_gpu:.6e}", trunc_err_ref=f"{tr_ref:.6e}")
    assert O.ranks_of(got) == O.ranks_of(ref) == (1,) + (32,) * 11 + (1,)
    assert meta["error_bound_violated"]
    assert abs(tr_gpu - tr_ref) <= 1e-8 * max(tr_ref, 1e-300)
    assert diff <= 1e-6
