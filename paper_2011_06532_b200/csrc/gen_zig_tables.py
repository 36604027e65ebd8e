"""Generate zig_tables.cuh: the 256-level ziggurat tables that numpy's
Generator.standard_normal uses, so the device generator (rng.cu) reproduces
the reference's seeded inputs bit for bit (core.py:250-266 draws every core
slice with Generator(Philox(SeedSequence(seed, spawn_key=(n, i))))
.standard_normal).

    python paper_2011_06532_b200/csrc/gen_zig_tables.py   (build-time tool, needs numpy)

The method is Marsaglia & Tsang's ziggurat ("The Ziggurat Method for
Generating Random Variables", JSS 2000) with 256 strips and 52-bit
mantissas: a draw u (uint64) picks strip idx = u & 0xff, a sign bit and a
52-bit magnitude m; x = m * w[idx] is returned when m < k[idx]; otherwise
the wedge test against f = exp(-x^2/2) (strips 1..255) or the exponential
tail beyond r (strip 0) decides.  Strip edges x_i satisfy
x_i (f(x_{i-1}) - f(x_i)) = v; w[i] = x_i / 2^52, k[i] = floor(2^52 x_{i-1}/x_i),
f[i] = f(x_i).

The exact bits of numpy's w[] are not reproduced by solving the edge
recursion in either double or 50-digit arithmetic (the recursion amplifies
the last bits of r and v differently per method), so this script MEASURES
them: whenever a fresh stream's first draw u is accepted (fast path or
wedge), standard_normal() == +-m * w[idx] exactly; intersecting the doubles
consistent with a few such draws per strip pins every w[idx] to one value.  k[] and f[] are then derived from the measured
edges (k and f only steer accept/reject decisions, where a last-bit
difference could matter only at an exact tie).  r = x_255 and 1/r come from
the same edges.  The script re-checks the tables against numpy on a few
hundred thousand draws before writing the header.
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "zig_tables.cuh")
M52 = 2.0 ** 52


def first_draws(n_streams, key):
    """(raw uint64 of draw 0, standard_normal() of a fresh stream) pairs."""
    for s in range(n_streams):
        ss = np.random.SeedSequence(20201111, spawn_key=(key, s))
        u = int(np.random.Philox(ss).random_raw(1)[0])
        z = float(np.random.Generator(np.random.Philox(ss)).standard_normal(1)[0])
        yield u, z


def split(u):
    idx = u & 0xFF
    u >>= 8
    return idx, u & 1, (u >> 1) & 0x000FFFFFFFFFFFFF


def consistent(m, z):
    """Doubles w within two ulps of |z|/m with fl(m * w) == |z|."""
    c = abs(z) / m
    lo = [c]
    for _ in range(2):
        lo.append(float(np.nextafter(lo[-1], -np.inf)))
    hi = [c]
    for _ in range(2):
        hi.append(float(np.nextafter(hi[-1], np.inf)))
    return {w for w in lo + hi if float(m) * w == abs(z)}


def approx_edges():
    """Double-precision edge recursion (good to a few hundred ulps) used only
    to tell draws returned from the first uint64 apart from the rest."""
    r = 3.6541528853610088
    f = lambda t: math.exp(-0.5 * t * t)
    v = r * f(r) + math.sqrt(math.pi / 2) * math.erfc(r / math.sqrt(2))
    x = [0.0] * 256
    x[255] = r
    for i in range(254, 0, -1):
        x[i] = math.sqrt(-2.0 * math.log(v / x[i + 1] + f(x[i + 1])))
    x[0] = v / f(r)  # pseudo-width of the base strip (rectangle + tail)
    return x


def measure_w():
    """A fresh stream's first output equals +-m * w[idx] of its first uint64
    whenever that draw is accepted (fast path or wedge); a rejected draw
    returns a value unrelated to m * w[idx], which the 1e-10 closeness test
    to the approximate edge filters out."""
    x = approx_edges()
    cand = {}
    for key in range(1, 40):
        for u, z in first_draws(20000, key):
            idx, _, m = split(u)
            if m == 0 or abs(abs(z) / m / (x[idx] / M52) - 1.0) > 1e-10:
                continue
            c = consistent(m, z)
            cand[idx] = cand[idx] & c if idx in cand else c
        if len(cand) == 256 and all(len(c) == 1 for c in cand.values()):
            break
    bad = [i for i in range(256) if len(cand.get(i, ())) != 1]
    if bad:
        raise SystemExit(f"could not pin w[] for strips {bad}")
    return [next(iter(cand[i])) for i in range(256)]


def derive(w):
    x = [wi * M52 for wi in w]  # exact: scaling by a power of two
    k = [0] * 256
    k[0] = int((x[255] / x[0]) * M52)
    for i in range(2, 256):
        k[i] = int((x[i - 1] / x[i]) * M52)
    f = [1.0] + [math.exp(-0.5 * x[i] * x[i]) for i in range(1, 256)]
    return k, f, x[255], 1.0 / x[255]


def normals(raw, n, w, k, f, r, rinv):
    """The ziggurat draw loop over a raw uint64 stream (Python restatement,
    used only for the self-check below)."""
    it = iter(raw)
    nd = lambda: (int(next(it)) >> 11) * (1.0 / 9007199254740992.0)
    out = []
    while len(out) < n:
        while True:
            idx, sign, m = split(int(next(it)))
            x = float(m) * w[idx]
            if sign:
                x = -x
            if m < k[idx]:
                out.append(x)
                break
            if idx == 0:
                while True:
                    xx = -rinv * math.log1p(-nd())
                    yy = -math.log1p(-nd())
                    if yy + yy > xx * xx:
                        out.append(-(r + xx) if (m >> 8) & 1 else r + xx)
                        break
                break
            if (f[idx - 1] - f[idx]) * nd() + f[idx] < math.exp(-0.5 * x * x):
                out.append(x)
                break
    return np.array(out)


def self_check(w, k, f, r, rinv, streams=40, n=8000):
    for s in range(streams):
        ss = np.random.SeedSequence(77, spawn_key=(s, 3))
        raw = np.random.Philox(ss).random_raw(3 * n)
        ref = np.random.Generator(np.random.Philox(ss)).standard_normal(n)
        got = normals(raw, n, w, k, f, r, rinv)
        if not np.array_equal(ref, got):
            j = int(np.nonzero(ref != got)[0][0])
            raise SystemExit(f"self-check failed: stream {s} draw {j}: {ref[j]!r} vs {got[j]!r}")


def main():
    w = measure_w()
    k, f, r, rinv = derive(w)
    self_check(w, k, f, r, rinv)
    lines = [
        "// GENERATED by gen_zig_tables.py -- do not edit.",
        "// 256-strip ziggurat tables of numpy's Generator.standard_normal:",
        "// w measured from numpy draws, k and f derived from the measured edges.",
        "#pragma once",
                "",
        "namespace ttb {",
        f"constexpr double kZigR = {r.hex()};     // {r!r}",
        f"constexpr double kZigRinv = {rinv.hex()};  // {rinv!r}",
        "__device__ const double kZigW[256] = {",
    ]
    lines += ["    " + ", ".join(v.hex() for v in w[i:i + 4]) + "," for i in range(0, 256, 4)]
    lines += ["};", "__device__ const unsigned long long kZigK[256] = {"]
    lines += ["    " + ", ".join("0x%013xull" % v for v in k[i:i + 4]) + "," for i in range(0, 256, 4)]
    lines += ["};", "__device__ const double kZigF[256] = {"]
    lines += ["    " + ", ".join(v.hex() for v in f[i:i + 4]) + "," for i in range(0, 256, 4)]
    lines += ["};", "}  // namespace ttb", ""]
    with open(OUT, "w") as fh:
        fh.write("\n".join(lines))
    print(OUT)


if __name__ == "__main__":
    sys.exit(main())
