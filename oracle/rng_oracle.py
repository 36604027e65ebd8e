"""Pure-Python restatement of the reference's seeded generator -- TEST
INFRASTRUCTURE ONLY (tests/ may import it; the product never does).

The reference draws slice i of core n from
``Generator(Philox(SeedSequence(seed, spawn_key=(n, i)))).standard_normal``
(core.py:250-253, fill_random_slab core.py:256-266).  The arithmetic lives in
numpy (pinned here: numpy 2.3): this module restates the three published
algorithms numpy implements, step for step, so the device generator
(paper_2011_06532_b200/csrc/rng.cu) has a readable spec to be checked
against, and the restatement itself is pinned to numpy's output and to the
reference's golden vectors in tests/test_rng_oracle.py:

- SeedSequence entropy mixing and generate_state (M. O'Neill's seed_seq
  design as adopted by numpy.random.bit_generator);
- Philox4x64-10 (Salmon, Moraes, Dror, Shaw, SC'11), numpy's counter
  incremented before each 4-word block;
- the 256-strip ziggurat of Generator.standard_normal (Marsaglia & Tsang
  2000) with the tables of paper_2011_06532_b200/csrc/zig_tables.cuh.
"""

from __future__ import annotations

import math
import os
import re

M32 = 0xFFFFFFFF
M64 = (1 << 64) - 1
INIT_A, MULT_A = 0x43B0D7E5, 0x931E8875
INIT_B, MULT_B = 0x8B51F9DD, 0x58F38DED
MIX_L, MIX_R = 0xCA01F9DD, 0x4973F715
PH_M0, PH_M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
PH_W0, PH_W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B

TABLES = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "paper_2011_06532_b200", "csrc", "zig_tables.cuh")


def words32(x: int) -> list:
    """Non-negative int -> little-endian uint32 words (0 -> [0])."""
    out = [x & M32]
    x >>= 32
    while x:
        out.append(x & M32)
        x >>= 32
    return out


def _hashmix(v, hc):
    v = (v ^ hc[0]) & M32
    hc[0] = (hc[0] * MULT_A) & M32
    v = (v * hc[0]) & M32
    return v ^ (v >> 16)


def _mix(x, y):
    r = (MIX_L * x - MIX_R * y) & M32
    return r ^ (r >> 16)


def seed_pool(seed: int, spawn_key=()) -> list:
    """SeedSequence(seed, spawn_key).pool (4 uint32 words)."""
    run = words32(seed)
    spawn = [w for k in spawn_key for w in words32(k)]
    if spawn and len(run) < 4:
        run = run + [0] * (4 - len(run))
    ent = run + spawn
    hc = [INIT_A]
    pool = [_hashmix(ent[i] if i < len(ent) else 0, hc) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = _mix(pool[d], _hashmix(pool[s], hc))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = _mix(pool[d], _hashmix(ent[s], hc))
    return pool


def generate_state_u64(pool, n_words: int) -> list:
    """SeedSequence.generate_state(n_words, np.uint64)."""
    hc = INIT_B
    w32 = []
    for i in range(2 * n_words):
        v = pool[i % 4] ^ hc
        hc = (hc * MULT_B) & M32
        v = (v * hc) & M32
        w32.append(v ^ (v >> 16))
    return [w32[2 * i] | (w32[2 * i + 1] << 32) for i in range(n_words)]


def philox4x64_10(ctr, key) -> list:
    c, k = list(ctr), list(key)
    for r in range(10):
        p0, p1 = PH_M0 * c[0], PH_M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & M64, (p0 >> 64) ^ c[3] ^ k[1], p0 & M64]
        if r < 9:
            k = [(k[0] + PH_W0) & M64, (k[1] + PH_W1) & M64]
    return c


def raw_stream(seed: int, spawn_key=()):
    """The uint64 stream of Philox(SeedSequence(seed, spawn_key))."""
    key = generate_state_u64(seed_pool(seed, spawn_key), 2)
    ctr = 0
    while True:
        ctr = (ctr + 1) & M64  # the 256-bit counter never carries in practice
        yield from philox4x64_10([ctr, 0, 0, 0], key)


def load_tables(path: str = TABLES):
    """(w, k, f, r, rinv) parsed from the generated CUDA header."""
    src = open(path).read()

    def block(name):
        return src.split(name + "[256] = {")[1].split("};")[0]

    fl = lambda s: [float.fromhex(t) for t in re.findall(r"0x[0-9a-f.]+p[-+]\d+", s)]
    w, f = fl(block("kZigW")), fl(block("kZigF"))
    k = [int(t, 16) for t in re.findall(r"0x([0-9a-f]+)ull", block("kZigK"))]
    r = float.fromhex(re.search(r"kZigR = (\S+);", src).group(1))
    rinv = float.fromhex(re.search(r"kZigRinv = (\S+);", src).group(1))
    assert len(w) == len(k) == len(f) == 256
    return w, k, f, r, rinv


def standard_normal(stream, n: int, tables) -> list:
    """n draws of Generator.standard_normal from a raw uint64 stream."""
    w, k, f, r, rinv = tables
    nd = lambda: (next(stream) >> 11) * (1.0 / 9007199254740992.0)
    out = []
    while len(out) < n:
        while True:
            u = next(stream)
            idx = u & 0xFF
            u >>= 8
            m = (u >> 1) & 0x000FFFFFFFFFFFFF
            x = float(m) * w[idx]
            if u & 1:
                x = -x
            if m < k[idx]:
                out.append(x)
                break
            if idx == 0:  # exponential tail beyond r; log1p from the host libm
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
    return out


def slice_normals(seed: int, n: int, i: int, count: int, tables=None) -> list:
    """The draws of slice i of core n (core.py:250-266)."""
    return standard_normal(raw_stream(seed, (n, i)), count, tables or load_tables())
