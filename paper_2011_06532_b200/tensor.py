"""TT containers: host-side TTCore/TTTensor (the reference's sequential
containers, core.py:40-131) and the device-resident DistTTTensor whose
per-rank slabs live in HBM (parallel.py:49-111).

Layout contract (core.py:1-23): a core is Fortran-ordered (r_left, dim,
r_right) float64.  On the device a slab is a torch float64 tensor with the
F-order strides (1, r_left, r_left*dim) over a flat buffer, so V(X) and
H(X) are zero-copy column-major views exactly as in the reference and the
native kernels receive a single base pointer per core.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from math import prod

import numpy as np

from .errors import BoundsError, ShapeError

# ----------------------------------------------------------------------------
# block rule and chain validation
# ----------------------------------------------------------------------------


def block_bounds(extent: int, nranks: int, rank: int) -> tuple:
    """Contiguous ceil-sized row block of ``rank`` (parallel.py:42-46)."""
    step = -(-int(extent) // int(nranks))
    lo = min(int(rank) * step, int(extent))
    return lo, min(lo + step, int(extent))


def check_chain(dims, ranks):
    """Validate a (dims, ranks) chain (core.py:236-247)."""
    dims = tuple(int(d) for d in dims)
    ranks = tuple(int(r) for r in ranks)
    if not dims or any(d < 1 for d in dims):
        raise ShapeError(f"dims must be positive, got {dims}")
    if len(ranks) != len(dims) + 1:
        raise ShapeError(f"need {len(dims) + 1} ranks for {len(dims)} modes, got {len(ranks)}")
    if ranks[0] != 1 or ranks[-1] != 1:
        raise ShapeError(f"end ranks must be 1, got {ranks[0]} and {ranks[-1]}")
    if any(r < 1 for r in ranks):
        raise ShapeError(f"ranks must be positive, got {ranks}")
    return dims, ranks


# ----------------------------------------------------------------------------
# host containers
# ----------------------------------------------------------------------------


class TTCore:
    """One 3-way core (r_left, dim, r_right), Fortran-ordered float64 (host)."""

    __slots__ = ("array",)

    def __init__(self, array):
        arr = np.asarray(array, dtype=np.float64)
        if arr.ndim != 3:
            raise ShapeError(f"core must be 3-way, got ndim={arr.ndim}")
        if arr.shape[0] < 1 or arr.shape[2] < 1:
            raise ShapeError(f"core ranks must be positive, got shape {arr.shape}")
        self.array = np.asfortranarray(arr)

    @property
    def r_left(self):
        return self.array.shape[0]

    @property
    def dim(self):
        return self.array.shape[1]

    @property
    def r_right(self):
        return self.array.shape[2]

    def slice(self, i):
        if not 0 <= i < self.dim:
            raise BoundsError(f"slice index {i} out of range [0, {self.dim})")
        return self.array[:, i, :]

    def vertical(self):
        rl, d, rr = self.array.shape
        return self.array.reshape((rl * d, rr), order="F")

    def horizontal(self):
        rl, d, rr = self.array.shape
        return self.array.reshape((rl, d * rr), order="F")

    def copy(self):
        return TTCore(self.array.copy(order="F"))


class TTTensor:
    """A host tensor train: chain of TTCore with matching bond ranks."""

    __slots__ = ("cores",)

    def __init__(self, cores):
        cores = [c if isinstance(c, TTCore) else TTCore(c) for c in cores]
        if not cores:
            raise ShapeError("a TT tensor needs at least one core")
        if cores[0].r_left != 1 or cores[-1].r_right != 1:
            raise ShapeError("end ranks must be 1")
        for k in range(len(cores) - 1):
            if cores[k].r_right != cores[k + 1].r_left:
                raise ShapeError(f"rank mismatch between cores {k} and {k + 1}: "
                                 f"{cores[k].r_right} != {cores[k + 1].r_left}")
        self.cores = cores

    @property
    def ndim(self):
        return len(self.cores)

    @property
    def dims(self):
        return tuple(c.dim for c in self.cores)

    @property
    def ranks(self):
        return (1,) + tuple(c.r_right for c in self.cores)

    def copy(self):
        return TTTensor([c.copy() for c in self.cores])

    def __repr__(self):  # pragma: no cover
        return f"TTTensor(dims={self.dims}, ranks={self.ranks})"


# ----------------------------------------------------------------------------
# seeded generation (core.py:250-282): per-slice Philox, P-invariant
# ----------------------------------------------------------------------------


def slice_rng(seed: int, n: int, i: int) -> np.random.Generator:
    """The dedicated stream of slice i of core n (0-based), core.py:250-253."""
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed, spawn_key=(n, i))))


def fill_random_slab(out: np.ndarray, n: int, lo: int, seed: int) -> None:
    """out[:, k, :] <- stream of global slice lo + k, left rank fastest."""
    rl, d_loc, rr = out.shape
    for k in range(d_loc):
        out[:, k, :] = slice_rng(seed, n, lo + k).standard_normal(rl * rr).reshape((rl, rr), order="F")


def random_tt(dims, ranks, seed: int) -> TTTensor:
    """i.i.d. N(0,1) cores, bitwise equal to the reference's random_tt."""
    dims, ranks = check_chain(dims, ranks)
    cores = []
    for n, d in enumerate(dims):
        arr = np.empty((ranks[n], d, ranks[n + 1]), order="F")
        fill_random_slab(arr, n, 0, seed)
        cores.append(TTCore(arr))
    return TTTensor(cores)


def seed_words(seed) -> list:
    """A non-negative int seed as little-endian uint32 words, numpy's
    SeedSequence entropy coercion (0 -> [0])."""
    import operator

    v = operator.index(seed)
    if v < 0:
        raise ValueError(f"expected non-negative integer seed, got {v}")
    words = [v & 0xFFFFFFFF]
    v >>= 32
    while v:
        words.append(v & 0xFFFFFFFF)
        v >>= 32
    return words


def fill_random_slabs(comm, slabs, cores, lo, seed) -> None:
    """Device form of fill_random_slab (core.py:256-266) for several slabs in
    one call: slabs[k][:, j, :] <- stream of global slice lo[k] + j of core
    cores[k].  Slabs must be F-order float64 on comm's device."""
    import ctypes as C

    from . import _lib

    for t in slabs:
        if not is_f_slab(t) or t.dtype.itemsize != 8 or not t.dtype.is_floating_point:
            raise ShapeError("fill_random_slabs needs F-order float64 device slabs")
    w = seed_words(seed)
    lib = _lib.load()
    _lib.check(lib.ttb_fill_random(
        comm.ctx(), (C.c_uint32 * len(w))(*w), len(w), len(slabs), _lib.i64_array(cores), _lib.i64_array(lo),
        _lib.i64_array([t.shape[0] for t in slabs]), _lib.i64_array([t.shape[1] for t in slabs]),
        _lib.i64_array([t.shape[2] for t in slabs]), _lib.ptr_array([t.data_ptr() for t in slabs])))


# ----------------------------------------------------------------------------
# device slabs
# ----------------------------------------------------------------------------


def f_empty(rl, d, rr, device):
    """Uninitialised F-order (rl, d, rr) float64 slab on the device."""
    import torch

    return torch.empty_strided((rl, d, rr), (1, rl, rl * d), dtype=torch.float64, device=device)


def f_view(flat, rl, d, rr):
    """(rl, d, rr) F-order view over the first rl*d*rr entries of a flat buffer."""
    return flat.as_strided((rl, d, rr), (1, rl, rl * d), 0)


def is_f_slab(t):
    rl, d, rr = t.shape
    if t.numel() == 0:
        return True
    want = (1, rl, rl * d)
    return all(s == w or n == 1 for s, w, n in zip(t.stride(), want, t.shape))


def to_device_slab(a, device):
    """Upload / convert to an F-contiguous float64 device slab."""
    import torch

    if isinstance(a, torch.Tensor):
        t = a.to(device=device, dtype=torch.float64)
        if t.dim() != 3:
            raise ShapeError(f"slab must be 3-way, got ndim={t.dim()}")
        if is_f_slab(t):
            return t
        out = f_empty(*t.shape, device)
        out.copy_(t)
        return out
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 3:
        raise ShapeError(f"slab must be 3-way, got ndim={arr.ndim}")
    out = f_empty(*arr.shape, device)
    if arr.size:
        out.copy_(torch.from_numpy(np.asfortranarray(arr)))
    return out


def to_host_array(t):
    """F-order numpy copy of a device slab."""
    if isinstance(t, np.ndarray):
        return np.asfortranarray(t)
    return np.asfortranarray(t.detach().cpu().numpy())


@dataclass
class DistTTTensor:
    """A TT tensor whose cores are row blocks of one global chain, resident in
    the HBM of this rank's GPU.  ``local[n]`` has shape
    (ranks[n], hi - lo, ranks[n+1]) for this rank's block of mode n
    (parallel.py:49-79)."""

    comm: object
    dims: tuple
    ranks: tuple
    local: list
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        self.dims, self.ranks = check_chain(self.dims, self.ranks)
        if len(self.local) != len(self.dims):
            raise ShapeError(f"{len(self.local)} slabs for {len(self.dims)} modes")
        slabs = []
        for n, slab in enumerate(self.local):
            lo, hi = self.local_bounds(n)
            want = (self.ranks[n], hi - lo, self.ranks[n + 1])
            t = to_device_slab(slab, self.comm.device)
            if tuple(t.shape) != want:
                raise ShapeError(f"mode {n} slab on rank {self.comm.rank} has shape "
                                 f"{tuple(t.shape)}, block rule wants {want}")
            slabs.append(t)
        self.local = slabs

    @property
    def ndim(self):
        return len(self.dims)

    def local_bounds(self, n):
        return block_bounds(self.dims[n], self.comm.size, self.comm.rank)

    def local_dims(self):
        return tuple(hi - lo for lo, hi in (self.local_bounds(n) for n in range(self.ndim)))

    @classmethod
    def random(cls, comm, dims, ranks, seed: int):
        """This rank's slabs straight from the per-slice streams (parallel.py:88-102),
        generated on the device by ttb_fill_random: bitwise equal to
        distribute(random_tt(...)) for every P."""
        dims, ranks = check_chain(dims, ranks)
        slabs, lo = [], []
        for n, d in enumerate(dims):
            a, b = block_bounds(d, comm.size, comm.rank)
            slabs.append(f_empty(ranks[n], b - a, ranks[n + 1], comm.device))
            lo.append(a)
        fill_random_slabs(comm, slabs, list(range(len(dims))), lo, seed)
        return cls(comm, dims, ranks, slabs)

    def copy(self):
        return DistTTTensor(self.comm, self.dims, self.ranks, [s.clone() for s in self.local], dict(self.meta))

    def nbytes(self):
        return sum(int(s.numel()) * 8 for s in self.local)

    def __repr__(self):  # pragma: no cover
        return f"DistTTTensor(P={self.comm.size}, dims={self.dims}, ranks={self.ranks})"
