"""TT files (TTPAR1) -- drop-in for ttpar's save_tt / load_tt (core.py:364-398)
plus the distributed form that moves each rank's slabs straight between the
file and HBM (``load_tt_dist`` / ``save_tt_dist``, native ttb_read_slabs /
ttb_write_slabs: page-locked double buffering, host pread/pwrite overlapped
with the copy engine, every rank touching only its own slice runs).

Layout: b"TTPAR1", little-endian u64 N, dims[N], ranks[N+1], then each core's
raw little-endian f8 entries in F order (r_left, dim, r_right).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .errors import ShapeError
from .tensor import DistTTTensor, TTCore, TTTensor, block_bounds, check_chain, f_empty

MAGIC = b"TTPAR1"


def _header_bytes(dims, ranks):
    return MAGIC + np.array((len(dims),) + tuple(dims) + tuple(ranks), dtype="<u8").tobytes()


def data_offset(ndim: int) -> int:
    return len(MAGIC) + 8 * (1 + ndim + ndim + 1)


def save_tt(path, t) -> None:
    """Write a TT tensor: magic, u64 header (N, dims, ranks), raw f8 cores
    (core.py:364-372).  A DistTTTensor is written by all its ranks in
    parallel (save_tt_dist)."""
    if isinstance(t, DistTTTensor):
        save_tt_dist(path, t)
        return
    with open(path, "wb") as f:
        f.write(_header_bytes(t.dims, t.ranks))
        for c in t.cores:
            f.write(np.ascontiguousarray(c.array.ravel(order="F"), dtype="<f8").tobytes())


def read_header(path):
    """(dims, ranks, data offset, file size) of a TTPAR1 file, validated as
    load_tt does (core.py:375-387)."""
    with open(path, "rb") as f:
        magic = f.read(len(MAGIC))
        if magic != MAGIC:
            raise ShapeError(f"{path!r} is not a TT file (bad magic {magic!r})")
        raw = f.read(8)
        if len(raw) != 8:
            raise ShapeError("TT file header truncated")
        ndim = int(np.frombuffer(raw, dtype="<u8")[0])
        if ndim < 1:
            raise ShapeError("TT file header declares zero modes")
        raw = f.read(8 * (2 * ndim + 1))
        if len(raw) != 8 * (2 * ndim + 1):
            raise ShapeError("TT file header truncated")
        vals = np.frombuffer(raw, dtype="<u8").astype(int)
        dims, ranks = check_chain(vals[:ndim], vals[ndim:])
    return dims, ranks, data_offset(ndim), os.path.getsize(path)


def _payload_end(dims, ranks):
    return data_offset(len(dims)) + 8 * sum(ranks[n] * dims[n] * ranks[n + 1] for n in range(len(dims)))


def load_tt(path) -> TTTensor:
    """Read a TT tensor written by `save_tt` (bitwise round trip, core.py:375-398)."""
    dims, ranks, off, size = read_header(path)
    cores = []
    with open(path, "rb") as f:
        f.seek(off)
        for k in range(len(dims)):
            count = ranks[k] * dims[k] * ranks[k + 1]
            raw = f.read(8 * count)
            if len(raw) != 8 * count:
                raise ShapeError(f"TT file truncated in core {k}")
            flat = np.frombuffer(raw, dtype="<f8").copy()
            cores.append(TTCore(flat.reshape((ranks[k], dims[k], ranks[k + 1]), order="F")))
        if f.read(1):
            raise ShapeError("trailing bytes after last core")
    return TTTensor(cores)


def load_tt_dist(path, comm=None) -> DistTTTensor:
    """This rank's block_bounds slices of every core of a TTPAR1 file, read
    straight into HBM (the distributed counterpart of load_tt)."""
    from .comm import default_comm

    comm = default_comm() if comm is None else comm
    dims, ranks, off, size = read_header(path)
    end = _payload_end(dims, ranks)
    if size < end:
        raise ShapeError("TT file truncated")
    if size > end:
        raise ShapeError("trailing bytes after last core")
    lo, hi, slabs = [], [], []
    for n, d in enumerate(dims):
        a, b = block_bounds(d, comm.size, comm.rank)
        lo.append(a)
        hi.append(b)
        slabs.append(f_empty(ranks[n], b - a, ranks[n + 1], comm.device))
    lib = _lib.load()
    _lib.check(lib.ttb_read_slabs(comm.ctx(), os.fsencode(str(path)), off, len(dims), _lib.i64_array(dims),
                                  _lib.i64_array(ranks), _lib.i64_array(lo), _lib.i64_array(hi),
                                  _lib.ptr_array([s.data_ptr() for s in slabs])))
    return DistTTTensor(comm, dims, ranks, slabs)


def save_tt_dist(path, dt: DistTTTensor) -> None:
    """Rank 0 writes the header and sizes the file; then every rank writes
    its own slice runs in place (no gather)."""
    comm = dt.comm
    if comm.rank == 0:
        with open(path, "wb") as f:
            f.write(_header_bytes(dt.dims, dt.ranks))
            f.truncate(_payload_end(dt.dims, dt.ranks))
    comm.barrier()
    lo, hi = zip(*(dt.local_bounds(n) for n in range(dt.ndim)))
    lib = _lib.load()
    _lib.check(lib.ttb_write_slabs(comm.ctx(), os.fsencode(str(path)), data_offset(dt.ndim), dt.ndim,
                                   _lib.i64_array(dt.dims), _lib.i64_array(dt.ranks), _lib.i64_array(lo),
                                   _lib.i64_array(hi), _lib.ptr_array([s.data_ptr() for s in dt.local])))
    comm.barrier()
