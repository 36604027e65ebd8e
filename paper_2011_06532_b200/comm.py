"""Device-group endpoints: the B200 stand-in for ttpar's Communicator
(comm.py:134-160).

One process drives one GPU (torch.distributed launches the ranks).  The
communicator owns the native context (stream binding, NCCL communicator for
the in-kernel-path collectives: the TSQR R allgather and the Gram / norm
allreduces) and offers the host-side collectives the harness needs
(gather of slabs, object exchange) through torch.distributed.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from .errors import CapabilityError, ContractError


class Communicator:
    """Endpoint of a P-rank device group.  ``size``/``rank`` as in ttpar."""

    size = 1
    rank = 0
    # every rank takes part in every exchange (in-process groups rendezvous
    # even with an empty peer list; NCCL ranks without peers skip the call)
    rendezvous = False

    def __init__(self, device=None):
        import torch

        if not torch.cuda.is_available():
            raise CapabilityError("no CUDA device: the B200 path has no CPU fallback")
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise CapabilityError("communicator device must be a CUDA device")
        self._ctx = None
        self.trace = DeviceTrace()

    # -- native context ------------------------------------------------------
    def ctx(self):
        """Native context handle bound to the current torch stream."""
        import torch

        lib = _lib.load()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        if self._ctx is None:
            h = C.c_void_p()
            with torch.cuda.device(self.device):
                _lib.check(lib.ttb_ctx_create(self.device.index, C.c_void_p(stream), C.byref(h)))
            self._ctx = h
            self._init_comm()
        else:
            _lib.check(lib.ttb_ctx_set_stream(self._ctx, C.c_void_p(stream)))
        return self._ctx

    def _init_comm(self):
        _lib.check(_lib.load().ttb_ctx_init_comm(self._ctx, 1, 0, None))

    def empty_cache(self):
        """Hand the library's cached device workspace back to the driver
        (ttb_ctx_trim; the analogue of torch.cuda.empty_cache())."""
        if self._ctx is not None:
            _lib.check(_lib.load().ttb_ctx_trim(self._ctx))

    def close(self):
        if self._ctx is not None:
            _lib.load().ttb_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):  # pragma: no cover - interpreter teardown order varies
        try:
            self.close()
        except Exception:
            pass

    # -- point-to-point exchange of device buffers ---------------------------
    def exchange(self, peers, sends, recvs):
        """Swap device buffers with peers in one grouped NCCL send/recv
        (ttb_exchange): sends[k] (a float64 tensor or None) goes to
        peers[k], recvs[k] (a float64 tensor view, possibly empty) is filled
        from it.  Stream-ordered on the current stream."""
        if not peers and not self.rendezvous:
            return
        lib = _lib.load()
        ctx = self.ctx()
        sp = [0 if t is None else t.data_ptr() for t in sends]
        sn = [0 if t is None else t.numel() for t in sends]
        rp = [t.data_ptr() if t.numel() else 0 for t in recvs]
        rn = [t.numel() for t in recvs]
        _lib.check(lib.ttb_exchange(ctx, len(peers), (C.c_int * max(1, len(peers)))(*peers), _lib.ptr_array(sp),
                                    _lib.i64_array(sn), _lib.ptr_array(rp), _lib.i64_array(rn)))

    # -- host-side collectives (harness / gather) ----------------------------
    def allreduce_sum(self, arr):
        return np.asarray(arr, dtype=np.float64).copy()

    def allgather_object(self, obj):
        return [obj]

    def barrier(self):
        pass


class SerialComm(Communicator):
    """One-rank group on the current device (ttpar SerialComm, comm.py:163-181)."""


class HostGroup:
    """Host-side collectives over a torch.distributed group (any backend,
    gloo included): the harness-level exchange (gather of slabs, object
    broadcast).  Deterministic rank-ascending reductions (comm.py:220-225)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise ContractError("HostGroup needs an initialised torch.distributed process group")
        self.group = group
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allgather_object(self, obj):
        import torch.distributed as dist

        box = [None] * self.size
        dist.all_gather_object(box, obj, group=self.group)
        return box

    def broadcast_object(self, obj, src=0):
        import torch.distributed as dist

        box = [obj]
        dist.broadcast_object_list(box, src=src, group=self.group)
        return box[0]

    def allreduce_sum(self, arr):
        a = np.asarray(arr, dtype=np.float64)
        out = np.zeros_like(a)
        for part in self.allgather_object(a):  # rank-ascending, deterministic
            out = out + part
        return out

    def barrier(self):
        import torch.distributed as dist

        dist.barrier(group=self.group)


class DistComm(Communicator):
    """Rank of a torch.distributed process group, one GPU per process.

    The NCCL communicator the native collectives use is bootstrapped with a
    unique id created on rank 0 and broadcast over the torch group.
    """

    def __init__(self, group=None, device=None):
        import torch

        self.host = HostGroup(group)
        self.group = group
        self.size = self.host.size
        self.rank = self.host.rank
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        super().__init__(device)

    def _init_comm(self):
        lib = _lib.load()
        if self.size == 1:
            _lib.check(lib.ttb_ctx_init_comm(self._ctx, 1, 0, None))
            return
        uid = C.create_string_buffer(128)
        if self.rank == 0:
            _lib.check(lib.ttb_comm_unique_id(uid))
        raw = self.host.broadcast_object(bytes(uid.raw), src=0)
        uid = C.create_string_buffer(raw, 128)
        _lib.check(lib.ttb_ctx_init_comm(self._ctx, self.size, self.rank, uid))

    def allreduce_sum(self, arr):
        return self.host.allreduce_sum(arr)

    def allgather_object(self, obj):
        return self.host.allgather_object(obj)

    def barrier(self):
        self.host.barrier()


class LocalGroup:
    """P ranks inside ONE process, one host thread each (ttb_group): the
    native multi-rank path -- allgathered TSQR triangles and redundant global
    trees, rank-offset applies, allreduced Gram / norm partials, operator halo
    exchanges -- runs with stream-ordered device copies and a host rendezvous
    in place of NCCL, at the same call sites.  The B200 stand-in for the
    reference's thread simulator (SimComm / run_spmd, comm.py:184-356): it
    lets one GPU execute the code a P-GPU job executes.  Reductions are
    rank-ascending sums; a rank that fails breaks the group (DeadlockError
    for its peers instead of a hang)."""

    def __init__(self, size, timeout=300.0):
        if size < 1:
            raise ContractError("group size must be >= 1")
        self.size = size
        self.timeout = timeout
        h = C.c_void_p()
        _lib.check(_lib.load().ttb_group_create(size, C.byref(h)))
        self._h = h
        self._bar = threading.Barrier(size)
        self._box = [None] * size

    def comm(self, rank, device=None):
        return LocalComm(self, rank, device)

    def barrier(self):
        from .errors import DeadlockError

        try:
            self._bar.wait(self.timeout)
        except threading.BrokenBarrierError as e:
            raise DeadlockError("in-process group: a peer failed or timed out") from e

    def abort(self):
        self._bar.abort()
        if self._h is not None:
            _lib.load().ttb_group_abort(self._h)

    def close(self):
        if self._h is not None:
            _lib.load().ttb_group_destroy(self._h)
            self._h = None


class LocalComm(Communicator):
    """Rank ``rank`` of a LocalGroup (ttpar's SimComm endpoint)."""

    rendezvous = True

    def __init__(self, group, rank, device=None):
        if not 0 <= rank < group.size:
            raise ContractError(f"rank {rank} outside a group of {group.size}")
        super().__init__(device)
        self.group = group
        self.size = group.size
        self.rank = rank

    def _init_comm(self):
        _lib.check(_lib.load().ttb_ctx_join_group(self._ctx, self.group._h, self.rank))

    def allgather_object(self, obj):
        g = self.group
        g._box[self.rank] = obj
        g.barrier()
        out = list(g._box)
        g.barrier()
        return out

    def allreduce_sum(self, arr):
        out = None
        for part in self.allgather_object(np.asarray(arr, dtype=np.float64)):  # rank-ascending
            out = part.copy() if out is None else out + part
        return out

    def barrier(self):
        self.group.barrier()


def run_local_ranks(size, fn, device=None, timeout=600.0):
    """Run ``fn(comm)`` for every rank of a fresh ``size``-rank LocalGroup,
    one host thread and one CUDA stream per rank (the run_spmd analogue,
    comm.py:338-356); returns the per-rank results in rank order and
    re-raises the first failure."""
    import torch

    g = LocalGroup(size)
    out, err = [None] * size, []
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

    def run(p):
        comm = None
        try:
            torch.cuda.set_device(dev)
            s = torch.cuda.Stream(dev)
            with torch.cuda.stream(s):
                comm = LocalComm(g, p, dev)
                out[p] = fn(comm)
                s.synchronize()
        except BaseException as e:  # surfaced below
            err.append((p, e))
            g.abort()
        finally:
            if comm is not None:
                comm.close()

    th = [threading.Thread(target=run, args=(p,), daemon=True) for p in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    alive = [t for t in th if t.is_alive()]
    if not alive:
        g.close()
    if err:
        from .errors import DeadlockError

        err.sort(key=lambda pe: isinstance(pe[1], DeadlockError))  # the root cause first
        raise err[0][1]
    if alive:
        from .errors import DeadlockError

        raise DeadlockError(f"{len(alive)} rank thread(s) still running after {timeout} s")
    return out


class DeviceTrace:
    """ttpar's per-rank Trace (comm.py:57-124) for the device path.

    ``reset()`` starts per-kernel-class CUDA-event timing in the native
    library; ``rows()`` / ``total()`` report it in the reference's phases --
    ``TSQR`` (leaf and tree factorisations), ``AppQ`` (implicit-Q applies),
    ``Other`` (folds, SVDs, Gram sweeps, construction) -- with the collective
    traffic of each phase (TSQR: the allgathers of R factors; Other:
    allreduces and operator exchanges).  Seconds are summed device time of
    the kernels, not wall time; flops come from the cost model, not counters.
    """

    PHASE = {"tsqr_leaf": "TSQR", "tsqr_tree": "TSQR", "apply_tree": "AppQ", "apply_chain": "AppQ",
             "apply_product": "AppQ"}

    def __init__(self):
        self._on = False
        self._seconds = {}
        self._flops = {}
        self._base = (0, 0, 0, 0)

    def reset(self):
        _lib.prof_enable(True)
        _lib.prof_dump()
        self._on = True
        self._seconds = {}
        self._flops = {}
        self._base = _lib.comm_stats()

    def freeze(self):
        """Fold the timings recorded so far into the phase totals."""
        if not self._on:
            return
        import torch

        torch.cuda.synchronize()
        for name, (cnt, ms) in _lib.prof_dump().items():
            if name.startswith("svd_sweeps"):
                continue
            ph = self.PHASE.get(name, "Other")
            self._seconds[ph] = self._seconds.get(ph, 0.0) + ms * 1e-3

    def stop(self):
        self.freeze()
        _lib.prof_enable(False)
        self._on = False

    def _traffic(self):
        now = _lib.comm_stats()
        d = [a - b for a, b in zip(now, self._base)]
        return {"TSQR": (float(d[1]), float(d[0])), "Other": (float(d[3]), float(d[2]))}

    def rows(self):
        """``(phase, seconds, flops, words, messages)`` per touched phase."""
        self.freeze()
        traffic = self._traffic()
        phases = sorted(set(self._seconds) | set(self._flops) | {p for p, (w, m) in traffic.items() if m})
        return [(ph, self._seconds.get(ph, 0.0), self._flops.get(ph, 0.0), traffic.get(ph, (0.0, 0.0))[0],
                 traffic.get(ph, (0.0, 0.0))[1]) for ph in phases]

    def total(self, counter):
        idx = {"seconds": 1, "flops": 2, "words": 3, "messages": 4}[counter]
        return float(sum(r[idx] for r in self.rows()))

    def add_flops(self, f, phase="Other"):
        """Cost-model flops of a host-issued operation (the reference's
        tr.add_flops calls, e.g. ops.py:151, 193-201); counted while tracing."""
        if self._on:
            self._flops[phase] = self._flops.get(phase, 0.0) + float(f)


_default = {}


def empty_cache():
    """Release the cached device workspace of every default communicator."""
    for comm in _default.values():
        comm.empty_cache()


def default_comm():
    """Process-wide SerialComm on the current CUDA device."""
    import torch

    if not torch.cuda.is_available():
        raise CapabilityError("no CUDA device: the B200 path has no CPU fallback")
    dev = torch.cuda.current_device()
    if dev not in _default:
        _default[dev] = SerialComm(torch.device("cuda", dev))
    return _default[dev]
