"""Multi-rank host logic on CPU (gloo, world_size 2): slicing, gather,
P-invariant seeded generation, and the collective compositions the native
driver uses (allgather of TSQR triangles + redundant stacked QR; allreduce of
per-core Gram partials).  The per-rank arithmetic here is the oracle's (test
infrastructure), the multi-rank plumbing is the package's."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import tt_oracle as O
        from paper_2011_06532_b200.comm import HostGroup
        from paper_2011_06532_b200.tensor import block_bounds, fill_random_slab
        from paper_2011_06532_b200.cost import rounding_bytes
        g = HostGroup()
        res = {}
        # 1. collectives: deterministic rank-ascending sums, object gather
        s = g.allreduce_sum(np.array([rank + 0.5, 2.0 * rank]))
        res["allreduce"] = s.tolist()
        res["gather"] = g.allgather_object(("r", rank))
        # 2. P-invariant generation + gather assembly (DistTTTensor.random)
        dims, ranks = (7, 5, 9), (1, 3, 4, 1)
        mine = []
        for n, d in enumerate(dims):
            lo, hi = block_bounds(d, world, rank)
            a = np.empty((ranks[n], hi - lo, ranks[n + 1]), order="F")
            fill_random_slab(a, n, lo, 11)
            mine.append(a)
        parts = g.allgather_object(mine)
        full = []
        for n, d in enumerate(dims):
            c = np.zeros((ranks[n], d, ranks[n + 1]), order="F")
            for p, sl in enumerate(parts):
                lo, hi = block_bounds(d, world, p)
                c[:, lo:hi, :] = sl[n]
            full.append(c)
        ref = O.random_cores(dims, ranks, 11)
        res["rng_bitwise"] = all(np.array_equal(a, b) for a, b in zip(full, ref))
        # 3. TSQR: local R, allgather, redundant stacked QR == global R
        rng = np.random.default_rng(3)
        A = rng.standard_normal((101, 6))
        lo, hi = block_bounds(101, world, rank)
        local = O.HouseholderQR(A[lo:hi])
        rs = g.allgather_object(local.r)
        top = O.HouseholderQR(np.vstack(rs))
        rg = np.linalg.qr(A)[1]
        rg = rg * np.where(np.diag(rg) < 0, -1.0, 1.0)[:, None]
        res["tsqr_err"] = float(np.abs(top.r - rg).max())
        # the apply needs no communication: this rank's rows of Q [c; 0]
        c = rng.standard_normal((6, 2))
        both = top.apply(c)
        qloc = local.apply(both[rank * 6:(rank + 1) * 6])
        qall = g.allgather_object(qloc)
        qfull = np.vstack(qall)
        res["apply_err"] = float(np.abs(qfull - A @ np.linalg.solve(top.r, c)).max())  # Q c = A R^-1 c
        # 4. Gram sweep: per-core partial over own slices, allreduce, next core
        x = O.random_cores((6, 8, 5), (1, 3, 2, 1), 1)
        y = O.random_cores((6, 8, 5), (1, 2, 4, 1), 2)
        w = np.ones((1, 1))
        for a, b in zip(x, y):
            lo, hi = block_bounds(a.shape[1], world, rank)
            aa, bb = a[:, lo:hi, :], b[:, lo:hi, :]
            z = np.einsum("ca,aib->cib", w, aa)
            part = np.einsum("cid,cib->db", bb, z)
            w = g.allreduce_sum(part)
        res["inner"] = float(w[0, 0])
        res["inner_ref"] = O.inner(x, y)
        res["bytes"] = rounding_bytes((4, 4), (1, 2, 1), (1, 1, 1))
        # 5. Kronecker-operator halo exchange (ops.py:270-311): the package's
        #    transfer plan, payloads swapped point to point over the group
        #    (the device path packs with ttb_gather_slices and swaps them with
        #    one grouped NCCL send/recv), renumbered CSR rows applied locally
        import scipy.sparse as sp
        import torch
        from paper_2011_06532_b200.operator import exchange_plan
        core = O.random_cores((13,), (1, 1), 5)[0]
        core = np.asfortranarray(np.repeat(core, 6, axis=0).reshape(2, 13, 3, order="F") * 1.5)
        ok = True
        for a in (sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(13, 13), format="csr"),
                  sp.csr_matrix((np.ones(13), (np.arange(13), (np.arange(13) + 5) % 13)), shape=(13, 13)),
                  sp.random(13, 13, density=0.3, random_state=9, format="csr")):
            pl = exchange_plan(a, world, rank)
            mine = core[:, pl.lo:pl.hi, :]
            reqs, bufs = [], []
            for qq, idx in sorted(pl.send.items()):
                payload = np.concatenate([mine[:, int(i), :].ravel(order="F") for i in idx])
                reqs.append(dist.isend(torch.from_numpy(payload), dst=qq))
            for qq, idx in sorted(pl.recv.items()):
                buf = torch.empty(idx.size * 6, dtype=torch.float64)
                reqs.append(dist.irecv(buf, src=qq))
                bufs.append(buf)
            for r_ in reqs:
                r_.wait()
            halo = [b.numpy().reshape(-1, 6) for b in bufs]
            src = np.concatenate([np.stack([mine[:, i, :].ravel(order="F") for i in range(pl.nloc)])] + halo)
            m = sp.csr_matrix((pl.vals, pl.cols, pl.indptr), shape=(pl.nloc, src.shape[0]))
            rows = np.asarray(m @ src).reshape(pl.nloc, 3, 2).transpose(2, 0, 1)
            got = np.concatenate(g.allgather_object(np.asfortranarray(rows)), axis=1)
            ok = ok and np.array_equal(got, O.mode2_multiply(core, a))
        res["operator_exchange"] = ok
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_host_logic():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        res = out[r]
        assert res["allreduce"] == [0.5 + 1.5, 0.0 + 2.0]
        assert res["gather"] == [("r", 0), ("r", 1)]
        assert res["rng_bitwise"]
        assert res["tsqr_err"] < 1e-12
        assert res["apply_err"] < 1e-12
        assert res["inner"] == pytest.approx(res["inner_ref"], rel=1e-12)
        assert res["operator_exchange"]
    # the redundant results are identical on every rank
    assert out[0]["inner"] == out[1]["inner"]
    assert out[0]["tsqr_err"] == out[1]["tsqr_err"]


def test_block_bounds_rule():
    from paper_2011_06532_b200.tensor import block_bounds
    assert [b - a for a, b in (block_bounds(5, 4, r) for r in range(4))] == [2, 2, 1, 0]
    for extent in (1, 2, 5, 7, 16, 33):
        for p in (1, 2, 3, 4, 8):
            marks = np.zeros(extent, dtype=int)
            for r in range(p):
                lo, hi = block_bounds(extent, p, r)
                marks[lo:hi] += 1
            assert (marks == 1).all()
