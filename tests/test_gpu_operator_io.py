"""GPU parity for the Kronecker-operator apply (ops.py:238-342, core.py:285-297)
and TTPAR1 files straight into HBM (core.py:364-398), against the
reference's own outputs (tests/golden, written by gen_golden.py).

Bars: sparse mode-2 products and the operator apply bitwise (the device
kernel follows scipy's CSR accumulation order); apply + round with ranks
identical and TT-form error <= 1e-10; file round trips bitwise, byte-equal
to the reference's writer.

P > 1 is emulated on the one GPU by threads, one rank each, whose exchange
hands device buffers over directly instead of through NCCL (everything
else -- plans, payload packing, halo renumbering, block-diagonal assembly
-- is the product code).
"""
import threading

import numpy as np
import pytest
import scipy.sparse as sp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2011_06532_b200 as T  # noqa: E402
from oracle import tt_oracle as O  # noqa: E402
from tests._golden import golden, tt  # noqa: E402
from tests.test_operator_io import kron_sum_terms, lap, shift_terms  # noqa: E402


def cores_of(t):
    return [c.array for c in t.cores]


def bitwise(xs, ys):
    assert len(xs) == len(ys)
    for a, b in zip(xs, ys):
        assert a.shape == b.shape and np.array_equal(a, b)


class _Group:
    def __init__(self, size):
        self.size = size
        self.cv = threading.Condition()
        self.box = {}       # (src, dst, seq) -> tensor
        self.taken = set()  # (src, dst, seq) consumed
        self.seq = {}
        self.bar = threading.Barrier(size)


class ThreadRank(T.SerialComm):
    """Rank `rank` of an emulated P-rank group on the one GPU."""

    def __init__(self, group, rank):
        super().__init__()
        self.g, self.size, self.rank = group, group.size, rank

    def exchange(self, peers, sends, recvs):
        g = self.g
        keys = []
        with g.cv:
            for q, s in zip(peers, sends):
                k = (self.rank, q, g.seq.get((self.rank, q), 0))
                g.seq[(self.rank, q)] = k[2] + 1
                if s is not None:
                    g.box[k] = s
                    keys.append(k)
            g.cv.notify_all()
            for q, r in zip(peers, recvs):
                if r.numel() == 0:
                    continue
                k = (q, self.rank, g.seq.get(("r", q, self.rank), 0))
                g.seq[("r", q, self.rank)] = k[2] + 1
                g.cv.wait_for(lambda: k in g.box)
                r.copy_(g.box.pop(k))  # same stream: ordered after the peer's packing kernel
                g.taken.add(k)
            g.cv.notify_all()
            g.cv.wait_for(lambda: all(k in g.taken for k in keys))

    def barrier(self):
        self.g.bar.wait()


def run_ranks(size, body):
    g = _Group(size)
    out, err = [None] * size, []

    def run(p):
        try:
            out[p] = body(ThreadRank(g, p))
        except BaseException as e:  # pragma: no cover - surfaced below
            err.append(e)
            g.bar.abort()
            with g.cv:
                g.cv.notify_all()

    th = [threading.Thread(target=run, args=(p,)) for p in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if err:
        raise err[0]
    return out


def gather_blocks(parts):
    """Concatenate per-rank host slab lists along the mode index."""
    return [np.asfortranarray(np.concatenate([p[n] for p in parts], axis=1)) for n in range(len(parts[0]))]


def distributed(comm, cores):
    dims = tuple(c.shape[1] for c in cores)
    ranks = (1,) + tuple(c.shape[2] for c in cores)
    local = []
    for n, c in enumerate(cores):
        lo, hi = T.block_bounds(dims[n], comm.size, comm.rank)
        local.append(np.asfortranarray(c[:, lo:hi, :]))
    return T.DistTTTensor(comm, dims, ranks, local)


# ------------------------------------------------------------- mode-2 products

def test_mode2_multiply_sparse_bitwise_dense_close():
    g = golden()
    a = sp.csr_matrix(g["m2_a_dense"])
    got = T.mode2_multiply(T.TTCore(g["m2_core"]), a)
    assert np.array_equal(got.array, g["m2_out"])
    dense = T.mode2_multiply(T.TTCore(g["m2_core"]), g["m2_a_dense"])
    assert np.allclose(dense.array, g["m2_out"], rtol=1e-13, atol=1e-14)
    with pytest.raises(T.ShapeError):
        T.mode2_multiply(T.TTCore(g["m2_core"]), np.ones((10, 10)))


def test_mode2_multiply_random_shapes():
    rng = np.random.default_rng(8)
    for _ in range(10):
        rl, d, rr = (int(v) for v in rng.integers(1, 40, size=3))
        core = np.asfortranarray(rng.standard_normal((rl, d, rr)))
        a = sp.random(d, d, density=0.3, random_state=int(rng.integers(1 << 30)), format="csr")
        got = T.mode2_multiply(T.TTCore(core), a).array
        assert np.array_equal(got, O.mode2_multiply(core, a))


# ------------------------------------------------------------ operator apply

def test_apply_operator_serial_bitwise():
    x = T.TTTensor(tt("op_x"))
    op = T.KroneckerOperator((6, 5, 7), kron_sum_terms((6, 5, 7)))
    z = T.apply_operator(op, x)
    assert z.ranks == (1, 9, 12, 1)
    bitwise(cores_of(z), tt("op_lap"))
    bitwise(cores_of(T.apply_operator(T.KroneckerOperator((6, 5, 7), shift_terms((6, 5, 7))), x)), tt("op_shift"))
    one = T.KroneckerOperator((8,), [[lap(8)], [sp.identity(8, format="csr")]])
    bitwise(cores_of(T.apply_operator(one, T.TTTensor(tt("op1_x")))), tt("op1_lap"))
    ident = T.apply_operator(T.KroneckerOperator.identity(x.dims), x)
    bitwise(cores_of(ident), tt("op_x"))


def test_apply_operator_many_terms():
    """More terms than the fused one-pass kernel takes (16): per-term launches."""
    dims = (5, 4, 6)
    x = O.random_cores(dims, (1, 2, 2, 1), 40)
    rng = np.random.default_rng(41)
    terms = [[sp.random(d, d, density=0.5, random_state=int(rng.integers(1 << 30)), format="csr") for d in dims]
             for _ in range(18)]
    op = T.KroneckerOperator(dims, terms)
    z = T.apply_operator(op, T.TTTensor(x))
    bitwise(cores_of(z), O.apply_operator(op.terms, x))
    x1 = O.random_cores((7,), (1, 1), 42)
    op1 = T.KroneckerOperator((7,), [[sp.random(7, 7, density=0.5, random_state=k, format="csr")] for k in range(20)])
    bitwise(cores_of(T.apply_operator(op1, T.TTTensor(x1))), O.apply_operator(op1.terms, x1))


def test_apply_operator_device_tensor_and_dims_check():
    x = T.TTTensor(tt("op_x"))
    op = T.KroneckerOperator((6, 5, 7), kron_sum_terms((6, 5, 7)))
    dz = T.apply_operator(op, T.serial_tt(x))
    assert isinstance(dz, T.DistTTTensor)
    bitwise(cores_of(T.gather(dz)), tt("op_lap"))
    with pytest.raises(T.ShapeError, match="dims"):
        T.apply_operator(T.KroneckerOperator.identity((4, 5, 4)), x)


def test_apply_operator_with_rounding():
    x = T.TTTensor(tt("op_x"))
    op = T.KroneckerOperator((6, 5, 7), kron_sum_terms((6, 5, 7)))
    z = T.apply_operator(op, x, round_eps=1e-10)
    ref = tt("op_lap_round")
    assert z.ranks == O.ranks_of(ref)
    assert O.rel_diff(cores_of(z), ref) <= 1e-10


@pytest.mark.parametrize("size", [2, 3])
def test_apply_operator_distributed_bitwise(size):
    op = T.KroneckerOperator((6, 5, 7), kron_sum_terms((6, 5, 7)))

    def body(comm):
        z = T.apply_operator(op, distributed(comm, tt("op_x")))
        torch.cuda.synchronize()
        return [T.tensor.to_host_array(s) for s in z.local]

    bitwise(gather_blocks(run_ranks(size, body)), tt(f"op_lap_p{size}"))


def test_apply_operator_distributed_coupled_slices():
    """4 ranks, tridiagonal factor on one mode (test_ops.py:324-346).  (The
    distributed apply + round needs the native NCCL collectives of the
    rounding, which the one-GPU thread emulation cannot provide.)"""
    x = O.random_cores((8, 8), (1, 2, 1), 28)
    op = T.KroneckerOperator((8, 8), [[lap(8), sp.identity(8, format="csr")]])
    want = O.apply_operator(op.terms, x)

    def body(comm):
        z = T.apply_operator(op, distributed(comm, x))
        torch.cuda.synchronize()
        return [T.tensor.to_host_array(s) for s in z.local]

    bitwise(gather_blocks(run_ranks(4, body)), want)



# ------------------------------------------------------------------- TT files

def test_load_tt_dist_reference_file_bitwise(tmp_path):
    p = tmp_path / "ref.tt"
    p.write_bytes(golden()["file_tt_bytes"].tobytes())
    ref = tt("file_tt")
    dt = T.load_tt_dist(p)
    bitwise([T.tensor.to_host_array(s) for s in dt.local], ref)
    for size in (2, 3, 4):
        parts = []
        for r in range(size):
            comm = ThreadRank(_Group(size), r)
            parts.append([T.tensor.to_host_array(s) for s in T.load_tt_dist(p, comm).local])
        bitwise(gather_blocks(parts), ref)
    bad = tmp_path / "short.tt"
    bad.write_bytes(golden()["file_tt_bytes"].tobytes()[:-8])
    with pytest.raises(T.ShapeError, match="truncated"):
        T.load_tt_dist(bad)


def test_save_tt_dist_matches_reference_writer(tmp_path):
    ref_bytes = golden()["file_tt_bytes"].tobytes()
    for size in (1, 3):
        p = tmp_path / f"out{size}.tt"

        def body(comm):
            T.save_tt_dist(p, distributed(comm, tt("file_tt")))

        run_ranks(size, body)
        assert p.read_bytes() == ref_bytes


def test_tt_file_large_roundtrip(tmp_path):
    """~150 MB: several 64 MB staging groups, multi-threaded pread, partial
    slice runs at P = 3."""
    dims, ranks = (3001, 4000, 2003), (1, 48, 50, 1)
    p = tmp_path / "big.tt"

    def write(comm):
        T.save_tt_dist(p, T.DistTTTensor.random(comm, dims, ranks, 5))

    run_ranks(3, write)
    full = T.load_tt_dist(p)
    want = T.DistTTTensor.random(T.default_comm(), dims, ranks, 5)
    for a, b in zip(full.local, want.local):
        assert torch.equal(a, b)
    host = T.load_tt(p)
    for a, b in zip(host.cores, want.local):
        assert np.array_equal(a.array, T.tensor.to_host_array(b))
