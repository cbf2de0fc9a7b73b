"""Multi-process (world_size 2 and 3, gloo, CPU) test of the slice-range sharding logic in
paper_1210_0084_b200/dist.py: partition, halo exchange, spill exchange and overlap-add.
The per-rank compute is the oracle's range functions (the CUDA range kernels are covered
by tests/test_gpu_parity.py::test_range_api_matches_full); this checks the host logic
that moves data between ranks, which has no GPU dependency."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cqplan
from oracle import slicq as oslicq

ARGS = (8000.0, 150.0, None, 6, 128, 16, 0)
ARGS_TR2 = (8000.0, 150.0, None, 6, 128, 2, 0)  # tr = 2 mod 4: odd slicq_halo


class OracleBackend:
    """RangeBackend with the oracle's fp64 range functions on CPU tensors."""

    def __init__(self, args=ARGS):
        self.p = cqplan.make_plan(*args)
        self.N = self.p.N
        h = (self.p.N + self.p.tr) // 2
        self.halo = h + (h & 1)  # as LibBackend: the range calls take an even halo

    def num_slices(self, n):
        return oslicq.num_slices(n, self.p.sl_len)

    def forward_range(self, x_local, halo, slice0, nslices, total_slices, out=None):
        res = [oslicq.forward_range(x_local[b].contiguous().numpy(), halo, slice0, nslices,
                                    self.p) for b in range(x_local.shape[0])]
        res = torch.from_numpy(np.stack(res))
        if out is not None:
            out.copy_(res)
            return out
        return res

    def inverse_range(self, c_local, slice0, nslices, total_slices, halo, y_local=None):
        ys, sps = [], []
        for b in range(c_local.shape[0]):
            y, sp = oslicq.inverse_range(c_local[b].contiguous().numpy(), slice0, nslices,
                                         self.p, halo)
            ys.append(y)
            sps.append(sp)
        y = torch.from_numpy(np.stack(ys))
        if y_local is not None:
            y_local.copy_(y)
            y = y_local
        return y, torch.from_numpy(np.stack(sps))

    def overlap_add(self, y_tail, spill):
        y_tail += spill


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, q, args=ARGS):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1210_0084_b200.dist import SliceRangeShard
        be = OracleBackend(args)
        rng = np.random.default_rng(123)
        x = torch.from_numpy(rng.standard_normal((2, n)))
        sh = SliceRangeShard(be, n, batch=2)
        xl = sh.local_input(x)
        c = sh.forward(xl)
        y = sh.inverse(c)
        full = sh.gather_output(y)
        # coefficients of every rank, gathered for the check
        cs = [torch.zeros(2, sh.S, c.shape[-1], dtype=c.dtype) for _ in range(world)]
        cpad = torch.zeros(2, sh.S, c.shape[-1], dtype=c.dtype)
        cpad[:, sh.s0:sh.s1] = c
        dist.all_gather(cs, cpad)
        if rank == 0:
            q.put((full.numpy(), sum(t.numpy() for t in cs)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,args", [(2, 1500, ARGS), (3, 1234, ARGS), (2, 128, ARGS),
                                         (2, 1500, ARGS_TR2), (3, 700, ARGS_TR2)])
def test_sharded_equals_unsharded(world, n, args):
    """Includes tr = 2 mod 4 (odd (N + tr)/2, rounded up to an even halo like LibBackend)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q, args)) for r in range(world)]
    for p in procs:
        p.start()
    y, c = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    p = cqplan.make_plan(*args)
    rng = np.random.default_rng(123)
    x = rng.standard_normal((2, n))
    c_ref = oslicq.forward(x, p)
    y_ref = oslicq.inverse(c_ref, p, n)
    np.testing.assert_allclose(c, c_ref, rtol=0, atol=1e-11)
    np.testing.assert_allclose(y, y_ref, rtol=0, atol=1e-11)
    np.testing.assert_allclose(y, x, rtol=0, atol=1e-10)  # Prop. 3: perfect reconstruction


def test_partition_bounds():
    from paper_1210_0084_b200.dist import slice_bounds
    for S, G in ((21094, 8), (8, 8), (28, 3), (10, 4)):
        b = slice_bounds(S, G)
        assert b[0] == 0 and b[-1] == S and all(b[i] < b[i + 1] for i in range(G))
        sizes = [b[i + 1] - b[i] for i in range(G)]
        assert max(sizes) - min(sizes) <= 1


def test_batch_shard_partition_covers_rows_once():
    """BatchShard (independent signals, no collective): every row is owned by exactly one
    rank, ranks get contiguous, balanced row ranges, and the per-rank transform is the
    plan's whole-signal transform of those rows."""
    from paper_1210_0084_b200.dist import BatchShard

    class FakePlan:  # records calls; the transform itself is covered by the GPU tests
        def forward(self, x, out=None):
            return x * 2

        def inverse(self, c, n, out=None):
            return c / 2

    B, n = 16, 100
    x = torch.arange(B * n, dtype=torch.float32).reshape(B, n)
    for world in (1, 2, 3, 8, 16):
        owned = []
        for r in range(world):
            sh = BatchShard(FakePlan(), n, B, rank=r, world=world)
            xl = sh.local_input(x)
            assert torch.equal(xl, x[sh.r0:sh.r1])
            assert torch.equal(sh.inverse(sh.forward(xl)), xl)
            owned += list(range(sh.r0, sh.r1))
            assert B // world <= sh.r1 - sh.r0 <= -(-B // world)
        assert owned == list(range(B))
    with pytest.raises(ValueError):
        BatchShard(FakePlan(), n, 4, rank=0, world=8)
