"""Multi-GPU partition of one long stream into contiguous slice ranges.

One process per GPU.  Rank r of G owns slices [s_r, s_{r+1}), s_r = floor(r S / G), and the
input samples [s_r N, s_{r+1} N).  The only data exchanged between ranks is the overlap of
neighbouring slices (the paper's hop-N overlap, with circular indices P:328):

* forward: slice s_r's Tukey window reaches (N+tr)/2 - 1 samples to the left of s_r N, so
  rank r receives that left halo from rank r-1 (rank 0 from rank G-1: circular wrap);
* inverse: slice s_r's overlap-add output spills onto the same samples, so rank r sends
  that spill to rank r-1, which adds it (slicq_overlap_add kernel).

Both exchanges are one grouped point-to-point send/recv pair per call
(torch.distributed.batch_isend_irecv; NCCL over NVLink on GPUs, gloo in the CPU tests).
Batches of independent signals are split by rows instead (BatchShard: no exchange at all).
All transform arithmetic runs in the backend's range calls (libslicq.so for the product;
the tests substitute the oracle to check this host logic without a GPU).
"""
from __future__ import annotations

from typing import Optional, Protocol

import torch
import torch.distributed as dist


class RangeBackend(Protocol):
    N: int
    halo: int

    def num_slices(self, n: int) -> int: ...

    def forward_range(self, x_local, halo, slice0, nslices, total_slices, out=None): ...

    def inverse_range(self, c_local, slice0, nslices, total_slices, halo, y_local=None): ...

    def overlap_add(self, y_tail, spill) -> None: ...


def slice_bounds(S: int, world: int):
    return [r * S // world for r in range(world + 1)]


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class SliceRangeShard:
    """This rank's share of a sliCQ forward/inverse over one long stream."""

    def __init__(self, backend: RangeBackend, n: int, batch: int = 1, rank: Optional[int] = None,
                 world: Optional[int] = None, group=None):
        self.b = backend
        self.n = n
        self.batch = batch
        self.group = group
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        self.N = backend.N
        self.S = backend.num_slices(n)
        if self.S < self.world:
            raise ValueError(f"{self.S} slices cannot be split over {self.world} ranks")
        self.halo = backend.halo
        bnd = slice_bounds(self.S, self.world)
        self.s0, self.s1 = bnd[self.rank], bnd[self.rank + 1]
        self.ns = self.s1 - self.s0
        self.L = self.S * self.N
        if self.ns * self.N < self.halo:
            raise ValueError("local range shorter than the halo")

    # ------------------------------------------------------------ data placement
    @property
    def own(self):
        """Global sample range [a, b) this rank holds (before trimming to n)."""
        return self.s0 * self.N, self.s1 * self.N

    def local_input(self, x_full: torch.Tensor, device=None) -> torch.Tensor:
        """[batch][halo + ns N] buffer: own samples at [halo:], zeros for padding positions
        >= n; the first `halo` entries are filled by :meth:`exchange_halo`."""
        a, b = self.own
        xl = torch.zeros((self.batch, self.halo + self.ns * self.N), dtype=x_full.dtype,
                         device=device if device is not None else x_full.device)
        hi = min(b, self.n)
        if hi > a:
            xl[:, self.halo:self.halo + hi - a] = x_full[:, a:hi].to(xl.device)
        return xl

    def _p2p_start(self, send: torch.Tensor, dst: int, recv: torch.Tensor, src: int):
        """Post one grouped send/recv pair; returns the works (NCCL: work.wait() makes the
        current stream wait for the transfer, the host does not block)."""
        if self.world == 1:
            recv.copy_(send)
            return []
        ops = [dist.P2POp(dist.isend, send, self._g(dst), group=self.group),
               dist.P2POp(dist.irecv, recv, self._g(src), group=self.group)]
        return dist.batch_isend_irecv(ops)

    @staticmethod
    def _wait(works):
        for w in works:
            w.wait()

    def _g(self, r: int) -> int:
        return dist.get_global_rank(self.group, r) if self.group is not None else r

    def exchange_halo(self, xl: torch.Tensor) -> None:
        """Left halo <- last `halo` own samples of rank r-1 (rank G-1 for rank 0)."""
        h = self.halo
        tail = xl[:, -h:].contiguous()
        head = torch.empty_like(tail)
        self._wait(self._p2p_start(tail, (self.rank + 1) % self.world, head,
                                   (self.rank - 1) % self.world))
        xl[:, :h] = head

    def exchange_spill(self, spill: torch.Tensor) -> torch.Tensor:
        """Send my left spill to rank r-1, receive rank r+1's spill (circularly)."""
        recv = torch.empty_like(spill)
        self._wait(self._p2p_start(spill.contiguous(), (self.rank - 1) % self.world, recv,
                                   (self.rank + 1) % self.world))
        return recv

    # ------------------------------------------------------------ transform
    def forward(self, xl: torch.Tensor) -> torch.Tensor:
        """Coefficients of slices [s0, s1): [batch][ns][C].  The halo transfer is posted first;
        the interior slices [s0 + 1, s1) -- which read own samples only, since the window
        reaches (N + tr)/2 - 1 < N samples left of a slice -- are transformed while it is in
        flight.  On the GPU the boundary slice s0 runs on a side stream gated
        on the halo's arrival, so its kernels overlap the interior's instead of following
        them; on CPU tensors (gloo tests) it simply goes last."""
        h, N, B = self.halo, self.N, self.batch
        tail = xl[:, -h:].contiguous()
        head = torch.empty_like(tail)
        c = None
        if B == 1 and hasattr(self.b, "C"):  # both slice ranges are views of one buffer
            c = torch.empty((B, self.ns, self.b.C), dtype=torch.complex64, device=xl.device)
        side = torch.cuda.Stream(device=xl.device) if xl.is_cuda else None
        if side is not None:
            side.wait_stream(torch.cuda.current_stream(xl.device))
            with torch.cuda.stream(side):  # halo exchange + boundary slice
                works = self._p2p_start(tail, (self.rank + 1) % self.world, head,
                                        (self.rank - 1) % self.world)
                self._wait(works)
                xl[:, :h] = head
                cb = self.b.forward_range(xl[:, :h + N], h, self.s0, 1, self.S,
                                          out=c[:, :1] if c is not None else None)
        else:
            works = self._p2p_start(tail, (self.rank + 1) % self.world, head,
                                    (self.rank - 1) % self.world)
        ci = None
        if self.ns > 1:  # interior: entry i of xl[:, N:] is sample (s0 + 1) N - h + i
            ci = self.b.forward_range(xl[:, N:], h, self.s0 + 1, self.ns - 1, self.S,
                                      out=c[:, 1:] if c is not None else None)
        if side is not None:
            torch.cuda.current_stream(xl.device).wait_stream(side)
            for t in (xl, head, tail, cb):
                t.record_stream(side)
        else:
            self._wait(works)
            xl[:, :h] = head
            cb = self.b.forward_range(xl[:, :h + N], h, self.s0, 1, self.S,
                                      out=c[:, :1] if c is not None else None)
        if c is not None:
            return c
        return cb if ci is None else torch.cat([cb, ci], dim=1)

    def inverse(self, c_local: torch.Tensor) -> torch.Tensor:
        """Overlap-added output of samples [s0 N, s1 N): [batch][ns N].  The boundary slice s0
        is synthesised first (on the GPU: on a side stream, concurrently with the interior)
        so that its left spill travels to rank r-1 while the interior slices are
        synthesised; the interior's own left spill lands on slice s0's tail, and rank r+1's
        spill on this range's tail last."""
        h, N = self.halo, self.N
        rdt = torch.float64 if c_local.dtype == torch.complex128 else torch.float32
        y = torch.empty((self.batch, self.ns * N), dtype=rdt, device=c_local.device)
        side = torch.cuda.Stream(device=c_local.device) if c_local.is_cuda else None
        cur = torch.cuda.current_stream(c_local.device) if side is not None else None
        if side is not None:
            side.wait_stream(cur)
        ctx = torch.cuda.stream(side) if side is not None else _nullctx()
        with ctx:  # boundary slice, then its spill to rank r-1
            cb = c_local[:, :1] if self.batch == 1 else c_local[:, :1].contiguous()
            yb, spill0 = self.b.inverse_range(cb, self.s0, 1, self.S, h, y_local=y[:, :N])
            if yb.data_ptr() != y.data_ptr():
                y[:, :N] = yb
            recv = torch.empty_like(spill0)
            works = self._p2p_start(spill0.contiguous(), (self.rank - 1) % self.world, recv,
                                    (self.rank + 1) % self.world)
        spill1 = None
        if self.ns > 1:
            ci = c_local[:, 1:] if self.batch == 1 else c_local[:, 1:].contiguous()
            yi, spill1 = self.b.inverse_range(ci, self.s0 + 1, self.ns - 1, self.S, h,
                                              y_local=y[:, N:])
            if yi.data_ptr() != y[:, N:].data_ptr():
                y[:, N:] = yi
        if side is not None:
            cur.wait_stream(side)  # (slice s0's samples complete before the spill lands)
            for t in (y, recv, spill0, c_local):
                t.record_stream(side)
        if spill1 is not None:
            self.b.overlap_add(y[:, N - h:N], spill1)
        self._wait(works)
        self.b.overlap_add(y[:, -h:], recv)
        return y

    def gather_output(self, y_local: torch.Tensor) -> Optional[torch.Tensor]:
        """Concatenate every rank's y_local on rank 0 (tests/diagnostics only), trimmed to n."""
        parts = [torch.empty_like(y_local) for _ in range(self.world)] if self.rank == 0 else None
        if self.world == 1:
            return y_local[:, :self.n]
        sizes = [(slice_bounds(self.S, self.world)[r + 1] - slice_bounds(self.S, self.world)[r])
                 for r in range(self.world)]
        mx = max(sizes) * self.N
        pad = torch.zeros((self.batch, mx), dtype=y_local.dtype, device=y_local.device)
        pad[:, :y_local.shape[1]] = y_local
        out = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(out, pad, group=self.group)
        if self.rank != 0:
            return None
        full = torch.cat([o[:, :sizes[r] * self.N] for r, o in enumerate(out)], dim=1)
        return full[:, :self.n]


class BatchShard:
    """Independent signals (cfg3's 128 channel-signals, cfg5's 16 signals): rank r
    owns rows [floor(r B / G), floor((r+1) B / G)) and transforms them whole with no data-path
    collective (slicq_forward / slicq_inverse on its rows)."""

    def __init__(self, plan, n: int, batch: int, rank: Optional[int] = None,
                 world: Optional[int] = None, group=None):
        self.plan = plan
        self.n = n
        self.batch = batch
        self.group = group
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        if batch < self.world:
            raise ValueError(f"{batch} signals cannot be split over {self.world} ranks")
        b = slice_bounds(batch, self.world)
        self.r0, self.r1 = b[self.rank], b[self.rank + 1]

    def local_input(self, x_full: torch.Tensor, device=None) -> torch.Tensor:
        return x_full[self.r0:self.r1].to(device if device is not None else x_full.device)

    def forward(self, xl: torch.Tensor, out=None) -> torch.Tensor:
        return self.plan.forward(xl, out=out)

    def inverse(self, c: torch.Tensor, out=None) -> torch.Tensor:
        return self.plan.inverse(c, self.n, out=out)


class LibBackend:
    """RangeBackend over libslicq.so (api.Plan).  The range calls take an even halo
    (slicq_forward_range; slicq_halo = (N + tr)/2 is odd when tr = 2 mod 4), so the halo is
    rounded up to even."""

    def __init__(self, plan):
        self.plan = plan
        self.N = plan.N
        self.C = plan.coeffs_per_slice
        self.halo = plan.halo + (plan.halo & 1)

    def num_slices(self, n):
        return self.plan.num_slices(n)

    def forward_range(self, x_local, halo, slice0, nslices, total_slices, out=None):
        return self.plan.forward_range(x_local, halo, slice0, nslices, total_slices, out=out)

    def inverse_range(self, c_local, slice0, nslices, total_slices, halo, y_local=None):
        return self.plan.inverse_range(c_local, slice0, nslices, total_slices, halo,
                                       y_local=y_local)

    def overlap_add(self, y_tail, spill):
        self.plan.overlap_add(y_tail, spill)
