"""Real-time (streaming) sliCQ over an unbounded signal — SURVEY 8(f) NEXT-3.

The paper motivates the sliCQ by bounded delay: slices of length 2N with
hop N can be transformed as soon as their samples have arrived.  A finite signal is sliced
with circular indices; a stream has no end to wrap to, so here the history before
sample 0 is zero instead (S:293-301's streaming head).  Everything else — slicing window,
CQ-NSGT per slice, dual window, overlap-add — is the same transform, computed by the
backend's slice-range calls (libslicq.so's slicq_forward_range / slicq_inverse_range /
slicq_overlap_add for the product, see dist.LibBackend; the tests also drive it with the
oracle), so a stream cut into arbitrary chunks gives exactly the coefficients and samples
of one range call over the whole (zero-headed) signal.

* ForwardStream.push(x) returns the coefficients of every slice whose windowed frame has
  fully arrived: slice m needs samples up to m N + Bw - 1 (Bw = (N + tr)/2, the window's
  half support), i.e. a delay of Bw samples after the slice centre.
* InverseStream.push(c) returns every output sample that no later slice can still change:
  all but the last `halo` samples of the pushed slices' span (those wait for the next
  slice's overlap-add contribution); flush() releases them at the end of the stream.
"""
from __future__ import annotations

import torch

_TOTAL = 1 << 40  # "total slices" of an unbounded stream (even; no circular wrap is used)


class ForwardStream:
    """Streaming analysis: push sample chunks, receive coefficients slice by slice."""

    def __init__(self, backend, batch: int = 1, device=None, dtype=torch.float32):
        self.b = backend
        self.N = backend.N
        self.halo = backend.halo + (backend.halo & 1)  # even, >= (N + tr)/2 - 1
        self.reach = backend.halo                       # Bw: slice m needs samples < m N + Bw
        self.batch = batch
        self.next = 0          # next slice to emit
        self.received = 0      # samples pushed so far
        # samples [next N - halo, received); zeros before sample 0 (streaming head)
        self.hist = torch.zeros((batch, self.halo), dtype=dtype, device=device)

    def ready(self) -> int:
        """Slices whose frames are complete but not yet emitted."""
        if self.received < self.reach:
            return 0
        return max(0, (self.received - self.reach) // self.N + 1 - self.next)

    def _emit(self, k: int):
        need = self.halo + k * self.N
        xl = self.hist[:, :need]
        if xl.shape[1] < need:  # samples not received yet lie outside every emitted window
            pad = torch.zeros((self.batch, need - xl.shape[1]), dtype=xl.dtype, device=xl.device)
            xl = torch.cat([xl, pad], dim=1)
        c = self.b.forward_range(xl.contiguous(), self.halo, self.next, k, _TOTAL)
        self.hist = self.hist[:, k * self.N:]
        self.next += k
        return c

    def push(self, x: torch.Tensor):
        """x: [batch][m] new samples.  Returns coefficients [batch][k][C] of the k >= 0 slices
        completed by this chunk (k = 0: None)."""
        if x.dim() == 1:
            x = x[None]
        self.hist = torch.cat([self.hist, x.to(self.hist.dtype)], dim=1)
        self.received += x.shape[1]
        k = self.ready()
        return self._emit(k) if k > 0 else None

    def flush(self):
        """End of stream: the remaining slices whose windows reach received samples (the
        signal continues with zeros).  Returns [batch][k][C] or None."""
        last = (self.received + self.reach - 1) // self.N  # largest m with m N - Bw < received
        k = last + 1 - self.next
        return self._emit(k) if k > 0 else None


class InverseStream:
    """Streaming synthesis: push coefficients slice by slice, receive final samples."""

    def __init__(self, backend, batch: int = 1):
        self.b = backend
        self.N = backend.N
        self.halo = backend.halo + (backend.halo & 1)
        self.batch = batch
        self.next = 0        # next slice expected
        self.pending = None  # partial sums of samples [next N - halo, next N)

    def push(self, c):
        """c: [batch][k][C] coefficients of slices [next, next + k).  Returns the samples that
        became final ([batch][m], consecutive from sample 0 over successive calls)."""
        if c is None:
            return None
        k = c.shape[1]
        y, sp = self.b.inverse_range(c, self.next, k, _TOTAL, self.halo)
        parts = []
        if self.pending is not None:
            self.b.overlap_add(self.pending, sp)  # the new first slice completes the tail
            parts.append(self.pending)
        # (the first slice's spill falls before sample 0: outside the stream, dropped)
        cut = k * self.N - self.halo
        parts.append(y[:, :cut])
        self.pending = y[:, cut:].contiguous()
        self.next += k
        return torch.cat(parts, dim=1)

    def flush(self):
        """End of stream: the held-back tail is final."""
        out, self.pending = self.pending, None
        return out
