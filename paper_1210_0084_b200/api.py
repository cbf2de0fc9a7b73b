"""Thin Python binding of the C ABI (include/slicq.h) over torch tensors.

Names follow the C ABI: ``plan_create`` -> :class:`Plan`, ``slicq_forward`` ->
:meth:`Plan.forward`, ``slicq_inverse`` -> :meth:`Plan.inverse`, ... .  This module
only marshals arguments (shapes, dtypes, device pointers, the current CUDA stream);
every arithmetic step of the transform runs in libslicq.so's kernels.  There is
no CPU fallback: without the built library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import check, lib


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> Optional[int]:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Plan:
    """plan_create(fs, fmin, fmax, bins_per_octave, sl_len, tr_area, rasterize)."""

    def __init__(self, fs: float, fmin: float, fmax: float, bins_per_octave: int, sl_len: int,
                 tr_area: int, rasterize: int = 0, host_only: bool = False):
        L = lib()
        h = C.c_void_p()
        flags = _lib.PLAN_HOST_ONLY if host_only else 0
        check(L.plan_create_ex(float(fs), float(fmin), float(fmax), int(bins_per_octave),
                               int(sl_len), int(tr_area), int(rasterize), flags, C.byref(h)),
              "plan_create")
        self._h = h
        self.host_only = host_only
        self.params = (fs, fmin, fmax, bins_per_octave, sl_len, tr_area, rasterize)
        self._ws = {}

    # ------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().plan_destroy(self._h)
            self._h = C.c_void_p()
        self._ws = {}

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------ queries
    @property
    def num_channels(self) -> int:
        return check(lib().slicq_num_channels(self._h), "slicq_num_channels")

    @property
    def K(self) -> int:
        return check(lib().slicq_num_cq_channels(self._h), "slicq_num_cq_channels")

    @property
    def sl_len(self) -> int:
        return check(lib().slicq_sl_len(self._h), "slicq_sl_len")

    @property
    def N(self) -> int:
        return self.sl_len // 2

    @property
    def coeffs_per_slice(self) -> int:
        return check(lib().slicq_coeffs_per_slice(self._h), "slicq_coeffs_per_slice")

    @property
    def halo(self) -> int:
        return check(lib().slicq_halo(self._h), "slicq_halo")

    def channel_lengths(self) -> np.ndarray:
        M = np.zeros(self.num_channels, dtype=np.int32)
        check(lib().slicq_channel_lengths(self._h, M.ctypes.data), "slicq_channel_lengths")
        return M

    def channel_offsets(self) -> np.ndarray:
        off = np.zeros(self.num_channels + 1, dtype=np.int64)
        check(lib().slicq_channel_offsets(self._h, off.ctypes.data), "slicq_channel_offsets")
        return off

    def padded_length(self, n: int) -> int:
        return check(lib().slicq_padded_length(self._h, int(n)), "slicq_padded_length")

    def num_slices(self, n: int) -> int:
        return check(lib().slicq_num_slices(self._h, int(n)), "slicq_num_slices")

    def workspace_bytes(self, nslices: int, batch: int) -> int:
        return int(lib().slicq_workspace_bytes(self._h, int(nslices), int(batch)))

    def kernel_launches(self, direction: str, nslices: int, batch: int) -> int:
        """Kernels one forward / inverse call launches (slicq_kernel_launches)."""
        d = {"forward": 0, "inverse": 1}[direction]
        return int(lib().slicq_kernel_launches(self._h, d, int(nslices), int(batch)))

    def export(self) -> dict:
        """Host copies of the plan tables (slicq_plan_export) for plan-parity tests."""
        K2 = self.num_channels
        tot = check(lib().slicq_filter_total_length(self._h), "slicq_filter_total_length")
        N2 = self.sl_len
        lo = np.zeros(K2, np.int32)
        ln = np.zeros(K2, np.int32)
        g = np.zeros(tot, np.float64)
        gd = np.zeros(tot, np.float64)
        h0 = np.zeros(N2, np.float64)
        h0d = np.zeros(N2, np.float64)
        xi = np.zeros(K2 - 2, np.float64)
        check(lib().slicq_plan_export(self._h, lo.ctypes.data, ln.ctypes.data, g.ctypes.data,
                                      gd.ctypes.data, h0.ctypes.data, h0d.ctypes.data,
                                      xi.ctypes.data), "slicq_plan_export")
        return dict(lo=lo, len=ln, g=g, gdual=gd, h0=h0, h0dual=h0d, xi=xi,
                    M=self.channel_lengths(), off=self.channel_offsets())

    # ------------------------------------------------------------ workspace
    def workspace(self, nslices: int, batch: int, device=None, tag=None) -> torch.Tensor:
        """Zero-initialised once, then reused (it carries the overlap-add pairing counters).
        One workspace per (device, shape, tag): calls that may run concurrently use tags."""
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        key = (str(dev), nslices, batch, tag)
        ws = self._ws.get(key)
        if ws is None:
            nb = self.workspace_bytes(nslices, batch)
            ws = torch.zeros((nb + 15) // 16 * 4, dtype=torch.float32, device=dev)
            self._ws[key] = ws
        return ws

    # ------------------------------------------------------------ hot path
    def forward(self, x: torch.Tensor, out: Optional[torch.Tensor] = None,
                stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """slicq_forward: x float32 [batch][n] (cuda) -> complex64 [batch][S][C]."""
        if x.dim() == 1:
            x = x[None]
        _check_tensor(x, torch.float32, "x")
        B, n = x.shape
        S = self.num_slices(n)
        if out is None:
            out = torch.empty((B, S, self.coeffs_per_slice), dtype=torch.complex64, device=x.device)
        else:
            _check_tensor(out, torch.complex64, "out", (B, S, self.coeffs_per_slice))
        ws = self.workspace(S, B, x.device)
        check(lib().slicq_forward(self._h, x.data_ptr(), n, B, out.data_ptr(), ws.data_ptr(),
                                  ws.numel() * 4, _stream_ptr(stream)), "slicq_forward")
        return out

    def inverse(self, c: torch.Tensor, n: int, out: Optional[torch.Tensor] = None,
                stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """slicq_inverse: complex64 [batch][S][C] -> float32 [batch][n]."""
        if c.dim() == 2:
            c = c[None]
        B = c.shape[0]
        S = self.num_slices(n)
        _check_tensor(c, torch.complex64, "coeffs", (B, S, self.coeffs_per_slice))
        if out is None:
            out = torch.empty((B, n), dtype=torch.float32, device=c.device)
        else:
            _check_tensor(out, torch.float32, "out", (B, n))
        ws = self.workspace(S, B, c.device)
        check(lib().slicq_inverse(self._h, c.data_ptr(), n, B, out.data_ptr(), ws.data_ptr(),
                                  ws.numel() * 4, _stream_ptr(stream)), "slicq_inverse")
        return out

    def forward_range(self, x_local: torch.Tensor, halo: int, slice0: int, nslices: int,
                      total_slices: int, out: Optional[torch.Tensor] = None,
                      x_len: Optional[int] = None,
                      stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """slicq_forward_range: x_local float32 [batch][x_len] whose entry i is global sample
        slice0*N - halo + i  ->  complex64 [batch][nslices][C]."""
        if x_local.dim() == 1:
            x_local = x_local[None]
        _check_tensor(x_local, torch.float32, "x_local")
        B, xl = x_local.shape
        xl = xl if x_len is None else x_len
        if out is None:
            out = torch.empty((B, nslices, self.coeffs_per_slice), dtype=torch.complex64,
                              device=x_local.device)
        ws = self.workspace(nslices, B, x_local.device)
        check(lib().slicq_forward_range(self._h, x_local.data_ptr(), xl, x_local.stride(0), halo,
                                        slice0, nslices, total_slices, B, out.data_ptr(),
                                        ws.data_ptr(), ws.numel() * 4, _stream_ptr(stream)),
              "slicq_forward_range")
        return out

    def inverse_range(self, c_local: torch.Tensor, slice0: int, nslices: int, total_slices: int,
                      halo: int, y_local: Optional[torch.Tensor] = None,
                      spill: Optional[torch.Tensor] = None,
                      stream: Optional[torch.cuda.Stream] = None):
        """slicq_inverse_range -> (y_local float32 [batch][nslices*N], left_spill [batch][halo])."""
        if c_local.dim() == 2:
            c_local = c_local[None]
        B = c_local.shape[0]
        _check_tensor(c_local, torch.complex64, "coeffs", (B, nslices, self.coeffs_per_slice))
        if y_local is None:
            y_local = torch.empty((B, nslices * self.N), dtype=torch.float32, device=c_local.device)
        if spill is None:
            spill = torch.empty((B, halo), dtype=torch.float32, device=c_local.device)
        ws = self.workspace(nslices, B, c_local.device)
        check(lib().slicq_inverse_range(self._h, c_local.data_ptr(), slice0, nslices, total_slices,
                                        B, y_local.data_ptr(), y_local.stride(0), spill.data_ptr(),
                                        halo, ws.data_ptr(), ws.numel() * 4, _stream_ptr(stream)),
              "slicq_inverse_range")
        return y_local, spill

    @staticmethod
    def overlap_add(y_tail: torch.Tensor, spill: torch.Tensor,
                    stream: Optional[torch.cuda.Stream] = None) -> None:
        """slicq_overlap_add: y_tail[b][:count] += spill[b][:count] (y_tail may be a view)."""
        if y_tail.dim() == 1:
            y_tail, spill = y_tail[None], spill[None]
        B, count = spill.shape
        assert spill.is_contiguous() and y_tail.stride(1) == 1
        check(lib().slicq_overlap_add(y_tail.data_ptr(), y_tail.stride(0), spill.data_ptr(), count,
                                      B, _stream_ptr(stream)), "slicq_overlap_add")


def _check_tensor(t: torch.Tensor, dtype, name: str, shape=None):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def plan_for_config(cfg) -> Plan:
    """Plan for a synth.configs.SlicqConfig."""
    return Plan(cfg.fs, cfg.fmin, cfg.fmax_eff, cfg.bins_per_octave, cfg.sl_len, cfg.tr_area,
                cfg.rasterize)


def process_host(plan: Plan, x_host: torch.Tensor, y_host: Optional[torch.Tensor] = None,
                 fn=None, pieces: int = 8, device=None) -> torch.Tensor:
    """Host-to-host sliCQ round trip of a (long) signal, pipelined over slice ranges.

    x_host: pinned float32 [batch][n] (CPU).  The S slices are cut into `pieces` contiguous
    ranges; for each range the input (plus its left halo, circular for range 0) is
    copied host->device on one stream, slicq_forward_range / optional `fn(coeffs_local,
    slice0)` (in-place coefficient processing on the device) / slicq_inverse_range run on a
    second stream, and the synthesised samples go device->host on a third stream as soon as
    the right neighbour's overlap-add spill has been added (slicq_overlap_add).  Copies of
    range r+1 / r-1 overlap the kernels of range r.  Returns y_host [batch][n].
    The arithmetic is exactly that of slicq_forward + slicq_inverse (same kernels)."""
    if x_host.dim() == 1:
        x_host = x_host[None]
    if x_host.is_cuda or x_host.dtype != torch.float32:
        raise ValueError("x_host must be a float32 CPU tensor (pinned for overlap)")
    B, n = x_host.shape
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    if y_host is None:
        y_host = torch.empty((B, n), dtype=torch.float32, pin_memory=True)
    N, halo = plan.N, plan.halo
    S = plan.num_slices(n)
    L = S * N
    P = max(1, min(pieces, S // 2))
    bounds = [r * S // P for r in range(P + 1)]
    C = plan.coeffs_per_slice
    st_in, st_k, st_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    cur = torch.cuda.current_stream(dev)
    for s_ in (st_in, st_k, st_out):
        s_.wait_stream(cur)
    xl, co, yl, sp, ev_in, ev_inv = [], [], [], [], [], []
    for r in range(P):
        ns = bounds[r + 1] - bounds[r]
        xl.append(torch.empty((B, halo + ns * N), dtype=torch.float32, device=dev))
        co.append(torch.empty((B, ns, C), dtype=torch.complex64, device=dev))
        yl.append(torch.empty((B, ns * N), dtype=torch.float32, device=dev))
        sp.append(torch.empty((B, halo), dtype=torch.float32, device=dev))
        ev_in.append(torch.cuda.Event())
        ev_inv.append(torch.cuda.Event())

    def copy_in(dst, a, b):  # global samples [a, b) (circular, zero beyond n) -> dst[:, :b-a]
        pos, o = a, 0
        while pos < b:
            g = pos % L
            seg = min(b - pos, L - g)
            hi = min(g + seg, n)
            if hi > g:
                dst[:, o:o + hi - g].copy_(x_host[:, g:hi], non_blocking=True)
            if g + seg > max(g, n):
                dst[:, o + max(hi - g, 0):o + seg].zero_()
            pos += seg
            o += seg

    def copy_out(r):
        a = bounds[r] * N
        hi = min(bounds[r + 1] * N, n)
        if hi > a:
            y_host[:, a:hi].copy_(yl[r][:, :hi - a], non_blocking=True)

    with torch.cuda.stream(st_in):
        for r in range(P):
            copy_in(xl[r], bounds[r] * N - halo, bounds[r + 1] * N)
            ev_in[r].record(st_in)
    ev_out = [torch.cuda.Event() for _ in range(P)]
    with torch.cuda.stream(st_k):
        for r in range(P):
            s0, ns = bounds[r], bounds[r + 1] - bounds[r]
            st_k.wait_event(ev_in[r])
            plan.forward_range(xl[r], halo, s0, ns, S, out=co[r], stream=st_k)
            if fn is not None:
                fn(co[r], s0)
            plan.inverse_range(co[r], s0, ns, S, halo, y_local=yl[r], spill=sp[r], stream=st_k)
            if r > 0:  # range r's spill completes range r-1's tail
                Plan.overlap_add(yl[r - 1][:, -halo:], sp[r], stream=st_k)
                ev_out[r - 1].record(st_k)
        Plan.overlap_add(yl[P - 1][:, -halo:], sp[0], stream=st_k)  # circular wrap
        ev_out[P - 1].record(st_k)
    with torch.cuda.stream(st_out):
        for r in range(P):
            st_out.wait_event(ev_out[r])
            copy_out(r)
    for s_ in (st_in, st_k, st_out):
        cur.wait_stream(s_)
    # keep the buffers alive until the work is done
    for t in xl + co + yl + sp:
        t.record_stream(cur)
    return y_host
