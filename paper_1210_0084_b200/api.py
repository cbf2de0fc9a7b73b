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
from ._lib import COEFF_FN, check, lib


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> Optional[int]:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Plan:
    """plan_create(fs, fmin, fmax, bins_per_octave, sl_len, tr_area, rasterize)."""

    def __init__(self, fs: float, fmin: float, fmax: float, bins_per_octave: int, sl_len: int,
                 tr_area: int, rasterize: int = 0, host_only: bool = False,
                 window: str = "hann", min_width: float = 4.0, sampled_from: int = 0):
        """window / min_width / sampled_from: plan_create_ex2 (the filter options of the
        paper's approximation experiments; sampled_from = 2N builds Prop. 4's full-length
        system for slices of 2N)."""
        L = lib()
        h = C.c_void_p()
        flags = _lib.PLAN_HOST_ONLY if host_only else 0
        check(L.plan_create_ex2(float(fs), float(fmin), float(fmax), int(bins_per_octave),
                                int(sl_len), int(tr_area), int(rasterize), flags,
                                _lib.WINDOWS[window], float(min_width), int(sampled_from),
                                C.byref(h)),
              "plan_create")
        self._h = h
        self.host_only = host_only
        self.params = (fs, fmin, fmax, bins_per_octave, sl_len, tr_area, rasterize)
        self.options = dict(window=window, min_width=min_width, sampled_from=sampled_from)
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

    @property
    def coeffs_per_slice_full(self) -> int:
        """sum of M_k over all 2K+2 channels (complex-input layout)."""
        return check(lib().slicq_coeffs_per_slice_full(self._h), "slicq_coeffs_per_slice_full")

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
    _WS_CACHE = 8  # workspaces kept per plan (least recently used are dropped)

    def workspace(self, nslices: int, batch: int, device=None, tag=None,
                  stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Cached per (device, shape, stream, tag): calls on different streams get different
        workspaces (the library resets the inverse's pairing counters at every call, so reuse
        on one stream is safe); a non-current stream gets record_stream.  At most _WS_CACHE
        workspaces are kept (least recently used dropped)."""
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        sid = stream.cuda_stream if stream is not None else None
        key = (str(dev), nslices, batch, sid, tag)
        ws = self._ws.pop(key, None)
        if ws is None:
            nb = self.workspace_bytes(nslices, batch)
            ws = torch.zeros((nb + 15) // 16 * 4, dtype=torch.float32, device=dev)
            while len(self._ws) >= self._WS_CACHE:
                self._ws.pop(next(iter(self._ws)))
        self._ws[key] = ws  # (most recently used last)
        if stream is not None and stream != torch.cuda.current_stream(dev):
            ws.record_stream(stream)
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
        ws = self.workspace(S, B, x.device, stream=stream)
        check(lib().slicq_forward(self._h, x.data_ptr(), n, B, out.data_ptr(), ws.data_ptr(),
                                  ws.numel() * 4, _stream_ptr(stream)), "slicq_forward")
        return out

    def inverse(self, c: torch.Tensor, n: int, out: Optional[torch.Tensor] = None,
                stream: Optional[torch.cuda.Stream] = None, mask: Optional[torch.Tensor] = None,
                mask_db: bool = True) -> torch.Tensor:
        """slicq_inverse: complex64 [batch][S][C] -> float32 [batch][n].  With `mask` (float32
        [batch][S][C]), slicq_inverse_masked: the coefficient mask (dB-scaled unless
        mask_db=False, paper §VI) is applied inside the inverse's coefficient loads."""
        if c.dim() == 2:
            c = c[None]
        B = c.shape[0]
        S = self.num_slices(n)
        _check_tensor(c, torch.complex64, "coeffs", (B, S, self.coeffs_per_slice))
        if out is None:
            out = torch.empty((B, n), dtype=torch.float32, device=c.device)
        else:
            _check_tensor(out, torch.float32, "out", (B, n))
        ws = self.workspace(S, B, c.device, stream=stream)
        if mask is not None:
            _check_tensor(mask, torch.float32, "mask", (B, S, self.coeffs_per_slice))
            check(lib().slicq_inverse_masked(self._h, c.data_ptr(), mask.data_ptr(),
                                             1 if mask_db else 0, n, B, out.data_ptr(),
                                             ws.data_ptr(), ws.numel() * 4, _stream_ptr(stream)),
                  "slicq_inverse_masked")
            return out
        check(lib().slicq_inverse(self._h, c.data_ptr(), n, B, out.data_ptr(), ws.data_ptr(),
                                  ws.numel() * 4, _stream_ptr(stream)), "slicq_inverse")
        return out

    def _workspace_complex(self, nslices: int, batch: int, n: int, device) -> torch.Tensor:
        key = (str(device), nslices, batch, ("complex", n))
        ws = self._ws.get(key)
        if ws is None:
            nb = int(lib().slicq_workspace_bytes_complex(self._h, nslices, batch, n))
            ws = torch.zeros((nb + 15) // 16 * 4, dtype=torch.float32, device=device)
            self._ws[key] = ws
        return ws

    def forward_complex(self, x: torch.Tensor, out: Optional[torch.Tensor] = None,
                        stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """slicq_forward_complex: complex64 [batch][n] -> complex64 [batch][S][Cf] over all
        2K+2 channels (Table-1 order: stored 0..K+1, then the mirrors of K..1)."""
        if x.dim() == 1:
            x = x[None]
        _check_tensor(x, torch.complex64, "x")
        B, n = x.shape
        S = self.num_slices(n)
        if out is None:
            out = torch.empty((B, S, self.coeffs_per_slice_full), dtype=torch.complex64,
                              device=x.device)
        else:
            _check_tensor(out, torch.complex64, "out", (B, S, self.coeffs_per_slice_full))
        ws = self._workspace_complex(S, B, n, x.device)
        check(lib().slicq_forward_complex(self._h, x.data_ptr(), n, B, out.data_ptr(),
                                          ws.data_ptr(), ws.numel() * 4, _stream_ptr(stream)),
              "slicq_forward_complex")
        return out

    def inverse_complex(self, c: torch.Tensor, n: int, out: Optional[torch.Tensor] = None,
                        stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """slicq_inverse_complex: complex64 [batch][S][Cf] -> complex64 [batch][n]."""
        if c.dim() == 2:
            c = c[None]
        B, S = c.shape[0], self.num_slices(n)
        _check_tensor(c, torch.complex64, "coeffs", (B, S, self.coeffs_per_slice_full))
        if out is None:
            out = torch.empty((B, n), dtype=torch.complex64, device=c.device)
        else:
            _check_tensor(out, torch.complex64, "out", (B, n))
        ws = self._workspace_complex(S, B, n, c.device)
        check(lib().slicq_inverse_complex(self._h, c.data_ptr(), n, B, out.data_ptr(),
                                          ws.data_ptr(), ws.numel() * 4, _stream_ptr(stream)),
              "slicq_inverse_complex")
        return out

    def nsgt_forward_complex(self, x: torch.Tensor, out: Optional[torch.Tensor] = None,
                             stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """slicq_nsgt_forward_complex: full-length CQ-NSGT of complex64 [batch][n], n <= sl_len
        -> complex64 [batch][Cf] (all 2K+2 channels)."""
        if x.dim() == 1:
            x = x[None]
        _check_tensor(x, torch.complex64, "x")
        B, n = x.shape
        if out is None:
            out = torch.empty((B, self.coeffs_per_slice_full), dtype=torch.complex64,
                              device=x.device)
        else:
            _check_tensor(out, torch.complex64, "out", (B, self.coeffs_per_slice_full))
        ws = self._workspace_complex(1, B, n, x.device)
        check(lib().slicq_nsgt_forward_complex(self._h, x.data_ptr(), n, B, out.data_ptr(),
                                               ws.data_ptr(), ws.numel() * 4, _stream_ptr(stream)),
              "slicq_nsgt_forward_complex")
        return out

    def nsgt_inverse_complex(self, c: torch.Tensor, n: int, out: Optional[torch.Tensor] = None,
                             stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """slicq_nsgt_inverse_complex: complex64 [batch][Cf] -> complex64 [batch][n]."""
        if c.dim() == 1:
            c = c[None]
        B = c.shape[0]
        _check_tensor(c, torch.complex64, "coeffs", (B, self.coeffs_per_slice_full))
        if out is None:
            out = torch.empty((B, n), dtype=torch.complex64, device=c.device)
        else:
            _check_tensor(out, torch.complex64, "out", (B, n))
        ws = self._workspace_complex(1, B, n, c.device)
        check(lib().slicq_nsgt_inverse_complex(self._h, c.data_ptr(), n, B, out.data_ptr(),
                                               ws.data_ptr(), ws.numel() * 4, _stream_ptr(stream)),
              "slicq_nsgt_inverse_complex")
        return out

    def nsgt_forward(self, x: torch.Tensor, out: Optional[torch.Tensor] = None,
                     stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """slicq_nsgt_forward: full-length CQ-NSGT (Alg. 1) of x float32 [batch][n],
        n <= sl_len -> complex64 [batch][C]."""
        if x.dim() == 1:
            x = x[None]
        _check_tensor(x, torch.float32, "x")
        B, n = x.shape
        if out is None:
            out = torch.empty((B, self.coeffs_per_slice), dtype=torch.complex64, device=x.device)
        else:
            _check_tensor(out, torch.complex64, "out", (B, self.coeffs_per_slice))
        ws = self.workspace(1, B, x.device, stream=stream)
        check(lib().slicq_nsgt_forward(self._h, x.data_ptr(), n, B, out.data_ptr(), ws.data_ptr(),
                                       ws.numel() * 4, _stream_ptr(stream)), "slicq_nsgt_forward")
        return out

    def nsgt_inverse(self, c: torch.Tensor, n: int, out: Optional[torch.Tensor] = None,
                     stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """slicq_nsgt_inverse: full-length CQ-NSGT synthesis (Alg. 2) -> float32 [batch][n]."""
        if c.dim() == 1:
            c = c[None]
        B = c.shape[0]
        _check_tensor(c, torch.complex64, "coeffs", (B, self.coeffs_per_slice))
        if out is None:
            out = torch.empty((B, n), dtype=torch.float32, device=c.device)
        else:
            _check_tensor(out, torch.float32, "out", (B, n))
        ws = self.workspace(1, B, c.device, stream=stream)
        check(lib().slicq_nsgt_inverse(self._h, c.data_ptr(), n, B, out.data_ptr(), ws.data_ptr(),
                                       ws.numel() * 4, _stream_ptr(stream)), "slicq_nsgt_inverse")
        return out

    def forward_range(self, x_local: torch.Tensor, halo: int, slice0: int, nslices: int,
                      total_slices: int, out: Optional[torch.Tensor] = None,
                      x_len: Optional[int] = None,
                      stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """slicq_forward_range: x_local float32 [batch][x_len] whose entry i is global sample
        slice0*N - halo + i  ->  complex64 [batch][nslices][C]."""
        if x_local.dim() == 1:
            x_local = x_local[None]
        # rows may be strided (a view into a wider buffer: the shard's boundary slice)
        _check_rows(x_local, torch.float32, "x_local", tuple(x_local.shape))
        B, xl = x_local.shape
        if x_len is not None:
            if not 0 < x_len <= xl:
                raise ValueError(f"x_len {x_len} outside (0, {xl}]")
            xl = x_len
        if out is None:
            out = torch.empty((B, nslices, self.coeffs_per_slice), dtype=torch.complex64,
                              device=x_local.device)
        else:
            _check_tensor(out, torch.complex64, "out", (B, nslices, self.coeffs_per_slice))
        ws = self.workspace(nslices, B, x_local.device, stream=stream)
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
        else:
            _check_rows(y_local, torch.float32, "y_local", (B, nslices * self.N))
        if spill is None:
            spill = torch.empty((B, halo), dtype=torch.float32, device=c_local.device)
        else:
            _check_tensor(spill, torch.float32, "spill", (B, halo))
        ws = self.workspace(nslices, B, c_local.device, stream=stream)
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


def _check_rows(t: torch.Tensor, dtype, name: str, shape):
    """A caller-provided [rows][cols] output whose rows may be strided (a view into a wider
    buffer): CUDA, dtype, shape, unit stride along a row, non-overlapping rows."""
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.stride(1) != 1 or (t.shape[0] > 1 and t.stride(0) < t.shape[1]):
        raise ValueError(f"{name} rows must be unit-stride and non-overlapping")


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


def approximation_error(x: torch.Tensor, ps: Plan, pl: Plan, stream=None):
    """Prop. 4 / Sec. V-A: how closely the sliCQ
    with plan ps (slices 2N) approximates the full-length CQ-NSGT with pl (created with
    sampled_from = 2N, sl_len L).  x: float32 [batch][L] (stored channels) or complex64
    [batch][L] (all 2K+2 channels, the paper's Set 1) on the device.  Runs the sliCQ, the
    full-length CQ-NSGT and slicq_approx_error(_complex); returns (snr_db [batch] float64
    tensor, sums [batch][channels][2] float64: per channel sum |c|^2 and sum |c - (s^0 + s^1)|^2
    in the Prop. 4 normalisation)."""
    if x.dim() == 1:
        x = x[None]
    B, L = x.shape
    if L != pl.sl_len:
        raise ValueError("x must hold L = pl.sl_len samples per row")
    if x.is_complex():  # the paper's Set 1: all 2K+2 channels (slicq_approx_error_complex)
        _check_tensor(x, torch.complex64, "x")
        s = ps.forward_complex(x, stream=stream)
        c = pl.nsgt_forward_complex(x, stream=stream)
        out = torch.empty((B, 2 * ps.K + 2, 2), dtype=torch.float64, device=x.device)
        fn, name = lib().slicq_approx_error_complex, "slicq_approx_error_complex"
    else:
        _check_tensor(x, torch.float32, "x")
        s = ps.forward(x, stream=stream)
        c = pl.nsgt_forward(x, stream=stream)
        out = torch.empty((B, ps.num_channels, 2), dtype=torch.float64, device=x.device)
        fn, name = lib().slicq_approx_error, "slicq_approx_error"
    check(fn(ps._h, pl._h, s.data_ptr(), c.data_ptr(), B, out.data_ptr(), _stream_ptr(stream)),
          name)
    tot = out.sum(dim=1)
    return 10.0 * torch.log10(tot[:, 0] / tot[:, 1]), out


def _rows(plan: Plan, c: torch.Tensor) -> torch.Tensor:
    if c.dim() == 2:
        c = c[None]
    _check_tensor(c, torch.complex64, "coeffs")
    if c.shape[-1] != plan.coeffs_per_slice:
        raise ValueError("coefficient rows must hold C = plan.coeffs_per_slice entries")
    return c


def apply_mask(plan: Plan, c: torch.Tensor, mask, db: bool = True, inplace: bool = False,
               stream=None) -> torch.Tensor:
    """Coefficient masking (paper §VI) on the device (slicq_apply_mask): c * a,
    a = 10^(-5 (1 - mask)) for dB-scaled masks ("0 in the mask corresponds to 10^-5 (-100 dB)
    and 1 corresponds to 1 (0 dB)"), else a = mask.  c: complex64 [batch][S][C]; mask: a
    number, a per-column [C] or a full [batch][S][C] real grid.  The fused alternative is
    Plan.inverse(c, n, mask=...)."""
    c = _rows(plan, c)
    m = torch.as_tensor(mask, dtype=torch.float32, device=c.device)
    C = plan.coeffs_per_slice
    if m.dim() == 0:
        m = m.expand(C)
    m = m.contiguous()
    if tuple(m.shape) == (C,):
        full = 0
    elif tuple(m.shape) == tuple(c.shape):
        full = 1
    else:
        raise ValueError("mask must be a number, [C] or the coefficients' shape")
    out = c if inplace else c.clone()
    check(lib().slicq_apply_mask(plan._h, out.data_ptr(), m.data_ptr(), out.numel() // C, full,
                                 1 if db else 0, _stream_ptr(stream)), "slicq_apply_mask")
    return out


def spectrogram(plan: Plan, c: torch.Tensor, stream=None):
    """The paper's sliCQ spectrogram |s^0 + s^1|^2 per channel (slicq_spectrogram):
    a list of [batch][S M_k / 2] float32 views into one device buffer, time-ordered with hop
    2N/M_k samples per entry."""
    c = _rows(plan, c)
    B, S, C = c.shape
    out = torch.empty((B, S * C // 2), dtype=torch.float32, device=c.device)
    check(lib().slicq_spectrogram(plan._h, c.data_ptr(), S, B, out.data_ptr(),
                                  _stream_ptr(stream)), "slicq_spectrogram")
    Ms, offs = plan.channel_lengths(), plan.channel_offsets()
    return [out[:, S * int(o) // 2: S * (int(o) + int(M)) // 2] for M, o in zip(Ms, offs)]


def transpose_bins(plan: Plan, c: torch.Tensor, shift: int, stream=None) -> torch.Tensor:
    """Pitch transposition by `shift` CQ bins (B bins = one octave, SURVEY
    NEXT-4) on the device (slicq_transpose_bins): CQ channel k takes channel (k - shift)'s
    coefficients, vacated channels are zero, the DC / Nyquist plateaus are kept.  Needs one
    coefficient count M for all CQ channels (a rasterised plan, C10; the paper's
    "rectangular representation").

    The library's coefficients carry absolute phase (C6): channel k's content at bin j sits
    at folded frequency j mod M.  Moving it to channel k' is the demodulated ("verbatim")
    copy of the paper's toolbox, which in absolute phase is a modulation by the difference
    of the two channels' centre bins: c'_{k'}[n] = c_k[n] e^{2 pi i (w_k' - w_k) n / M}."""
    c = _rows(plan, c)
    out = torch.empty_like(c)
    check(lib().slicq_transpose_bins(plan._h, c.data_ptr(), out.data_ptr(),
                                     c.numel() // plan.coeffs_per_slice, int(shift),
                                     _stream_ptr(stream)), "slicq_transpose_bins")
    return out


def two_layer(plan: Plan, c: torch.Tensor):
    """The paper's coefficient array s = {s^0, s^1} as a view of the
    slice-major coefficients c [batch][S][C]: per channel k a tensor [batch][2][S M_k / 2]
    with s^{m mod 2}_k[((m-1) M_k/2 + n) mod (S M_k/2)] = c^m_k[n].  Layer l holds the
    slices m = l, l+2, ... back to back, rotated by (l-1) M_k / 2 -- index arithmetic only
    (torch slicing / roll on the tensor's device)."""
    if c.dim() == 2:
        c = c[None]
    B, S, _ = c.shape
    if S % 2:
        raise ValueError("a sliced stream has an even number of slices")
    Ms, offs = plan.channel_lengths(), plan.channel_offsets()
    out = []
    for M, off in zip(Ms, offs):
        layers = []
        for layer in (0, 1):
            blk = c[:, layer::2, off:off + M].reshape(B, -1)   # slices m = layer + 2i
            layers.append(torch.roll(blk, shifts=(layer - 1) * (M // 2), dims=1))
        out.append(torch.stack(layers, dim=1))
    return out


def from_two_layer(plan: Plan, s) -> torch.Tensor:
    """Inverse of :func:`two_layer` (the partition of Alg. 4): per-channel
    [batch][2][S M_k / 2] tensors -> c [batch][S][C]."""
    Ms, offs = plan.channel_lengths(), plan.channel_offsets()
    B, _, W0 = s[0].shape
    S = 2 * W0 // Ms[0]
    c = torch.empty((B, S, plan.coeffs_per_slice), dtype=s[0].dtype, device=s[0].device)
    for sk, M, off in zip(s, Ms, offs):
        for layer in (0, 1):
            blk = torch.roll(sk[:, layer], shifts=-(layer - 1) * (M // 2), dims=1)
            c[:, layer::2, off:off + M] = blk.reshape(B, S // 2, M)
    return c


class _DeviceView:
    """__cuda_array_interface__ view of library-owned device memory (no copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 2}


def process_host(plan: Plan, x_host: torch.Tensor, y_host: Optional[torch.Tensor] = None,
                 fn=None, pieces: int = 32, device=None) -> torch.Tensor:
    """Host-to-host sliCQ round trip of a (long) signal: slicq_process_host, the library's
    native streaming executor (csrc/stream_exec.cpp), pipelined over `pieces` slice ranges
    on three streams so host<->device copies overlap the kernels.

    x_host: float32 [batch][n] CPU tensor (pinned for overlap).  fn(coeffs, slice0), if
    given, is called once per range with a torch view of that range's device coefficients
    [batch][nslices][C] under the stream it must enqueue its work on (in-place processing).
    Returns y_host [batch][n]; asynchronous: synchronise the current stream before use.
    The arithmetic is exactly that of slicq_forward + slicq_inverse (same kernels)."""
    if x_host.dim() == 1:
        x_host = x_host[None]
    if x_host.is_cuda or x_host.dtype != torch.float32 or not x_host.is_contiguous():
        raise ValueError("x_host must be a contiguous float32 CPU tensor (pinned for overlap)")
    B, n = x_host.shape
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    if y_host is None:
        y_host = torch.empty((B, n), dtype=torch.float32, pin_memory=True)
    elif y_host.is_cuda or y_host.dtype != torch.float32 or tuple(y_host.shape) != (B, n) \
            or not y_host.is_contiguous():
        raise ValueError("y_host must be a contiguous float32 CPU tensor of x_host's shape")
    key = (str(dev), "process_host", n, B, pieces)
    ws = plan._ws.get(key)
    if ws is None:
        nb = int(lib().slicq_process_host_workspace_bytes(plan._h, n, B, pieces))
        if nb == 0:
            raise ValueError("slicq_process_host_workspace_bytes: invalid arguments")
        ws = torch.zeros((nb + 15) // 16 * 4, dtype=torch.float32, device=dev)
        plan._ws[key] = ws
    cb = None
    if fn is not None:
        C_ = plan.coeffs_per_slice

        def _hook(user, ptr, slice0, nslices, batch, stream):
            try:
                t = torch.as_tensor(_DeviceView(ptr, (batch, nslices, C_), "<c8"), device=dev)
                with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=dev)):
                    fn(t, int(slice0))
                return 0
            except Exception:  # reported through the library's error path
                import traceback
                traceback.print_exc()
                return 1
        cb = COEFF_FN(_hook)
    with torch.cuda.device(dev):
        check(lib().slicq_process_host(plan._h, x_host.data_ptr(), y_host.data_ptr(), n, B,
                                       int(pieces), cb, None, ws.data_ptr(), ws.numel() * 4,
                                       _stream_ptr(None)), "slicq_process_host")
    return y_host
