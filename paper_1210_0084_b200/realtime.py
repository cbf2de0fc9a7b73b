"""Per-hop real-time sliCQ: one slice in, one hop of samples out, as one CUDA graph replay
(latency mode; the paper's motivation for slicing is bounded delay,
P:83).

Every hop of N new samples completes exactly one slice: slice h needs samples
[hN - Bw + 1, hN + Bw) with Bw = (N + tr)/2 < N, all of which have arrived once samples
[hN, (h+1)N) are in.  One hop step is

    H2D copy of the hop (pinned host -> window[:, halo:])
    slicq_forward_range  (1 slice; window = last `halo` samples + the hop)
    hook(c)              (optional in-place coefficient processing, captured with the rest)
    slicq_inverse_range  (1 slice -> y [N], left spill [halo])
    slicq_overlap_add    (held-back tail of the previous hop += spill: now final)
    D2H copy of the completed N samples [hN - halo, (h+1)N - halo)
    window shift, tail <- y[N - halo:]

so the output lags the input by `halo` samples plus the step's own time.  Only the window's
relative position matters to the range kernels (global sample index slice0*N - halo + i,
every offset taken relative to slice0*N; no circular wrap in range mode), so one graph,
captured with slice0 = 1, is exact for every hop: the output stream is bit-identical to
stream.ForwardStream / InverseStream over the same zero-headed signal.

All arithmetic runs in libslicq.so's kernels; the graph holds them plus plain copies.
Run `python -m paper_1210_0084_b200.realtime --config 1` on a GPU for per-hop p50 / p99
latency (graph replay vs eager launches).
"""
from __future__ import annotations

import argparse
import json
import time
from typing import Callable, Optional

import numpy as np
import torch

_TOTAL = 1 << 40


class RealtimeSliCQ:
    """push(hop) -> the N samples that became final; the step is a CUDA graph when graph=True.

    hook: optional fn(c) modifying the coefficients [batch][1][C] (complex64, device) in
    place with torch/CUDA work on the current stream; it is captured into the graph, so it
    must be shape-static and must not synchronise."""

    def __init__(self, plan, batch: int = 1, hook: Optional[Callable] = None,
                 graph: bool = True, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("RealtimeSliCQ needs a CUDA device (libslicq.so path only)")
        self.p = plan
        self.N = N = plan.N
        self.halo = h = plan.halo + (plan.halo & 1)  # even (slicq_forward_range)
        self.batch = B = batch
        self.hook = hook
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.stream = torch.cuda.Stream(device=dev)
        f32 = dict(dtype=torch.float32, device=dev)
        self.win = torch.zeros((B, h + N), **f32)      # samples [hN - halo, (h+1)N)
        self.c = torch.empty((B, 1, plan.coeffs_per_slice), dtype=torch.complex64, device=dev)
        self.y = torch.empty((B, N), **f32)
        self.spill = torch.empty((B, h), **f32)
        self.tail = torch.zeros((B, h), **f32)         # partial sums of the last halo samples
        self.out = torch.empty((B, N), **f32)
        self.x_host = torch.zeros((B, N), dtype=torch.float32).pin_memory()
        self.y_host = torch.empty((B, N), dtype=torch.float32).pin_memory()
        self.hops = 0
        self.graph = None
        with torch.cuda.stream(self.stream):
            # the range calls' workspace (cached per stream) is allocated outside the capture;
            # holding it keeps the captured pointer alive if the plan's cache drops it
            self.ws = plan.workspace(1, B, dev, stream=self.stream)
        if graph:
            self._capture()

    # one hop on the current stream (eager, or being captured)
    def _step(self):
        s = self.stream
        N, h, p = self.N, self.halo, self.p
        self.win[:, h:].copy_(self.x_host, non_blocking=True)
        p.forward_range(self.win, h, 1, 1, _TOTAL, out=self.c, stream=s)
        if self.hook is not None:
            self.hook(self.c)
        p.inverse_range(self.c, 1, 1, _TOTAL, h, y_local=self.y, spill=self.spill,
                        stream=s)
        p.overlap_add(self.tail, self.spill, stream=s)
        self.out[:, :h].copy_(self.tail)
        self.out[:, h:].copy_(self.y[:, :N - h])
        self.y_host.copy_(self.out, non_blocking=True)
        self.tail.copy_(self.y[:, N - h:])
        self.win[:, :h].copy_(self.win[:, N:])

    def _capture(self):
        # warm up outside the capture on a throwaway state, then restore
        saved = [t.clone() for t in (self.win, self.tail)]
        with torch.cuda.stream(self.stream):
            self._step()
        self.stream.synchronize()
        self.win.copy_(saved[0])
        self.tail.copy_(saved[1])
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._step()
        torch.cuda.synchronize()

    def push_async(self, hop) -> None:
        """Enqueue one hop (array/tensor [batch][N] or [N], host).  Read result() after
        synchronize(); the previous hop must have completed (its input buffer is reused)."""
        hop = torch.as_tensor(hop, dtype=torch.float32)
        self.x_host.copy_(hop.reshape(self.batch, self.N))
        with torch.cuda.stream(self.stream):  # replay() launches on the current stream
            if self.graph is not None:
                self.graph.replay()
            else:
                self._step()
        self.hops += 1

    def synchronize(self) -> None:
        self.stream.synchronize()

    def result(self) -> torch.Tensor:
        """The hop's final samples [batch][N] = output samples [hN - halo, (h+1)N - halo) of
        the (zero-headed) stream; a view of a pinned host buffer, overwritten by the next
        hop."""
        return self.y_host

    def push(self, hop) -> torch.Tensor:
        self.push_async(hop)
        self.synchronize()
        return self.y_host.clone()

    def launches_per_hop(self) -> int:
        """libslicq.so kernels one hop launches (forward + inverse + overlap-add)."""
        return (self.p.kernel_launches("forward", 1, self.batch)
                + self.p.kernel_launches("inverse", 1, self.batch) + 1)


def measure(cfg: int, hops: int, batch: int, graph: bool, seed: int = 1) -> dict:
    from paper_1210_0084_b200 import api
    from synth.configs import CONFIGS
    from synth.signals import random_signal
    plan = api.plan_for_config(CONFIGS[cfg])
    rt = RealtimeSliCQ(plan, batch=batch, graph=graph)
    N = plan.N
    warm = 20
    x = random_signal(seed, batch, (hops + warm) * N).astype(np.float32)
    lat, dev_ms = [], []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(hops + warm):
        hop = x[:, k * N:(k + 1) * N]
        t0 = time.perf_counter()
        ev0.record(rt.stream)
        rt.push_async(hop)
        ev1.record(rt.stream)
        rt.synchronize()
        t1 = time.perf_counter()
        if k >= warm:
            lat.append((t1 - t0) * 1e6)
            dev_ms.append(ev0.elapsed_time(ev1) * 1e3)
    lat, dev = np.array(lat), np.array(dev_ms)
    c = CONFIGS[cfg]
    return {"config": c.name, "N": N, "halo": rt.halo, "batch": batch, "hops": hops,
            "graph": graph, "launches_per_hop": rt.launches_per_hop(),
            "hop_ms_of_audio": 1e3 * N / c.fs,
            "algorithmic_delay_samples": rt.halo,
            "host_latency_us": {"p50": float(np.percentile(lat, 50)),
                                "p99": float(np.percentile(lat, 99)),
                                "max": float(lat.max())},
            "device_us": {"p50": float(np.percentile(dev, 50)),
                          "p99": float(np.percentile(dev, 99))}}


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--config", type=int, nargs="+", default=[1, 4])
    ap.add_argument("--hops", type=int, default=2000)
    ap.add_argument("--batch", type=int, default=1)
    args = ap.parse_args()
    for cfg in args.config:
        for graph in (True, False):
            print(json.dumps(measure(cfg, args.hops, args.batch, graph)), flush=True)


if __name__ == "__main__":
    main()
