"""Per-hop real-time sliCQ (paper_1210_0084_b200/realtime.py, SURVEY 8(f) NEXT-3 latency
mode): one CUDA-graph replay per hop of N samples gives exactly the samples of the chunked
streaming transform (stream.py) and reconstructs the input with a delay of `halo` samples
(Prop. 3)."""
import numpy as np
import pytest
import torch

from paper_1210_0084_b200.stream import ForwardStream, InverseStream
from synth.signals import random_signal


def _plan(cfg):
    from paper_1210_0084_b200 import api
    from synth.configs import CONFIGS
    return api.plan_for_config(CONFIGS[cfg])


def _run_rt(plan, x, graph, hook=None):
    from paper_1210_0084_b200.realtime import RealtimeSliCQ
    B, n = x.shape
    rt = RealtimeSliCQ(plan, batch=B, hook=hook, graph=graph)
    N = plan.N
    return torch.cat([rt.push(x[:, k * N:(k + 1) * N]) for k in range(n // N)], dim=1), rt


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,batch", [(1, 2), (4, 1)])
def test_realtime_matches_stream_and_reconstructs(cfg, batch):
    from paper_1210_0084_b200.dist import LibBackend
    plan = _plan(cfg)
    N = plan.N
    H = 12
    x = torch.from_numpy(random_signal(31 + cfg, batch, H * N))
    y_rt, rt = _run_rt(plan, x, graph=True)
    h = rt.halo
    assert y_rt.shape == (batch, H * N)
    # hop k's output = samples [kN - halo, (k+1)N - halo): the first halo samples lie before
    # sample 0 (the zero head, reconstructed as ~0)
    assert y_rt[:, :h].abs().max().item() <= 1e-5 * x.abs().max().item()
    err = ((y_rt[:, h:] - x[:, :H * N - h]).norm() / x[:, :H * N - h].norm()).item()
    assert err <= 1e-5, err
    # the chunked stream (one slice-range call per hop at the true slice index) over the same
    # zero-headed signal: identical samples, i.e. the captured slice0 = 1 graph is exact
    be = LibBackend(plan)
    xd = x.cuda()
    fs, inv = ForwardStream(be, batch=batch, device=xd.device), InverseStream(be, batch=batch)
    ys = [inv.push(fs.push(xd[:, k * N:(k + 1) * N])) for k in range(H)]
    y_st = torch.cat([t for t in ys if t is not None], dim=1).cpu()
    m = min(y_st.shape[1], H * N - h)
    assert torch.equal(y_rt[:, h:h + m], y_st[:, :m])


@pytest.mark.gpu
def test_realtime_graph_equals_eager_and_hook_is_applied():
    plan = _plan(1)
    N = plan.N
    x = torch.from_numpy(random_signal(77, 1, 6 * N))
    y_g, _ = _run_rt(plan, x, graph=True)
    y_e, _ = _run_rt(plan, x, graph=False)
    assert torch.equal(y_g, y_e)
    # a captured in-place coefficient hook: scaling by 2 is exact in floating point, so the
    # output is exactly twice the unprocessed one
    y_2, _ = _run_rt(plan, x, graph=True, hook=lambda c: c.mul_(2.0))
    assert torch.equal(y_2, 2 * y_g)


@pytest.mark.gpu
def test_realtime_latency_report_fields():
    from paper_1210_0084_b200.realtime import measure
    r = measure(1, hops=50, batch=1, graph=True)
    assert r["launches_per_hop"] > 0 and r["algorithmic_delay_samples"] == r["halo"]
    assert 0 < r["host_latency_us"]["p50"] <= r["host_latency_us"]["p99"]
    assert r["device_us"]["p50"] > 0


def test_realtime_requires_cuda():
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    from paper_1210_0084_b200.realtime import RealtimeSliCQ
    with pytest.raises(RuntimeError):
        RealtimeSliCQ(object())
