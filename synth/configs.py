"""Workload registry: the five BASELINE.json configurations.

Plain parameters only (no transform arithmetic).  Shared by the CUDA path's
tests/bench and by the oracle's tests, so both sides transform the same
problem.  The transform parameters are BASELINE.json `configs[i]`; the
signal recipes are SURVEY.md §8(d) "Synthetic inputs" (items marked
*(proposed)* there are this repo's readings, listed in DESIGN.md).
"""
from dataclasses import dataclass, field
from typing import Optional

SEED_BASE = 12100084  # seed = 12100084 + cfg


@dataclass(frozen=True)
class SlicqConfig:
    cfg: int
    name: str
    fs: float
    fmin: float
    fmax: Optional[float]  # None -> fs/2
    bins_per_octave: int
    sl_len: int  # 2N
    tr_area: int  # tr (the paper's transition length "M")
    rasterize: int  # 0 none, 1 per octave, 2 full (C10)
    batch: int  # independent fp32 signals (stereo = 2 per signal)
    n: int  # samples per signal
    seed: int = field(default=0)

    @property
    def fmax_eff(self) -> float:
        return self.fs / 2 if self.fmax is None else self.fmax


CONFIGS = {
    1: SlicqConfig(1, "cfg1-mono-65536", 44100.0, 65.4, 22050.0, 12, 16384, 2048, 0,
                   1, 65536, SEED_BASE + 1),
    2: SlicqConfig(2, "cfg2-mono-10s-octave-raster", 44100.0, 32.7, None, 48, 32768, 4096, 1,
                   1, 441000, SEED_BASE + 2),
    3: SlicqConfig(3, "cfg3-64stereo-2^20-full-raster", 44100.0, 55.0, None, 24, 16384, 2048, 2,
                   128, 1 << 20, SEED_BASE + 3),
    4: SlicqConfig(4, "cfg4-1h-stream-48k", 48000.0, 32.7, 24000.0, 48, 16384, 2048, 0,
                   1, 172_800_000, SEED_BASE + 4),
    5: SlicqConfig(5, "cfg5-16x2^22-B96-2N131072", 44100.0, 27.5, None, 96, 131072, 16384, 0,
                   16, 1 << 22, SEED_BASE + 5),
}


def plan_args(c: SlicqConfig):
    """Arguments of plan_create(fs, fmin, fmax, bins_per_octave, sl_len, tr_area, rasterize)."""
    return (c.fs, c.fmin, c.fmax_eff, c.bins_per_octave, c.sl_len, c.tr_area, c.rasterize)
