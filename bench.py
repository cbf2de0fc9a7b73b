#!/usr/bin/env python
"""sliCQ forward+inverse throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl reference]

A *step* is one pass of the whole hot path — slicq_forward then slicq_inverse (every row
of SURVEY.md §8(a)) — over the config's whole synthetic workload.  Default workload:
BASELINE configs[3] ("cfg4": one hour of 48 kHz mono, 172.8 M samples, 21 094 slices of
2N = 16384), the config the north_star's multi-GPU target is stated on; configs[0..1]
are microsecond-scale (8 / 28 slices) and serve as parity cases.

N = 1: one process, slicq_forward + slicq_inverse on the whole stream (circular slices).
N > 1 (torchrun): contiguous slice ranges per rank with the NCCL halo / spill exchange
(paper_1210_0084_b200/dist.py), total work fixed => "scaling": "strong".

Timing: W warm-up steps; barrier + synchronize; CUDA events on the launching stream around
exactly K steps; barrier + synchronize; max over ranks.  Inputs (691 MB) and coefficients
(3 GB) are far larger than the 126 MB L2, so no flush is needed between steps.
`--impl reference` times the fp64 oracle (oracle/, the test oracle) on the host cores
instead — a deliberately slow reference, reported, not a target.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "sliCQ fwd+inv input samples/s"
UNIT = "samples/s"
E2E_PIECES = 32  # slice ranges of the end-to-end (host-to-host) pipeline


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during the timed region."""
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.ok = False
        self.samples, self.reasons = [], set()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


_ORACLE = {}


def _oracle_init(cfg_id: int):
    """Pool worker: build the oracle plan once (plan creation is not timed)."""
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import cqplan
    from synth.configs import CONFIGS, plan_args
    cfg = CONFIGS[cfg_id]
    _ORACLE["cfg"] = cfg
    _ORACLE["plan"] = cqplan.make_plan(*plan_args(cfg))
    _ORACLE["x"] = _workload_row(cfg_id, _ORACLE["plan"])


def _workload_row(cfg_id: int, ref, slices: int = 256) -> np.ndarray:
    """Row 0 of the workload's own seeded signal (the input the GPU arm transforms, VERDICT
    round 1 "baseline hygiene"), as fp64; for the long stream only the prefix the sample
    uses (cfg4_signal's prefixes are exact)."""
    from synth.configs import CONFIGS
    from synth.signals import cfg3_signal, cfg4_signal, cfg5_signal, make_signal
    cfg = CONFIGS[cfg_id]
    need = (ref.N + ref.tr) // 2 + (slices + 2) * ref.N
    if cfg_id == 3:
        x = cfg3_signal(cfg, batch=1)
    elif cfg_id == 4:
        x = cfg4_signal(cfg, n=min(cfg.n, need))
    elif cfg_id == 5:
        x = cfg5_signal(cfg, batch=1)
    else:
        x = make_signal(cfg_id)
    return x[0].astype(np.float64)


def _oracle_chunk(args):
    """Pool worker: forward + inverse of `nsl` consecutive slices (oracle slice-range
    functions, fp64 NumPy) of a distinct part of the stream; returns the seconds it took."""
    slice0, nsl = args
    from oracle import slicq as oslicq
    ref, xw = _ORACLE["plan"], _ORACLE["x"]
    N = ref.N
    halo = (N + ref.tr) // 2
    # the slices [slice0, slice0 + nsl) of the workload's signal (cyclically where the
    # signal is shorter than the sample: cfg1 has 8 slices)
    s0 = 1 + slice0 % max(1, (len(xw) - halo) // N - nsl - 1)
    idx = (s0 * N - halo + np.arange(halo + nsl * N)) % len(xw)
    x = xw[idx]
    t0 = time.perf_counter()
    c = oslicq.forward_range(x, halo, slice0, nsl, ref)
    oslicq.inverse_range(c, slice0, nsl, ref, halo)
    return time.perf_counter() - t0


class OracleTimer:
    """The fp64 oracle as it stands, timed on the host's cores: one process per core
    (os.sched_getaffinity), each transforming its own run of consecutive slices (SURVEY
    8(d)).  Wall time from dispatch to the last result."""

    def __init__(self, cfg, nsl: int = 12):
        import multiprocessing as mp
        self.cfg, self.nsl = cfg, nsl
        self.cores = max(1, len(os.sched_getaffinity(0)))
        # spawn: the bench process holds a CUDA context (never fork it)
        self.pool = mp.get_context("spawn").Pool(self.cores, _oracle_init, (cfg.cfg,))
        self.run()  # warm the workers (plan build, imports)

    def run(self):
        jobs = [(w * self.nsl, self.nsl) for w in range(self.cores)]
        t0 = time.perf_counter()
        self.pool.map(_oracle_chunk, jobs, chunksize=1)
        return time.perf_counter() - t0

    def samples_per_run(self):
        return self.cores * self.nsl * (self.cfg.sl_len // 2)

    def describe(self):
        return (f"{self.nsl} consecutive slices of {self.cfg.name}'s own signal (row 0) per "
                f"process ({self.nsl * (self.cfg.sl_len // 2)} input samples each), {self.cores} "
                f"processes on {self.cores} host cores, oracle.slicq.forward_range + "
                f"inverse_range, fp64 NumPy")

    def one_core(self, reps: int = 2) -> float:
        """samples/s of one process alone (the same job in this process, 1 core)."""
        _oracle_init(self.cfg.cfg)
        _oracle_chunk((0, self.nsl))  # warm
        dt = min(_oracle_chunk((0, self.nsl)) for _ in range(reps))
        return self.nsl * (self.cfg.sl_len // 2) / dt

    def close(self):
        self.pool.terminate()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def oracle_sample_rate(cfg, reps: int = 3):
    """(samples/s, seconds per run, cores, description, 1-core samples/s) of the oracle on
    all host cores and on one."""
    t = OracleTimer(cfg)
    try:
        dts = [t.run() for _ in range(reps)]
        dt = sum(dts) / len(dts)
        v1 = t.one_core()
        return t.samples_per_run() / dt, dt, t.cores, t.describe(), v1
    finally:
        t.close()


def run_reference(args, cfg):
    rank, world, _ = _env_rank()
    if rank != 0:
        return  # rank 0 alone runs and prints the reference arm
    t = OracleTimer(cfg)
    try:
        for _ in range(args.warmup):
            t.run()
        per = [t.run() for _ in range(args.steps)]
    finally:
        t.close()
    value = t.samples_per_run() / (sum(per) / len(per))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(per) / len(per), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": t.cores, "kind": "oracle",
                             "sample": t.describe(), "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def padded_len(cfg):
    return -(-cfg.n // cfg.sl_len) * cfg.sl_len


def config_dict(cfg, world):
    return {"workload": f"BASELINE configs[{cfg.cfg - 1}] ({cfg.name})", "batch": cfg.batch,
            "samples_per_row": cfg.n, "fs": cfg.fs, "fmin": cfg.fmin, "fmax": cfg.fmax_eff,
            "bins_per_octave": cfg.bins_per_octave, "sl_len": cfg.sl_len, "tr_area": cfg.tr_area,
            "rasterize": cfg.rasterize,
            "parallelism": ("single GPU" if world == 1 else
                            f"signals split over {world} ranks (no exchange)"
                            if cfg.batch >= world and cfg.batch > 1 else
                            f"slice ranges x{world} (NCCL halo)"),
            "l2": "no flush: inputs and coefficients exceed the 126 MB L2"}


def run_gpu(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1210_0084_b200 import api
    from paper_1210_0084_b200.dist import BatchShard, LibBackend, SliceRangeShard
    from synth.signals import make_signal

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    plan = api.plan_for_config(cfg)
    x_np = make_signal(cfg.cfg)
    B_all, n = x_np.shape
    # batches of independent signals split by rows across ranks (no collective);
    # a single long stream is split into slice ranges with the NCCL halo / spill exchange
    batch_mode = world > 1 and B_all >= world and B_all > 1
    if batch_mode:
        bsh = BatchShard(plan, n, B_all, rank, world)
        x_np = np.ascontiguousarray(x_np[bsh.r0:bsh.r1])
    B = x_np.shape[0]
    C = plan.coeffs_per_slice
    stream = torch.cuda.current_stream()

    sharded = (world > 1 and not batch_mode) or args.force_shard
    if not sharded:
        x = torch.from_numpy(x_np).to(dev)
        c = torch.empty((B, plan.num_slices(n), C), dtype=torch.complex64, device=dev)
        y = torch.empty((B, n), dtype=torch.float32, device=dev)
        S_local = c.shape[1]
        L_local = plan.padded_length(n)
        # forward: spectrum + channel kernel(s); inverse: channel kernel(s) + spectrum
        launches_per_step = (plan.kernel_launches("forward", S_local, B)
                             + plan.kernel_launches("inverse", S_local, B))

        def fwd():
            plan.forward(x, out=c)

        def inv():
            plan.inverse(c, n, out=y)
    else:
        shard = SliceRangeShard(LibBackend(plan), n, B, rank, world)
        xl = shard.local_input(torch.from_numpy(x_np), device=dev)
        S_local = shard.ns
        L_local = shard.ns * plan.N
        state = {}
        # forward_range, inverse_range, overlap_add
        launches_per_step = (plan.kernel_launches("forward", S_local, B)
                             + plan.kernel_launches("inverse", S_local, B) + 1)

        def fwd():
            state["c"] = shard.forward(xl)

        def inv():
            state["y"] = shard.inverse(state["c"])

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for _ in range(args.warmup):
        fwd()
        inv()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e_f0, e_f1, e_i1 = [ev() for _ in range(args.steps)], [ev() for _ in range(args.steps)], \
        [ev() for _ in range(args.steps)]
    t_start, t_end = ev(), ev()
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for k in range(args.steps):
            e_f0[k].record(stream)
            fwd()
            e_f1[k].record(stream)
            inv()
            e_i1[k].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms_total = t_start.elapsed_time(t_end)
    per_f = [e_f0[k].elapsed_time(e_f1[k]) for k in range(args.steps)]
    per_i = [e_f1[k].elapsed_time(e_i1[k]) for k in range(args.steps)]
    ms_f = sum(per_f) / args.steps
    ms_i = sum(per_i) / args.steps
    # SURVEY 8(d) (as the paper): spread of the per-step times besides the mean
    step_stats = {"forward_ms_median": statistics.median(per_f),
                  "forward_ms_std": statistics.pstdev(per_f),
                  "inverse_ms_median": statistics.median(per_i),
                  "inverse_ms_std": statistics.pstdev(per_i)}
    t = torch.tensor([ms_total, ms_f, ms_i], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total, ms_f, ms_i = t.tolist()
    ms_step = ms_total / args.steps
    samples = B_all * n  # whole job: all ranks' signals
    value = samples / (ms_step / 1e3)

    # parity spot-check of this run's output (reconstruction, C17)
    if not sharded:
        nd = torch.stack([torch.sum((y - x).double() ** 2), torch.sum(x.double() ** 2)])
        if world > 1:
            dist.all_reduce(nd)  # batch mode: every rank's rows
        rec = float((nd[0] / nd[1]).sqrt())
    else:
        yl = state["y"]
        a, b = shard.own
        hi = min(b, n) - a
        xs = torch.from_numpy(x_np[:, a:a + hi]).to(dev) if hi > 0 else None
        num = torch.tensor([0.0, 0.0], dtype=torch.float64, device=dev)
        if hi > 0:
            num[0] = torch.sum((yl[:, :hi] - xs).double() ** 2)
            num[1] = torch.sum(xs.double() ** 2)
        if world > 1:
            dist.all_reduce(num)
        rec = float((num[0] / num[1]).sqrt())

    # roofline for the dominant kernel (algorithmic bytes)
    peak, peak_src = peaks()
    bytes_fwd = B * (4 * L_local + 8 * S_local * C)  # read x once, write complex64 coefficients
    bytes_inv = bytes_fwd                             # read coefficients, write y
    # the dominant direction; each C-ABI call is one spectrum kernel + the channel kernel
    # variants its packets need (lite <16,3> and full <32,2>)
    dom = "slicq_inverse" if ms_i >= ms_f else "slicq_forward"
    # (the spectrum kernel by slice length: persistent single-CTA for 2N = 2^12..2^15, the
    # mixed-radix generic kernel, four-step for 2^16, 16-CTA cluster for 2^17)
    spec = {"slicq_inverse": ("slicq_inv_spec_persist_kernel", "slicq_inv_spec_generic",
                              "inv_large_pack/col/row + inv_large_bnd",
                              "inv_large_cluster + inv_large_bnd"),
            "slicq_forward": ("slicq_fwd_spec_kernel", "slicq_fwd_spec_generic",
                              "fwd_large_col/row", "fwd_large_cluster")}[dom]
    sl = plan.sl_len
    si = 3 if sl == 131072 else 2 if sl == 65536 else 0 if sl & (sl - 1) == 0 else 1
    kernels = (f"slicq_inv_chan_kernel (lite + full variants) + {spec[si]}"
               if dom == "slicq_inverse"
               else f"{spec[si]} + slicq_fwd_chan_kernel (lite + full variants)")
    ms_dom = max(ms_i, ms_f)
    achieved = (bytes_inv if dom == "slicq_inverse" else bytes_fwd) / (ms_dom / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            t = json.load(open(tp)).get(f"cfg{cfg.cfg}", {}).get(dom)
            traffic = None if t is None else t * (L_local * B) / (cfg.batch * padded_len(cfg))
        except Exception:
            traffic = None

    # end to end through the public API with host buffers (pinned), copies timed
    e2e = None
    if not sharded and not args.no_e2e:
        # end to end through the public API with host buffers: api.process_host streams the
        # signal host->device, runs forward + inverse (slice ranges) and device->host,
        # pipelined over E2E_PIECES ranges on three streams; copies are inside the timed region
        xh = torch.from_numpy(x_np).pin_memory()
        yh = torch.empty((B, n), dtype=torch.float32).pin_memory()
        ke = max(2, min(args.steps, 5))
        api.process_host(plan, xh, yh, pieces=E2E_PIECES)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a0, a1 = ev(), ev()
        a0.record(stream)
        for _ in range(ke):
            api.process_host(plan, xh, yh, pieces=E2E_PIECES)
        a1.record(stream)
        torch.cuda.synchronize()
        ms_e2e = a0.elapsed_time(a1) / ke
        if world > 1:  # batch mode: ranks stream their own rows; the job ends with the last
            tm = torch.tensor([ms_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            ms_e2e = float(tm[0])
        e2e_err = float(np.linalg.norm(yh.numpy().astype(np.float64) - x_np) / np.linalg.norm(x_np))
        e2e = {"value": samples / (ms_e2e / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 4 * B_all * n, "d2h_bytes_per_step": 4 * B_all * n,
               "ms_per_step": ms_e2e, "recon_rel_l2": e2e_err,
               "api": f"paper_1210_0084_b200.api.process_host -> slicq_process_host (native executor, {E2E_PIECES} slice ranges, 3 streams)"}

    if sharded and not args.no_e2e:
        # end to end at N ranks through the public multi-GPU API (dist.SliceRangeShard): each
        # step copies this rank's input samples from pinned host memory, runs the sharded
        # forward + inverse (NCCL halo / spill exchange) and copies its output samples back
        a, b = shard.own
        hi = max(0, min(b, n) - a)
        xh = shard.local_input(torch.from_numpy(x_np)).pin_memory()
        yh = torch.empty((B, hi), dtype=torch.float32).pin_memory()

        def e2e_step():
            xl.copy_(xh, non_blocking=True)
            c_ = shard.forward(xl)
            y_ = shard.inverse(c_)
            if hi > 0:
                yh.copy_(y_[:, :hi], non_blocking=True)

        ke = max(2, min(args.steps, 5))
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a0, a1 = ev(), ev()
        a0.record(stream)
        for _ in range(ke):
            e2e_step()
        a1.record(stream)
        torch.cuda.synchronize()
        tt = torch.tensor([a0.elapsed_time(a1) / ke, 4.0 * B * xh.shape[1], 4.0 * B * hi],
                          dtype=torch.float64, device=dev)
        mx = tt[:1].clone()
        if world > 1:
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(tt)
        ms_e2e = float(mx[0])
        e2e = {"value": samples / (ms_e2e / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(tt[1]), "d2h_bytes_per_step": int(tt[2]),
               "ms_per_step": ms_e2e,
               "api": "paper_1210_0084_b200.dist.SliceRangeShard (pinned host copies of each "
                      "rank's range + sharded forward/inverse, max over ranks)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, dt, cores, desc, v1 = oracle_sample_rate(cfg)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
               "value_1core": v1, "cpu_model": cpu_model()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic", "config": config_dict(cfg, world),
            "forward_samples_per_s": samples / (ms_f / 1e3),
            "inverse_samples_per_s": samples / (ms_i / 1e3),
            "ms_forward": ms_f, "ms_inverse": ms_i, "step_stats": step_stats,
            "recon_rel_l2": rec,
            "roofline": {"bound": "hbm", "kernel": f"{dom} ({kernels})", "achieved": achieved,
                         "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch":
                             bytes_inv if dom == "slicq_inverse" else bytes_fwd},
            "roofline_step_frac": (bytes_fwd + bytes_inv) / (ms_step / 1e3) / 1e9 / peak,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def torchrun_cmd(argv, ngpus: int, port: int):
    """The command that re-launches this script with one process per GPU (torchrun, rendezvous
    on 127.0.0.1), for `--gpus N > 1` started without a launcher (no WORLD_SIZE)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={ngpus}", "--master-addr", "127.0.0.1", f"--master-port={port}",
            os.path.abspath(__file__), *argv]


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--force-shard", action="store_true",
                    help="run the multi-GPU slice-range code path even at N=1 (testing)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (rank 0 prints the JSON line)
        import subprocess
        sys.exit(subprocess.call(torchrun_cmd(sys.argv[1:], args.gpus, _free_port())))
    _, world, _ = _env_rank()
    if args.gpus > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    args.warmup = max(args.warmup, 3) if args.impl == "cuda" else args.warmup
    from synth.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
