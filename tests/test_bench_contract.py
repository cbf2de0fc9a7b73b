"""bench.py's JSON-line contract (the driver parses it): the reference arm on CPU, the CUDA
arm on a GPU (small config, few steps)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"]


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "1"], 600)
    for k in BASE:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_gpus_flag_relaunches_one_process_per_gpu():
    """`bench.py --gpus N` without a launcher re-executes itself under torchrun with N
    processes on one node (rendezvous on 127.0.0.1), forwarding every argument."""
    sys.path.insert(0, ROOT)
    import bench
    cmd = bench.torchrun_cmd(["--gpus", "8", "--steps", "3"], 8, 29511)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "8", "--steps", "3"] and cmd[-5].endswith("bench.py")


def test_reference_arm_under_launcher_world_2():
    """The reference arm launched with --gpus 2 (re-launched under torchrun): rank 0 alone runs
    and prints one line with n_gpus = 2; the other rank exits 0 without work."""
    d = _run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0",
              "--gpus", "2"], 900)
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


@pytest.mark.gpu
def test_cuda_arm_line():
    d = _run(["--config", "1", "--steps", "5", "--warmup", "3"], 1200)
    for k in BASE + ["roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"]:
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    rf = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert 0 < rf["frac"] < 1
    assert d["gpu_launches"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["recon_rel_l2"] <= 1e-5
    assert e["recon_rel_l2"] <= 1e-5  # the host round trip reconstructs too
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
