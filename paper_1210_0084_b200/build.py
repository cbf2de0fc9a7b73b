"""Build libslicq.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache).

    python -m paper_1210_0084_b200.build          # or __graft_entry__.build()

The per-size kernel instantiations (kernels_spec.cu for 2N = 4096 .. 32768, kernels_large.cu
for 2N = 65536, 131072) are one source compiled once per size (-DSLICQ_LOGN=...) in parallel;
the host plan (plan.cpp) and the dispatch (kernels_host.cu, fused_host.cu) are linked with
them into one shared library with a static CUDA runtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libslicq.so")
OBJ = os.path.join(PKG, "_build")

# (source, object name, extra defines)
SOURCES = [("plan.cpp", "plan", ()), ("kernels_host.cu", "kernels_host", ()),
           ("fused_host.cu", "fused_host", ())]
SOURCES += [("kernels_spec.cu", f"kernels_spec_l{n}", (f"SLICQ_LOGN={n}",)) for n in (11, 12, 13, 14)]
SOURCES += [("kernels_large.cu", f"kernels_large_l{n}", (f"SLICQ_LOGN={n}",)) for n in (15, 16)]
SOURCES += [("kernels_generic.cu", "kernels_generic", ())]
SOURCES += [("kernels_long.cu", "kernels_long", ()), ("kernels_complex.cu", "kernels_complex", ()),
            ("kernels_coeff.cu", "kernels_coeff", ()), ("stream_exec.cpp", "stream_exec", ())]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v"]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def _compile(unit, objdir: str = OBJ, extra=()) -> tuple[str, str]:
    src, name, defines = unit
    obj = os.path.join(objdir, name + ".o")
    cmd = [nvcc(), *ARCH, *FLAGS, *extra, *[f"-D{d}" for d in defines], "-x", "cu", "-c",
           os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}:\n{r.stderr}")
    return obj, r.stderr


def _stale(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(PKG, "..", "include", "slicq.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, debug_timing: bool = False,
          variant: str = "", defines=(), only=()) -> str:
    """Build libslicq.so (or, with debug_timing, libslicq_dbg.so with per-phase clock64
    instrumentation for tools/phase_timing.py; or, with variant, libslicq_<variant>.so with
    extra -D defines for tuning experiments, selected via SLICQ_LIB; never used by the
    product path)."""
    tag = "dbg" if debug_timing else variant
    out = OUT if not tag else os.path.join(PKG, f"libslicq_{tag}.so")
    if not force and not _stale(out):
        return out
    objdir = OBJ if not tag else OBJ + "_" + tag
    os.makedirs(objdir, exist_ok=True)
    extra = (["-DSLICQ_PHASE_TIMING"] if debug_timing else []) + [f"-D{d}" for d in defines]
    # only: object names a tuning variant recompiles; the rest is linked from the main build
    def one(s):
        if only and s[1] not in only:
            return os.path.join(OBJ, s[1] + ".o"), ""
        return _compile(s, objdir, extra)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(one, SOURCES))
    log = "\n".join(r[1] for r in results)
    with open(os.path.join(objdir, "ptxas.log"), "w") as f:
        f.write(log)
    if verbose:
        print(log)
    tmp = out + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *[r[0] for r in results]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                debug_timing="--debug-timing" in sys.argv))
