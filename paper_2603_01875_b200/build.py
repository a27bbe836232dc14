"""Build libkdfused.so in-tree: nvcc, sm_100a only (no other targets, no JIT).

    python -m paper_2603_01875_b200.build [--verbose]
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libkdfused.so")
SOURCES = ["kd_pass.cu", "kd_gemm.cu", "kd_aux.cu", "kd_stage.cu", "kd_api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def flags(verbose: bool = False) -> list[str]:
    f = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
                "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    if verbose:
        f += ["-Xptxas", "-v"]
    return f


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, s) for s in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "kdfused.h"),
                                                                  os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: str = OUT) -> str:
    """defines: extra -D macros for instrumented variants (e.g. ("KD_EPI_TIMING",) -> libkdfused_tim.so, used by
    scripts/probe_epi.py); the product library is built without any."""
    if not force and out == OUT and not _stale():
        return OUT
    bdir = os.path.join(HERE, "_build" + ("_" + "_".join(defines).lower() if defines else ""))
    os.makedirs(bdir, exist_ok=True)
    cc = nvcc()
    objs = []
    procs = []
    for s in SOURCES:
        o = os.path.join(bdir, s.replace(".cu", ".o"))
        objs.append(o)
        cmd = [cc, *flags(verbose), *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, s), "-o", o]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for cmd, p in procs:
        log, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{log}")
        if verbose and log:
            print(log)
    tmp = os.path.join(bdir, os.path.basename(out) + ".link")  # link output under _build/, then moved into place
    link = [cc, *ARCH, "-shared", "-o", tmp, *objs, "-lcuda"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        # libcuda may be absent on a CPU box: link against the driver stub instead
        stub = "/usr/local/cuda/lib64/stubs"
        link = [cc, *ARCH, "-shared", "-o", tmp, *objs, "-L", stub, "-lcuda"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(link)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    if "--timing" in sys.argv:
        print(build(force=True, defines=("KD_EPI_TIMING",), out=os.path.join(HERE, "libkdfused_tim.so")))
    else:
        print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
