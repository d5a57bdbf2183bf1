"""Build the engine shared library in-tree (nvcc / g++, no JIT cache).

    python -m paper_2107_05337_b200.build

Produces ``paper_2107_05337_b200/_lib/libphi_engine.so`` for sm_100a.  CUDA
sources are compiled with ``-fmad=false`` and host sources with
``-ffp-contract=off``: the engine reproduces the reference's (non-fused)
floating-point evaluation order, which is what makes its results
bit-identical to the CPU reference on identical inputs.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# developer trace builds go to their own directory (PHI_TRACE=1 -> _lib_trace)
# developer A/B builds: PHI_VARIANT=name PHI_VARIANT_FLAGS="-DX=1 ..." -> _lib_<name>
_VARIANT = os.environ.get("PHI_VARIANT", "")
OUT_DIR = os.path.join(HERE, "_lib_trace" if os.environ.get("PHI_TRACE") == "1"
                       else ("_lib_" + _VARIANT if _VARIANT else "_lib"))
LIB = os.path.join(OUT_DIR, "libphi_engine.so")
ROOT = os.path.dirname(HERE)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_INC = "/usr/local/cuda/include"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-ffp-contract=off", "-Xptxas", "-v", "--expt-relaxed-constexpr"]
if os.environ.get("PHI_TRACE") == "1":  # developer timing stamps (tools/probe_*.py)
    NVCC_FLAGS += ["-DPHI_TRACE_ON=1"]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wno-unused-function",
             f"-I{CUDA_INC}"]
if _VARIANT:
    NVCC_FLAGS += os.environ.get("PHI_VARIANT_FLAGS", "").split()
    CXX_FLAGS += os.environ.get("PHI_VARIANT_FLAGS", "").split()

CU = ["phi_launch.cu", "assembly.cu", "spmm.cu", "ilut.cu"]
DEGREES = range(1, 9)  # phi_deg.cu is compiled once per spline degree (-DPHI_DEG=d)
CPP = ["setup_host.cpp", "engine.cpp", "capi.cpp", "timeshard.cpp"]
HEADERS = ["common.hpp", "device_types.cuh", "phi_kernels.cuh", "phi_device.cuh", "setup_host.hpp", "engine.hpp",
           "timeshard.hpp"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], log: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")


def build(verbose: bool = False) -> str:
    os.makedirs(os.path.join(OUT_DIR, "obj"), exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "phi_engine.h")]
    # a change of compiler flags (e.g. PHI_TRACE) invalidates every object
    stamp = os.path.join(OUT_DIR, "obj", "flags.txt")
    flags = " ".join(NVCC_FLAGS + CXX_FLAGS)
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        for f in os.listdir(os.path.join(OUT_DIR, "obj")):
            if f.endswith(".o"):
                os.remove(os.path.join(OUT_DIR, "obj", f))
        with open(stamp, "w") as fh:
            fh.write(flags)
    jobs, objs = [], []  # compile commands still to run; every object of the library
    for src in CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT_DIR, "obj", src + ".o")
        objs.append(o)
        if _newer(o, [s] + hdrs):
            jobs.append([NVCC] + NVCC_FLAGS + ["-c", s, "-o", o])
    for d in DEGREES:
        s = os.path.join(CSRC, "phi_deg.cu")
        o = os.path.join(OUT_DIR, "obj", f"phi_deg{d}.cu.o")
        objs.append(o)
        if _newer(o, [s] + hdrs):
            jobs.append([NVCC] + NVCC_FLAGS + [f"-DPHI_DEG={d}", "-c", s, "-o", o])
    for src in CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT_DIR, "obj", src + ".o")
        objs.append(o)
        if _newer(o, [s] + hdrs):
            jobs.append(["g++"] + CXX_FLAGS + ["-c", s, "-o", o])
    def compile_one(cmd: list[str]) -> list[str]:
        out: list[str] = []
        _run(cmd, out)
        return out

    log: list[str] = []
    with ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
        for part in ex.map(compile_one, jobs):
            log += part
    if jobs or _newer(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-ldl"], log)
    with open(os.path.join(OUT_DIR, "build.log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
