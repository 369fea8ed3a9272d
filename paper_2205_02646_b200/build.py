"""Build libtqsb.so in-tree: nvcc for the sm_100a kernels, g++ for the host C++.

    python paper_2205_02646_b200/build.py        (or __graft_entry__.build())

Incremental (rebuilds an object only when its sources are newer). The .so is
git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libtqsb.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU = ["tables.cu", "solve_f32.cu", "solve_f64.cu", "solve_f64r.cu", "solve_ljsde.cu", "sensor.cu", "probe.cu"]
CPP = ["plan.cpp", "io.cpp"]
HEADERS = [os.path.join(CSRC, "tqsb_internal.hpp"), os.path.join(CSRC, "solve_common.cuh"),
           os.path.join(INCLUDE, "tqsb", "tqsb.h"),
           os.path.abspath(__file__)]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))


def build(verbose: bool = False, defines: list[str] | None = None, lib: str | None = None,
          tag: str = "") -> str:
    """defines/lib/tag: experiment variants (e.g. -DTQSB_WARPS_F32=8 into libtqsb_w8.so)."""
    defines = [f"-D{d}" for d in (defines or [])]
    build_dir = BUILD + tag
    lib = lib or LIB
    os.makedirs(build_dir, exist_ok=True)
    jobs = []
    objs = []
    for f in CU:
        src = os.path.join(CSRC, f)
        obj = os.path.join(build_dir, f + ".o")
        objs.append(obj)
        if _newer(obj, [src] + HEADERS):
            jobs.append([NVCC, *ARCH, *defines, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                         "-Xptxas", "-warn-spills", "-I", INCLUDE, "-c", src, "-o", obj])
    for f in CPP:
        src = os.path.join(CSRC, f)
        obj = os.path.join(build_dir, f + ".o")
        objs.append(obj)
        if _newer(obj, [src] + HEADERS):
            # x86-64-v3 + contraction: the input generators then round exactly like the
            # reference build (g++ -O3 -march=native contracts a*b+c into FMA)
            jobs.append(["g++", "-std=c++17", "-O3", "-march=x86-64-v3", "-ffp-contract=fast",
                         "-fPIC", "-Wall", "-Wextra", "-pthread", *defines,
                         "-I", os.path.join(CUDA, "include"), "-I", INCLUDE, "-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for cmd in jobs:
            if verbose:
                print(" ".join(cmd))
        list(ex.map(_run, jobs))
    if _newer(lib, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib + ".tmp", *objs,
              "-Xcompiler", "-pthread"])
        os.replace(lib + ".tmp", lib)
    if lib == LIB:
        build_cli(lib)
    return lib


def build_cli(lib: str = LIB) -> str:
    """bin/tqsb: the command-line toolbox (csrc/cli/tqsb_cli.cpp) over libtqsb.so."""
    src = os.path.join(CSRC, "cli", "tqsb_cli.cpp")
    out = os.path.join(HERE, "bin", "tqsb")
    deps = [src, lib, os.path.join(INCLUDE, "tqsb", "reconstruct.hpp"),
            os.path.join(INCLUDE, "tqsb", "io.hpp"), os.path.join(INCLUDE, "tqsb", "tqsb.h")]
    if _newer(out, deps):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        _run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", INCLUDE, src, "-L", HERE,
              "-l:" + os.path.basename(lib), "-Wl,-rpath,$ORIGIN/..", "-o", out + ".tmp"])
        os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    # python build.py [VARIANT_TAG DEFINE ...]  e.g.  python build.py w8 TQSB_WARPS_F32=8
    if len(sys.argv) > 1:
        tag = sys.argv[1]
        print(build(verbose=True, defines=sys.argv[2:], tag="_" + tag,
                    lib=os.path.join(HERE, f"libtqsb_{tag}.so")))
    else:
        print(build(verbose=True))
