"""In-tree build of libmrf_cuda.so for sm_100a (nvcc cross-compiles; no GPU needed).

Translation units are compiled in parallel to objects under build/, then
linked into paper_1910_10892_b200/libmrf_cuda.so.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
UNITS = ["mrf_cuda.cu", "misc.cu", "head.cu", "sgm.cu", "topology.cpp", "fwd_generic.cu", "fwd_band2_isgmr.cu", "fwd_band2_trwp.cu", "fwd_bandw.cu", "fwd_small.cu",
         "bwd_isgmr.cu", "bwd_trwp.cu"]
OUT = os.path.join(HERE, "libmrf_cuda.so")
OBJDIR = os.path.join(ROOT, "build", "mrf_cuda")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-lineinfo", "-O3", "-std=c++17",
    # Bit-exact argmins need one rounding per operation: no FMA contraction,
    # IEEE division/sqrt, no flush-to-zero (SURVEY.md §7 hard part 1).
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
] + os.environ.get("MRF_NVCC_EXTRA", "").split()


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def _deps():
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".hpp", ".cpp"))]
    return deps + [os.path.join(ROOT, "include", "mrf_cuda.h"), __file__]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in _deps())


def _compile(unit: str):
    src = os.path.join(CSRC, unit)
    obj = os.path.join(OBJDIR, unit + ".o")
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    return obj, res.stderr


CLI_SRC = os.path.join(HERE, "cli", "mrfmp_cuda.cpp")
CLI_OUT = os.path.join(HERE, "bin", "mrfmp_cuda")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build_cli() -> str:
    """The reference CLI's `run` driver over the C++ drop-in header
    (cli/mrfmp_cuda.cpp), linked against the in-tree libmrf_cuda.so."""
    deps = [CLI_SRC, OUT, os.path.join(ROOT, "include", "mrf", "mp_cuda.hpp"), os.path.join(ROOT, "include", "mrf", "io.hpp")]
    if os.path.exists(CLI_OUT) and all(os.path.getmtime(d) <= os.path.getmtime(CLI_OUT) for d in deps):
        return CLI_OUT
    os.makedirs(os.path.dirname(CLI_OUT), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA_HOME, "include"),
           CLI_SRC, "-o", CLI_OUT + ".tmp", "-L", HERE, "-lmrf_cuda", "-L", os.path.join(CUDA_HOME, "lib64"), "-lcudart",
           "-Wl,-rpath,$ORIGIN/..:" + os.path.join(CUDA_HOME, "lib64")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("CLI build failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    os.replace(CLI_OUT + ".tmp", CLI_OUT)
    return CLI_OUT


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        build_cli()
        return OUT
    os.makedirs(OBJDIR, exist_ok=True)
    workers = max(1, min(len(UNITS), os.cpu_count() or 1))
    with cf.ThreadPoolExecutor(workers) as ex:
        results = list(ex.map(_compile, UNITS))
    objs = [o for o, _ in results]
    cmd = [nvcc(), *ARCH, "-shared", "-o", OUT + ".tmp", *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    os.replace(OUT + ".tmp", OUT)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write("".join(log for _, log in results))
    if verbose:
        print("".join(log for _, log in results), file=sys.stderr)
    build_cli()
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
