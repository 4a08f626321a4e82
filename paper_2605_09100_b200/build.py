"""Builds libhpa.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python paper_2605_09100_b200/build.py [--force] [-v] [-DNAME=VAL ... --out=path]

(run by path: importing the package would load the library it is building)

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo; the CUDA runtime
is linked statically and the driver is reached through
cudaGetDriverEntryPoint, so the library loads on hosts without a driver.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libhpa.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["decode.cu", "prefill.cu", "copy_kernels.cu"]
CPP_SOURCES = ["runtime.cpp"]
HEADERS = ["hpa_kernels.h", "ptx.cuh"]


def _newest_dep() -> float:
    deps = [os.path.join(CSRC, f) for f in CU_SOURCES + CPP_SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "hpa.h"))
    deps.append(os.path.abspath(__file__))
    return max(os.path.getmtime(p) for p in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout, r.stderr, flush=True)
    return r


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """defines: extra -D flags (variant builds for A/B experiments go to `out`)."""
    if not force and not defines and os.path.exists(out) and os.path.getmtime(out) >= _newest_dep():
        return out
    build_dir = BUILD if not defines else BUILD + "_" + "_".join(d.replace("=", "") for d in defines)
    os.makedirs(build_dir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    common += [f"-D{d}" for d in defines]
    jobs = []
    for f in CU_SOURCES:
        obj = os.path.join(build_dir, f + ".o")
        jobs.append(([NVCC, *ARCH, *common, "-lineinfo", "-Xptxas", "-v", "--expt-relaxed-constexpr",
                      "-c", os.path.join(CSRC, f), "-o", obj], obj))
    for f in CPP_SOURCES:
        obj = os.path.join(build_dir, f + ".o")
        jobs.append(([NVCC, *common, "-x", "c++", "-c", os.path.join(CSRC, f), "-o", obj], obj))
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        results = list(ex.map(lambda j: _run(j[0], verbose), jobs))
    with open(os.path.join(build_dir, "ptxas.log"), "w") as f:
        for (cmd, _), r in zip(jobs, results):
            f.write(f"## {cmd[-3]}\n{r.stderr}\n")
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", out + ".tmp", *[o for _, o in jobs]], verbose)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                out=outs[0] if outs else LIB))
