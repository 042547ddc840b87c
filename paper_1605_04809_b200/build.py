"""Build libnmt.so in-tree for sm_100a with nvcc (no JIT cache; the .so travels with the repo)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libnmt.so")
SOURCES = ["gemm.cu", "kernels.cu", "api.cu", "ensemble.cu", "randparams.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "nmt.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, diag: bool = False, variant: str = "",
          defines: tuple = ()) -> str:
    """diag: a separate libnmt_diag.so with the -DNMT_DIAG switches (stage skipping, traces, ...) for
    measurements only; the product library ignores the environment.  variant + defines: an A/B build
    libnmt_var_<variant>.so (libnmt_diag_<variant>.so with diag) with extra -D flags, for measurements."""
    if variant:
        lib = os.path.join(HERE, f"libnmt_{'diag' if diag else 'var'}_{variant}.so")
        bdir = os.path.join(BUILD, f"{'diag' if diag else 'var'}_{variant}")
    else:
        lib = os.path.join(HERE, "libnmt_diag.so") if diag else LIB
        bdir = os.path.join(BUILD, "diag") if diag else BUILD
    if not diag and not variant and not force and not _stale():
        return LIB
    os.makedirs(bdir, exist_ok=True)

    def compile_one(src: str) -> str:
        obj = os.path.join(bdir, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *FLAGS, *(["-DNMT_DIAG"] if diag else []), *[f"-D{x}" for x in defines], "-Xptxas", "-v" if verbose else "-O3", "-c",
               os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-ldl",
           "-Xcompiler", "-fvisibility=hidden"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, diag="--diag" in sys.argv))
