"""Build librba.so in-tree: nvcc for sm_100a (B200), linked against the NCCL that ships with torch."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librba.so")
SOURCES = ["rba_kernels.cu", "rba_sc.cu", "rba_factored.cu", "rba_sqrtba64.cu", "rba_lm.cu", "rba_api.cu", "rba_bal.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for base in spec.submodule_search_locations:
            cands.append(os.path.join(base, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc():
    for p in (os.environ.get("CUDA_HOME", ""), "/usr/local/cuda"):
        cand = os.path.join(p, "bin", "nvcc")
        if p and os.path.exists(cand):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile librba.so (or, with `defines` / `out`, a tuning variant of it for tools/)."""
    lib = out or LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in ("rba_internal.cuh", "rba_model.cuh")] + \
        [os.path.join(ROOT, "include", "rba.h")]
    if not force and os.path.exists(lib) and all(os.path.getmtime(lib) >= os.path.getmtime(d) for d in deps):
        return lib
    inc, libdir = _nccl_dirs()
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", os.path.join(ROOT, "include"), "-I", inc] + [f"-D{x}" for x in defines]
    if verbose:
        common += ["-Xptxas", "-v"]
    objs = []

    def comp(src):
        obj = os.path.join(CSRC, os.path.basename(src) + f".{os.path.basename(lib)}.o")
        r = subprocess.run(common + ["-c", src, "-o", obj], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(len(srcs)) as ex:
        objs = list(ex.map(comp, srcs))
    link = [nvcc(), *ARCH, "-shared", "-o", lib, *objs, "-L", libdir, "-l:libnccl.so.2", "-lz",
            "-Xlinker", f"-rpath,{libdir}"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv))
