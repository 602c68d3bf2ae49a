"""Build libspinsim_b200.so in-tree with nvcc for sm_100a (and only sm_100a).

    python -m paper_2204_05586_b200.build        # or __graft_entry__.build()

Each .cu in csrc/ compiles to an object in parallel (-O3 -lineinfo, -Xptxas -v logged to build/ptxas.log), then
nvcc links them into a shared library with the CUDA runtime linked statically (no libcudart.so dependency).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libspinsim_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I", INCLUDE]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "spinsim_b200.h")]


def _compile(src: str, variant: str = "", defines=()) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + (f".{variant}" if variant else "") + ".o")
    newest = max(os.path.getmtime(d) for d in _deps())
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build the library; a non-empty `variant` (tuning experiments only) builds libspinsim_b200.<variant>.so with
    extra -D `defines`, loadable through SPINSIM_LIB."""
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    lib = LIB if not variant else LIB[:-3] + f".{variant}.so"
    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, variant, defines), srcs))
    objs = [o for o, _ in results]
    log = "".join(l for _, l in results)
    if log:
        with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
            f.write(log)
    if not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", *objs, "-o", lib]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(lib)
    return lib


if __name__ == "__main__":
    if len(sys.argv) > 2:          # python -m paper_2204_05586_b200.build <variant> NAME=VALUE ...
        build(verbose=True, variant=sys.argv[1], defines=sys.argv[2:])
    else:
        build(verbose=True)
    sys.exit(0)
