"""Build tools/libfp64peak.so (FP64 DFMA throughput probe, sm_100a)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "fp64_peak.cu")
LIB = os.path.join(HERE, "libfp64peak.so")


def build() -> str:
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", SRC, "-o", LIB])
    return LIB


def probe(blocks_per_sm: int = 8, iters: int = 20000, reps: int = 5):
    import ctypes
    lib = ctypes.CDLL(build())
    t, ms = ctypes.c_double(), ctypes.c_double()
    rc = lib.fp64_peak_probe(blocks_per_sm, iters, reps, ctypes.byref(t), ctypes.byref(ms))
    if rc != 0:
        raise RuntimeError("fp64 probe failed")
    return t.value, ms.value
