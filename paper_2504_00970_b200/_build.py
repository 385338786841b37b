"""Build libsentencekv.so in-tree with nvcc for sm_100a (B200).  No JIT, no torch extension:
the product is a plain C-ABI shared library (include/sentencekv.h)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
TRACE = os.environ.get("SKV_TRACE", "") == "1"  # phase-timestamp build for kernel studies
# A/B experiments: SKV_VARIANT=<name> SKV_DEFS="-DX=1 ..." builds libsentencekv_<name>.so beside the
# product library (selected at run time with SKV_LIB); never the product path
VARIANT = os.environ.get("SKV_VARIANT", "trace" if TRACE else "")
DEFS = os.environ.get("SKV_DEFS", "").split()
BUILD = os.path.join(HERE, f"build_{VARIANT}" if VARIANT else "build")
LIB = os.path.join(HERE, f"libsentencekv_{VARIANT}.so" if VARIANT else "libsentencekv.so")
SOURCES = ["prefill.cu", "retain.cu", "variants.cu", "local.cu", "decode_select.cu", "decode_attend_mma.cu", "decode_unit.cu", "abi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v"] + (
    ["-DSKV_TRACE"] if TRACE else []) + DEFS


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "sentencekv.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        with open(os.path.join(BUILD, src + ".ptxas.txt"), "w") as f:
            f.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    os.replace(tmp, LIB)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
