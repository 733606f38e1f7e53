"""Build libf3s.so in-tree with nvcc for sm_100a (no GPU needed: nvcc cross-compiles)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libf3s.so")
SOURCES = ["f3s_api.cu", "plan.cu", "attention_simt.cu", "attention_sm100.cu", "backward.cu", "backward_sm100.cu"]
HEADERS = ["internal.h", "sm100.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC,-O2"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "f3s.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, defines=(), variant: str = "") -> str:
    """variant/defines: experiment builds libf3s_<variant>.so with extra -D flags (selected at run
    time by F3S_LIB_VARIANT; diagnostics only, the product library is libf3s.so)."""
    lib = LIB if not variant else os.path.join(HERE, f"libf3s_{variant}.so")
    if not force and not variant and not _stale():
        return LIB
    objs = []
    build_dir = os.path.join(HERE, "build" + (f"_{variant}" if variant else ""))
    os.makedirs(build_dir, exist_ok=True)
    for src in SOURCES:
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys
    args = [a for a in sys.argv[1:] if a != "-v"]
    if args:  # python _build.py VARIANT DEF1=1 DEF2=3 ...
        print(build(force=True, verbose="-v" in sys.argv, variant=args[0], defines=args[1:]))
    else:
        print(build(force=True, verbose="-v" in sys.argv))
