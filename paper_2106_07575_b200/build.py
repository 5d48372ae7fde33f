"""Build libptyger.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_2106_07575_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libptyger.so")
OBJ = os.path.join(PKG, "_build")
SOURCES = ["kernels_frame.cu", "kernels_ls128.cu", "kernels_c256.cu", "kernels_p2p.cu", "kernels_n256.cu", "kernels_misc.cu", "kernels_fft.cu", "kernels_peak.cu", "ctx.cu",
           "host.cpp"]
HEADERS = ["fft.cuh", "dev.cuh", "tma.cuh", "internal.h", "host.h", "p2p.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    try:
        import nvidia  # type: ignore
        for p in nvidia.__path__:
            inc = os.path.join(p, "nccl", "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    return "/usr/include"


def _nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "ptyger.h"),
                                                                  __file__]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    nvcc = _nvcc()
    common = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
              "-I" + CSRC, "-I" + _nccl_include()]
    procs = []
    objs = []
    for src in SOURCES:
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        cmd = [nvcc] + ARCH + common + ["-c", os.path.join(CSRC, src), "-o", o]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if os.environ.get("PTYGER_PTXAS_V") else []
        procs.append((src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for src, cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((src, cmd, out.decode(errors="replace")))
        elif verbose and out:
            sys.stdout.write(out.decode(errors="replace"))
    if failed:
        msg = "\n".join(f"--- {s}: {' '.join(c)}\n{o}" for s, c, o in failed)
        raise RuntimeError("libptyger build failed:\n" + msg)
    tmp = LIB + ".tmp"
    link = [nvcc] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl"]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("libptyger link failed:\n" + r.stdout.decode(errors="replace"))
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
