"""Build liblopa.so (sm_100a only) in-tree with nvcc.  No CPU fallback, no other archs.

    python -m paper_2512_16229_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import site
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblopa.so")
SOURCES = ["lopa_core.cu", "lopa_syn.cu", "lopa_bp.cu", "lopa_lmhead.cu", "lopa_d2f.cu", "lopa_graph.cu"]
HEADERS = ["lopa_ptx.cuh", "lopa_decide.cuh", "lopa_internal.h", "lopa_k1_ldg.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    """The NCCL that torch loads (nvidia-nccl wheel); the system copy is older."""
    for sp in site.getsitepackages() + [site.getusersitepackages()]:
        base = os.path.join(sp, "nvidia", "nccl")
        if os.path.exists(os.path.join(base, "include", "nccl.h")):
            return os.path.join(base, "include"), os.path.join(base, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "liblopa.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines: tuple = ()) -> str:
    """Build liblopa.so, or liblopa_<variant>.so with extra -D defines (tuning A/B builds;
    select at run time with LOPA_LIB_VARIANT=<variant>)."""
    out = LIB if not variant else os.path.join(PKG, f"liblopa_{variant}.so")
    if not variant and not force and not stale():
        return LIB
    inc, lib = _nccl_dirs()
    cmd = [
        _nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--shared", "-Xcompiler", "-fPIC",
        "-Xcompiler", "-fvisibility=hidden", "-cudart", "static",
        "-I", os.path.join(ROOT, "include"), "-I", inc,
        *[os.path.join(CSRC, f) for f in SOURCES],
        "-L", lib, "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}",
        *[f"-D{d}" for d in defines],
        "-o", out + ".tmp",
    ]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--variant")
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, variant=a.variant, defines=tuple(a.D)))
