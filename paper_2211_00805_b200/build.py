"""Build recipe for libgeosink_b200.so (nvcc, sm_100a) -- used by __graft_entry__.build().

Flags: -gencode arch=compute_100a,code=sm_100a; -lineinfo for ncu source attribution;
-fmad=false so the only fused operations are the explicit fma() calls mirrored by the oracle; the
32-bit mode computes in fp64 with the same chains (only its stored words are narrower) and its
kernels are tested bit-identical to one another, so the flag covers every translation unit.
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2211_00805_b200")
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib", "libgeosink_b200.so")
SOURCES = ["gs_core.cu", "gs_cheb.cu", "gs_graph.cu", "gs_reorder.cu", "gs_part.cu", "gs_euler.cu", "gs_dense.cu", "gs_win.cu", "gs_sell.cu", "gs_lane.cu", "gs_nccl.cu", "gs_knn_tc.cu", "gs_rng.cpp", "gs_io.cpp"]
HEADERS = ["gs_internal.cuh", "gs_step.cuh", "gs_win.cuh", "gs_sell.cuh", "gs_persist.cuh"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-fmad=false", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
              "-diag-suppress", "550"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "geosink_b200.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every source and link lib/libgeosink_b200.so (or `out`, for tuning variants
    built with extra -D defines)."""
    lib = out or LIB
    if not force and out is None and not defines and not _stale():
        return LIB
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    tag = "" if out is None else "_" + os.path.basename(out).replace(".so", "")
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(PKG, "lib", src.rsplit(".", 1)[0] + tag + ".o")
        cmd = ["nvcc", *NVCC_FLAGS, *["-D" + d for d in defines], "-c", "-I",
               os.path.join(ROOT, "include"), "-o", obj, os.path.join(CSRC, src)]
        cmd = [c for c in cmd if c != "-shared"]
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), cmd))
        objs.append(obj)
    logs = []
    for p, cmd in procs:
        out, _ = p.communicate()
        logs.append(out.decode())
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    link = ["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib, *objs, "-ldl"]
    subprocess.run(link, check=True)
    with open(os.path.join(PKG, "lib", "ptxas" + tag + ".log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                out=outs[0] if outs else None))
