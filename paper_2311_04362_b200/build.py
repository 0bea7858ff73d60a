"""Build libitsk_b200.so (sm_100a) in-tree with nvcc.

    python -m paper_2311_04362_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libitsk_b200.so")
SOURCES = ["capi.cu", "pattern.cu", "sketch.cu", "qr.cu", "qr2.cu", "qr_far.cu", "trsv.cu", "pass.cu", "loop.cu", "sparse.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-I" + CSRC, "-I" + os.path.join(ROOT, "include")]


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in deps)


def build(verbose: bool = False, jobs: int | None = None, probe: str | None = None) -> str:
    """probe="timeline": a diagnostic variant (libitsk_b200_timeline.so,
    -DITSK_TIMELINE: %globaltimer stamps of the loop's kernels) for
    scripts/loop_timeline.py; the product library is unchanged."""
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = os.path.join(HERE, "build" if probe is None else f"build_{probe}")
    lib_out = LIB if probe is None else os.path.join(HERE, f"libitsk_b200_{probe}.so")
    extra = [] if probe is None else [f"-DITSK_{probe.upper()}"]
    os.makedirs(objdir, exist_ok=True)
    # every header under csrc/ (a header missing from a hand-kept list left stale objects behind)
    hdrs = sorted(os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h")))
    hdrs.append(os.path.join(ROOT, "include", "itsk_b200.h"))
    objs, procs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if _stale(o, [s] + hdrs):
            cmd = [nvcc, *ARCH, *FLAGS, *extra, "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((src, out.decode()))
        elif verbose and out:
            print(out.decode())
    if failed:
        msg = "\n".join(f"--- {s}\n{o}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    if _stale(lib_out, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", lib_out, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return lib_out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, probe="timeline" if "--timeline" in sys.argv else None))
