"""Build libcascade_b200.so in-tree for sm_100a (nvcc; no torch extension
machinery -- the library is a plain C-ABI shared object)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcascade_b200.so")
AB_LIB = os.path.join(HERE, "libcascade_b200_ab.so")
SOURCES = ["host.cpp", "eam_kernels.cu", "store_kernels.cu", "capi.cu", "peak.cu", "slab.cu", "comm.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC,-fvisibility=hidden,-ffp-contract=off",
         "-Xptxas", "-v", "-cudart", "static", "-ldl"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "cascade_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, ab: bool = False) -> str:
    """ab: the experiment build (-DCBX_AB, the A/B environment switches live)
    into libcascade_b200_ab.so, loaded with CBX_LIB=<path>"""
    out = AB_LIB if ab else LIB
    if not ab and not force and not stale():
        return LIB
    # one object per translation unit, compiled in parallel, then linked
    import concurrent.futures as cf
    import tempfile
    tmp = tempfile.mkdtemp(prefix="cbx_build_")
    extra = ["-DCBX_AB"] if ab else []
    objs = [os.path.join(tmp, os.path.splitext(s)[0] + ".o") for s in SOURCES]
    cmds = [[nvcc()] + ARCH + FLAGS + extra + ["-c", "-o", o, os.path.join(CSRC, s)]
            for s, o in zip(SOURCES, objs)]
    link = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-ldl", "-o", out] + objs
    with cf.ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        rs = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds))
    log = os.path.join(HERE, "build.log")
    text = "".join(" ".join(c) + "\n" + r.stdout + r.stderr for c, r in zip(cmds, rs))
    bad = [r for r in rs if r.returncode != 0]
    if not bad:
        r = subprocess.run(link, capture_output=True, text=True)
        text += " ".join(link) + "\n" + r.stdout + r.stderr
        if r.returncode != 0:
            bad = [r]
    with open(log, "w") as f:
        f.write(text)
    if bad:
        sys.stderr.write(bad[0].stderr[-6000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(text)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, ab="--ab" in sys.argv))
