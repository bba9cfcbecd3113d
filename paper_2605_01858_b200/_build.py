"""Build libdscache.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2605_01858_b200._build [--verbose]

The shared library is the C-ABI boundary (include/dscache.h); the Python
binding (dscache.py) loads it with ctypes.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdscache.so")
SOURCES = ["dscache_api.cu", "kernels_common.cu", "attn_fa.cu", "sched.cu", "decode.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "dscache.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), out: str = LIB) -> str:
    """Compile the library.  `defines` (e.g. ["DSC_POLY=2"]) build a tuning variant into `out`."""
    if not force and not defines and not needs_build():
        return LIB
    objs = []
    tag = "_".join(d.replace("=", "") for d in defines)
    tmp = os.path.join(PKG, "build", tag) if tag else os.path.join(PKG, "build")
    os.makedirs(tmp, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(tmp, src.replace(".cu", ".o"))
        cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
               "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src), "-o", obj]
        cmd += [f"-D{d}" for d in defines]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for cmd, p in procs:
        log, _ = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(log)
        if p.returncode:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    os.makedirs(os.path.dirname(out), exist_ok=True)
    link = [nvcc(), *ARCH, "-shared", "-o", out, *objs, "-lcudart_static"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    return out


def build_variant(name: str, defines) -> str:
    return build(force=True, defines=list(defines), out=os.path.join(PKG, "variants", f"libdscache_{name}.so"))


if __name__ == "__main__":
    if "--checked" in sys.argv:      # the DSC_CHECK bounds-check build (scripts/gpu_checked.sh)
        print(build_variant("checked", ["DSC_CHECK=1"]))
    elif "--variant" in sys.argv:      # --variant NAME DEF1 DEF2 ...
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:]))
    else:
        build(verbose="--verbose" in sys.argv, force=True)
        print(LIB)
