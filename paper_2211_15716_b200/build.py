"""Build libigg.so in-tree for sm_100a with nvcc (no JIT, no torch extension).

The library links cudart statically and libnccl.so.2 from the torch wheel's
nvidia-nccl package (rpath), so it loads on a box without a GPU (symbol
checks) and on the B200 boxes (same image).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libigg.so")
SOURCES = ["topology.cpp", "plan.cpp", "grid.cpp", "kernels.cu", "fused.cu", "halo26.cu", "acoustic.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_root() -> str:
    import nvidia.nccl  # the NCCL that torch itself loads
    return os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "igg.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, extra=()) -> str:
    """out / extra: another build of the same sources (e.g. an A/B variant with -D flags, loaded with
    IGG_LIBRARY=<out>); the default is the product library in-tree."""
    if out is None and not force and not needs_build():
        return OUT
    target = out or OUT
    os.makedirs(os.path.dirname(os.path.abspath(target)), exist_ok=True)
    nr = nccl_root()
    inc = os.path.join(nr, "include")
    lib = os.path.join(nr, "lib")
    objs = []
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden,-ffp-contract=off",
              "-I", inc, "-I", os.path.join(HERE, "..", "include")]
    for src in SOURCES:
        obj = os.path.join(CSRC, src + (".%d.o" % os.getpid()))
        cmd = [nvcc()] + ARCH + common + list(extra) + ["-fmad=false", "-Xptxas", "-v" if verbose else "-O3",
                                          "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    link = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", target] + objs + [
        "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libigg.so failed")
    for o in objs:
        os.remove(o)
    return target


if __name__ == "__main__":
    # python build.py [--force] [-v] [--out PATH -DFLAG ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    extra = [x for x in args if x.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, out=out, extra=extra))
