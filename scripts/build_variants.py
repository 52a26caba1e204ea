"""Build timing variants of libigg.so (experiment infrastructure): copies the package to /tmp, applies a
source transform to csrc/fused.cu, builds, and drops the library into ab/libigg_<name>.so, to be loaded with
IGG_LIBRARY=... for A/B timing of several builds on one box."""
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def inline_all(s):
    """the tile decode and the face epilogue written inline in the kernel body"""
    a = s.index("template <bool XS>\n__device__ __forceinline__ void fused_faces(")
    b = s.index("\n}\n", a) + 3
    body = s[a:b]
    hdr_end = body.index("    __syncthreads();          // the CTA's T2 stores are visible to the CTA\n")
    inner = body[hdr_end:body.rindex("}")]
    s = s[:a] + s[b:]
    s = s.replace("    if (face_tile) fused_faces<XS>(F, td, zs, ze);   // CTA-uniform\n",
                  "    if (!face_tile) return;   // CTA-uniform\n    double *__restrict__ T2 = F.T2;\n" + inner)
    return s


def noinline(s):
    return s.replace("template <bool XS>\n__device__ __forceinline__ void fused_faces(",
                     "template <bool XS>\n__device__ __noinline__ void fused_faces(")


def lb9(s):
    return s.replace("__launch_bounds__(32 * kFTY, 10) heat_fused_kernel", "__launch_bounds__(32 * kFTY, 9) heat_fused_kernel")


def stcs(s):
    return s.replace("                *reinterpret_cast<double2 *>(T2 + i) = make_double2(r0, r1);",
                     "                __stcs(reinterpret_cast<double2 *>(T2 + i), make_double2(r0, r1));")


VARIANTS = {"cur": [], "lb9": [lb9], "stcs": [stcs]}   # (inline_all/noinline applied to an older layout)


def build(name, fns):
    d = f"/tmp/var_{name}"
    shutil.rmtree(d, ignore_errors=True)
    shutil.copytree(os.path.join(ROOT, "paper_2211_15716_b200"), os.path.join(d, "paper_2211_15716_b200"),
                    ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(d, "include"))
    p = os.path.join(d, "paper_2211_15716_b200", "csrc", "fused.cu")
    s = open(p).read()
    for f in fns:
        s2 = f(s)
        assert s2 != s, (name, f.__name__)
        s = s2
    open(p, "w").write(s)
    r = subprocess.run([sys.executable, "-c", "from paper_2211_15716_b200 import build as b; b.build(force=True)"],
                       cwd=d, capture_output=True, text=True)
    if r.returncode:
        print(r.stdout, r.stderr)
        raise SystemExit(name)
    os.makedirs(os.path.join(ROOT, "ab"), exist_ok=True)
    shutil.copy(os.path.join(d, "paper_2211_15716_b200", "libigg.so"), os.path.join(ROOT, "ab", f"libigg_{name}.so"))
    r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                        "-Xptxas", "-v", "-fmad=false", "-c", p, "-o", "/tmp/x.o", "-I",
                        os.path.join(d, "paper_2211_15716_b200", "csrc")], capture_output=True, text=True)
    props = re.findall(r"heat_fused_kernelILb0E.*?\n.*?\n(.*?)\n(.*?)\n", r.stderr)
    print(name, props[:1])


if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        build(n, VARIANTS[n])
