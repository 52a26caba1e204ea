"""Build acoustic tiling variants of libigg.so (experiment infrastructure): copies the package to /tmp,
changes kAcTY (rows per CTA) / kAcKC (planes per CTA) in csrc/acoustic.cu, builds, and drops the library
into ab/libigg_ac_<TY>_<KC>.so, loaded with IGG_LIBRARY=... for A/B timing on one box."""
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build(ty, kc):
    name = f"ac_{ty}_{kc}"
    d = f"/tmp/var_{name}"
    shutil.rmtree(d, ignore_errors=True)
    shutil.copytree(os.path.join(ROOT, "paper_2211_15716_b200"), os.path.join(d, "paper_2211_15716_b200"),
                    ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(d, "include"))
    p = os.path.join(d, "paper_2211_15716_b200", "csrc", "acoustic.cu")
    s = open(p).read()
    s2 = s.replace("constexpr int kAcTY = 4;", f"constexpr int kAcTY = {ty};").replace(
        "constexpr int kAcKC = 32;", f"constexpr int kAcKC = {kc};")
    assert (ty, kc) == (4, 32) or s2 != s
    open(p, "w").write(s2)
    r = subprocess.run([sys.executable, "-c", "from paper_2211_15716_b200 import build as b; b.build(force=True)"],
                       cwd=d, capture_output=True, text=True)
    if r.returncode:
        print(r.stdout, r.stderr)
        raise SystemExit(name)
    os.makedirs(os.path.join(ROOT, "ab"), exist_ok=True)
    shutil.copy(os.path.join(d, "paper_2211_15716_b200", "libigg.so"), os.path.join(ROOT, "ab", f"libigg_{name}.so"))
    return name


if __name__ == "__main__":
    cfgs = [tuple(map(int, a.split(","))) for a in sys.argv[1:]]
    with ThreadPoolExecutor(len(cfgs)) as ex:
        for n in ex.map(lambda c: build(*c), cfgs):
            print("built", n)
