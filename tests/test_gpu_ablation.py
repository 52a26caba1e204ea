"""The tuning variants of the stencil kernels (IGG_OPT_STENCIL_KERNEL 2..56 binary64, 100..126 binary32)
and the binary32 schedule bits live in a separate ablation build (ablation/libigg_ablation.so, built by
__graft_entry__.build()); the product library has only the defaults.  This runs the tests marked
`ablation` against that build in a subprocess: every variant must compute the same cells."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ablation_variants_bit_exact():
    lib = os.path.join(ROOT, "ablation", "libigg_ablation.so")
    if not os.path.exists(lib):
        from paper_2211_15716_b200 import build as B
        B.build(out=lib, extra=["-DIGG_ABLATION=1"])
    env = dict(os.environ, IGG_LIBRARY=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu and ablation", os.path.join(ROOT, "tests")],
                       capture_output=True, text=True, timeout=1200, env=env, cwd=ROOT)
    sys.stdout.write(r.stdout[-3000:])
    sys.stderr.write(r.stderr[-3000:])
    assert r.returncode == 0
    assert " passed" in r.stdout and "skipped" not in r.stdout
