"""Shared pytest setup: the `gpu` marker and the repo root on sys.path."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run through gpurun)")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")
    config.addinivalue_line("markers", "ablation: needs the ablation build (IGG_LIBRARY=ablation/libigg_ablation.so); "
                                       "run by tests/test_gpu_ablation.py in a subprocess")


def pytest_collection_modifyitems(config, items):
    # the `ablation` tests need the ablation build: with the product library they are deselected (not
    # skipped); tests/test_gpu_ablation.py runs them against the ablation build in a subprocess
    if "ablation" in os.environ.get("IGG_LIBRARY", ""):
        return
    keep = [it for it in items if "ablation" not in it.keywords]
    if len(keep) != len(items):
        config.hook.pytest_deselected(items=[it for it in items if "ablation" in it.keywords])
        items[:] = keep


def pytest_sessionstart(session):
    # test infrastructure: make sure the in-tree library and the C oracle are
    # built (the product itself never builds or falls back; it raises)
    from paper_2211_15716_b200 import build as B
    if B.needs_build():
        B.build()
    from oracle import heat3d as OH
    OH.build()
