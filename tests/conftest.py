import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _ensure_built():
    """The suites load the in-tree libraries; build them when missing."""
    import subprocess
    lib = os.path.join(ROOT, "paper_1608_08658_b200", "libsfdb200.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1608_08658_b200", "csrc"),
                        "-j4"], check=True)
    if not os.path.exists(os.path.join(ROOT, "oracle", "libsfdoracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"], check=True)


def pytest_configure(config):
    _ensure_built()
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libsfdb200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
