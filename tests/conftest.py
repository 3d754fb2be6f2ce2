import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    # build every native artefact in-tree (no-op when up to date)
    if os.environ.get("TGS_SKIP_MAKE") != "1":
        r = subprocess.run(["make", "-s", "-C", ROOT], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("make failed:\n" + r.stdout + r.stderr)


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
