import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def _ensure_built():
    """Build the in-tree libraries if stale (nvcc / gcc are in the image)."""
    import importlib.util
    import shutil
    spec = importlib.util.spec_from_file_location(
        "_pgc_build", os.path.join(ROOT, "paper_2008_11321_b200", "_build.py"))
    pb = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(pb)   # without importing the package (it needs the .so)
    if pb.stale() and (os.path.exists(os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"))
                       or shutil.which("nvcc")):
        pb.build()


def pytest_configure(config):
    _ensure_built()
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    # GPU tests are skipped (not failed) when no device is present, so that
    # `-m "not gpu"` and a plain run behave on the CPU-only build box.
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
