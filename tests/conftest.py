import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        from paper_2306_01369_b200._native import cuda_device_count

        return cuda_device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    # an explicit `-m gpu` run must fail loudly without a device, never skip
    expr = config.getoption("-m") or ""
    if os.environ.get("GG_FORCE_GPU_TESTS") or (expr.strip() == "gpu"):
        return
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
