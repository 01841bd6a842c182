"""Test configuration.

Markers:
  gpu   -- needs a CUDA device (B200); run with `pytest -m gpu` on the GPU box.
  slow  -- CPU tests that need >10 GB host RAM / minutes (config 4/5 oracle pins);
           run with STARMM_SLOW=1.
"""
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long CPU oracle pins (set STARMM_SLOW=1)")


def pytest_collection_modifyitems(config, items):
    import torch
    has_gpu = torch.cuda.is_available()
    slow = os.environ.get("STARMM_SLOW") == "1"
    for it in items:
        if "gpu" in it.keywords and not has_gpu:
            it.add_marker(pytest.mark.skip(reason="no CUDA device"))
        if "slow" in it.keywords and not slow:
            it.add_marker(pytest.mark.skip(reason="set STARMM_SLOW=1"))
