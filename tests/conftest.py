import functools
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

GOLDEN_DIR = os.path.join(TESTS, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@functools.lru_cache(maxsize=1)
def golden_small():
    return np.load(os.path.join(GOLDEN_DIR, "small.npz"))


def golden_configs(cfg_id):
    """All committed per-realization records of a BASELINE config."""
    import glob
    import json

    recs = []
    full = os.path.join(GOLDEN_DIR, f"config{cfg_id}_full.json")
    paths = [full] if os.path.exists(full) else sorted(glob.glob(os.path.join(GOLDEN_DIR, f"config{cfg_id}_*.json")))
    for path in paths:
        recs.extend(json.load(open(path))["records"])
    recs.sort(key=lambda r: r["m"])
    return recs


@functools.lru_cache(maxsize=1)
def golden_generic():
    """Reference outputs at grid sizes that are not powers of two (n = 12, 20, 24, 28)."""
    return np.load(os.path.join(GOLDEN_DIR, "generic.npz"))
