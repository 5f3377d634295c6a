import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through libpss.so)")
    config.addinivalue_line("markers", "slow: full-size parity cases (minutes)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "worked_examples.json")) as f:
        return json.load(f)


LETTERS = {c: i + 1 for i, c in enumerate("abcdefghijklmnopqrstuvwxyz")}


def letters(s):
    import numpy as np
    return np.array([LETTERS[c] for c in s], dtype=np.uint64)


def build_lib():
    """Build libpss.so without importing the package (its __init__ loads the library)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_pss_build", os.path.join(ROOT, "paper_1606_04669_b200", "_build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()
