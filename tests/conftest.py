# SPDX-License-Identifier: Apache-2.0
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_1611_07819_b200", "libgridmath_b200.so")
    if not os.path.exists(lib):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "paper_1611_07819_b200"), "-j8"])
    c = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
    if not os.path.exists(c):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "_build/liboracle.so"])


_ensure_built()


@pytest.fixture(scope="session")
def golden_index():
    import json
    with open(os.path.join(GOLDEN, "index.json")) as fh:
        return json.load(fh)


def load_case(name):
    import numpy as np
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))
