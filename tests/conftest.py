import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_cases():
    d = os.path.join(REPO, "tests", "golden")
    return sorted(f[:-4] for f in os.listdir(d) if f.endswith(".npz"))


def load_golden(case):
    import numpy as np
    z = np.load(os.path.join(REPO, "tests", "golden", case + ".npz"))
    return {k: z[k] for k in z.files}
