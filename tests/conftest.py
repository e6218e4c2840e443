import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    meta = json.load(open(os.path.join(GOLDEN_DIR, "golden.json")))
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def oracle_mod():
    lib = os.path.join(ROOT, "oracle", "liboracle.so")
    src = os.path.join(ROOT, "oracle", "dgswe_oracle.c")
    if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    from oracle import oracle
    return oracle


def perturb_nz2(X):
    """The second-level perturbation used by tests/golden/make_golden.py."""
    X[0, :, :, 1, 0] += 25.0
    X[0, :, :, 1, 1:] *= 0.9
    X[1, :, :, 1, :] *= 1.1
    return X


def oracle_case(oracle, e):
    t, orc, X = oracle.build_case(e["case"], e["nx"], e["ny"], e["p"], e["nz"], *e["rusanov"])
    if e["nz"] == 2:
        perturb_nz2(X)
    return t, orc, X
