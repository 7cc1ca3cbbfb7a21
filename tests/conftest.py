import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    d = {k: g[k] for k in g.files}
    if "meta" in d:
        d["meta"] = json.loads(str(d["meta"]))
    return d


def golden_names(prefix=""):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, f"{prefix}*.npz")))


@pytest.fixture(scope="session")
def refmod():
    from oracle import ref

    if not ref.available():
        pytest.skip("reference oracle library (oracle/_ref) not built here")
    return ref


@pytest.fixture(scope="session")
def oc():
    from paper_1806_05896_b200 import optcon

    return optcon


@pytest.fixture(scope="session")
def ctx(oc):
    return oc.Context(0)


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
