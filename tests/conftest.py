import json
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


@pytest.fixture(scope="session")
def golden():
    """(arrays, metadata) produced by tests/golden/make_golden.py from the reference."""
    arrs = np.load(GOLDEN / "golden.npz")
    meta = json.loads((GOLDEN / "golden.json").read_text())
    return arrs, meta


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_15082_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def golden_graph(arrs, name):
    from paper_2211_15082_b200.storage import CscGraph

    ip = arrs[f"g/{name}/indptr"]
    ix = arrs[f"g/{name}/indices"]
    return CscGraph(len(ip) - 1, len(ix), ip, ix)
