import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size (config C1/C2) parity runs")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.build()
    return o


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    g = ROOT / "tests" / "golden"
    out = {
        "generators": json.loads((g / "generators.json").read_text()),
        "kats": json.loads((g / "kats.json").read_text()),
        "corpus": dict(np.load(g / "corpus.npz")),
        "split": dict(np.load(g / "split.npz")),
        "scan": dict(np.load(g / "scan.npz")),
    }
    big = g / "big.json"
    out["big"] = json.loads(big.read_text()) if big.exists() else None
    return out
