import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")
    config.addinivalue_line("markers", "slow: takes more than a few seconds on CPU")


def _have_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _have_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def gold_small():
    """name -> dict(centers, radii, meta, k0..k3, optional p1..p3) from the real reference."""
    data = np.load(os.path.join(GOLD, "complex_small.npz"))
    index = json.load(open(os.path.join(GOLD, "complex_small.json")))
    out = {}
    for name, meta in index.items():
        rec = dict(meta=meta, centers=data[name + "__centers"], radii=data[name + "__radii"])
        for d in range(4):
            rec[f"k{d}"] = data[f"{name}__k{d}"]
        if meta["potentials_stored"]:
            for d in (1, 2, 3):
                rec[f"p{d}"] = (data[f"{name}__p{d}_rows"], data[f"{name}__p{d}_centers"], data[f"{name}__p{d}_sizes"])
        out[name] = rec
    return out


@pytest.fixture(scope="session")
def gold_config1():
    data = np.load(os.path.join(GOLD, "config1.npz"))
    meta = json.load(open(os.path.join(GOLD, "config1.json")))
    return data, meta


@pytest.fixture(scope="session")
def gold_errors():
    return json.load(open(os.path.join(GOLD, "error_cases.json")))


@pytest.fixture(scope="session")
def gold_large():
    path = os.path.join(GOLD, "large_configs.json")
    return json.load(open(path)) if os.path.exists(path) else {}
