import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (str(ROOT), str(ROOT / "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device and the built libcmb200.so")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


def parse_case(key):
    """'<series>_E<E>_t<tau>' -> (E, tau)."""
    E = int(key.split("_E")[1].split("_")[0])
    tau = int(key.split("_t")[-1])
    return E, tau


def parse_edim_case(key):
    """'<series>_M<Emax>_t<tau>_p<Tp>' -> (E_max, tau, Tp)."""
    E_max = int(key.split("_M")[1].split("_")[0])
    tau = int(key.split("_t")[-1].split("_")[0])
    Tp = int(key.split("_p")[-1])
    return E_max, tau, Tp


@pytest.fixture(scope="session")
def golden():
    return load_golden
