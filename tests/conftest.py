import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLD / "ref_small_cases.npz")


@pytest.fixture(scope="session")
def kats():
    return json.loads((GOLD / "reference_kats.json").read_text())


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.build(with_reference=False)
    return oracle.oracle()


@pytest.fixture(scope="session")
def ref81():
    import oracle

    lib = oracle.reference(81)
    if lib is None:
        pytest.skip("compiled reference (oracle/_ref) not available")
    return lib


@pytest.fixture(scope="session")
def ref47():
    import oracle

    lib = oracle.reference(47)
    if lib is None:
        pytest.skip("compiled reference (oracle/_ref) not available")
    return lib


def rel_err(got, ref, axis=-1):
    """max |got - ref| / max(|ref|, ||ref_row||_inf) (SURVEY §8d tolerance rule)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    row = np.max(np.abs(ref), axis=axis, keepdims=True) if ref.ndim > 1 else np.abs(ref)
    den = np.maximum(np.maximum(np.abs(ref), row), 1e-30)
    return float(np.max(np.abs(got - ref) / den)) if ref.size else 0.0


def max_abs(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref))) if ref.size else 0.0
