"""Shared fixtures: golden vectors, marker registration, repo on sys.path."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"
LCRWMD_CASES = ["small_m16", "m300", "clustered", "self_queries", "dup_rows", "ragged_m37"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C ABI)")
    config.addinivalue_line("markers", "slow: full-size (BASELINE configs[1]) GPU parity, ~1 min")


def load_case(name):
    from paper_1711_07227_b200.corpus import HistogramSet

    z = np.load(GOLDEN / f"{name}.npz")

    def hs(p):
        return HistogramSet(z[f"{p}_offsets"], z[f"{p}_ids"], z[f"{p}_vals"], int(z[f"{p}_ncols"]))

    return z, hs("x1"), hs("x2")


@pytest.fixture(params=LCRWMD_CASES)
def golden_case(request):
    return (request.param, *load_case(request.param))


def rel_close(a, b, rtol=1e-4, atol=1e-6):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.all(np.abs(a - b) <= rtol * np.abs(b) + atol), float(
        np.max(np.abs(a - b) / (np.abs(b) + atol / rtol)) if a.size else 0.0)


WIDEN_CASES = ["small_m16", "m300", "clustered", "dup_rows"]


def load_widen(name):
    """(base golden, widen golden, x1, x2, dyadic xd1, dyadic xd2) for SURVEY §8f rows."""
    from paper_1711_07227_b200.corpus import HistogramSet

    z, x1, x2 = load_case(name)
    w = np.load(GOLDEN / f"widen_{name}.npz")

    def hs(p):
        return HistogramSet(w[f"{p}_offsets"], w[f"{p}_ids"], w[f"{p}_vals"], int(w[f"{p}_ncols"]))

    return z, w, x1, x2, hs("xd1"), hs("xd2")


@pytest.fixture(params=WIDEN_CASES)
def widen_case(request):
    return (request.param, *load_widen(request.param))
