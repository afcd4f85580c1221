"""Shared test fixtures.

Markers: ``gpu`` (needs a CUDA device and libmbgpu.so; run on the B200 box)
and ``slow`` (long CPU oracle runs, deselected by default with -m "not slow").
"""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "oracle"))

import paper_2005_05412_b200 as gpu  # noqa: E402

from paper_2005_05412_b200.reference import mblight as mb  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmbgpu.so")
    config.addinivalue_line("markers", "slow: long-running CPU oracle comparison")


@pytest.fixture(autouse=True)
def fresh_material_library():
    mb.clear_material_library()
    yield
    mb.clear_material_library()


def load_golden(name):
    """Records of a reference run: list of (name, data, axes dict)."""
    path = GOLDEN / f"{name}.npz"
    if not path.exists():
        pytest.skip(f"golden fixture {path.name} not generated")
    z = np.load(path)
    meta = json.loads(bytes(z["meta"]).decode())
    recs = []
    for k, m in enumerate(meta["records"]):
        recs.append((m["name"], z[f"r{k}"], m))
    return meta, recs


def rel_err(got, ref):
    """max_t |got - ref| / max_t |ref|  (inf when ref is all-zero and got is not)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    scale = float(np.max(np.abs(ref))) if ref.size else 0.0
    diff = float(np.max(np.abs(got - ref))) if ref.size else 0.0
    if scale == 0.0:
        return 0.0 if diff == 0.0 else float("inf")
    return diff / scale


def build_case(name, api=mb):
    from cases import CASES

    build, stepper = CASES[name]
    dev, sce = build(api)
    return dev, sce, stepper
