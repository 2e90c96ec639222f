import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

FIELD_KEYS = ("positions", "log_scales", "rotations", "raw_amplitude", "raw_relax")
GRAD_KEYS = ("raw_amplitude", "raw_relax", "positions", "log_scales", "rotations")

SWEEP_GRIDS = [((8, 8, 8), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)),
               ((16, 16, 16), (0.7, 1.0, 1.3), (-2.0, 0.0, 1.0)),
               ((32, 24, 16), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)),
               ((32, 32, 32), (0.5, 0.5, 0.5), (1.0, 1.0, 1.0)),
               ((24, 24, 24), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def field_dict(arrays, relax_enabled=True, amplitude_enabled=True):
    d = {k: np.array(a, dtype=np.float64, order="C", copy=True) for k, a in zip(FIELD_KEYS, arrays)}
    d["relax_enabled"] = relax_enabled
    d["amplitude_enabled"] = amplitude_enabled
    return d


@pytest.fixture
def unit_grid():
    from paper_2603_09621_b200 import GridSpec
    return GridSpec((8, 8, 8), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
