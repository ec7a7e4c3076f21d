import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the product kernels")
    config.addinivalue_line("markers", "slow: larger CPU or GPU cases")


def golden_cases():
    # small-graph goldens only: parser vectors and the full-size fixtures
    # (full_*.json, sample_*.json from make_scale_golden.py) have their own tests
    names = sorted(f[:-5] for f in os.listdir(GOLDEN)
                   if f.endswith(".json") and f != "parser.json" and not f.startswith(("full_", "sample_")))
    return names


def scale_goldens(prefix):
    return sorted(f[:-5] for f in os.listdir(GOLDEN) if f.startswith(prefix) and f.endswith(".json"))


def load_golden(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return 0
