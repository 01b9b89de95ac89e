import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN, allow_pickle=True)


def make_spec(**overrides):
    """reference tests/conftest.py:7-21 defaults."""
    from paper_2410_23317_b200.trace import GenSpec

    base = dict(num_layers=2, num_query_heads=4, num_kv_heads=2, head_dim=32, prompt_len=96,
                post_vision_len=12, decode_len=4, seed=11, heavy_fraction=0.05, noise_scale=0.1)
    base.update(overrides)
    return GenSpec(**base)


TOY = dict(num_layers=4, num_query_heads=8, num_kv_heads=8, head_dim=64, prompt_len=624,
           post_vision_len=32, decode_len=100, seed=0)
