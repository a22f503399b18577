"""Shared test configuration: the ``gpu`` marker and common helpers."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA extension")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN, allow_pickle=False)


def conftest_cfg(**over):
    """pkg/tests/conftest.py:12-19 (the reference's toy config)."""
    base = dict(n_layers=2, d_model=64, n_heads=4, n_kv_heads=2, d_ff=128, vocab_size=256,
                max_seq_len=96, rope_theta=10000.0, norm_eps=1e-5, group_size=32)
    base.update(over)
    return base


TINY = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, d_ff=768, vocab_size=1024,
            max_seq_len=160, group_size=128)

MODEL_SPECS = [  # pkg/tests/test_acceptance.py:47-68 (first 8 shapes; mirrors make_golden.py)
    dict(n_layers=2, d_model=64, n_heads=4, n_kv_heads=2, d_ff=128, vocab_size=256, group_size=32),
    dict(n_layers=2, d_model=64, n_heads=4, n_kv_heads=4, d_ff=128, vocab_size=512, group_size=16),
    dict(n_layers=2, d_model=64, n_heads=2, n_kv_heads=1, d_ff=192, vocab_size=1024, group_size=64),
    dict(n_layers=2, d_model=96, n_heads=4, n_kv_heads=2, d_ff=192, vocab_size=512, group_size=32),
    dict(n_layers=2, d_model=128, n_heads=8, n_kv_heads=2, d_ff=256, vocab_size=1024, group_size=64),
    dict(n_layers=3, d_model=64, n_heads=4, n_kv_heads=1, d_ff=128, vocab_size=256, group_size=16),
    dict(n_layers=3, d_model=96, n_heads=6, n_kv_heads=3, d_ff=192, vocab_size=768, group_size=48),
    dict(n_layers=2, d_model=96, n_heads=2, n_kv_heads=2, d_ff=192, vocab_size=1024, group_size=96),
]
