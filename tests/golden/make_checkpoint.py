"""Golden QSPC checkpoints written by the UNMODIFIED reference (run here, where /root/reference exists).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_checkpoint.py

toy_seed0.qspc: reference random_init(toy config, seed 0) -> save_checkpoint (storage.py:315-349).
tests/test_checkpoint.py loads it into the device layout, checks it equals our random_init, and that
our save_checkpoint reproduces the file byte for byte.
"""
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from qspec import ModelConfig  # noqa: E402
from qspec.storage import random_init, save_checkpoint  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
cfg = ModelConfig(n_layers=2, d_model=64, n_heads=4, n_kv_heads=2, d_ff=128, vocab_size=256, max_seq_len=96,
                  rope_theta=10000.0, norm_eps=1e-5, group_size=32)
save_checkpoint(random_init(cfg, 0), os.path.join(HERE, "toy_seed0.qspc"))
print("wrote", os.path.join(HERE, "toy_seed0.qspc"))
