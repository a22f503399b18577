"""QSPC checkpoints (storage.py:1-28 format, 300-422 save/load) -- against a file the
unmodified reference wrote (tests/golden/make_checkpoint.py)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import ROOT

import paper_2410_11305_b200 as Q
from paper_2410_11305_b200 import storage as S

CKPT = os.path.join(ROOT, "tests", "golden", "toy_seed0.qspc")


def test_header_round_trip_and_errors():
    cfg, recs = S.read_checkpoint(CKPT)
    assert cfg.d_model == 64 and cfg.group_size == 32 and cfg.n_kv_heads == 2
    assert S.config_from_text(S.config_to_text(cfg)) == cfg
    assert len(recs) == 1 + 2 * (2 + 7 * 2) + 1 + 2
    assert recs["layers.0.q_proj.codes"][1] == (64, 64)
    with pytest.raises(Q.CheckpointError):
        S.config_from_text("n_layers=2\n")
    with pytest.raises(Q.CheckpointError):
        S.config_from_text(S.config_to_text(cfg) + "bogus=1\n")


@pytest.mark.parametrize("cut", [3, 20, 5000])
def test_truncated_and_bad_magic(tmp_path, cut):
    data = open(CKPT, "rb").read()
    p = tmp_path / "t.qspc"
    p.write_bytes(data[:cut])
    with pytest.raises(Q.CheckpointError):
        S.read_checkpoint(str(p))
    p.write_bytes(b"XXXX" + data[4:])
    with pytest.raises(Q.CheckpointError):
        S.read_checkpoint(str(p))


@pytest.mark.gpu
def test_load_equals_random_init_and_saves_byte_identical(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    m = S.load_checkpoint(CKPT)
    r = Q.random_init(m.config, 0)
    for a, b in ((m.layers[1].gate_up, r.layers[1].gate_up), (m.layers[0].qkv, r.layers[0].qkv),
                 (m.lm_head.store, r.lm_head.store)):
        assert torch.equal(a.codes, b.codes) and torch.equal(a.scales, b.scales)
    out = tmp_path / "again.qspc"
    S.save_checkpoint(m, str(out))
    assert out.read_bytes() == open(CKPT, "rb").read()
    prompt = [5, 9, 100, 3, 77]
    cfg = Q.GenerationConfig(gamma=3, max_new_tokens=16)
    assert Q.generate_qspec(m, prompt, cfg).new_tokens == Q.generate_qspec(r, prompt, cfg).new_tokens


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -0.5])
def test_corrupt_scales_rejected(tmp_path, bad):
    # quant.py:138-139 + storage.py:390-397: a NaN / infinite / negative scale is a
    # CheckpointError naming the record, raised before any device work
    data = bytearray(open(CKPT, "rb").read())
    _, recs = S.read_checkpoint(CKPT)
    payload = recs["layers.1.down_proj.scales"][2]
    off = bytes(data).find(payload)
    assert off > 0
    data[off + 8:off + 12] = np.array([bad], dtype="<f4").tobytes()
    p = tmp_path / "bad.qspc"
    p.write_bytes(bytes(data))
    with pytest.raises(Q.CheckpointError, match="layers.1.down_proj.codes"):
        S.load_checkpoint(str(p))
