"""Opt-in Hadamard rotation (ModelConfig.hadamard; default OFF -- the reference has no
rotation, so the default path is what every other parity test pins).

CPU: the oracle's wht128 is the orthonormal Sylvester-Hadamard transform; the flag
round-trips through the checkpoint header and is validated like the reference's fields.
GPU: device rotation, rotated weight codes and rotated activation codes are bit-exact with
the oracle; a rotated model's logits and QSpec tokens follow the oracle's rotated model.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2410_11305_b200 as Q
from oracle import qspec_oracle as O

TINY_H = dict(n_layers=2, d_model=256, n_heads=2, n_kv_heads=2, d_ff=768, vocab_size=1024, max_seq_len=160,
              group_size=128)


def _hadamard_matrix(n):
    h = np.array([[1.0]])
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    return h / np.sqrt(n)


def test_oracle_wht128_is_orthonormal_hadamard():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 256)).astype(np.float32)
    y = O.wht128(x)
    H = _hadamard_matrix(128)
    ref = np.concatenate([x[:, :128] @ H, x[:, 128:] @ H], axis=1)
    assert np.abs(y - ref).max() < 1e-5
    assert np.abs(O.wht128(y) - x).max() < 1e-5          # H is symmetric and orthonormal


def test_config_flag_validation_and_header_roundtrip():
    from paper_2410_11305_b200.storage import config_from_text, config_to_text
    with pytest.raises(Q.ConfigError):
        Q.ModelConfig(**dict(TINY_H, group_size=64), hadamard=True)
    cfg = Q.ModelConfig(**TINY_H, hadamard=True)
    assert config_from_text(config_to_text(cfg)) == cfg
    plain = Q.ModelConfig(**TINY_H)
    assert "hadamard" not in config_to_text(plain)           # default header = the reference's
    assert config_from_text(config_to_text(plain)).hadamard is False


@pytest.mark.gpu
def test_device_rotation_and_rotated_codes_bit_exact():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2410_11305_b200.quant import hadamard_rows, linear_group_dots
    rng = np.random.default_rng(1)
    x = rng.standard_normal((7, 512)).astype(np.float32)
    assert np.array_equal(hadamard_rows(torch.from_numpy(x)).cpu().numpy(), O.wht128(x))
    w = (rng.standard_normal((384, 512)) * 0.02).astype(np.float32)
    q = Q.quantize_groupwise(torch.from_numpy(w), 128, hadamard=True)
    wc, ws = O.quantize_rows(O.wht128(w), 128)
    assert np.array_equal(q.unpacked_codes(), wc) and np.array_equal(q.scales, ws)
    lin = O.OracleLinear(wc, ws, 128, rotated=True)
    for low in (True, False):
        mode = Q.ExecutionMode.LOW_PRECISION if low else Q.ExecutionMode.HIGH_PRECISION
        ref = O.qlinear(lin, x, low)
        y = Q.qlinear_forward(q, torch.from_numpy(x), mode).cpu().numpy()
        assert np.abs(y - ref).max() <= 2e-5 * np.abs(ref).max()


@pytest.mark.gpu
@pytest.mark.parametrize("T", [1, 5])
def test_rotated_model_forward_and_qspec_follow_oracle(T):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg = Q.ModelConfig(**TINY_H, hadamard=True)
    model = Q.random_init(cfg, 0)
    om = O.random_model(O.OracleConfig(**TINY_H, hadamard=True), 0)
    # rotated weights are bit-exact with the oracle's rotate-then-quantise
    assert np.array_equal(model.layers[1].down_proj.unpacked_codes(), om.layers[1]["down_proj"].codes)
    ids = [int(t) for t in np.random.default_rng(T).integers(0, 1024, T)]
    kv = Q.KVCache(cfg)
    got = Q.forward(model, ids, kv, Q.ExecutionMode.HIGH_PRECISION, Q.WriteTarget.VERIFY).logits.cpu().numpy()
    ref = O.forward(om, ids, O.OracleKV(om.cfg), False, "verify")
    assert np.abs(got - ref).max() <= 1e-4 * np.abs(ref).max()
    prompt = [int(t) for t in np.random.default_rng(42).integers(0, 1024, 16)]
    res = Q.generate_qspec(model, prompt, Q.GenerationConfig(gamma=3, max_new_tokens=24))
    oref = O.generate(om, prompt, gamma=3, max_new=24)
    assert res.new_tokens == oref.new_tokens
