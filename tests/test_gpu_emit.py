"""Fused next-operand emits (linear_tc.cu emit_rms / emit_silu) against the separate
act_pack path: every forward output must be bit-identical -- the emits restate the
pack's RMSNorm (numpy pairwise order, numerics.py:46-62) and quantiser (quant.py:179-194)
exactly, only the kernel that runs them changes."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import TINY

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2410_11305_b200 as Q  # noqa: E402
from paper_2410_11305_b200 import _lib  # noqa: E402
from paper_2410_11305_b200.model import run_forward_chunks  # noqa: E402

C7B2 = dict(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=32, d_ff=11008, vocab_size=32000, max_seq_len=256,
            group_size=128)
C8B2 = dict(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=8, d_ff=14336, vocab_size=4096, max_seq_len=256,
            rope_theta=500000.0, group_size=128)


def _run(model, ids, low, mask):
    _lib.call("qs_set_emit", mask)
    try:
        kv = Q.KVCache(model.config)
        logits, arg = run_forward_chunks(model, kv, ids, 0, low)
        n = _lib.load().qs_forward_launches()
        torch.cuda.synchronize()
        return logits.cpu().numpy(), arg.cpu().numpy(), [k.clone() for k in kv.k[:1]], n
    finally:
        _lib.call("qs_set_emit", 3)


@pytest.mark.parametrize("cfg", ["tiny", "7b2", "8b2"])
@pytest.mark.parametrize("T", [1, 4, 16])
@pytest.mark.parametrize("low", [False, True])
def test_emit_bit_identical_to_pack(cfg, T, low):
    kw = {"tiny": TINY, "7b2": C7B2, "8b2": C8B2}[cfg]
    model = Q.random_init(Q.ModelConfig(**kw), 0)
    ids = [int(t) for t in np.random.default_rng(T).integers(0, model.config.vocab_size, T)]
    l0, a0, k0, n0 = _run(model, ids, low, 0)
    L = model.config.n_layers
    assert n0 == 9 * L + 2
    l1, a1, k1, n1 = _run(model, ids, low, 3)
    assert np.array_equal(a1, a0)
    assert np.array_equal(l1, l0), np.abs(l1 - l0).max()
    assert all(torch.equal(x, y) for x, y in zip(k1, k0))
    assert n1 == 6 * L + 2, n1   # qkv, attention, attention-merge pack, o, gate_up, down per layer


def test_emit_decode_tokens_match_pack_path():
    model = Q.random_init(Q.ModelConfig(**C7B2), 0)
    prompt = [int(t) for t in np.random.default_rng(42).integers(0, 32000, 24)]
    gc = Q.GenerationConfig(gamma=3, max_new_tokens=16)
    _lib.call("qs_set_emit", 0)
    try:
        ref = Q.generate_qspec(model, prompt, gc)
    finally:
        _lib.call("qs_set_emit", 3)
    got = Q.generate_qspec(model, prompt, gc)
    assert got.new_tokens == ref.new_tokens
    assert [c.accept_len for c in got.cycles] == [c.accept_len for c in ref.cycles]
