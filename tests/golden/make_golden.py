"""Freeze reference outputs into small fixtures (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the UNMODIFIED reference package (``/root/reference/pkg/src/qspec``)
and writes ``tests/golden/golden.npz``.  The GPU box never runs this (the
reference is not there); tests read the committed ``.npz``.  Large tensors are
pinned by sha256 digests, small ones are stored whole.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from qspec import (  # noqa: E402  (reference package)
    ExecutionMode, GenerationConfig, KVCache, ModelConfig, WriteTarget, forward,
    generate_greedy, generate_qspec, qlinear_forward, random_init,
)
from qspec.quant import _quantize_groups, fake_quantize_activations  # noqa: E402
from qspec.storage import Lcg64  # noqa: E402

HIGH, LOW = ExecutionMode.HIGH_PRECISION, ExecutionMode.LOW_PRECISION
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def conftest_cfg(**over) -> ModelConfig:   # pkg/tests/conftest.py:12-19
    base = dict(n_layers=2, d_model=64, n_heads=4, n_kv_heads=2, d_ff=128, vocab_size=256,
                max_seq_len=96, rope_theta=10000.0, norm_eps=1e-5, group_size=32)
    base.update(over)
    return ModelConfig(**base)


TINY = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, d_ff=768, vocab_size=1024,
            max_seq_len=160, group_size=128)

MODEL_SPECS = [  # pkg/tests/test_acceptance.py:47-68 (first 8 shapes)
    dict(n_layers=2, d_model=64, n_heads=4, n_kv_heads=2, d_ff=128, vocab_size=256, group_size=32),
    dict(n_layers=2, d_model=64, n_heads=4, n_kv_heads=4, d_ff=128, vocab_size=512, group_size=16),
    dict(n_layers=2, d_model=64, n_heads=2, n_kv_heads=1, d_ff=192, vocab_size=1024, group_size=64),
    dict(n_layers=2, d_model=96, n_heads=4, n_kv_heads=2, d_ff=192, vocab_size=512, group_size=32),
    dict(n_layers=2, d_model=128, n_heads=8, n_kv_heads=2, d_ff=256, vocab_size=1024, group_size=64),
    dict(n_layers=3, d_model=64, n_heads=4, n_kv_heads=1, d_ff=128, vocab_size=256, group_size=16),
    dict(n_layers=3, d_model=96, n_heads=6, n_kv_heads=3, d_ff=192, vocab_size=768, group_size=48),
    dict(n_layers=2, d_model=96, n_heads=2, n_kv_heads=2, d_ff=192, vocab_size=1024, group_size=96),
]


def main() -> None:
    g: dict[str, np.ndarray] = {}
    # -- LCG (storage.py:62-101)
    g["lcg_seed1234_first64"] = Lcg64(1234).fill(64)
    r = Lcg64(77)
    r.fill(10_000)
    g["lcg_seed77_after10000_state"] = np.array([r.state], dtype=np.uint64)

    # -- conftest model, seed 0: every quantized store whole (small)
    m = random_init(conftest_cfg(), 0)
    for name, q in m.quantized_tensors():
        g[f"toy0.{name}.codes"] = q.codes
        g[f"toy0.{name}.scales"] = q.scales
    g["toy0.token_embedding"] = m.token_embedding

    # -- tiny C0 model, seed 0: digests of every store
    tiny = random_init(ModelConfig(**TINY), 0)
    g["tiny.digests"] = np.array([f"{n}:{sha(q.codes)}:{sha(q.scales)}" for n, q in tiny.quantized_tensors()])
    g["tiny.emb_digest"] = np.array([sha(tiny.token_embedding)])

    # -- activation quantizer (quant.py:179-194, 229-245)
    rng = np.random.default_rng(5)
    for gs in (16, 32, 128):
        x = (rng.standard_normal((5, 256)) * 3).astype(np.float32)
        x[1, :gs] = 0.0                                   # an all-zero group
        codes, scales = _quantize_groups(x, gs)
        g[f"aq{gs}.x"], g[f"aq{gs}.codes"], g[f"aq{gs}.scales"] = x, codes, scales
        g[f"aq{gs}.fq"] = fake_quantize_activations(x, gs)

    # -- qlinear both modes on a conftest store
    x = rng.standard_normal((3, 64)).astype(np.float32)
    q = m.layers[0].q_proj
    g["ql.x"] = x
    g["ql.high"] = qlinear_forward(q, x, HIGH)
    g["ql.low"] = qlinear_forward(q, x, LOW)

    # -- forward logits (model.py:255-348) on the conftest model
    toks = [5, 9, 200, 3, 77]
    for mode, tag in ((HIGH, "high"), (LOW, "low")):
        kv = KVCache(m.config)
        g[f"fwd.{tag}"] = forward(m, toks, kv, mode, WriteTarget.VERIFY).logits
        g[f"fwd.{tag}.k0"] = kv.verify_k[0][:5].copy()

    # -- generation streams on the tiny C0 config
    prompts = np.random.default_rng(42).integers(0, 1024, size=(8, 16))
    g["tiny.prompts"] = prompts
    greedy, qs, acc = [], [], []
    for p in prompts:
        p = [int(t) for t in p]
        gr = generate_greedy(tiny, p, HIGH, GenerationConfig(max_new_tokens=64))
        qq = generate_qspec(tiny, p, GenerationConfig(gamma=3, max_new_tokens=64))
        assert gr.tokens == qq.tokens
        greedy.append(gr.new_tokens)
        qs.append(qq.new_tokens)
        acc.append([qq.acceptance_rate, qq.tokens_per_cycle, len(qq.cycles)])
    g["tiny.greedy"] = np.array(greedy)
    g["tiny.qspec_stats"] = np.array(acc)
    g["tiny.qspec_accept_lens"] = np.array(
        [c.accept_len for p in prompts[:1]
         for c in generate_qspec(tiny, [int(t) for t in p], GenerationConfig(gamma=3, max_new_tokens=64)).cycles])
    gl = generate_greedy(tiny, [int(t) for t in prompts[0]], LOW, GenerationConfig(max_new_tokens=64))
    g["tiny.greedy_low0"] = np.array(gl.new_tokens)

    # -- conftest toy models: QSpec == greedy streams, gamma sweep (test_specdec.py:166-174)
    toy6 = random_init(conftest_cfg(vocab_size=512), 6)
    g["toy6.greedy"] = np.array(generate_greedy(toy6, [4, 9, 100, 3], HIGH,
                                                GenerationConfig(max_new_tokens=14)).new_tokens)
    for gm in (1, 2, 3, 5, 7):
        res = generate_qspec(toy6, [4, 9, 100, 3], GenerationConfig(gamma=gm, max_new_tokens=14))
        g[f"toy6.qspec.g{gm}"] = np.array(res.new_tokens)
        g[f"toy6.qspec.g{gm}.acc"] = np.array([res.acceptance_rate])

    # -- acceptance-gate shapes (test_acceptance.py:47-68), 3 prompts each
    rng = np.random.default_rng(20241)
    for mi, spec in enumerate(MODEL_SPECS):
        cfg = conftest_cfg(max_seq_len=48, **spec)
        mod = random_init(cfg, seed=1000 + mi)
        for pi in range(3):
            p = [int(t) for t in rng.integers(0, cfg.vocab_size, size=int(rng.integers(3, 7)))]
            g[f"spec{mi}.p{pi}.prompt"] = np.array(p)
            g[f"spec{mi}.p{pi}.greedy"] = np.array(
                generate_greedy(mod, p, HIGH, GenerationConfig(max_new_tokens=12)).new_tokens)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
