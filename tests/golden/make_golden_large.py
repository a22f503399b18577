"""Freeze reference outputs at the BASELINE shapes (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_large.py <case>

Cases (each writes ``tests/golden/large_<case>.npz``):

  7b2l   Llama-2-7B shape (d=4096, H=KV=32, ff=11008, V=32000), 2 layers, seed 0
  8b2l   Llama-3-8B shape (GQA 32/8, ff=14336, V=128256, theta=5e5), 2 layers, seed 0
  ctx    SURVEY C0 tiny config with 8 prompts of 270 tokens: context >= 256 (>= 5 split-KV
         chunks of 64 keys) for greedy HIGH / LOW and QSpec
  7b32   the full 32-layer 7B shape, seed 0 (the BASELINE model itself; ~15 min, ~35 GB)

Everything comes from the UNMODIFIED reference (``/root/reference/pkg/src/qspec``):
``random_init`` weights, ``forward`` logits (model.py:255-348), ``generate_greedy`` in
both modes and ``generate_qspec`` (specdec.py:395-427) with its per-cycle accept lengths
(specdec.py:371-392).  Logit rows are pinned by argmax, max|logit| and their 256 largest
entries (indices + values), which keeps the fixtures small at V = 128256.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from qspec import (  # noqa: E402  (reference package)
    ExecutionMode, GenerationConfig, KVCache, ModelConfig, WriteTarget, forward,
    generate_greedy, generate_qspec, random_init,
)
from qspec.model import kv_commit  # noqa: E402

HIGH, LOW = ExecutionMode.HIGH_PRECISION, ExecutionMode.LOW_PRECISION
HERE = os.path.dirname(os.path.abspath(__file__))

C7B = dict(d_model=4096, n_heads=32, n_kv_heads=32, d_ff=11008, vocab_size=32000, max_seq_len=512,
           group_size=128)
C8B = dict(d_model=4096, n_heads=32, n_kv_heads=8, d_ff=14336, vocab_size=128256, max_seq_len=512,
           rope_theta=500000.0, group_size=128)
TINY = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, d_ff=768, vocab_size=1024, group_size=128)
TOPK = 256


def pin_rows(g: dict, key: str, logits: np.ndarray) -> None:
    logits = np.asarray(logits, dtype=np.float32)
    idx = np.argsort(-logits, axis=-1, kind="stable")[:, :TOPK]
    g[f"{key}.argmax"] = np.argmax(logits, axis=-1).astype(np.int64)
    g[f"{key}.absmax"] = np.abs(logits).max(-1).astype(np.float32)
    g[f"{key}.top_idx"] = idx.astype(np.int32)
    g[f"{key}.top_val"] = np.take_along_axis(logits, idx, -1)


def gen_streams(g: dict, m, prompt: list[int], n_new: int, gamma: int = 3, low_new: int | None = None) -> None:
    g["prompt"] = np.array(prompt)
    t = time.time()
    gr = generate_greedy(m, prompt, HIGH, GenerationConfig(max_new_tokens=n_new))
    g["greedy_high"] = np.array(gr.new_tokens)
    print(f"  greedy HIGH {time.time() - t:.0f}s", flush=True)
    t = time.time()
    gl = generate_greedy(m, prompt, LOW, GenerationConfig(max_new_tokens=low_new or n_new))
    g["greedy_low"] = np.array(gl.new_tokens)
    print(f"  greedy LOW {time.time() - t:.0f}s", flush=True)
    t = time.time()
    qs = generate_qspec(m, prompt, GenerationConfig(gamma=gamma, max_new_tokens=n_new))
    assert qs.new_tokens == gr.new_tokens
    g["qspec_accept_lens"] = np.array([c.accept_len for c in qs.cycles])
    g["qspec_drafted"] = np.array([len(c.drafted) for c in qs.cycles])
    g["qspec_stats"] = np.array([qs.acceptance_rate, qs.tokens_per_cycle, len(qs.cycles)])
    print(f"  qspec {time.time() - t:.0f}s", flush=True)


def shape_case(cfg_kw: dict, n_layers: int, n_new: int) -> dict:
    g: dict[str, np.ndarray] = {}
    t = time.time()
    m = random_init(ModelConfig(n_layers=n_layers, **cfg_kw), 0)
    print(f"  init {time.time() - t:.0f}s", flush=True)
    V = cfg_kw["vocab_size"]
    toks = [int(x) for x in np.random.default_rng(7).integers(0, V, size=4)]
    g["fwd_tokens"] = np.array(toks)
    # T=4 HIGH (verify shape) from an empty cache, then commit and one T=1 LOW (draft shape)
    kv = KVCache(m.config)
    pin_rows(g, "fwd.high4", forward(m, toks, kv, HIGH, WriteTarget.VERIFY).logits)
    kv_commit(kv, 3)
    nxt = int(g["fwd.high4.argmax"][-1])
    g["fwd.low1_token"] = np.array([nxt])
    pin_rows(g, "fwd.low1", forward(m, [nxt], kv, LOW, WriteTarget.DRAFT).logits)
    # T=4 LOW from an empty cache (draft arithmetic at several positions)
    pin_rows(g, "fwd.low4", forward(m, toks, KVCache(m.config), LOW, WriteTarget.VERIFY).logits)
    prompt = [int(x) for x in np.random.default_rng(42).integers(0, V, size=8)]
    gen_streams(g, m, prompt, n_new)
    return g


def main() -> None:
    case = sys.argv[1]
    t0 = time.time()
    if case == "7b2l":
        g = shape_case(C7B, 2, 8)
    elif case == "8b2l":
        g = shape_case(C8B, 2, 8)
    elif case == "7b32":
        g = shape_case(C7B, 32, 8)
    elif case == "ctx":
        m = random_init(ModelConfig(max_seq_len=400, **TINY), 0)
        g = {}
        prompts = np.random.default_rng(42).integers(0, 1024, size=(8, 270))
        for i, p in enumerate(prompts):
            gi: dict[str, np.ndarray] = {}
            gen_streams(gi, m, [int(x) for x in p], 40)
            g.update({f"p{i}.{k}": v for k, v in gi.items()})
    else:
        raise SystemExit(f"unknown case {case}")
    out = os.path.join(HERE, f"large_{case}.npz")
    np.savez_compressed(out, **g)
    print(f"wrote {out}: {len(g)} arrays, {os.path.getsize(out)} bytes, {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
