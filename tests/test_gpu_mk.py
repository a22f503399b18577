"""The persistent forward kernel (qs_forward_mk, forward_mk.cu) against the per-step
launch sequence (qs_forward): same logits, argmax and KV-cache writes BIT FOR BIT
(same stream-K partition and reduction orders), and identical decode streams
through the engine -- so every oracle-parity test of the per-step path carries
over to the persistent one."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import MODEL_SPECS, TINY

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2410_11305_b200 as Q  # noqa: E402
from paper_2410_11305_b200 import _lib  # noqa: E402
from paper_2410_11305_b200.engine import DecodeEngine  # noqa: E402

SEVEN_B_2L = dict(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=32, d_ff=11008, vocab_size=32000,
                  max_seq_len=256, group_size=128)
GQA_8B_2L = dict(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=8, d_ff=14336, vocab_size=4096,
                 max_seq_len=256, group_size=128)
SHAPES = {"tiny": TINY, "spec0": dict(MODEL_SPECS[0], max_seq_len=96), "spec6": dict(MODEL_SPECS[6], max_seq_len=96),
          "spec2": dict(MODEL_SPECS[2], max_seq_len=96), "7b2l": SEVEN_B_2L, "8b2l": GQA_8B_2L}
_models: dict = {}


def model_of(name):
    if name not in _models:
        _models[name] = Q.random_init(Q.ModelConfig(**SHAPES[name]), 0)
    return _models[name]


def _engine(model, B, gamma=3, prompt_len=20):
    eng = DecodeEngine(model, B, gamma=gamma, max_new_cap=48, use_graphs=False)
    rng = np.random.default_rng(7)
    for b in range(B):
        eng.prefill(b, [int(t) for t in rng.integers(0, model.config.vocab_size, prompt_len + 3 * b)], 40)
    return eng


def _forward_both(eng, per_seq, low):
    """Stage one draft (per_seq=1) or verify (per_seq=gamma+1) batch, run both forwards."""
    cfg = eng.cfg
    B = eng.B
    committed = eng.t["committed"].clone()
    toks = torch.randint(0, cfg.vocab_size, (B * per_seq,), dtype=torch.int32, device="cuda")
    pos = (committed.repeat_interleave(per_seq) + torch.arange(per_seq, device="cuda").repeat(B)).int()
    eng.t["tok"][:B * per_seq].copy_(toks)
    eng.t["pos"][:B * per_seq].copy_(pos)
    eng.t["slot"][:B * per_seq].copy_(torch.arange(B, device="cuda").repeat_interleave(per_seq).int())
    batches = eng.draft_batches if per_seq == 1 else eng.verify_batches
    mode = _lib.QS_MODE_LOW if low else _lib.QS_MODE_HIGH
    st = _lib.stream_ptr()
    out = []
    for fn in ("qs_forward", "qs_forward_mk"):
        logits = torch.full((64, cfg.vocab_size), float("nan"), device="cuda")
        arg = torch.full((64,), -1, dtype=torch.int32, device="cuda")
        for b, off in batches:
            T = b.T
            lg = logits[off // 4: off // 4 + T]
            _lib.call(fn, eng.cm, b, mode, eng.ws, lg.data_ptr(), arg.data_ptr() + off, st)
        torch.cuda.synchronize()
        kv = [(k.clone(), v.clone()) for k, v in zip(eng.kv.k, eng.kv.v)]
        out.append((logits[:B * per_seq].clone(), arg[:B * per_seq].clone(), kv))
    return out


@pytest.mark.parametrize("name", ["tiny", "spec0", "spec2", "spec6", "7b2l", "8b2l"])
@pytest.mark.parametrize("low", [True, False], ids=["low", "high"])
def test_forward_mk_bit_identical(name, low):
    model = model_of(name)
    B = 4 if name not in ("7b2l", "8b2l") else 16
    eng = _engine(model, B)
    per_seq = 1 if low else eng.gamma + 1
    (l0, a0, kv0), (l1, a1, kv1) = _forward_both(eng, per_seq, low)
    assert torch.equal(a0, a1)
    assert torch.equal(l0, l1), float((l0 - l1).abs().max())
    for (k0, v0), (k1, v1) in zip(kv0, kv1):
        assert torch.equal(k0, k1) and torch.equal(v0, v1)


@pytest.mark.parametrize("B", [1, 3, 16])
def test_forward_mk_batch_sizes(B):
    model = model_of("tiny")
    eng = _engine(model, B)
    for low, per_seq in ((True, 1), (False, eng.gamma + 1)):
        (l0, a0, _), (l1, a1, _) = _forward_both(eng, per_seq, low)
        assert torch.equal(a0, a1) and torch.equal(l0, l1)


@pytest.mark.parametrize("name", ["tiny", "spec6"])
@pytest.mark.parametrize("algorithm", ["qspec", "greedy"])
def test_engine_persistent_equals_per_step(name, algorithm):
    model = model_of(name)
    res = []
    for persistent in (False, True):
        eng = DecodeEngine(model, 4, gamma=3, max_new_cap=40, algorithm=algorithm, persistent=persistent)
        rng = np.random.default_rng(3)
        for b in range(4):
            eng.prefill(b, [int(t) for t in rng.integers(0, model.config.vocab_size, 12 + b)], 32)
        eng.run()
        res.append([eng.result(b) for b in range(4)])
    for r0, r1 in zip(*res):
        assert r0.new_tokens == r1.new_tokens
        assert np.array_equal(r0.trace, r1.trace)


def test_forward_mk_graph_replay_counters_reset():
    """Counters are reset by the kernel itself: many graph replays stay correct."""
    model = model_of("tiny")
    eng = DecodeEngine(model, 2, gamma=3, max_new_cap=64, persistent=True)
    ref = DecodeEngine(model, 2, gamma=3, max_new_cap=64, persistent=False, use_graphs=False)
    for e in (eng, ref):
        for b in range(2):
            e.prefill(b, [5 + b, 17, 99, 3], 60)
        e.run()
    for b in range(2):
        assert eng.result(b).new_tokens == ref.result(b).new_tokens


@pytest.mark.parametrize("name", ["spec6", "7b2l"])
@pytest.mark.parametrize("algorithm", ["qspec", "greedy"])
def test_engine_persistent_b1(name, algorithm):
    """B = 1: the smallest token buckets (T = 1 draft / AR, T = 4 verify)."""
    model = model_of(name)
    res = []
    for persistent in (False, True):
        eng = DecodeEngine(model, 1, gamma=3, max_new_cap=24, algorithm=algorithm, persistent=persistent)
        eng.prefill(0, [3, 14, 15, 92, 65, 35], 20)
        eng.run()
        res.append(eng.result(0))
    assert res[0].new_tokens == res[1].new_tokens
    assert np.array_equal(res[0].trace, res[1].trace)
