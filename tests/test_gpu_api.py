"""GPU ports of the reference's API-level tests (pkg/tests/test_model.py, test_specdec.py,
test_acceptance.py C5/C7): KV bookkeeping, mode purity, weight sharing, EOS, batching."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import conftest_cfg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2410_11305_b200 as Q  # noqa: E402
from paper_2410_11305_b200.engine import DecodeEngine  # noqa: E402
from oracle import qspec_oracle as O  # noqa: E402

HIGH, LOW = Q.ExecutionMode.HIGH_PRECISION, Q.ExecutionMode.LOW_PRECISION
_models: dict = {}


def toy(seed=0, **over):
    key = (seed, tuple(sorted(over.items())))
    if key not in _models:
        _models[key] = Q.random_init(Q.ModelConfig(**conftest_cfg(**over)), seed)
    return _models[key]


def test_forward_errors():
    m = toy(0)
    kv = Q.KVCache(m.config)
    with pytest.raises(Q.TokenIdError):
        Q.forward(m, [m.config.vocab_size], kv, HIGH, Q.WriteTarget.VERIFY)
    with pytest.raises(Q.ShapeError):
        Q.forward(m, [], kv, HIGH, Q.WriteTarget.VERIFY)
    with pytest.raises(Q.SequenceOverflowError):
        Q.forward(m, [1, 2, 3, 4], Q.KVCache(m.config, gamma_max=2), HIGH, Q.WriteTarget.VERIFY)


def test_zero_model_logits_and_tiebreak():
    cfg = Q.ModelConfig(**conftest_cfg(n_layers=1))
    tensors = {n: (np.ones(s, np.float32) if len(s) == 1 else np.zeros(s, np.float32))
               for n, s in Q.storage.float_tensor_shapes(cfg)}
    m = Q.model_from_float_tensors(cfg, tensors)
    blk = Q.forward(m, [1, 2, 3], Q.KVCache(cfg), HIGH, Q.WriteTarget.VERIFY)
    assert np.array_equal(blk.numpy(), np.zeros_like(blk.numpy()))
    assert int(blk.argmax[-1]) == 0
    lo = Q.forward(m, [1, 2, 3], Q.KVCache(cfg), LOW, Q.WriteTarget.VERIFY)
    assert np.array_equal(lo.numpy(), blk.numpy())
    r = Q.generate_qspec(m, [1, 2], Q.GenerationConfig(max_new_tokens=8, eos_token=0))
    assert r.new_tokens == [0] and r.finish_reason == "eos" and r.cycles == [] and r.acceptance_rate == 1.0


def test_kv_commit_semantics_and_report():
    m = toy(0)
    kv = Q.KVCache(m.config)
    Q.forward(m, [1, 2, 3], kv, HIGH, Q.WriteTarget.VERIFY)
    Q.kv_commit(kv, 2)
    assert kv.committed_len == 3 and kv.verify_len == 0
    Q.forward(m, [7], kv, LOW, Q.WriteTarget.DRAFT)
    Q.forward(m, [3, 4, 5], kv, HIGH, Q.WriteTarget.VERIFY)
    Q.kv_commit(kv, 1)
    assert kv.committed_len == 5 and kv.draft_len == 0 and kv.verify_len == 0
    with pytest.raises(Q.SequenceOverflowError):
        Q.forward(m, [3], kv, HIGH, Q.WriteTarget.VERIFY)
        Q.kv_commit(kv, 1)
    rep = Q.kv_memory_report(kv)
    cfg = m.config
    assert rep["per_position_bytes"] == cfg.n_layers * 2 * cfg.n_kv_heads * cfg.head_dim * 4
    assert rep["scratch_bytes"] <= 2 * (kv.gamma_max + 1) * rep["per_position_bytes"]


def test_committed_kv_matches_oracle_sequential():
    # C2 spirit: committed KV after batched verify-style commits == sequential oracle decode
    m = toy(2)
    cfg_o = O.OracleConfig(**conftest_cfg())
    om = O.random_model(cfg_o, 2)
    seq = [1, 2, 3, 4, 5, 6]
    okv = O.OracleKV(cfg_o)
    for t in seq:
        O.forward(om, [t], okv, False, "verify")
        okv.commit(0)
    kv = Q.KVCache(m.config)
    Q.forward(m, seq[:3], kv, HIGH, Q.WriteTarget.VERIFY)
    Q.kv_commit(kv, 2)
    Q.forward(m, seq[3:], kv, HIGH, Q.WriteTarget.VERIFY)
    Q.kv_commit(kv, 2)
    for li in range(m.config.n_layers):
        got = kv.committed_k[li].cpu().numpy()
        ref = okv.ck[li][:6]
        assert np.abs(got - ref).max() <= 1e-4 * np.abs(ref).max()


def test_mode_purity_and_weight_sharing():
    m = toy(0)
    Q.reset_activation_quant_calls()
    Q.forward(m, [1, 2, 3], Q.KVCache(m.config), HIGH, Q.WriteTarget.VERIFY)
    assert Q.activation_quant_calls() == 0
    Q.forward(m, [1], Q.KVCache(m.config), LOW, Q.WriteTarget.DRAFT)
    assert Q.activation_quant_calls() == 7 * m.config.n_layers + 1
    weights = m.quantized_tensors()
    ids = {id(q) for _, q in weights}
    assert len(weights) == 7 * m.config.n_layers + 1 == len(ids)
    for _, q in weights:
        assert q.packed_bytes == q.out_features * q.in_features // 2
    eng = Q.SequenceEngine(m, [1, 2, 3], Q.GenerationConfig(gamma=3, max_new_tokens=8))
    eng.prefill()
    Q.start_qlinear_log()
    eng.run_draft_phase()
    eng.run_verify_phase()
    log = Q.stop_qlinear_log()
    assert {i for i, md in log if md is LOW} == ids == {i for i, md in log if md is HIGH}


def _eos_case():
    m = toy(9, vocab_size=512)
    om = O.random_model(O.OracleConfig(**conftest_cfg(vocab_size=512)), 9)
    prompt = [7, 8, 9]
    golden = O.generate(om, prompt, max_new=16, qspec=False).new_tokens
    eos = next(golden[i] for i in range(3, len(golden) - 1) if golden.index(golden[i]) == i)
    return m, om, prompt, eos


@pytest.mark.parametrize("gamma", [1, 3, 7])
def test_eos_truncation_matches_oracle(gamma):
    m, om, prompt, eos = _eos_case()
    ref = O.generate(om, prompt, gamma=gamma, max_new=16, eos=eos)
    r = Q.generate_qspec(m, prompt, Q.GenerationConfig(gamma=gamma, max_new_tokens=16, eos_token=eos))
    assert r.tokens == ref.tokens and r.finish_reason == "eos" and r.new_tokens[-1] == eos


def test_batched_engine_independent_of_batch():
    # C7: every request's tokens equal its standalone generation, for B in {1, 2, 4}
    m = toy(7, vocab_size=512, max_seq_len=48)
    rng = np.random.default_rng(707)
    reqs = [([int(t) for t in rng.integers(0, 512, size=int(rng.integers(2, 6)))], int(rng.integers(4, 11)))
            for _ in range(8)]
    alone = [Q.generate_greedy(m, p, HIGH, Q.GenerationConfig(max_new_tokens=n)).new_tokens for p, n in reqs]
    for B in (2, 4):
        for s0 in range(0, len(reqs), B):
            eng = DecodeEngine(m, B, gamma=3, max_new_cap=16)
            chunk = reqs[s0:s0 + B]
            for b, (p, n) in enumerate(chunk):
                eng.prefill(b, p, n)
            eng.run()
            for b in range(len(chunk)):
                assert eng.result(b).new_tokens == alone[s0 + b], (B, s0 + b)


def test_qspec_equals_w4a16_ar_on_device_batched():
    m = toy(6, vocab_size=512)
    prompts = [[4, 9, 100, 3], [5, 6], [11, 12, 13, 14, 15], [1]]
    eng = DecodeEngine(m, 4, gamma=3, max_new_cap=24)
    ar = DecodeEngine(m, 4, gamma=3, max_new_cap=24, algorithm="greedy")
    for b, p in enumerate(prompts):
        eng.prefill(b, p, 20)
        ar.prefill(b, p, 20)
    eng.run()
    ar.run()
    for b in range(4):
        assert eng.result(b).new_tokens == ar.result(b).new_tokens


def test_cycle_accounting():
    m = toy(8)
    r = Q.generate_qspec(m, [5, 6], Q.GenerationConfig(gamma=4, max_new_tokens=17))
    assert sum(len(c.emitted) for c in r.cycles) == len(r.new_tokens) - 1
    for rec in r.cycles:
        assert 1 <= len(rec.emitted) <= 5 and rec.accept_len <= len(rec.drafted)
    txt = Q.format_trace(r.cycles)
    assert len(Q.parse_trace(txt)) == len(r.cycles)


@pytest.mark.parametrize("algorithm", ["qspec", "greedy"])
def test_attention_context_bound_matches_full_grid(algorithm):
    """The engine sizes the attention grid from a host bound on the committed lengths
    (engine._ctx_cap); runs crossing several 64-key chunk boundaries, with and without
    poll() tightening the bound mid-run, give the tokens and per-cycle traces of a run over
    the full KV capacity."""
    m = toy(9, vocab_size=512, max_seq_len=320)
    prompts = [[3, 1, 4, 1, 5] * 12, [2, 7], [9] * 130]
    runs = []
    for mode in ("full", "bound", "bound_nopoll"):
        eng = DecodeEngine(m, 3, gamma=3, max_new_cap=160, algorithm=algorithm)
        if mode == "full":
            eng._ctx_cap = lambda hi, e=eng: e.kv.capacity
        for b, p in enumerate(prompts):
            eng.prefill(b, p, 150)
        if mode == "bound_nopoll":
            for _ in range(200):
                eng.step()
            assert eng.all_done()
        else:
            eng.run()
        caps = sorted(eng.graphs)
        runs.append(([eng.result(b).new_tokens for b in range(3)], [eng.result(b).trace.tolist() for b in range(3)]))
        if mode != "full":
            assert len(caps) > 1 and min(caps) < eng.kv.capacity, caps
    assert runs[1] == runs[0] and runs[2] == runs[0]
