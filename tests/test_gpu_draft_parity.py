"""GPU parity of the W4A4 draft path and of the BASELINE shapes against the reference.

QSpec tokens equal W4A16 greedy tokens whatever the draft emits (specdec.py:159-176), so
token tests alone cannot see a broken draft.  What pins the draft:

* exact pieces, at full shapes: the RMSNorm feeding every draft operand (bit-exact with
  numpy's pairwise order, numerics.py:46-62), the activation codes / scales and the int32
  core (test_gpu_parity.py);
* the draft streams themselves -- LOW greedy tokens, per-cycle accept lengths,
  acceptance (specdec.py:103-133, 371-392) -- frozen from the UNMODIFIED reference by
  ``tests/golden/make_golden.py`` / ``make_golden_large.py``.

The W4A4 forward is chaotic under fp32 re-association: one activation code that lands
on the other side of a rounding boundary moves the next layer's inputs by ~1e-3 and
flips dozens of codes there.  The reference's own algorithm with float64-accurate
linear sums (``scripts/dev/low_flips.py``; ``tests/test_oracle_golden.py::
test_low_path_is_order_sensitive``) moves 2-layer 7B-shape LOW logits by ~20 %.  No
implementation that does not replay numpy's exact float32 operation order can match
LOW streams token for token everywhere, so stream-level draft checks are statistical,
with bounds calibrated on that float64 variant (``scripts/dev/low_calibrate.py``);
everything the HIGH path and QSpec emit is checked exactly.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import TINY, conftest_cfg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2410_11305_b200 as Q  # noqa: E402
from oracle import qspec_oracle as O  # noqa: E402

HIGH, LOW = Q.ExecutionMode.HIGH_PRECISION, Q.ExecutionMode.LOW_PRECISION
GOLD = os.path.join(os.path.dirname(__file__), "golden")

C7B = dict(d_model=4096, n_heads=32, n_kv_heads=32, d_ff=11008, vocab_size=32000, max_seq_len=512, group_size=128)
C8B = dict(d_model=4096, n_heads=32, n_kv_heads=8, d_ff=14336, vocab_size=128256, max_seq_len=512,
           rope_theta=500000.0, group_size=128)
LARGE = {"7b2l": (C7B, 2), "8b2l": (C8B, 2), "7b32": (C7B, 32)}


def large(case: str):
    path = os.path.join(GOLD, f"large_{case}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    return np.load(path)


# ----------------------------------------------------------------- RMSNorm (draft operand input)
@pytest.mark.parametrize("K", [7, 13, 64, 96, 200, 256, 1000, 4096, 5120])
def test_rmsnorm_bit_exact(K):
    rng = np.random.default_rng(K)
    x = (rng.standard_normal((5, K)) * rng.uniform(0.01, 40, size=(5, 1))).astype(np.float32)
    w = rng.uniform(0.5, 1.5, size=K).astype(np.float32)
    ref = O.rmsnorm(x, w, 1e-5)
    got = Q.rmsnorm(torch.from_numpy(x), torch.from_numpy(w), 1e-5).cpu().numpy()
    assert got.tobytes() == ref.tobytes()


# ----------------------------------------------------------------- draft streams on the toy configs
def _first_diff(a, b) -> int:
    return next((i for i, (x, y) in enumerate(zip(a, b)) if x != y), min(len(a), len(b)))


def test_tiny_greedy_low_stream(golden):
    m = Q.random_init(Q.ModelConfig(**TINY), 0)
    p = [int(t) for t in golden["tiny.prompts"][0]]
    r = Q.generate_greedy(m, p, LOW, Q.GenerationConfig(max_new_tokens=64))
    # float64-sum reference variant: identical for all 64 tokens
    assert _first_diff(r.new_tokens, [int(t) for t in golden["tiny.greedy_low0"]]) >= 32


def test_tiny_qspec_accept_traces(golden):
    m = Q.random_init(Q.ModelConfig(**TINY), 0)
    same, acc, drafted, ref_acc, ref_drafted = 0, 0, 0, 0.0, 0.0
    for i, p in enumerate(golden["tiny.prompts"]):
        r = Q.generate_qspec(m, [int(t) for t in p], Q.GenerationConfig(gamma=3, max_new_tokens=64))
        assert r.new_tokens == [int(t) for t in golden["tiny.greedy"][i]]
        a_ref, _, n_cyc = golden["tiny.qspec_stats"][i]
        same += int(len(r.cycles) == int(n_cyc) and r.acceptance_rate == a_ref)
        acc += sum(c.accept_len for c in r.cycles)
        drafted += sum(len(c.drafted) for c in r.cycles)
        ref_acc += a_ref * 3 * n_cyc  # every tiny cycle drafts gamma = 3 (64-token budget)
        ref_drafted += 3 * n_cyc
        if i == 0:
            assert [c.accept_len for c in r.cycles] == [int(a) for a in golden["tiny.qspec_accept_lens"]]
    assert same >= 6, same  # float64-sum variant: 8 / 8
    assert abs(acc / drafted - ref_acc / ref_drafted) <= 0.02


def test_toy6_acceptance_per_gamma(golden):
    m = Q.random_init(Q.ModelConfig(**conftest_cfg(vocab_size=512)), 6)
    d = []
    for gm in (1, 2, 3, 5, 7):
        r = Q.generate_qspec(m, [4, 9, 100, 3], Q.GenerationConfig(gamma=gm, max_new_tokens=14))
        assert r.new_tokens == [int(t) for t in golden[f"toy6.qspec.g{gm}"]], gm
        d.append(abs(r.acceptance_rate - float(golden[f"toy6.qspec.g{gm}.acc"][0])))
    assert np.mean(d) <= 0.05 and max(d) <= 0.15, d


def test_long_context_streams():
    # 8 prompts of 270 tokens: every attention pass merges >= 5 split-KV chunks of 64 keys
    g = large("ctx")
    m = Q.random_init(Q.ModelConfig(**dict(TINY, max_seq_len=400)), 0)
    low_full, acc, drafted, ref_acc, ref_drafted = 0, 0, 0, 0, 0
    for i in range(8):
        p = [int(t) for t in g[f"p{i}.prompt"]]
        hi = [int(t) for t in g[f"p{i}.greedy_high"]]
        assert Q.generate_greedy(m, p, HIGH, Q.GenerationConfig(max_new_tokens=40)).new_tokens == hi, i
        qs = Q.generate_qspec(m, p, Q.GenerationConfig(gamma=3, max_new_tokens=40))
        assert qs.new_tokens == hi, i
        acc += sum(c.accept_len for c in qs.cycles)
        drafted += sum(len(c.drafted) for c in qs.cycles)
        ref_acc += int(g[f"p{i}.qspec_accept_lens"].sum())
        ref_drafted += int(g[f"p{i}.qspec_drafted"].sum())
        lo = Q.generate_greedy(m, p, LOW, Q.GenerationConfig(max_new_tokens=40)).new_tokens
        low_full += int(lo == [int(t) for t in g[f"p{i}.greedy_low"]])
    assert low_full >= 5, low_full  # float64-sum variant: 6 / 8
    assert abs(acc / drafted - ref_acc / ref_drafted) <= 0.03, (acc / drafted, ref_acc / ref_drafted)


# ----------------------------------------------------------------- BASELINE shapes vs the reference
def _check_rows(got: np.ndarray, g, key: str, rel: float, rows=None) -> None:
    top_idx, top_val, absmax = g[f"{key}.top_idx"], g[f"{key}.top_val"], g[f"{key}.absmax"]
    rows = range(got.shape[0]) if rows is None else rows
    for r in rows:
        assert int(np.argmax(got[r])) == int(g[f"{key}.argmax"][r]), (key, r)
        assert abs(np.abs(got[r]).max() - absmax[r]) <= rel * absmax[r], (key, r)
        err = np.abs(got[r, top_idx[r]] - top_val[r]).max()
        assert err <= rel * absmax[r], (key, r, err / absmax[r])


_models: dict = {}


def _model(case: str):
    if case not in _models:
        _models.clear()
        cfg_kw, nl = LARGE[case]
        _models[case] = Q.random_init(Q.ModelConfig(n_layers=nl, **cfg_kw), 0)
    return _models[case]


@pytest.mark.parametrize("case", ["7b2l", "8b2l", "7b32"])
def test_shape_forward_logits(case):
    g = large(case)
    m = _model(case)
    toks = [int(t) for t in g["fwd_tokens"]]
    kv = Q.KVCache(m.config)
    # W4A16 verify shape (T = 4): every row, 1e-4 of max|logit|
    _check_rows(Q.forward(m, toks, kv, HIGH, Q.WriteTarget.VERIFY).numpy(), g, "fwd.high4", 1e-4)
    Q.kv_commit(kv, 3)
    if LARGE[case][1] > 2:
        return  # 32 W4A4 layers: the chaos (module docstring) reaches every row
    # W4A4 draft shape (T = 1) on the committed verify rows: the next draft token
    low1 = Q.forward(m, [int(g["fwd.low1_token"][0])], kv, LOW, Q.WriteTarget.DRAFT).numpy()
    assert int(np.argmax(low1[0])) == int(g["fwd.low1.argmax"][0])
    # W4A4 from an empty cache: position 0 sees no re-associated input before layer 0's
    # attention, so two layers of it are pinned tightly; later rows are chaotic
    low4 = Q.forward(m, toks, Q.KVCache(m.config), LOW, Q.WriteTarget.VERIFY).numpy()
    _check_rows(low4, g, "fwd.low4", 1e-3, rows=[0])


@pytest.mark.parametrize("case", ["7b2l", "8b2l", "7b32"])
def test_shape_streams(case):
    g = large(case)
    m = _model(case)
    p = [int(t) for t in g["prompt"]]
    gr = Q.generate_greedy(m, p, HIGH, Q.GenerationConfig(max_new_tokens=8))
    assert gr.new_tokens == [int(t) for t in g["greedy_high"]]
    qs = Q.generate_qspec(m, p, Q.GenerationConfig(gamma=3, max_new_tokens=8))
    assert qs.new_tokens == gr.new_tokens
