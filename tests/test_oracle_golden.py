"""Pin the CPU oracle to the reference: every golden fixture must match bit-exactly.

Fixtures come from ``tests/golden/make_golden.py`` (the unmodified reference
imported in the build container).  Frozen vectors from the reference's own
tests are checked verbatim (pkg/tests/test_storage_cli.py:31-57).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import MODEL_SPECS, TINY, conftest_cfg
from oracle import qspec_oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_lcg_known_recurrence():
    # pkg/tests/test_storage_cli.py:53-57
    assert O.lcg_jump(0, 1) == 1442695040888963407


def test_lcg_stream_and_jump(golden):
    assert np.array_equal(O.LcgStream(1234).floats(64), golden["lcg_seed1234_first64"])
    assert O.lcg_jump(77, 10_000) == int(golden["lcg_seed77_after10000_state"][0])


def test_golden_q_proj_codes():
    # pkg/tests/test_storage_cli.py:31-39,75-77
    cfg = O.OracleConfig(**conftest_cfg(max_seq_len=128))
    m = O.random_model(cfg, 42)
    assert m.layers[0]["q_proj"].packed()[:16].tobytes() == bytes(
        [147, 189, 11, 13, 82, 207, 165, 234, 188, 52, 201, 74, 195, 167, 86, 207])


def test_toy_model_stores(golden):
    m = O.random_model(O.OracleConfig(**conftest_cfg()), 0)
    assert np.array_equal(m.emb, golden["toy0.token_embedding"])
    for i, lw in enumerate(m.layers):
        for p in O.PROJ:
            assert np.array_equal(lw[p].packed(), golden[f"toy0.layers.{i}.{p}.codes"])
            assert np.array_equal(lw[p].scales, golden[f"toy0.layers.{i}.{p}.scales"])
    assert np.array_equal(m.lm_head.packed(), golden["toy0.lm_head.codes"])


def test_tiny_model_digests(golden):
    m = O.random_model(O.OracleConfig(**TINY), 0)
    got = [f"layers.{i}.{p}:{sha(lw[p].packed())}:{sha(lw[p].scales)}"
           for i, lw in enumerate(m.layers) for p in O.PROJ]
    got.append(f"lm_head:{sha(m.lm_head.packed())}:{sha(m.lm_head.scales)}")
    assert got == [str(s) for s in golden["tiny.digests"]]
    assert sha(m.emb) == str(golden["tiny.emb_digest"][0])


@pytest.mark.parametrize("gs", [16, 32, 128])
def test_activation_quantizer(golden, gs):
    x = golden[f"aq{gs}.x"]
    codes, scales = O.quantize_rows(x, gs)
    assert np.array_equal(codes, golden[f"aq{gs}.codes"])
    assert np.array_equal(scales, golden[f"aq{gs}.scales"])
    assert np.array_equal(O.fake_quant(x, gs), golden[f"aq{gs}.fq"])
    assert codes.min() >= -7 and codes.max() <= 7   # -8 is never produced


def test_pack_unpack_round_trip():
    c = np.random.default_rng(0).integers(-8, 8, size=513).astype(np.int8)
    assert np.array_equal(O.unpack_nibbles(O.pack_nibbles(c), 513), c)
    assert O.pack_nibbles(np.array([3, -2], np.int8))[0] == (3 & 0xF) | ((-2 & 0xF) << 4)


def test_qlinear_both_modes(golden):
    m = O.random_model(O.OracleConfig(**conftest_cfg()), 0)
    x = golden["ql.x"]
    assert np.array_equal(O.qlinear(m.layers[0]["q_proj"], x, False), golden["ql.high"])
    assert np.array_equal(O.qlinear(m.layers[0]["q_proj"], x, True), golden["ql.low"])


@pytest.mark.parametrize("tag,low", [("high", False), ("low", True)])
def test_forward_logits_and_kv(golden, tag, low):
    cfg = O.OracleConfig(**conftest_cfg())
    m = O.random_model(cfg, 0)
    kv = O.OracleKV(cfg)
    logits = O.forward(m, [5, 9, 200, 3, 77], kv, low, "verify")
    assert np.array_equal(logits, golden[f"fwd.{tag}"])
    assert np.array_equal(kv.reg["verify"][0][0][:5], golden[f"fwd.{tag}.k0"])


def test_tiny_generation_streams(golden):
    m = O.random_model(O.OracleConfig(**TINY), 0)
    prompts = golden["tiny.prompts"]
    for i in (0, 3):
        p = [int(t) for t in prompts[i]]
        gr = O.generate(m, p, max_new=64, qspec=False)
        assert gr.new_tokens == [int(t) for t in golden["tiny.greedy"][i]]
        qs = O.generate(m, p, gamma=3, max_new=64)
        assert qs.tokens == gr.tokens
        st = golden["tiny.qspec_stats"][i]
        assert qs.acceptance_rate == st[0] and qs.tokens_per_cycle == st[1] and len(qs.cycles) == st[2]
        if i == 0:
            assert [c[1] for c in qs.cycles] == [int(a) for a in golden["tiny.qspec_accept_lens"]]
    low = O.generate(m, [int(t) for t in prompts[0]], max_new=64, qspec=False, low_greedy=True)
    assert low.new_tokens == [int(t) for t in golden["tiny.greedy_low0"]]


def test_toy_gamma_sweep(golden):
    m = O.random_model(O.OracleConfig(**conftest_cfg(vocab_size=512)), 6)
    ref = [int(t) for t in golden["toy6.greedy"]]
    assert O.generate(m, [4, 9, 100, 3], max_new=14, qspec=False).new_tokens == ref
    for gm in (1, 2, 3, 5, 7):
        r = O.generate(m, [4, 9, 100, 3], gamma=gm, max_new=14)
        assert r.new_tokens == [int(t) for t in golden[f"toy6.qspec.g{gm}"]] == ref
        assert r.acceptance_rate == float(golden[f"toy6.qspec.g{gm}.acc"][0])


@pytest.mark.parametrize("mi", range(len(MODEL_SPECS)))
def test_acceptance_shapes(golden, mi):
    cfg = O.OracleConfig(**conftest_cfg(max_seq_len=48, **MODEL_SPECS[mi]))
    m = O.random_model(cfg, 1000 + mi)
    for pi in range(3):
        p = [int(t) for t in golden[f"spec{mi}.p{pi}.prompt"]]
        ref = [int(t) for t in golden[f"spec{mi}.p{pi}.greedy"]]
        assert O.generate(m, p, max_new=12, qspec=False).new_tokens == ref
        assert O.generate(m, p, gamma=3, max_new=12).new_tokens == ref


@pytest.mark.parametrize("n", [1, 5, 7, 8, 13, 64, 96, 127, 128, 200, 256, 1000, 4096, 5120])
def test_pairwise_sum_is_numpys_mean_order(n):
    # the device RMSNorm implements O.pairwise_sum_f32's order (csrc/pack_dev.cuh); pin it
    # to np.mean(x*x, dtype=float32) of numerics.py:60 on rows where the order matters
    rng = np.random.default_rng(n)
    x = (rng.standard_normal((6, n)) * rng.uniform(0.01, 50, size=(6, 1))).astype(np.float32)
    ref = np.mean(x * x, axis=-1, keepdims=True, dtype=np.float32)[:, 0]
    got = np.array([O.pairwise_sum_f32(r * r) / np.float32(n) for r in x], dtype=np.float32)
    assert got.tobytes() == ref.tobytes()


def test_pairwise_order_is_discriminating():
    # a plain sequential fp32 sum disagrees with numpy on 4096-wide rows (the 7B d_model):
    # the test above would catch a device reduction in the wrong order
    rng = np.random.default_rng(1)
    x = (rng.standard_normal((64, 4096)) * 3).astype(np.float32)
    ref = np.mean(x * x, axis=-1, dtype=np.float32)
    seq = []
    for r in x:
        acc = np.float32(0)
        for v in (r * r):
            acc = np.float32(acc + v)
        seq.append(np.float32(acc / np.float32(4096)))
    assert (np.array(seq, dtype=np.float32) != ref).any()


def test_long_context_streams():
    # tests/golden/large_ctx.npz: C0 tiny with 270-token prompts (>= 5 split-KV chunks)
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "large_ctx.npz"))
    m = O.random_model(O.OracleConfig(**dict(TINY, max_seq_len=400)), 0)
    for i in (0, 5):
        p = [int(t) for t in g[f"p{i}.prompt"]]
        gr = O.generate(m, p, max_new=40, qspec=False)
        assert gr.new_tokens == [int(t) for t in g[f"p{i}.greedy_high"]]
        qs = O.generate(m, p, gamma=3, max_new=40)
        assert qs.tokens == gr.tokens
        assert [c[1] for c in qs.cycles] == [int(a) for a in g[f"p{i}.qspec_accept_lens"]]
        assert qs.acceptance_rate == g[f"p{i}.qspec_stats"][0] and qs.tokens_per_cycle == g[f"p{i}.qspec_stats"][1]
        low = O.generate(m, p, max_new=40, qspec=False, low_greedy=True)
        assert low.new_tokens == [int(t) for t in g[f"p{i}.greedy_low"]]


def test_low_path_is_order_sensitive():
    # The reference's W4A4 forward with float64-accurate linear sums (what a device
    # integer core computes, up to its fp32 epilogue) instead of einsum's sequential
    # float32 sums: identical W4A16 tokens, but the W4A4 greedy stream parts ways within
    # a few tokens on this 270-token prompt -- one flipped activation code cascades.
    # This is why draft-stream parity is statistical (tests/test_gpu_draft_parity.py).
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "large_ctx.npz"))
    m = O.random_model(O.OracleConfig(**dict(TINY, max_seq_len=400)), 0)
    p = [int(t) for t in g["p0.prompt"]]
    ref_low = [int(t) for t in g["p0.greedy_low"]]
    orig = O.qlinear

    def f64_sums(lin, x, low):
        xq = O.fake_quant(x, lin.g) if low else x
        return (xq.astype(np.float64) @ lin.wt.astype(np.float64)).astype(np.float32)

    try:
        O.qlinear = f64_sums
        hi = O.generate(m, p, max_new=40, qspec=False).new_tokens
        lo = O.generate(m, p, max_new=40, qspec=False, low_greedy=True).new_tokens
    finally:
        O.qlinear = orig
    assert hi == [int(t) for t in g["p0.greedy_high"]]
    assert lo[:3] == ref_low[:3] and lo != ref_low
