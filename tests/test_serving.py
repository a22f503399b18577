"""FCFS continuous batching (serving.py) -- ports of the reference's serving tests
(pkg/tests/test_serving_costmodel.py): workload parsing, validation, rejection,
and the batching contract (a request's tokens equal its standalone generation)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import TINY, conftest_cfg

import paper_2410_11305_b200 as Q
from paper_2410_11305_b200 import serving as S


def test_parse_workload_and_errors():
    reqs = S.parse_workload("# comment\nr0 4 1 2 3\n\nr1 2 7\n")
    assert [r.id for r in reqs] == ["r0", "r1"]
    assert reqs[0].prompt == [1, 2, 3] and reqs[0].max_new_tokens == 4 and reqs[1].arrival_index == 1
    for bad in ("r0 4", "r0 x 1", "r0 0 1", "", "# only comment"):
        with pytest.raises(Q.WorkloadError):
            S.parse_workload(bad)


def test_validation_before_any_device_work():
    r = [S.Request("a", [1], 2, 0)]
    cfg = Q.GenerationConfig()
    with pytest.raises(Q.ConfigError):
        S.run_fcfs(r, 0, None, cfg)
    with pytest.raises(Q.ConfigError):
        S.run_fcfs([], 2, None, cfg)
    with pytest.raises(Q.ConfigError):
        S.run_fcfs(r, 2, None, cfg, mode="beam")
    with pytest.raises(Q.WorkloadError):
        S.run_fcfs(r + [S.Request("a", [2], 2, 1)], 2, None, cfg)


def test_latency_split_and_format():
    st = S.ServingStats(10, 1.0, 10.0, 3, 4, 1.0, 30.0, 20.0, 0.1, 0.2, 0.3, 0.4, [], [], ["a"], ["a"],
                        [S.RejectedRequest("b", "empty prompt")])
    sp = S.per_valid_token_latency(st)
    assert sp.draft_share == 3.0 and sp.verify_share == 2.0 and sp.total == 5.0
    txt = S.format_stats(st)
    assert "total_new_tokens: 10" in txt and "rejected: b empty prompt" in txt
    with pytest.raises(Q.ConfigError):
        S.per_valid_token_latency(S.ServingStats(0, 1.0, 0.0, 0, 0, 0, 0, 0, 0, 0, 0, 0, [], [], [], [], []))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["qspec", "greedy-high"])
def test_fcfs_matches_standalone(mode):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg_kw = dict(conftest_cfg(), max_seq_len=96)
    model = Q.random_init(Q.ModelConfig(**cfg_kw), 0)
    rng = np.random.default_rng(5)
    reqs = [S.Request(f"r{i}", [int(t) for t in rng.integers(0, cfg_kw["vocab_size"], 3 + i)], 6 + 3 * (i % 4), i)
            for i in range(7)]
    reqs.append(S.Request("empty", [], 4, 7))
    reqs.append(S.Request("toolong", [1] * 90, 20, 8))
    gcfg = Q.GenerationConfig(gamma=3, max_new_tokens=32)
    out, stats = S.run_fcfs(reqs, 3, model, gcfg, mode=mode)
    assert sorted(r.id for r in stats.rejected) == ["empty", "toolong"]
    assert stats.admission_order[:3] == ["r0", "r1", "r2"]
    assert set(stats.completion_order) == {f"r{i}" for i in range(7)}
    for r in reqs[:7]:
        c = Q.GenerationConfig(gamma=3, max_new_tokens=r.max_new_tokens)
        ref = Q.generate_qspec(model, r.prompt, c) if mode == "qspec" else \
            Q.generate_greedy(model, r.prompt, Q.ExecutionMode.HIGH_PRECISION, c)
        assert out[r.id].new_tokens == ref.new_tokens, r.id
    assert stats.total_new_tokens == sum(len(v.new_tokens) for v in out.values())
    # per-step cost units add up to the per-request totals (serving.py:182-187)
    assert sum(stats.step_draft_units) == pytest.approx(stats.draft_cost_units)
    assert sum(stats.step_verify_units) == pytest.approx(stats.verify_cost_units)


@pytest.mark.gpu
def test_fcfs_tiny_against_oracle():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from oracle import qspec_oracle as O
    model = Q.random_init(Q.ModelConfig(**TINY), 0)
    om = O.random_model(O.OracleConfig(**TINY), 0)
    rng = np.random.default_rng(42)
    reqs = [S.Request(f"q{i}", [int(t) for t in rng.integers(0, 1024, 16)], 12, i) for i in range(5)]
    out, _ = S.run_fcfs(reqs, 2, model, Q.GenerationConfig(gamma=3, max_new_tokens=12))
    for r in reqs:
        assert out[r.id].new_tokens == O.generate(om, r.prompt, gamma=3, max_new=12).new_tokens
