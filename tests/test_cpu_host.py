"""CPU-only checks: the C-ABI library loads and exports every symbol of include/qspec_b200.h,
the ctypes mirrors match the header, and host-side logic that needs no device."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "qspec_b200.h")


def header_functions() -> list[str]:
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(qs_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2410_11305_b200 import _lib
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)


def test_version_string_no_device_needed():
    from paper_2410_11305_b200 import _lib
    assert b"sm_100a" in _lib.load().qs_version()


def test_struct_sizes_match_header_layout():
    from paper_2410_11305_b200 import _lib
    assert ctypes.sizeof(_lib.QWeight) == 16 + 9 * 4 + 4     # two pointers, nine int32, tail padding
    assert ctypes.sizeof(_lib.Batch) == 4 + 4 + 3 * 8 + 8 + 2 * 8 + 8   # T(+pad), 3 ptrs, n_blk(+pad), 2 ptrs, 2 int
    assert ctypes.sizeof(_lib.Workspace) == 12 * 8


def test_geometry_and_errors():
    from paper_2410_11305_b200 import _lib
    from paper_2410_11305_b200.errors import ConfigError
    g = _lib.QWeight()
    _lib.call("qs_qweight_geometry", 11008, 4096, 128, g)
    assert (g.n_pad, g.n_tiles, g.G, g.gp, g.cpg, g.n_chunks) == (11008, 86, 32, 128, 1, 32)
    _lib.call("qs_qweight_geometry", 320, 192, 48, g)
    assert (g.n_pad, g.G, g.gp, g.n_chunks) == (384, 4, 128, 4)
    with pytest.raises(ConfigError):
        _lib.call("qs_qweight_geometry", 10, 100, 32, g)


def test_workspace_sizes_7b():
    from paper_2410_11305_b200 import _lib
    m = _lib.Model(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=32, d_ff=11008, vocab=32000, group_size=128,
                   rope_len=576)
    s = _lib.WorkspaceSizes()
    _lib.call("qs_workspace_size", m, 64, s)
    # two operand slots (the fused next-operand emits double-buffer the image), ascale +
    # acorr per slot, per-tile counters + emit counters + emit leaf sums
    assert s.img == 2 * 86 * 192 * 128 and s.ascale == 2 * 86 * 64 * 4 * 5
    assert s.counters == (4096 + 8 + 1024 + 2 * 64 * 128) * 4  # + two emit leaf buffers


def test_model_config_validation_mirrors_reference():
    from paper_2410_11305_b200 import ModelConfig
    from paper_2410_11305_b200.errors import ConfigError
    base = dict(n_layers=2, d_model=64, n_heads=4, n_kv_heads=2, d_ff=128, vocab_size=256, max_seq_len=96,
                group_size=32)
    ModelConfig(**base)
    for over in ({"d_model": 65}, {"n_heads": 3}, {"n_kv_heads": 3}, {"d_ff": 100}, {"n_layers": 0},
                 {"norm_eps": 0.0}):   # pkg/tests/test_model.py:22-36
        with pytest.raises(ConfigError):
            ModelConfig(**{**base, **over})


def test_generation_config_validation():
    from paper_2410_11305_b200 import GenerationConfig
    from paper_2410_11305_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        GenerationConfig(gamma=0)
    with pytest.raises(ConfigError):
        GenerationConfig(max_new_tokens=0)


def test_pack_unpack_layout():
    from paper_2410_11305_b200 import pack_int4, unpack_int4
    codes = np.arange(-8, 8, dtype=np.int8)
    assert np.array_equal(unpack_int4(pack_int4(codes), 16), codes)
    assert pack_int4(np.array([3, -2], np.int8))[0] == (3 & 0xF) | ((-2 & 0xF) << 4)


def test_accept_greedy_hand_cases():
    # pkg/tests/test_specdec.py:123-157 with host logits blocks
    import torch
    from paper_2410_11305_b200 import ExecutionMode, LogitsBlock, accept_greedy
    from paper_2410_11305_b200.errors import ShapeError

    def oh(ids, vocab):
        rows = torch.zeros(len(ids), vocab)
        for j, t in enumerate(ids):
            rows[j, t] = 1.0
        return LogitsBlock(rows, ExecutionMode.HIGH_PRECISION)

    assert accept_greedy([5, 6, 7], oh([5, 6, 7, 8], 16)) == (3, 8, True)
    assert accept_greedy([5, 6, 7], oh([9, 6, 7, 8], 16)) == (0, 9, False)
    assert accept_greedy([5, 6, 7], oh([5, 6, 12, 8], 16)) == (2, 12, False)
    with pytest.raises(ShapeError):
        accept_greedy([1, 2], oh([1, 2], 8))


def test_trace_round_trip():
    from paper_2410_11305_b200 import CycleRecord, TokenSource, format_trace, parse_trace
    from paper_2410_11305_b200.errors import TraceError
    rec = CycleRecord([1, 2], 1, [1, 9], TokenSource.RESAMPLED, 2.0, 3.0)
    txt = format_trace([rec], request_id="r7")
    assert "request=r7" in txt and parse_trace(txt)[0].drafted == [1, 2]
    with pytest.raises(TraceError):
        parse_trace("cycle=0 drafted=1 accept_len=2 emitted=1 source=bonus draft_cost_units=1.0 verify_cost_units=1.0")


def test_lcg_offsets_match_oracle():
    from paper_2410_11305_b200.model import ModelConfig
    from paper_2410_11305_b200.storage import draw_offsets
    from oracle import qspec_oracle as O
    kw = dict(n_layers=3, d_model=96, n_heads=6, n_kv_heads=3, d_ff=192, vocab_size=768, max_seq_len=48,
              group_size=48)
    assert draw_offsets(ModelConfig(**kw)) == O.lcg_offsets(O.OracleConfig(**kw))


def test_device_ops_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2410_11305_b200 as Q
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        Q.random_init(Q.ModelConfig(n_layers=1, d_model=64, n_heads=4, n_kv_heads=4, d_ff=128, vocab_size=64,
                                    max_seq_len=32, group_size=32), 0)
