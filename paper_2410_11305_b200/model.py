"""Decoder model, shared paged KV cache and the forward step (drop-in for pkg/src/qspec/model.py).

Device layout:
  * per layer four fused int4 stores: q|k|v, o, gate/up (rows interleaved so
    the linear epilogue computes silu(gate)*up), down; plus lm_head;
  * fp32 embedding, norms and RoPE tables (tables built on the host exactly as
    numerics.py:97-116, f64 angles cast to f32);
  * one paged fp32 KV pool per cache, [layer][page][kv_head][page_size][head_dim].

KV semantics: the reference keeps committed rows plus separate DRAFT / VERIFY
scratch regions and copies verify rows on commit (model.py:152-229).  Here the
draft and verify passes of a cycle write the SAME positions committed_len + j
of one paged cache, verify overwriting draft in place, so ``kv_commit`` is a
length update with no copy.  The committed prefix is bit-identical to the
reference's (it always holds verify-produced rows); the only observable
difference is that a DRAFT pass issued after an uncommitted VERIFY pass
overwrites those verify rows -- an order the QSpec loop never produces.
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .errors import ConfigError, SequenceOverflowError, ShapeError, TokenIdError
from .quant import (DEFAULT_GROUP_SIZE, DeviceStore, ExecutionMode, QuantizedTensor, _count_act_quant,
                    _log_qlinear)

DEFAULT_GAMMA_MAX = 8
PAGE_SIZE = 16


@dataclass
class ModelConfig:
    """model.py:32-69 (same fields, defaults and validation)."""

    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    d_ff: int
    vocab_size: int
    max_seq_len: int
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    group_size: int = DEFAULT_GROUP_SIZE
    # Opt-in, default off (the reference has no rotation): rotate
    # every linear's input groups and weight rows by the orthonormal 128-point Hadamard
    # transform before quantising (x H . (W H)^T = x W^T; spreads activation outliers for the
    # W4A4 draft).  Off, every result is the reference's; on, it needs group_size 128.
    hadamard: bool = False

    def __post_init__(self) -> None:
        for name in ("n_layers", "d_model", "n_heads", "n_kv_heads", "d_ff", "vocab_size", "max_seq_len",
                     "group_size"):
            if int(getattr(self, name)) < 1:
                raise ConfigError(f"{name} must be >= 1, got {getattr(self, name)}")
        if self.d_model % self.n_heads:
            raise ConfigError("d_model must be divisible by n_heads")
        if self.n_heads % self.n_kv_heads:
            raise ConfigError("n_heads must be divisible by n_kv_heads")
        if self.d_model % self.group_size or self.d_ff % self.group_size:
            raise ConfigError("d_model and d_ff must be divisible by group_size")
        if (self.d_model // self.n_heads) % 2:
            raise ConfigError("head dimension must be even for rotary embeddings")
        if self.rope_theta <= 0 or self.norm_eps <= 0:
            raise ConfigError("rope_theta and norm_eps must be positive")
        if self.hadamard and self.group_size != 128:
            raise ConfigError("the Hadamard rotation works on 128-wide groups (group_size must be 128)")

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads


def rope_tables(n_pos: int, hd: int, theta: float) -> tuple[np.ndarray, np.ndarray]:
    """numerics.py:97-116: angles in float64, cast to float32 after cos/sin."""
    inv = 1.0 / (theta ** (np.arange(0, hd, 2, dtype=np.float64) / hd))
    ang = np.arange(n_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


@dataclass(eq=False)
class LayerWeights:
    """model.py:72-84: per-projection handles are views of the fused device stores."""

    attn_norm: object
    ffn_norm: object
    qkv: DeviceStore = field(repr=False)
    o: DeviceStore = field(repr=False)
    gate_up: DeviceStore = field(repr=False)
    down: DeviceStore = field(repr=False)
    q_proj: QuantizedTensor = field(repr=False, default=None)
    k_proj: QuantizedTensor = field(repr=False, default=None)
    v_proj: QuantizedTensor = field(repr=False, default=None)
    o_proj: QuantizedTensor = field(repr=False, default=None)
    gate_proj: QuantizedTensor = field(repr=False, default=None)
    up_proj: QuantizedTensor = field(repr=False, default=None)
    down_proj: QuantizedTensor = field(repr=False, default=None)


def make_layer_stores(cfg: ModelConfig, attn_norm, ffn_norm) -> LayerWeights:
    H, KV, hd, d, ff, g = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.d_model, cfg.d_ff, cfg.group_size
    qkv = DeviceStore.empty((H + 2 * KV) * hd, d, g)
    o = DeviceStore.empty(d, d, g)
    gu = DeviceStore.empty(2 * ff, d, g)
    dn = DeviceStore.empty(d, ff, g)
    lw = LayerWeights(attn_norm, ffn_norm, qkv, o, gu, dn)
    lw.q_proj = QuantizedTensor(H * hd, d, g, qkv, 0, 1)
    lw.k_proj = QuantizedTensor(KV * hd, d, g, qkv, H * hd, 1)
    lw.v_proj = QuantizedTensor(KV * hd, d, g, qkv, (H + KV) * hd, 1)
    lw.o_proj = QuantizedTensor(d, d, g, o)
    lw.gate_proj = QuantizedTensor(ff, d, g, gu, 0, 2)
    lw.up_proj = QuantizedTensor(ff, d, g, gu, 1, 2)
    lw.down_proj = QuantizedTensor(d, ff, g, dn)
    for p in PROJ_NAMES:
        getattr(lw, p).rotated = cfg.hadamard
    return lw


PROJ_NAMES = ("q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj")


class TransformerModel:
    """model.py:87-121: immutable device weights, shareable by many caches / engines."""

    def __init__(self, config: ModelConfig, token_embedding, layers: list[LayerWeights], final_norm,
                 lm_head: QuantizedTensor) -> None:
        import torch
        if len(layers) != config.n_layers:
            raise ConfigError(f"expected {config.n_layers} layers, got {len(layers)}")
        if tuple(token_embedding.shape) != (config.vocab_size, config.d_model):
            raise ShapeError("token_embedding shape mismatch")
        self.config = config
        self.token_embedding = token_embedding
        self.layers = layers
        self.final_norm = final_norm
        self.lm_head = lm_head
        self.rope_len = config.max_seq_len + 64
        cos, sin = rope_tables(self.rope_len, config.head_dim, config.rope_theta)
        self.rope_cos = torch.from_numpy(cos).cuda()
        self.rope_sin = torch.from_numpy(sin).cuda()
        self._c_layers = (_lib.Layer * config.n_layers)()
        for i, lw in enumerate(layers):
            cl = self._c_layers[i]
            cl.attn_norm, cl.ffn_norm = lw.attn_norm.data_ptr(), lw.ffn_norm.data_ptr()
            cl.qkv, cl.o, cl.gate_up, cl.down = lw.qkv.geo, lw.o.geo, lw.gate_up.geo, lw.down.geo
        self._ws_cache: dict = {}

    def quantized_tensors(self) -> list[tuple[str, QuantizedTensor]]:
        out = []
        for i, lw in enumerate(self.layers):
            for p in PROJ_NAMES:
                out.append((f"layers.{i}.{p}", getattr(lw, p)))
        out.append(("lm_head", self.lm_head))
        return out

    @property
    def weight_bytes_per_forward(self) -> int:
        """Algorithmic weight bytes one forward streams (codes + scales of every store)."""
        tot = self.lm_head.store.weight_bytes
        for lw in self.layers:
            tot += lw.qkv.weight_bytes + lw.o.weight_bytes + lw.gate_up.weight_bytes + lw.down.weight_bytes
        return tot

    def c_model(self, kv: "KVCache") -> _lib.Model:
        cfg = self.config
        m = _lib.Model(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
                       n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab_size,
                       group_size=cfg.group_size, rope_len=self.rope_len, norm_eps=cfg.norm_eps,
                       tok_emb=self.token_embedding.data_ptr(), final_norm=self.final_norm.data_ptr(),
                       rope_cos=self.rope_cos.data_ptr(), rope_sin=self.rope_sin.data_ptr(),
                       lm_head=self.lm_head.store.geo, block_table=kv.block_table.data_ptr(),
                       bt_ld=kv.block_table.shape[1], page=kv.page, hadamard=int(cfg.hadamard))
        layers = (_lib.Layer * cfg.n_layers)()
        for i in range(cfg.n_layers):
            layers[i] = self._c_layers[i]
            layers[i].k_cache = kv.k[i].data_ptr()
            layers[i].v_cache = kv.v[i].data_ptr()
        m._layers_keepalive = layers
        m.layers = ctypes.cast(layers, ctypes.POINTER(_lib.Layer))
        return m

    def workspace(self, t_max: int = 64):
        """Cached scratch per (model, thread, device) -- allocated once; the kernels leave
        counters zeroed.  Engines over one shared model may run in threads,
        so no two threads ever share a workspace."""
        import torch
        key = (t_max, threading.get_ident(), torch.cuda.current_device())
        if key not in self._ws_cache:
            probe = _lib.Model(n_layers=self.config.n_layers, d_model=self.config.d_model,
                               n_heads=self.config.n_heads, n_kv_heads=self.config.n_kv_heads,
                               d_ff=self.config.d_ff, vocab=self.config.vocab_size,
                               group_size=self.config.group_size, rope_len=self.rope_len)
            sizes = _lib.WorkspaceSizes()
            _lib.call("qs_workspace_size", probe, t_max, sizes)
            bufs = {n: torch.zeros(max(16, getattr(sizes, n)), dtype=torch.uint8, device="cuda")
                    for n, _ in _lib.WorkspaceSizes._fields_}
            ws = _lib.Workspace(**{n: b.data_ptr() for n, b in bufs.items()})
            self._ws_cache[key] = (ws, bufs)
        return self._ws_cache[key]


class WriteTarget(Enum):
    DRAFT = "draft"
    VERIFY = "verify"


@dataclass
class LogitsBlock:
    """model.py:131-139; ``logits`` is a device float32 tensor [n, vocab]."""

    logits: object
    mode: ExecutionMode
    argmax: object = None

    def row(self, j: int):
        return self.logits[j]

    def numpy(self) -> np.ndarray:
        return self.logits.cpu().numpy()


@dataclass
class CostCounter:
    units: int = 0

    def add(self, macs: int) -> None:
        self.units += macs


class KVCache:
    """Paged fp32 KV cache of one sequence or of a batch of slots (model.py:152-201).

    ``slots`` > 1 gives the batched engine one block-table row per slot over a
    shared page pool.  Region lengths follow the reference's bookkeeping; both
    regions alias positions committed_len.. of the single paged cache.
    """

    def __init__(self, config: ModelConfig, gamma_max: int = DEFAULT_GAMMA_MAX, *, slots: int = 1,
                 page: int = PAGE_SIZE) -> None:
        import torch
        if gamma_max < 1:
            raise ConfigError("gamma_max must be >= 1")
        if page < 1 or page & (page - 1):
            raise ConfigError("KV page size must be a power of two")
        _lib.require_cuda()
        self.config = config
        self.gamma_max = gamma_max
        self.scratch_capacity = gamma_max + 1
        self.page = page
        self.capacity = config.max_seq_len + gamma_max + 1
        pages = -(-self.capacity // page)
        self.block_table = (torch.arange(slots * pages, dtype=torch.int32, device="cuda")
                            .reshape(slots, pages).contiguous())
        shape = (slots * pages, config.n_kv_heads, page, config.head_dim)
        self.k = [torch.zeros(shape, dtype=torch.float32, device="cuda") for _ in range(config.n_layers)]
        self.v = [torch.zeros(shape, dtype=torch.float32, device="cuda") for _ in range(config.n_layers)]
        self.committed_len = 0
        self.draft_len = 0
        self.verify_len = 0
        self.pending_token: int | None = None

    def region_len(self, target: WriteTarget) -> int:
        return self.draft_len if target is WriteTarget.DRAFT else self.verify_len

    def _set_region_len(self, target: WriteTarget, v: int) -> None:
        if target is WriteTarget.DRAFT:
            self.draft_len = v
        else:
            self.verify_len = v

    def clear_scratch(self) -> None:
        self.draft_len = 0
        self.verify_len = 0

    def rows(self, layer: int, start: int, stop: int, which: str = "k", slot: int = 0):
        """Gather positions [start, stop) of one slot as [n, kv_heads, head_dim] (device)."""
        import torch
        pos = torch.arange(start, stop, device="cuda")
        pages = self.block_table[slot, pos // self.page].long()
        buf = (self.k if which == "k" else self.v)[layer]
        return buf[pages, :, pos % self.page, :]

    @property
    def committed_k(self):
        return [self.rows(i, 0, self.committed_len, "k") for i in range(self.config.n_layers)]

    @property
    def committed_v(self):
        return [self.rows(i, 0, self.committed_len, "v") for i in range(self.config.n_layers)]


def kv_reset(kv: KVCache) -> None:
    kv.committed_len = 0
    kv.clear_scratch()
    kv.pending_token = None


def kv_commit(kv: KVCache, accept_len: int) -> None:
    """model.py:211-229: keep pending + accept_len verify rows.  In-place cache: no copy."""
    need = accept_len + 1
    if accept_len < 0 or need > kv.verify_len:
        raise SequenceOverflowError(f"accept_len {accept_len} exceeds verify-scratch contents ({kv.verify_len})")
    if kv.committed_len + need > kv.config.max_seq_len:
        raise SequenceOverflowError("commit would exceed max_seq_len")
    kv.committed_len += need
    kv.clear_scratch()


def kv_memory_report(kv: KVCache) -> dict[str, int]:
    cfg = kv.config
    per_position = cfg.n_layers * 2 * cfg.n_kv_heads * cfg.head_dim * 4
    return {"committed_bytes": kv.committed_len * per_position,
            "scratch_bytes": 2 * kv.scratch_capacity * per_position,
            "per_position_bytes": per_position}


def _macs(cfg: ModelConfig, n: int, base: int) -> int:
    """model.py:310,330,337,344: deterministic MAC count of one forward."""
    hd, kvd = cfg.head_dim, cfg.n_kv_heads * cfg.head_dim
    per_layer = n * cfg.d_model * (cfg.d_model + 2 * kvd) + n * cfg.d_model * (cfg.d_model + 3 * cfg.d_ff)
    attn = sum(2 * cfg.n_heads * hd * (base + j + 1) for j in range(n))
    return cfg.n_layers * (per_layer + attn) + n * cfg.d_model * cfg.vocab_size


class _BatchBuffers:
    """Device staging for one single-sequence forward chunk."""

    def __init__(self) -> None:
        import torch
        self.ids = torch.zeros(64, dtype=torch.int32, device="cuda")
        self.pos = torch.zeros(64, dtype=torch.int32, device="cuda")
        self.slot = torch.zeros(64, dtype=torch.int32, device="cuda")
        self.blk = torch.zeros(2, dtype=torch.int32, device="cuda")
        self.arg = torch.zeros(64, dtype=torch.int32, device="cuda")


_tls = threading.local()  # staging buffers per (thread, device): engines may run in threads


def _batch_buffers() -> _BatchBuffers:
    import torch
    per = getattr(_tls, "bb", None)
    if per is None:
        per = _tls.bb = {}
    dev = torch.cuda.current_device()
    if dev not in per:
        per[dev] = _BatchBuffers()
    return per[dev]


def run_forward_chunks(model: TransformerModel, kv: KVCache, ids: list[int], base: int, low: bool,
                       slot: int = 0):
    """Enqueue qs_forward over ``ids`` at positions base.. (chunks of <= 64 tokens)."""
    import torch
    _bb = _batch_buffers()
    cfg = model.config
    hpk = cfg.n_heads // cfg.n_kv_heads
    tmax = min(64, max(1, 64 // hpk), 8192 // (hpk * cfg.head_dim) or 1)
    ws, _ = model.workspace(64)
    cm = model.c_model(kv)
    n = len(ids)
    logits = torch.empty((n, cfg.vocab_size), dtype=torch.float32, device="cuda")
    argmax = torch.empty(n, dtype=torch.int32, device="cuda")
    mode = _lib.QS_MODE_LOW if low else _lib.QS_MODE_HIGH
    dev_ids = ids if torch.is_tensor(ids) else torch.tensor(ids, dtype=torch.int32).cuda()
    dev_ids = dev_ids.to(device="cuda", dtype=torch.int32)
    for s in range(0, n, tmax):
        T = min(tmax, n - s)
        _bb.ids[:T].copy_(dev_ids[s:s + T])
        torch.arange(base + s, base + s + T, dtype=torch.int32, out=_bb.pos[:T])
        _bb.slot[:T].fill_(slot)
        _bb.blk[0], _bb.blk[1] = 0, T
        b = _lib.Batch(T=T, tokens=_bb.ids.data_ptr(), positions=_bb.pos.data_ptr(), slots=_bb.slot.data_ptr(),
                       n_blk=1, blk_tok0=_bb.blk.data_ptr(), blk_ntok=_bb.blk[1:].data_ptr(), blk_qmax=T,
                       ctx_cap=base + s + T)
        _lib.call("qs_forward", cm, b, mode, ws, logits[s:].data_ptr(), argmax[s:].data_ptr(),
                  _lib.stream_ptr())
    return logits, argmax


def forward(model: TransformerModel, tokens: list[int], kv: KVCache, mode: ExecutionMode,
            write_target: WriteTarget, counter: CostCounter | None = None) -> LogitsBlock:
    """model.py:255-348: causal pass over ``tokens`` appended at the target region."""
    cfg = model.config
    n = len(tokens)
    if n == 0:
        raise ShapeError("forward requires a non-empty token sequence")
    ids = [int(t) for t in tokens]
    if min(ids) < 0 or max(ids) >= cfg.vocab_size:
        raise TokenIdError(f"token id out of vocab range [0, {cfg.vocab_size})")
    c, r = kv.committed_len, kv.region_len(write_target)
    base = c + r
    if base + n > cfg.max_seq_len:
        raise SequenceOverflowError(f"sequence overflow: {base} committed/scratch + {n} new > {cfg.max_seq_len}")
    if r + n > kv.scratch_capacity:
        raise SequenceOverflowError(f"scratch overflow: {r} + {n} new > capacity {kv.scratch_capacity}")
    low = mode is ExecutionMode.LOW_PRECISION
    for _, q in model.quantized_tensors():
        _log_qlinear(q, mode)
    if low:
        _count_act_quant(7 * cfg.n_layers + 1)
    logits, argmax = run_forward_chunks(model, kv, ids, base, low)
    kv._set_region_len(write_target, r + n)
    if counter is not None:
        counter.add(_macs(cfg, n, base))
    return LogitsBlock(logits=logits, mode=mode, argmax=argmax)
