"""Seeded model construction on the device (drop-in for storage.py:135-182 random_init et al.).

The reference draws every 2-D tensor from one 64-bit LCG stream in file order
(storage.py:104-124) and quantises group-wise.  Here each tensor's first draw
index is computed on the host and the GPU jumps straight to it (qs_init_weight /
qs_lcg_fill), so a 7B-shape model is built in well under a second instead of
minutes, bit-identical to the reference (tests pin it against the oracle).
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .model import ModelConfig, TransformerModel, make_layer_stores
from .quant import DeviceStore, QuantizedTensor


def float_tensor_shapes(cfg: ModelConfig) -> list[tuple[str, tuple[int, ...]]]:
    """Names and shapes in draw order (storage.py:104-124)."""
    hd = cfg.head_dim
    out: list[tuple[str, tuple[int, ...]]] = [("token_embedding", (cfg.vocab_size, cfg.d_model))]
    for i in range(cfg.n_layers):
        p = f"layers.{i}."
        out += [(p + "attn_norm", (cfg.d_model,)), (p + "q_proj", (cfg.n_heads * hd, cfg.d_model)),
                (p + "k_proj", (cfg.n_kv_heads * hd, cfg.d_model)), (p + "v_proj", (cfg.n_kv_heads * hd, cfg.d_model)),
                (p + "o_proj", (cfg.d_model, cfg.d_model)), (p + "ffn_norm", (cfg.d_model,)),
                (p + "gate_proj", (cfg.d_ff, cfg.d_model)), (p + "up_proj", (cfg.d_ff, cfg.d_model)),
                (p + "down_proj", (cfg.d_model, cfg.d_ff))]
    out += [("final_norm", (cfg.d_model,)), ("lm_head", (cfg.vocab_size, cfg.d_model))]
    return out


def draw_offsets(cfg: ModelConfig) -> dict[str, int]:
    off, res = 0, {}
    for name, shape in float_tensor_shapes(cfg):
        if len(shape) == 2:
            res[name] = off
            off += shape[0] * shape[1]
    return res


def _placement(cfg: ModelConfig, lw, proj: str):
    """(store, row_off, row_stride) of a projection inside the fused layer stores."""
    H, KV, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    return {"q_proj": (lw.qkv, 0, 1), "k_proj": (lw.qkv, H * hd, 1), "v_proj": (lw.qkv, (H + KV) * hd, 1),
            "o_proj": (lw.o, 0, 1), "gate_proj": (lw.gate_up, 0, 2), "up_proj": (lw.gate_up, 1, 2),
            "down_proj": (lw.down, 0, 1)}[proj]


def _empty_model(cfg: ModelConfig):
    import torch
    layers = []
    for _ in range(cfg.n_layers):
        ones = torch.ones(cfg.d_model, dtype=torch.float32, device="cuda")
        layers.append(make_layer_stores(cfg, ones, ones.clone()))
    lm = DeviceStore.empty(cfg.vocab_size, cfg.d_model, cfg.group_size)
    emb = torch.empty((cfg.vocab_size, cfg.d_model), dtype=torch.float32, device="cuda")
    return layers, lm, emb


def random_init(cfg: ModelConfig, seed: int) -> TransformerModel:
    """storage.py:180-182 on the device: LCG draws * f32(1/sqrt(d)), quantised group-wise."""
    import torch
    _lib.require_cuda()
    scale = float(np.float32(1.0 / math.sqrt(cfg.d_model)))
    offs = draw_offsets(cfg)
    layers, lm, emb = _empty_model(cfg)
    st = _lib.stream_ptr()
    _lib.call("qs_lcg_fill", emb.data_ptr(), seed, offs["token_embedding"], emb.numel(), scale, st)
    g = cfg.group_size
    for i, lw in enumerate(layers):
        for proj in ("q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj"):
            q: QuantizedTensor = getattr(lw, proj)
            store, off, stride = _placement(cfg, lw, proj)
            _lib.call("qs_init_weight", seed, offs[f"layers.{i}.{proj}"], scale, q.out_features, q.in_features, g,
                      store.codes.data_ptr(), store.scales.data_ptr(), store.geo.n_pad, off, stride, None, None, st)
    _lib.call("qs_init_weight", seed, offs["lm_head"], scale, cfg.vocab_size, cfg.d_model, g,
              lm.codes.data_ptr(), lm.scales.data_ptr(), lm.geo.n_pad, 0, 1, None, None, st)
    torch.cuda.synchronize()
    final = torch.ones(cfg.d_model, dtype=torch.float32, device="cuda")
    return TransformerModel(cfg, emb, layers, final, QuantizedTensor(cfg.vocab_size, cfg.d_model, g, lm))


def model_from_float_tensors(cfg: ModelConfig, tensors: dict) -> TransformerModel:
    """storage.py:152-177: quantise float tensors (numpy or torch) into the device layout."""
    import torch
    _lib.require_cuda()

    def dev(a):
        return torch.as_tensor(np.asarray(a, dtype=np.float32) if not torch.is_tensor(a) else a,
                               dtype=torch.float32).cuda().contiguous()

    layers, lm, emb = _empty_model(cfg)
    emb.copy_(dev(tensors["token_embedding"]))
    g, st = cfg.group_size, _lib.stream_ptr()
    keep = []
    for i, lw in enumerate(layers):
        lw.attn_norm.copy_(dev(tensors[f"layers.{i}.attn_norm"]))
        lw.ffn_norm.copy_(dev(tensors[f"layers.{i}.ffn_norm"]))
        for proj in ("q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj"):
            q = getattr(lw, proj)
            store, off, stride = _placement(cfg, lw, proj)
            w = dev(tensors[f"layers.{i}.{proj}"])
            keep.append(w)
            _lib.call("qs_quantize_weight", w.data_ptr(), q.out_features, q.in_features, g, store.codes.data_ptr(),
                      store.scales.data_ptr(), store.geo.n_pad, off, stride, None, None, st)
    w = dev(tensors["lm_head"])
    keep.append(w)
    _lib.call("qs_quantize_weight", w.data_ptr(), cfg.vocab_size, cfg.d_model, g, lm.codes.data_ptr(),
              lm.scales.data_ptr(), lm.geo.n_pad, 0, 1, None, None, st)
    torch.cuda.synchronize()
    final = dev(tensors["final_norm"])
    return TransformerModel(cfg, emb, layers, final, QuantizedTensor(cfg.vocab_size, cfg.d_model, g, lm))
