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
    if cfg.hadamard:  # opt-in rotation: float draws -> rotated rows -> quantise (not in the reference)
        def init(q_rows, q_cols, off, store, row_off, stride):
            w = torch.empty(q_rows * q_cols, dtype=torch.float32, device="cuda")
            _lib.call("qs_lcg_fill", w.data_ptr(), seed, off, w.numel(), scale, st)
            _lib.call("qs_hadamard_rows", w.data_ptr(), q_rows, q_cols, st)
            _lib.call("qs_quantize_weight", w.data_ptr(), q_rows, q_cols, g, store.codes.data_ptr(),
                      store.scales.data_ptr(), store.geo.n_pad, row_off, stride, None, None, st)
            torch.cuda.current_stream().synchronize()
        for i, lw in enumerate(layers):
            for proj in ("q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj"):
                q = getattr(lw, proj)
                store, off, stride = _placement(cfg, lw, proj)
                init(q.out_features, q.in_features, offs[f"layers.{i}.{proj}"], store, off, stride)
        init(cfg.vocab_size, cfg.d_model, offs["lm_head"], lm, 0, 1)
        final = torch.ones(cfg.d_model, dtype=torch.float32, device="cuda")
        return TransformerModel(cfg, emb, layers, final,
                                QuantizedTensor(cfg.vocab_size, cfg.d_model, g, lm, rotated=True))
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
    rot = (lambda w: _rotate(w)) if cfg.hadamard else (lambda w: w)
    for i, lw in enumerate(layers):
        lw.attn_norm.copy_(dev(tensors[f"layers.{i}.attn_norm"]))
        lw.ffn_norm.copy_(dev(tensors[f"layers.{i}.ffn_norm"]))
        for proj in ("q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj"):
            q = getattr(lw, proj)
            store, off, stride = _placement(cfg, lw, proj)
            w = rot(dev(tensors[f"layers.{i}.{proj}"]))
            keep.append(w)
            _lib.call("qs_quantize_weight", w.data_ptr(), q.out_features, q.in_features, g, store.codes.data_ptr(),
                      store.scales.data_ptr(), store.geo.n_pad, off, stride, None, None, st)
    w = rot(dev(tensors["lm_head"]))
    keep.append(w)
    _lib.call("qs_quantize_weight", w.data_ptr(), cfg.vocab_size, cfg.d_model, g, lm.codes.data_ptr(),
              lm.scales.data_ptr(), lm.geo.n_pad, 0, 1, None, None, st)
    torch.cuda.synchronize()
    final = dev(tensors["final_norm"])
    return TransformerModel(cfg, emb, layers, final,
                            QuantizedTensor(cfg.vocab_size, cfg.d_model, g, lm, rotated=cfg.hadamard))


def _rotate(w):
    from .quant import hadamard_rows
    return hadamard_rows(w)


# ---------------------------------------------------------------------------
# QSPC checkpoints (storage.py:1-28 format, 300-422 save / load)
# ---------------------------------------------------------------------------

MAGIC = b"QSPC"
FORMAT_VERSION = 1
_F32, _I4 = 0, 1
HEADER_FIELDS = ("n_layers", "d_model", "n_heads", "n_kv_heads", "d_ff", "vocab_size", "max_seq_len", "rope_theta",
                 "norm_eps", "group_size")
_FLOATS = {"rope_theta", "norm_eps"}
_PROJS = ("q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj")


def config_to_text(cfg: ModelConfig) -> str:
    """storage.py:189-194: key=value lines, fixed order, floats by repr."""
    txt = "".join(f"{f}={getattr(cfg, f)!r}\n" if f in _FLOATS else f"{f}={getattr(cfg, f)}\n"
                  for f in HEADER_FIELDS)
    # the opt-in rotation (not a reference field) is written only when on, so default
    # checkpoints stay byte-identical with the reference's
    return txt + ("hadamard=1\n" if getattr(cfg, "hadamard", False) else "")


def config_from_text(text: str) -> ModelConfig:
    """storage.py:197-222 (same errors)."""
    from .errors import CheckpointError, ConfigError
    vals: dict[str, str] = {}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        if "=" not in line:
            raise CheckpointError(f"header line {lineno}: expected key=value, got {line!r}")
        k, v = line.split("=", 1)
        vals[k.strip()] = v.strip()
    missing = [f for f in HEADER_FIELDS if f not in vals]
    if missing:
        raise CheckpointError(f"header missing fields: {', '.join(missing)}")
    hadamard = vals.pop("hadamard", "0") not in ("0", "False", "false")
    extra = [k for k in vals if k not in HEADER_FIELDS]
    if extra:
        raise CheckpointError(f"header has unknown fields: {', '.join(extra)}")
    try:
        kw = {f: (float(vals[f]) if f in _FLOATS else int(vals[f])) for f in HEADER_FIELDS}
    except ValueError as exc:
        raise CheckpointError(f"header value: {exc}") from exc
    try:
        return ModelConfig(**kw, hadamard=hadamard)
    except ConfigError as exc:
        raise CheckpointError(f"header config invalid: {exc}") from exc


def _records(model: TransformerModel):
    """(name, dtype, shape, payload) in the reference's record order (storage.py:317-336)."""
    def f32(name, t):
        a = t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)
        return (name, _F32, tuple(a.shape), a.astype("<f4").tobytes())

    def quant(name, q):
        return [(f"{name}.codes", _I4, (q.out_features, q.in_features), q.codes.tobytes()),
                (f"{name}.scales", _F32, tuple(q.scales.shape), q.scales.astype("<f4").tobytes())]

    out = [f32("token_embedding", model.token_embedding)]
    for i, lw in enumerate(model.layers):
        p = f"layers.{i}"
        out.append(f32(f"{p}.attn_norm", lw.attn_norm))
        for proj in _PROJS[:4]:
            out += quant(f"{p}.{proj}", getattr(lw, proj))
        out.append(f32(f"{p}.ffn_norm", lw.ffn_norm))
        for proj in _PROJS[4:]:
            out += quant(f"{p}.{proj}", getattr(lw, proj))
    out.append(f32("final_norm", model.final_norm))
    out += quant("lm_head", model.lm_head)
    return out


def save_checkpoint(model: TransformerModel, path: str) -> None:
    """storage.py:315-349: byte-deterministic QSPC file of a quantized model (device -> reference layout)."""
    import io
    import struct
    recs = _records(model)
    header = config_to_text(model.config).encode("utf-8")
    buf = io.BytesIO()
    buf.write(MAGIC + struct.pack("<II", FORMAT_VERSION, len(header)) + header + struct.pack("<I", len(recs)))
    for name, dtype, shape, payload in recs:
        nb = name.encode("utf-8")
        buf.write(struct.pack("<H", len(nb)) + nb + struct.pack("<BB", dtype, len(shape)))
        buf.write(b"".join(struct.pack("<I", d) for d in shape) + struct.pack("<Q", len(payload)) + payload)
    with open(path, "wb") as f:
        f.write(buf.getvalue())


def read_checkpoint(path: str):
    """Parse a QSPC file: (config, {name: (dtype, shape, payload)}), with the reference's checks."""
    import struct
    from .errors import CheckpointError

    with open(path, "rb") as f:
        data = f.read()
    pos = 0

    def take(n, what):
        nonlocal pos
        if pos + n > len(data):
            raise CheckpointError(f"truncated checkpoint while reading {what}")
        b = data[pos:pos + n]
        pos += n
        return b

    magic = take(4, "magic")
    if magic != MAGIC:
        raise CheckpointError(f"bad magic {magic!r}, expected {MAGIC!r}")
    (version,) = struct.unpack("<I", take(4, "version"))
    if version != FORMAT_VERSION:
        raise CheckpointError(f"unsupported format version {version}")
    (hlen,) = struct.unpack("<I", take(4, "header length"))
    cfg = config_from_text(take(hlen, "header").decode("utf-8"))
    (count,) = struct.unpack("<I", take(4, "record count"))
    recs: dict = {}
    for _ in range(count):
        (nl,) = struct.unpack("<H", take(2, "record name length"))
        name = take(nl, "record name").decode("utf-8")
        dtype, ndim = struct.unpack("<BB", take(2, f"record '{name}' dtype"))
        shape = tuple(struct.unpack("<I", take(4, f"record '{name}' dims"))[0] for _ in range(ndim))
        (plen,) = struct.unpack("<Q", take(8, f"record '{name}' payload length"))
        payload = take(plen, f"record '{name}' payload")
        n_el = int(np.prod(shape)) if shape else 1
        if dtype == _F32:
            want = 4 * n_el
        elif dtype == _I4:
            want = (n_el + 1) // 2
        else:
            raise CheckpointError(f"record '{name}': unknown dtype code {dtype}")
        if len(payload) != want:
            raise CheckpointError(f"record '{name}': payload is {len(payload)} bytes, expected {want} "
                                  f"for shape {shape}")
        if name in recs:
            raise CheckpointError(f"record '{name}': duplicated")
        recs[name] = (dtype, shape, payload)
    return cfg, recs


def load_checkpoint(path: str) -> TransformerModel:
    """storage.py:352-422: a reference QSPC checkpoint into the device layout (qs_repack_ref), bit-exact."""
    import torch
    from .errors import CheckpointError
    cfg, recs = read_checkpoint(path)
    # quant.py:138-139, reported by storage.py:390-397 as a CheckpointError naming the
    # codes record: every quantized store's scales must be finite and non-negative
    for name, (dtype, _, payload) in recs.items():
        if name.endswith(".scales") and name[:-7] + ".codes" in recs and dtype == _F32:
            sc = np.frombuffer(payload, dtype="<f4")
            if np.any(sc < 0) or not np.all(np.isfinite(sc)):
                raise CheckpointError(f"record '{name[:-7]}.codes': scales must be finite and non-negative")
    _lib.require_cuda()
    hd, g = cfg.head_dim, cfg.group_size

    def take_f32(name, shape):
        if name not in recs:
            raise CheckpointError(f"record '{name}': missing")
        dtype, rshape, payload = recs.pop(name)
        if dtype != _F32 or rshape != shape:
            raise CheckpointError(f"record '{name}': expected f32 {shape}, found dtype={dtype} shape={rshape}")
        return torch.from_numpy(np.frombuffer(payload, dtype="<f4").astype(np.float32).reshape(shape).copy())

    def take_quant(name, n, k):
        cname = f"{name}.codes"
        if cname not in recs:
            if name in recs:
                raise CheckpointError(f"record '{name}': stored as f32 (unquantized checkpoint); "
                                      f"run the quantize step first")
            raise CheckpointError(f"record '{cname}': missing")
        dtype, shape, payload = recs.pop(cname)
        if dtype != _I4 or shape != (n, k):
            raise CheckpointError(f"record '{cname}': expected i4-packed ({n}, {k}), found dtype={dtype} "
                                  f"shape={shape}")
        scales = take_f32(f"{name}.scales", (n, k // g))
        codes = torch.from_numpy(np.frombuffer(payload, dtype=np.uint8).copy()).cuda()
        return codes, scales.cuda()

    layers, lm, emb = _empty_model(cfg)
    emb.copy_(take_f32("token_embedding", (cfg.vocab_size, cfg.d_model)))
    st = _lib.stream_ptr()
    keep = []
    dims = {"q_proj": (cfg.n_heads * hd, cfg.d_model), "k_proj": (cfg.n_kv_heads * hd, cfg.d_model),
            "v_proj": (cfg.n_kv_heads * hd, cfg.d_model), "o_proj": (cfg.d_model, cfg.d_model),
            "gate_proj": (cfg.d_ff, cfg.d_model), "up_proj": (cfg.d_ff, cfg.d_model),
            "down_proj": (cfg.d_model, cfg.d_ff)}
    for i, lw in enumerate(layers):
        p = f"layers.{i}"
        lw.attn_norm.copy_(take_f32(f"{p}.attn_norm", (cfg.d_model,)))
        lw.ffn_norm.copy_(take_f32(f"{p}.ffn_norm", (cfg.d_model,)))
        for proj in _PROJS:
            n, k = dims[proj]
            codes, scales = take_quant(f"{p}.{proj}", n, k)
            keep += [codes, scales]
            store, off, stride = _placement(cfg, lw, proj)
            _lib.call("qs_repack_ref", codes.data_ptr(), scales.data_ptr(), n, k, g, store.codes.data_ptr(),
                      store.scales.data_ptr(), store.geo.n_pad, off, stride, st)
    final = take_f32("final_norm", (cfg.d_model,)).cuda()
    codes, scales = take_quant("lm_head", cfg.vocab_size, cfg.d_model)
    keep += [codes, scales]
    _lib.call("qs_repack_ref", codes.data_ptr(), scales.data_ptr(), cfg.vocab_size, cfg.d_model, g,
              lm.codes.data_ptr(), lm.scales.data_ptr(), lm.geo.n_pad, 0, 1, st)
    if recs:
        raise CheckpointError(f"unexpected records: {', '.join(sorted(recs))}")
    torch.cuda.synchronize()
    return TransformerModel(cfg, emb, layers, final, QuantizedTensor(cfg.vocab_size, cfg.d_model, g, lm))
