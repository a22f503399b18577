"""Group-wise int4 weight stores and the mode-routed linear (drop-in for pkg/src/qspec/quant.py).

One ``DeviceStore`` per fused projection holds packed int4 codes in the device
chunk layout plus fp32 per-(row, group) scales; both execution modes stream
the SAME bytes (QSpec's weight sharing):

  * ``ExecutionMode.LOW_PRECISION``  -> W4A4 draft linear (``qs_w4a4_linear``):
    activations quantised per (token, group) exactly as quant.py:179-194, then
    an int4 x int4 integer core on tcgen05 ``kind::i8``.
  * ``ExecutionMode.HIGH_PRECISION`` -> W4A16 verify linear (``qs_w4a16_linear``):
    fp32 activations as 24-bit fixed point per (token, group), three int8 limbs,
    same kernel and instruction.

``QuantizedTensor`` is the reference's per-projection handle; inside a model it
is a row-view (``row_off``, ``row_stride``) of a fused store, so the audit
surface (one instance per linear, shared by both modes) is preserved.
"""

from __future__ import annotations

import threading

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .errors import ConfigError, ShapeError

DEFAULT_GROUP_SIZE = 128
CODE_MIN, CODE_MAX = -8, 7


class ExecutionMode(Enum):
    """quant.py:37-41."""

    HIGH_PRECISION = "high"
    LOW_PRECISION = "low"


# ---------------------------------------------------------------- audit hooks (quant.py:48-73)
_act_quant_calls = 0
_qlinear_log: list | None = None


def activation_quant_calls() -> int:
    return _act_quant_calls


def reset_activation_quant_calls() -> None:
    global _act_quant_calls
    _act_quant_calls = 0


def _count_act_quant(n: int = 1) -> None:
    global _act_quant_calls
    _act_quant_calls += n


def start_qlinear_log() -> None:
    global _qlinear_log
    _qlinear_log = []


def stop_qlinear_log() -> list:
    global _qlinear_log
    log, _qlinear_log = (_qlinear_log or []), None
    return log


def _log_qlinear(q: "QuantizedTensor", mode: ExecutionMode) -> None:
    if _qlinear_log is not None:
        _qlinear_log.append((id(q), mode))


# ---------------------------------------------------------------- host byte helpers (quant.py:81-103)
def pack_int4(codes: np.ndarray) -> np.ndarray:
    """Reference packing: flat row-major, even index in the low nibble."""
    flat = np.asarray(codes, dtype=np.int8).reshape(-1)
    if flat.size % 2:
        flat = np.concatenate([flat, np.zeros(1, np.int8)])
    nib = flat.view(np.uint8) & 0x0F
    return (nib[0::2] | (nib[1::2] << 4)).astype(np.uint8)


def unpack_int4(packed: np.ndarray, count: int) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty(p.size * 2, dtype=np.int8)
    out[0::2] = ((p & 0x0F).astype(np.int8) ^ 8) - 8
    out[1::2] = ((p >> 4).astype(np.int8) ^ 8) - 8
    return out[:count]


# ---------------------------------------------------------------- device store
@dataclass
class DeviceStore:
    """Packed codes [n_tiles][n_chunks][4][128][16] + scales [n_tiles][n_chunks][128] on the device."""

    n: int
    k: int
    g: int
    codes: "object"   # torch.uint8 tensor
    scales: "object"  # torch.float32 tensor [n_tiles, n_chunks, 128] (per 128-wide chunk, tile-major)
    geo: _lib.QWeight = field(repr=False)

    @classmethod
    def empty(cls, n: int, k: int, g: int) -> "DeviceStore":
        import torch
        _lib.require_cuda()
        if g < 1 or k % g:
            raise ConfigError(f"in_features {k} not divisible by group_size {g}")
        geo = _lib.QWeight()
        _lib.call("qs_qweight_geometry", n, k, g, geo)
        codes = torch.zeros(geo.n_tiles * geo.n_chunks * 8192, dtype=torch.uint8, device="cuda")
        scales = torch.zeros((geo.n_tiles, geo.n_chunks, 128), dtype=torch.float32, device="cuda")
        geo.codes, geo.scales = codes.data_ptr(), scales.data_ptr()
        return cls(n, k, g, codes, scales, geo)

    @property
    def weight_bytes(self) -> int:
        """Algorithmic bytes one linear streams: n*k/2 packed codes + n*k/g fp32 scales."""
        return self.n * self.k // 2 + 4 * self.n * (self.k // self.g)

    def unpacked(self) -> np.ndarray:
        """int8 codes [n, k] in logical order (host copy; test/export path)."""
        geo = self.geo
        raw = self.codes.cpu().numpy().reshape(geo.n_tiles, geo.n_chunks, 4, 128, 16)
        rows = raw.transpose(0, 3, 1, 2, 4).reshape(geo.n_pad, geo.n_chunks, 64)
        # device nibbles are offset binary (code + 8; qs_common.cuh)
        lo = (rows & 0x0F).astype(np.int8) - 8
        hi = (rows >> 4).astype(np.int8) - 8
        full = np.concatenate([lo, hi], axis=2).reshape(geo.n_pad, geo.G, geo.gp)[:, :, :self.g]
        return full.reshape(geo.n_pad, self.k)[:self.n]


@dataclass(eq=False)
class QuantizedTensor:
    """Per-projection handle (quant.py:111-160): a row view of a DeviceStore."""

    out_features: int
    in_features: int
    group_size: int
    store: DeviceStore = field(repr=False)
    row_off: int = 0
    row_stride: int = 1
    rotated: bool = False   # weights Hadamard-rotated (ModelConfig.hadamard): inputs are rotated too

    def __post_init__(self) -> None:
        if self.in_features % self.group_size:
            raise ConfigError(f"in_features {self.in_features} not divisible by group_size {self.group_size}")

    @property
    def packed_bytes(self) -> int:
        return (self.out_features * self.in_features + 1) // 2

    def _rows(self) -> np.ndarray:
        return self.row_off + self.row_stride * np.arange(self.out_features)

    def unpacked_codes(self) -> np.ndarray:
        return self.store.unpacked()[self._rows()]

    @property
    def codes(self) -> np.ndarray:
        """Reference-layout packed bytes (host copy)."""
        return pack_int4(self.unpacked_codes())

    @property
    def scales(self) -> np.ndarray:
        geo = self.store.geo
        per_chunk = self.store.scales.cpu().numpy()[:, ::geo.cpg, :]          # [n_tiles, G, 128]
        per_row = per_chunk.transpose(0, 2, 1).reshape(geo.n_pad, geo.G)
        return per_row[self._rows()].copy()

    @property
    def is_view(self) -> bool:
        return not (self.row_off == 0 and self.row_stride == 1 and self.out_features == self.store.n)


# ---------------------------------------------------------------- construction
def hadamard_rows(x):
    """Orthonormal 128-point Walsh-Hadamard transform of every 128-block of every row (a new
    device float32 tensor): the opt-in rotation (ModelConfig.hadamard)."""
    import torch
    t = torch.as_tensor(x, dtype=torch.float32).to("cuda").clone().contiguous()
    if t.dim() != 2 or t.shape[1] % 128:
        raise ShapeError("hadamard_rows needs a [rows, 128*k] matrix")
    _lib.call("qs_hadamard_rows", t.data_ptr(), t.shape[0], t.shape[1], _lib.stream_ptr())
    return t


def quantize_groupwise(w, group_size: int = DEFAULT_GROUP_SIZE, *, hadamard: bool = False) -> QuantizedTensor:
    """quant.py:197-218 on the device: float32 [out, in] -> one standalone store.
    hadamard=True (opt-in, not in the reference): rotate the rows' 128-blocks first; the
    store then rotates its inputs in qlinear_forward."""
    import torch
    _lib.require_cuda()
    t = torch.as_tensor(w)
    if t.dtype != torch.float32 or t.dim() != 2:
        raise ShapeError("w must be a float32 matrix")
    if group_size < 1 or t.shape[1] % group_size:
        raise ConfigError(f"cols {t.shape[1]} not divisible by group_size {group_size}")
    t = t.to("cuda").contiguous()
    if hadamard:
        if group_size != 128:
            raise ConfigError("the Hadamard rotation works on 128-wide groups")
        t = hadamard_rows(t)
    n, k = t.shape
    st = DeviceStore.empty(n, k, group_size)
    _lib.call("qs_quantize_weight", t.data_ptr(), n, k, group_size, st.codes.data_ptr(),
              st.scales.data_ptr(), st.geo.n_pad, 0, 1, None, None, _lib.stream_ptr())
    return QuantizedTensor(n, k, group_size, st, rotated=hadamard)


def dequantize(q: QuantizedTensor) -> np.ndarray:
    """quant.py:221-226: f32 code*scale, [out, in] (host; audit/test helper)."""
    c = q.unpacked_codes().astype(np.float32)
    g = q.group_size
    return (c.reshape(q.out_features, -1, g) * q.scales[:, :, None]).reshape(q.out_features, q.in_features)


# ---------------------------------------------------------------- operators
def _as_rows(x):
    import torch
    t = torch.as_tensor(x)
    if t.dtype != torch.float32 or t.dim() != 2:
        raise ShapeError(f"x must be a float32 matrix, got {t.dtype} ndim={t.dim()}")
    return t.to("cuda").contiguous()


def fake_quantize_activations(x, group_size: int = DEFAULT_GROUP_SIZE, *, return_codes: bool = False):
    """quant.py:229-245 (bit-exact integer codes and scales on the device)."""
    import torch
    _lib.require_cuda()
    t = _as_rows(x)
    T, K = t.shape
    if group_size < 1 or K % group_size:
        raise ConfigError(f"cols {K} not divisible by group_size {group_size}")
    _count_act_quant()
    codes = torch.empty((T, K), dtype=torch.int8, device="cuda")
    scales = torch.empty((T, K // group_size), dtype=torch.float32, device="cuda")
    fq = torch.empty((T, K), dtype=torch.float32, device="cuda")
    _lib.call("qs_act_quant", t.data_ptr(), T, K, group_size, codes.data_ptr(), scales.data_ptr(),
              fq.data_ptr(), _lib.stream_ptr())
    return (fq, codes, scales) if return_codes else fq


class _LinearWorkspace:
    """Scratch for standalone qlinear_forward calls (one per process, grown on demand)."""

    def __init__(self) -> None:
        self.key = None
        self.ws = None
        self.bufs = []

    def get(self, n: int, k: int, g: int):
        import torch
        key = (n, k, g)
        if self.key != key:
            n_pad = -(-n // 128) * 128
            gp = -(-g // 128) * 128
            chunks = (k // g) * gp // 128
            sms = _lib.i32()
            _lib.call("qs_num_sms", C_byref(sms))
            sizes = dict(x=4, h=4, attn=4, q=4, img=chunks * 192 * 128, ascale=chunks * 64 * 4 * 5,  # ascale + acorr
                         part=(sms.value + n_pad // 128) * 64 * 128 * 4, counters=(4096 + 2) * 4,
                         arg_val=(n_pad // 128) * 64 * 4, arg_idx=(n_pad // 128) * 64 * 4, att_o=4, att_ml=4)
            self.bufs = {kk: torch.zeros(v, dtype=torch.uint8, device="cuda") for kk, v in sizes.items()}
            self.ws = _lib.Workspace(**{kk: b.data_ptr() for kk, b in self.bufs.items()})
            self.key = key
        return self.ws


def C_byref(x):
    import ctypes
    return ctypes.byref(x)


class _ThreadWorkspaces(threading.local):
    """One _LinearWorkspace per (thread, device): standalone qlinear_forward calls from
    several threads never share staging buffers."""

    def get(self, n: int, k: int, g: int):
        import torch
        per = self.__dict__.setdefault("per", {})
        dev = torch.cuda.current_device()
        if dev not in per:
            per[dev] = _LinearWorkspace()
        return per[dev].get(n, k, g)


_ws = _ThreadWorkspaces()


def qlinear_forward(q: QuantizedTensor, x, mode: ExecutionMode):
    """quant.py:248-261: x [m, in] -> [m, out] through the shared store, routed by mode."""
    import torch
    _lib.require_cuda()
    t = _as_rows(x)
    if t.shape[1] != q.in_features:
        raise ShapeError(f"qlinear input width {t.shape[1]} != in_features {q.in_features}")
    _log_qlinear(q, mode)
    if q.rotated:
        t = hadamard_rows(t)
    st = q.store
    low = mode is ExecutionMode.LOW_PRECISION
    if low:
        _count_act_quant()
    ws = _ws.get(st.n, st.k, st.g)
    tmax = _lib.load().qs_linear_max_tokens()
    y = torch.empty((t.shape[0], st.n), dtype=torch.float32, device="cuda")
    fn = "qs_w4a4_linear" if low else "qs_w4a16_linear"
    for s in range(0, t.shape[0], tmax):
        xs = t[s:s + tmax].contiguous()
        ys = y[s:s + tmax]
        _lib.call(fn, st.geo, xs.data_ptr(), xs.shape[0], ys.data_ptr(), ws, _lib.stream_ptr())
    if q.is_view:
        y = y[:, q.row_off: q.row_off + q.row_stride * q.out_features: q.row_stride].contiguous()
    return y


def linear_group_dots(q: QuantizedTensor, x, mode: ExecutionMode):
    """Raw int32 dots of the tensor-core integer core: [n_pad, G, r_pad] (parity tests)."""
    import torch
    t = _as_rows(x)
    st = q.store
    T = t.shape[0]
    L = 1 if mode is ExecutionMode.LOW_PRECISION else 3
    # linear_tmax_bucket(T, L) in linear_tc.cu
    tm = (2 if T <= 2 else 4) if (L == 3 and T <= 4) else 8 if T <= 8 else 16 if T <= 16 else 32 if T <= 32 else 64
    r = tm * L
    r_pad = 8 if r <= 8 else -(-r // 16) * 16
    dots = torch.zeros((st.geo.n_pad, st.geo.n_chunks, r_pad), dtype=torch.int32, device="cuda")
    ws = _ws.get(st.n, st.k, st.g)
    _lib.call("qs_linear_group_dots", st.geo, t.data_ptr(), T,
              _lib.QS_MODE_LOW if L == 1 else _lib.QS_MODE_HIGH, dots.data_ptr(), ws, _lib.stream_ptr())
    return dots
