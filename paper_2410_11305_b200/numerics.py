"""Dense float32 helpers on the device (drop-in for pkg/src/qspec/numerics.py where the
decode path needs them).

``rmsnorm`` runs the same kernel code the forward's operand producer uses
(``csrc/pack_dev.cuh`` token_inv_rms), so its bit-exactness test covers the
normalisation every RMSNorm'd linear operand goes through.
"""

from __future__ import annotations

from . import _lib
from .errors import ShapeError


def rmsnorm(x, weight, eps: float):
    """numerics.py:46-62: ``x * (1/sqrt(mean(x^2) + eps)) * weight`` per row, float32.

    The mean uses numpy's pairwise summation order, so the result is bit-identical to
    the reference for the same input.  ``x``: [n] or [rows, n]; returns a new device tensor.
    """
    import torch
    _lib.require_cuda()
    t = torch.as_tensor(x)
    w = torch.as_tensor(weight)
    if t.dtype != torch.float32 or w.dtype != torch.float32:
        raise ShapeError("rmsnorm expects float32 inputs")
    if t.dim() not in (1, 2) or w.dim() != 1:
        raise ShapeError(f"rmsnorm expects a vector or matrix, got ndim={t.dim()}")
    if t.shape[-1] != w.shape[0]:
        raise ShapeError(f"rmsnorm length mismatch: x {tuple(t.shape)} vs weight {tuple(w.shape)}")
    if eps <= 0:
        raise ShapeError("rmsnorm eps must be positive")
    rows = t.reshape(-1, t.shape[-1]).to("cuda").contiguous()
    wd = w.to("cuda").contiguous()
    y = torch.empty_like(rows)
    _lib.call("qs_rmsnorm", rows.data_ptr(), wd.data_ptr(), rows.shape[0], rows.shape[1], float(eps), y.data_ptr(),
              _lib.stream_ptr())
    return y.reshape(t.shape)
