"""ctypes binding of the C ABI in ``include/qspec_b200.h``.

The shared library is built in-tree by ``build.py``.  There is no fallback: if
the library is missing, or CUDA is unavailable when a device op is called, the
call raises -- the product path never routes through a CPU implementation.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, QSpecError, SequenceOverflowError, ShapeError, TokenIdError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QSPEC_LIB") or os.path.join(HERE, "libqspec_b200.so")

QS_OK, QS_ERR_SHAPE, QS_ERR_CONFIG, QS_ERR_OVERFLOW, QS_ERR_TOKEN, QS_ERR_CUDA = range(6)
QS_MODE_HIGH, QS_MODE_LOW = 0, 1

i32, u64, i64, f32 = C.c_int32, C.c_uint64, C.c_int64, C.c_float
vp = C.c_void_p


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


class TP(C.Structure):
    """qs_tp_t"""
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("vocab_off", C.c_int32), ("nccl_comm", C.c_void_p),
                ("allreduce", ALLREDUCE_FN), ("allgather", ALLGATHER_FN), ("user", C.c_void_p),
                ("scratch", C.c_void_p)]


class QWeight(C.Structure):
    _fields_ = [("codes", vp), ("scales", vp)] + [
        (n, i32) for n in ("n", "k", "g", "n_pad", "n_tiles", "G", "gp", "cpg", "n_chunks")]


class Layer(C.Structure):
    _fields_ = [("attn_norm", vp), ("ffn_norm", vp), ("qkv", QWeight), ("o", QWeight),
                ("gate_up", QWeight), ("down", QWeight), ("k_cache", vp), ("v_cache", vp)]


class Model(C.Structure):
    _fields_ = [(n, i32) for n in ("n_layers", "d_model", "n_heads", "n_kv_heads", "d_ff", "vocab",
                                   "group_size", "rope_len")] + [
        ("norm_eps", f32), ("tok_emb", vp), ("final_norm", vp), ("rope_cos", vp), ("rope_sin", vp),
        ("lm_head", QWeight), ("layers", C.POINTER(Layer)), ("block_table", vp), ("bt_ld", i32),
        ("page", i32), ("hadamard", i32)]


class Batch(C.Structure):
    _fields_ = [("T", i32), ("tokens", vp), ("positions", vp), ("slots", vp), ("n_blk", i32),
                ("blk_tok0", vp), ("blk_ntok", vp), ("blk_qmax", i32), ("ctx_cap", i32)]


WS_FIELDS = ("x", "h", "attn", "q", "img", "ascale", "part", "counters", "arg_val", "arg_idx", "att_o", "att_ml")


class Workspace(C.Structure):
    _fields_ = [(n, vp) for n in WS_FIELDS]


class WorkspaceSizes(C.Structure):
    _fields_ = [(n, C.c_size_t) for n in WS_FIELDS]


class Seq(C.Structure):
    _fields_ = [(n, vp) for n in ("pending", "committed", "n_out", "done", "finish", "max_new", "g_eff",
                                  "drafted", "out_tokens", "n_drafted", "n_accepted", "n_cycles",
                                  "dropped", "trace", "trace_tok")] + [
        (n, i32) for n in ("out_cap", "trace_cap", "B", "gamma", "eos", "max_seq")] + [
        ("tok", vp), ("pos", vp), ("slot", vp), ("argmax", vp)]


_SIGS = {
    "qs_version": ([], C.c_char_p),
    "qs_num_sms": ([C.POINTER(i32)], C.c_int),
    "qs_linear_max_tokens": ([], C.c_int),
    "qs_attention_chunk_len": ([], C.c_int),
    "qs_workspace_size": ([C.POINTER(Model), i32, C.POINTER(WorkspaceSizes)], C.c_int),
    "qs_qweight_geometry": ([i32, i32, i32, C.POINTER(QWeight)], C.c_int),
    "qs_init_weight": ([u64, u64, f32, i32, i32, i32, vp, vp, i32, i32, i32, vp, vp, vp], C.c_int),
    "qs_quantize_weight": ([vp, i32, i32, i32, vp, vp, i32, i32, i32, vp, vp, vp], C.c_int),
    "qs_lcg_fill": ([vp, u64, u64, i64, f32, vp], C.c_int),
    "qs_repack_ref": ([vp, vp, i32, i32, i32, vp, vp, i32, i32, i32, vp], C.c_int),
    "qs_ktrace_enable": ([vp, i32], C.c_int),
    "qs_ktrace_read": ([vp, i32, C.POINTER(i32)], C.c_int),
    "qs_rmsnorm": ([vp, vp, i32, i32, f32, vp, vp], C.c_int),
    "qs_act_quant": ([vp, i32, i32, i32, vp, vp, vp, vp], C.c_int),
    "qs_w4a4_linear": ([C.POINTER(QWeight), vp, i32, vp, C.POINTER(Workspace), vp], C.c_int),
    "qs_w4a16_linear": ([C.POINTER(QWeight), vp, i32, vp, C.POINTER(Workspace), vp], C.c_int),
    "qs_linear_prepacked": ([C.POINTER(QWeight), i32, i32, vp, C.POINTER(Workspace), vp], C.c_int),
    "qs_debug_timeline": ([vp], C.c_int),
    "qs_debug_select": ([i32], C.c_int),
    "qs_forward_launches": ([], C.c_int),
    "qs_hadamard_rows": ([vp, i64, i32, vp], C.c_int),
    "qs_tp_scratch_bytes": ([i32], C.c_size_t),
    "qs_tp_nccl_unique_id": ([C.POINTER(C.c_uint8)], C.c_int),
    "qs_tp_nccl_init": ([i32, i32, C.POINTER(C.c_uint8), C.POINTER(C.c_void_p)], C.c_int),
    "qs_tp_nccl_destroy": ([vp], C.c_int),
    "qs_forward_tp2": ([C.POINTER(Model), C.POINTER(Batch), i32, C.POINTER(Workspace), vp, vp, C.POINTER(TP), vp],
                       C.c_int),
    "qs_set_emit": ([i32], C.c_int),
    "qs_linear_group_dots": ([C.POINTER(QWeight), vp, i32, i32, vp, C.POINTER(Workspace), vp], C.c_int),
    "qs_profile_enable": ([i32], C.c_int),
    "qs_profile_reset": ([], C.c_int),
    "qs_profile_read": ([vp, vp, i32, C.POINTER(i32)], C.c_int),
    "qs_forward": ([C.POINTER(Model), C.POINTER(Batch), i32, C.POINTER(Workspace), vp, vp, vp], C.c_int),
    "qs_forward_tp": ([C.POINTER(Model), C.POINTER(Batch), i32, C.POINTER(Workspace), vp, vp, i32, vp, vp, vp],
                      C.c_int),
    "qs_draft_prep": ([C.POINTER(Seq), i32, vp], C.c_int),
    "qs_verify_prep": ([C.POINTER(Seq), vp], C.c_int),
    "qs_accept": ([C.POINTER(Seq), vp], C.c_int),
    "qs_ar_prep": ([C.POINTER(Seq), vp], C.c_int),
    "qs_ar_commit": ([C.POINTER(Seq), vp], C.c_int),
}

EXPORTED = tuple(_SIGS)

_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load the extension (no build, no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2410_11305_b200.build` "
                "(the QSpec hot path has no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


_ERRS = {QS_ERR_SHAPE: ShapeError, QS_ERR_CONFIG: ConfigError, QS_ERR_OVERFLOW: SequenceOverflowError,
         QS_ERR_TOKEN: TokenIdError}


def check(rc: int, what: str) -> None:
    if rc != QS_OK:
        raise _ERRS.get(rc, QSpecError)(f"{what} failed with status {rc}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


def require_cuda() -> None:
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("qspec_b200 device ops need a CUDA (sm_100a) device; there is no CPU fallback")
    load()
