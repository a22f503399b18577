"""CPU oracle for the QSpec decode hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's arithmetic
(``/root/reference/pkg/src/qspec``), written to reproduce its float32 results
bit-for-bit.  It exists so that ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` have a checker that
travels to the GPU box (``/root/reference`` does not).  Nothing in the product
path (``paper_2410_11305_b200``) may import it.

Parity status: PINNED.  ``tests/golden/make_golden.py`` imports the unmodified
reference in the build container and freezes its outputs (LCG draws, packed
codes, scales, activation codes, qlinear outputs, forward logits, greedy and
QSpec token streams); ``tests/test_oracle_golden.py`` checks this module
against every fixture bit-exactly, plus the reference's own frozen vectors
(``pkg/tests/test_storage_cli.py:31-57``).

Every function cites the reference ``file:line`` it restates.  The numpy call
shapes (einsum subscripts with optimize=False, float32 dtypes, operation order)
are kept identical because float32 bits depend on them.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32
SEVEN = np.float32(7.0)

# ---------------------------------------------------------------------------
# Configuration  (model.py:32-69, specdec.py:40-59)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class OracleConfig:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    d_ff: int
    vocab_size: int
    max_seq_len: int
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    group_size: int = 128
    hadamard: bool = False   # opt-in rotation of the B200 build (not in the reference; wht128)

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads


# ---------------------------------------------------------------------------
# 64-bit LCG weight stream  (storage.py:56-101, 104-149)
# ---------------------------------------------------------------------------

LCG_MUL = 6364136223846793005
LCG_INC = 1442695040888963407
MASK64 = (1 << 64) - 1


def lcg_jump(state: int, n: int) -> int:
    """State after ``n`` steps of s <- MUL*s + INC (mod 2^64), by affine squaring."""
    mul, inc = LCG_MUL, LCG_INC
    acc_mul, acc_inc = 1, 0
    while n:
        if n & 1:
            acc_mul, acc_inc = (acc_mul * mul) & MASK64, (acc_inc * mul + inc) & MASK64
        mul, inc = (mul * mul) & MASK64, (inc * mul + inc) & MASK64
        n >>= 1
    return (acc_mul * state + acc_inc) & MASK64


class LcgStream:
    """Block-vectorised draw of the documented generator (storage.py:62-98)."""

    BLOCK = 4096

    def __init__(self, seed: int) -> None:
        self.state = seed & MASK64
        m, c = 1, 0
        muls = np.empty(self.BLOCK, dtype=np.uint64)
        incs = np.empty(self.BLOCK, dtype=np.uint64)
        for j in range(self.BLOCK):
            m = (m * LCG_MUL) & MASK64
            c = (c * LCG_MUL + LCG_INC) & MASK64
            muls[j], incs[j] = m, c
        self._muls, self._incs = muls, incs

    def floats(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float32)
        pos = 0
        while pos < count:
            n = min(self.BLOCK, count - pos)
            st = self._muls[:n] * np.uint64(self.state) + self._incs[:n]
            self.state = int(st[-1])
            out[pos:pos + n] = (st >> np.uint64(40)).astype(np.float32) / np.float32(1 << 23) - np.float32(1.0)
            pos += n
        return out


def weight_file_order(cfg: OracleConfig) -> list[tuple[str, tuple[int, ...]]]:
    """Float tensors in draw order (storage.py:104-124)."""
    hd = cfg.head_dim
    order: list[tuple[str, tuple[int, ...]]] = [("token_embedding", (cfg.vocab_size, cfg.d_model))]
    for i in range(cfg.n_layers):
        p = f"layers.{i}."
        order += [
            (p + "attn_norm", (cfg.d_model,)),
            (p + "q_proj", (cfg.n_heads * hd, cfg.d_model)),
            (p + "k_proj", (cfg.n_kv_heads * hd, cfg.d_model)),
            (p + "v_proj", (cfg.n_kv_heads * hd, cfg.d_model)),
            (p + "o_proj", (cfg.d_model, cfg.d_model)),
            (p + "ffn_norm", (cfg.d_model,)),
            (p + "gate_proj", (cfg.d_ff, cfg.d_model)),
            (p + "up_proj", (cfg.d_ff, cfg.d_model)),
            (p + "down_proj", (cfg.d_model, cfg.d_ff)),
        ]
    order += [("final_norm", (cfg.d_model,)), ("lm_head", (cfg.vocab_size, cfg.d_model))]
    return order


def lcg_offsets(cfg: OracleConfig) -> dict[str, int]:
    """Draw index of the first element of every 2-D tensor (1-D norms draw nothing)."""
    off, out = 0, {}
    for name, shape in weight_file_order(cfg):
        if len(shape) == 2:
            out[name] = off
            off += shape[0] * shape[1]
    return out


def float_weights(cfg: OracleConfig, seed: int) -> dict[str, np.ndarray]:
    """storage.py:135-149: LCG draws * f32(1/sqrt(d_model)); norms are ones."""
    rng = LcgStream(seed)
    scale = np.float32(1.0 / math.sqrt(cfg.d_model))
    out: dict[str, np.ndarray] = {}
    for name, shape in weight_file_order(cfg):
        if len(shape) == 1:
            out[name] = np.ones(shape, dtype=np.float32)
        else:
            out[name] = (rng.floats(shape[0] * shape[1]) * scale).reshape(shape)
    return out


# ---------------------------------------------------------------------------
# Group-wise 4-bit quantization  (quant.py:81-103, 163-245)
# ---------------------------------------------------------------------------


def snap_max(m: np.ndarray) -> np.ndarray:
    """Fixed point of m -> f32(7*f32(m/7)) (quant.py:163-176)."""
    m = m.astype(np.float32, copy=True)
    for _ in range(8):
        nxt = SEVEN * (m / SEVEN)
        if np.array_equal(nxt, m):
            return m
        m = nxt
    raise AssertionError("snap did not converge")


def quantize_rows(x: np.ndarray, g: int) -> tuple[np.ndarray, np.ndarray]:
    """Symmetric int4 codes + f32 scales per (row, group) (quant.py:179-194)."""
    rows, cols = x.shape
    grp = x.reshape(rows, cols // g, g)
    m = snap_max(np.max(np.abs(grp), axis=-1))
    s = m / SEVEN
    with np.errstate(divide="ignore", invalid="ignore"):
        q = np.rint(grp / s[:, :, None])
    q = np.where(s[:, :, None] == 0, 0.0, q)
    return np.clip(q, -8, 7).astype(np.int8).reshape(rows, cols), s


def pack_nibbles(codes: np.ndarray) -> np.ndarray:
    """Two codes per byte, even flat index in the low nibble (quant.py:81-92)."""
    flat = codes.reshape(-1).astype(np.int8)
    if flat.size % 2:
        flat = np.concatenate([flat, np.zeros(1, np.int8)])
    u = flat.astype(np.uint8) & 0x0F
    return (u[0::2] | (u[1::2] << 4)).astype(np.uint8)


def unpack_nibbles(packed: np.ndarray, count: int) -> np.ndarray:
    """Inverse of pack_nibbles with 4-bit sign extension (quant.py:95-103)."""
    both = np.empty(packed.size * 2, dtype=np.int16)
    both[0::2] = packed & 0x0F
    both[1::2] = (packed >> 4) & 0x0F
    return ((both ^ 8) - 8).astype(np.int8)[:count]


def dequant(codes: np.ndarray, scales: np.ndarray, g: int) -> np.ndarray:
    """w = code*scale in f32, [out, in] (quant.py:221-226)."""
    n, k = codes.shape
    return (codes.astype(np.float32).reshape(n, k // g, g) * scales[:, :, None]).reshape(n, k)


def fake_quant(x: np.ndarray, g: int) -> np.ndarray:
    """Per-(token, group) quantize-dequantize (quant.py:229-245)."""
    codes, s = quantize_rows(x, g)
    rows, cols = x.shape
    return (codes.astype(np.float32).reshape(rows, cols // g, g) * s[:, :, None]).reshape(rows, cols)


@dataclass
class OracleLinear:
    """One shared 4-bit store (quant.py:111-160), with the transposed f32 cache."""

    codes: np.ndarray          # int8 [out, in]
    scales: np.ndarray         # f32 [out, in/g]
    g: int
    _wt: np.ndarray | None = field(default=None, repr=False)
    rotated: bool = False      # opt-in Hadamard rotation (inputs rotated by wht128 in qlinear)

    @property
    def wt(self) -> np.ndarray:
        if self._wt is None:
            self._wt = np.ascontiguousarray(dequant(self.codes, self.scales, self.g).T)
        return self._wt

    def packed(self) -> np.ndarray:
        return pack_nibbles(self.codes)


def wht128(x: np.ndarray) -> np.ndarray:
    """The opt-in rotation (ModelConfig.hadamard; NOT part of the reference, which has no
    rotation -- SPEC.md:17): orthonormal 128-point Walsh-Hadamard transform of every
    128-block along the last axis, float32 butterflies over index bits 0..6 in order
    (pair (i, i | 2^b) -> a + c, a - c), then * f32(1/sqrt(128)) -- csrc/pack_dev.cuh
    wht128_warp's order, so rotated codes compare bit for bit."""
    x = np.asarray(x, dtype=np.float32)
    shp = x.shape
    y = x.reshape(-1, 128).copy()
    h = 1
    while h < 128:
        y = y.reshape(-1, 128 // (2 * h), 2, h)
        a, c = y[:, :, 0, :], y[:, :, 1, :]
        y = np.stack([a + c, a - c], axis=2).reshape(-1, 128)
        h *= 2
    return (y * np.float32(1.0 / np.sqrt(128.0))).reshape(shp)


def qlinear(lin: OracleLinear, x: np.ndarray, low: bool) -> np.ndarray:
    """quant.py:248-261 with numerics.py:31-43 (einsum, optimize=False)."""
    if lin.rotated:
        x = wht128(x)
    if low:
        x = fake_quant(x, lin.g)
    return np.einsum("ik,kj->ij", x, lin.wt, optimize=False)


# ---------------------------------------------------------------------------
# Dense f32 helpers  (numerics.py:46-133)
# ---------------------------------------------------------------------------


def rmsnorm(x: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    ms = np.mean(x * x, axis=-1, keepdims=True, dtype=np.float32)
    return x * (F32(1.0) / np.sqrt(ms + F32(eps))) * w


def pairwise_sum_f32(v: np.ndarray) -> np.float32:
    """numpy's float32 add-reduce order along a contiguous row (the ``pairwise_sum`` of
    numpy/_core/src/umath/loops_utils.h.src), which ``np.mean(x * x, dtype=float32)`` in
    numerics.py:60 runs: n < 8 sequential from 0; n <= 128 eight strided accumulators in
    order, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8 tail; else split at
    n/2 - (n/2) % 8.  Explicit restatement of the order the device RMSNorm implements
    (``csrc/pack_dev.cuh`` token_inv_rms); ``rmsnorm`` above uses numpy itself."""
    v = np.asarray(v, dtype=np.float32)
    n = v.shape[0]
    if n < 8:
        r = F32(0.0)
        for x in v:
            r = F32(r + x)
        return r
    if n <= 128:
        r = [v[j] for j in range(8)]
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] = F32(r[j] + v[i + j])
            i += 8
        res = F32(F32(F32(r[0] + r[1]) + F32(r[2] + r[3])) + F32(F32(r[4] + r[5]) + F32(r[6] + r[7])))
        for k in range(i, n):
            res = F32(res + v[k])
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return F32(pairwise_sum_f32(v[:n2]) + pairwise_sum_f32(v[n2:]))


def softmax(s: np.ndarray) -> np.ndarray:
    e = np.exp(s - np.max(s, axis=-1, keepdims=True))
    return e / np.sum(e, axis=-1, keepdims=True, dtype=np.float32)


def silu(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return x / (F32(1.0) + np.exp(-x))


def rope_tables(n_pos: int, hd: int, theta: float) -> tuple[np.ndarray, np.ndarray]:
    """numerics.py:97-116: f64 angles, cast to f32 after cos/sin."""
    inv = 1.0 / (theta ** (np.arange(0, hd, 2, dtype=np.float64) / hd))
    ang = np.arange(n_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def rope_rows(x: np.ndarray, c: np.ndarray, s: np.ndarray) -> np.ndarray:
    """model.py:243-252: rotate interleaved pairs (2i, 2i+1)."""
    ev, od = x[..., 0::2], x[..., 1::2]
    c, s = c[:, None, :], s[:, None, :]
    out = np.empty_like(x)
    out[..., 0::2] = ev * c - od * s
    out[..., 1::2] = ev * s + od * c
    return out


# ---------------------------------------------------------------------------
# Model, KV cache and the forward step  (model.py:87-348, storage.py:152-182)
# ---------------------------------------------------------------------------

PROJ = ("q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj")


@dataclass
class OracleModel:
    cfg: OracleConfig
    emb: np.ndarray
    layers: list[dict]
    final_norm: np.ndarray
    lm_head: OracleLinear
    rope: tuple[np.ndarray, np.ndarray]


def build_model(cfg: OracleConfig, tensors: dict[str, np.ndarray]) -> OracleModel:
    def q(name: str) -> OracleLinear:
        w = wht128(tensors[name]) if cfg.hadamard else tensors[name]
        codes, s = quantize_rows(w, cfg.group_size)
        return OracleLinear(codes, s, cfg.group_size, rotated=cfg.hadamard)

    layers = []
    for i in range(cfg.n_layers):
        p = f"layers.{i}."
        d = {k: q(p + k) for k in PROJ}
        d["attn_norm"] = tensors[p + "attn_norm"]
        d["ffn_norm"] = tensors[p + "ffn_norm"]
        layers.append(d)
    return OracleModel(cfg, tensors["token_embedding"], layers, tensors["final_norm"],
                       q("lm_head"), rope_tables(cfg.max_seq_len, cfg.head_dim, cfg.rope_theta))


def random_model(cfg: OracleConfig, seed: int) -> OracleModel:
    return build_model(cfg, float_weights(cfg, seed))


class OracleKV:
    """Committed buffers + DRAFT/VERIFY scratch regions (model.py:152-229)."""

    def __init__(self, cfg: OracleConfig, gamma_max: int = 8) -> None:
        self.cfg, self.cap = cfg, gamma_max + 1
        shp_c = (cfg.max_seq_len, cfg.n_kv_heads, cfg.head_dim)
        shp_s = (self.cap, cfg.n_kv_heads, cfg.head_dim)
        L = cfg.n_layers
        self.ck = [np.zeros(shp_c, F32) for _ in range(L)]
        self.cv = [np.zeros(shp_c, F32) for _ in range(L)]
        self.reg = {t: ([np.zeros(shp_s, F32) for _ in range(L)], [np.zeros(shp_s, F32) for _ in range(L)])
                    for t in ("draft", "verify")}
        self.rlen = {"draft": 0, "verify": 0}
        self.clen = 0
        self.pending: int | None = None

    def commit(self, accept_len: int) -> None:
        need = accept_len + 1
        if accept_len < 0 or need > self.rlen["verify"] or self.clen + need > self.cfg.max_seq_len:
            raise ValueError("bad commit")
        vk, vv = self.reg["verify"]
        for li in range(self.cfg.n_layers):
            self.ck[li][self.clen:self.clen + need] = vk[li][:need]
            self.cv[li][self.clen:self.clen + need] = vv[li][:need]
        self.clen += need
        self.rlen = {"draft": 0, "verify": 0}


def forward(model: OracleModel, tokens: list[int], kv: OracleKV, low: bool, target: str) -> np.ndarray:
    """One causal step; returns f32 logits [n, V] (model.py:255-348)."""
    cfg = model.cfg
    n = len(tokens)
    c, r = kv.clen, kv.rlen[target]
    base = c + r
    if n == 0 or base + n > cfg.max_seq_len or r + n > kv.cap:
        raise ValueError("forward out of range")
    H, KV, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    inv_sqrt = F32(1.0) / np.sqrt(F32(hd))
    cos, sin = model.rope[0][base:base + n], model.rope[1][base:base + n]
    rk, rv = kv.reg[target]
    x = model.emb[np.asarray(tokens, dtype=np.int64)]
    for li, lw in enumerate(model.layers):
        h = rmsnorm(x, lw["attn_norm"], cfg.norm_eps)
        q = rope_rows(qlinear(lw["q_proj"], h, low).reshape(n, H, hd), cos, sin)
        k = rope_rows(qlinear(lw["k_proj"], h, low).reshape(n, KV, hd), cos, sin)
        v = qlinear(lw["v_proj"], h, low).reshape(n, KV, hd)
        ctx_k = np.concatenate([kv.ck[li][:c], rk[li][:r], k], axis=0)
        ctx_v = np.concatenate([kv.cv[li][:c], rv[li][:r], v], axis=0)
        qg = q.reshape(n, KV, H // KV, hd)
        att = np.empty((n, cfg.d_model), dtype=F32)
        for j in range(n):
            t = base + j + 1
            sc = np.einsum("ghd,tgd->ght", qg[j], ctx_k[:t], optimize=False) * inv_sqrt
            att[j] = np.einsum("ght,tgd->ghd", softmax(sc), ctx_v[:t], optimize=False).reshape(cfg.d_model)
        x = x + qlinear(lw["o_proj"], att, low)
        h2 = rmsnorm(x, lw["ffn_norm"], cfg.norm_eps)
        gate = silu(qlinear(lw["gate_proj"], h2, low))
        x = x + qlinear(lw["down_proj"], gate * qlinear(lw["up_proj"], h2, low), low)
        rk[li][r:r + n] = k
        rv[li][r:r + n] = v
    logits = qlinear(model.lm_head, rmsnorm(x, model.final_norm, cfg.norm_eps), low)
    kv.rlen[target] = r + n
    return logits


# ---------------------------------------------------------------------------
# Draft / verify / accept and the generation drivers  (specdec.py:103-427)
# ---------------------------------------------------------------------------


def argmax(row: np.ndarray) -> int:
    return int(np.argmax(row))   # first index of the maximum (numerics.py:81-86)


def accept(drafted: list[int], logits: np.ndarray) -> tuple[int, int, bool]:
    """Longest matching prefix + correction/bonus (specdec.py:159-176)."""
    a = 0
    while a < len(drafted) and drafted[a] == argmax(logits[a]):
        a += 1
    return a, argmax(logits[a]), a == len(drafted)


@dataclass
class OracleResult:
    tokens: list[int]
    new_tokens: list[int]
    cycles: list[tuple[list[int], int, list[int]]]   # (drafted, accept_len, kept)
    acceptance_rate: float
    tokens_per_cycle: float
    finish_reason: str


def _prefill(model: OracleModel, kv: OracleKV, prompt: list[int], low: bool) -> int:
    """specdec.py:234-254: chunks of scratch capacity through VERIFY, commit each."""
    last = None
    for s in range(0, len(prompt), kv.cap):
        chunk = prompt[s:s + kv.cap]
        last = forward(model, chunk, kv, low, "verify")
        kv.commit(len(chunk) - 1)
    return argmax(last[-1])


def generate(model: OracleModel, prompt: list[int], *, gamma: int = 3, max_new: int = 32,
             eos: int | None = None, qspec: bool = True, low_greedy: bool = False,
             draft_low: bool = True) -> OracleResult:
    """generate_qspec (specdec.py:395-408) when qspec else generate_greedy (411-427)."""
    cfg = model.cfg
    if not prompt or len(prompt) + max_new > cfg.max_seq_len:
        raise ValueError("bad request")
    kv = OracleKV(cfg, gamma_max=gamma)
    out: list[int] = []
    cycles = []
    n_draft = n_acc = n_kept = 0
    done, reason = False, ""

    def append(kept: list[int]) -> None:
        nonlocal done, reason
        out.extend(kept)
        kv.pending = kept[-1]
        if eos is not None and kept[-1] == eos:
            done, reason = True, "eos"
        elif len(out) >= max_new:
            done, reason = True, "max_new_tokens"

    append([_prefill(model, kv, prompt, False if qspec else low_greedy)])
    while not done:
        if not qspec:   # specdec.py:325-335
            logits = forward(model, [kv.pending], kv, low_greedy, "verify")
            kv.commit(0)
            append([argmax(logits[0])])
            continue
        remaining = max_new - len(out)                       # specdec.py:263-265
        g_eff = min(gamma, max(1, remaining - 1), cfg.max_seq_len - kv.clen - 1)
        drafted, tok = [], kv.pending                        # specdec.py:103-133
        for _ in range(g_eff):
            tok = argmax(forward(model, [tok], kv, draft_low, "draft")[0])
            drafted.append(tok)
            if eos is not None and tok == eos:
                break
        logits = forward(model, [kv.pending, *drafted], kv, False, "verify")
        a, nxt, _ = accept(drafted, logits)
        kept = (drafted[:a] + [nxt])[:remaining]             # specdec.py:294-300
        if eos is not None and eos in kept:
            kept = kept[:kept.index(eos) + 1]
        kv.commit(len(kept) - 1)
        n_draft += len(drafted)
        n_acc += a
        n_kept += len(kept)
        cycles.append((drafted, a, kept))
        append(kept)
    return OracleResult(
        tokens=list(prompt) + out, new_tokens=out, cycles=cycles,
        acceptance_rate=n_acc / n_draft if n_draft else 1.0,
        tokens_per_cycle=n_kept / len(cycles) if cycles else 0.0,
        finish_reason=reason)
