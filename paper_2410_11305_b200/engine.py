"""Batched, device-resident QSpec / autoregressive decode engine (the hot path).

B sequence slots share one immutable model and one paged KV pool.  A QSpec
cycle for the whole batch is

    gamma x [draft_prep(j) -> qs_forward(LOW, T=B)]          (W4A4 drafts, in-place KV)
    verify_prep -> qs_forward(HIGH, T=B*(gamma+1))            (W4A16 verify, overwrites draft KV)
    accept                                                    (greedy accept + commit + bookkeeping)

entirely on the device, captured once into a CUDA graph and replayed; the host
only polls the ``done`` flags.  The same engine runs plain W4A16 greedy decoding
(``ar_prep -> qs_forward(HIGH, T=B) -> ar_commit``) on the same kernels -- the
baseline QSpec is compared against.  Per-request outputs are independent of the
batch composition (every kernel is batch-invariant), which is the contract of
the reference's serving loop (serving.py:1-9).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, SequenceOverflowError, ShapeError, TokenIdError
from .model import KVCache, TransformerModel, run_forward_chunks


@dataclass
class SlotResult:
    new_tokens: list[int]
    finish_reason: str
    n_drafted: int
    n_accepted: int
    n_cycles: int
    dropped_after_eos: int
    trace: np.ndarray        # [cycles, 4]: drafted_len, accept_len, kept_len, is_bonus
    trace_tok: np.ndarray    # [cycles, gamma]


class DecodeEngine:
    def __init__(self, model: TransformerModel, batch: int, *, gamma: int = 3, max_new_cap: int = 256,
                 eos_token: int | None = None, draft_low: bool = True, algorithm: str = "qspec",
                 greedy_low: bool = False, use_graphs: bool = True) -> None:
        import torch
        _lib.require_cuda()
        if gamma < 1:
            raise ConfigError("gamma must be >= 1")
        cfg = model.config
        self.model, self.cfg, self.B, self.gamma = model, cfg, batch, gamma
        self.algorithm, self.draft_low, self.greedy_low = algorithm, draft_low, greedy_low
        self.eos = -1 if eos_token is None else int(eos_token)
        self._setup_storage(model, batch, gamma)
        self.cap = max_new_cap
        i32 = dict(dtype=torch.int32, device="cuda")
        B, G1 = batch, gamma + 1
        z = lambda n: torch.zeros(n, **i32)  # noqa: E731
        self.t = {n: z(B) for n in ("pending", "committed", "n_out", "done", "finish", "max_new", "g_eff",
                                    "n_drafted", "n_accepted", "n_cycles", "dropped")}
        self.t["drafted"] = z(B * gamma)
        self.t["out_tokens"] = z(B * self.cap)
        self.t["trace"] = z(B * self.cap * 4)
        self.t["trace_tok"] = z(B * self.cap * gamma)
        for n in ("tok", "pos", "slot", "argmax"):
            self.t[n] = z(B * G1)
        self.t["done"].fill_(1)
        self.seq = _lib.Seq(**{n: self.t[n].data_ptr() for n in (
            "pending", "committed", "n_out", "done", "finish", "max_new", "g_eff", "drafted", "out_tokens",
            "n_drafted", "n_accepted", "n_cycles", "dropped", "trace", "trace_tok", "tok", "pos", "slot",
            "argmax")}, out_cap=self.cap, trace_cap=self.cap, B=B, gamma=gamma, eos=self.eos,
            max_seq=cfg.max_seq_len)
        hpk = cfg.n_heads // cfg.n_kv_heads
        if G1 * hpk > 64:
            raise ConfigError("gamma+1 query rows per kv head exceed the attention block limit (64)")
        self.draft_batches = self._batches(1)
        self.verify_batches = self._batches(G1)
        self.use_graphs = use_graphs
        self.graphs: dict[int, object] = {}   # attention grid bound (ctx_cap) -> captured step
        self.graph = None
        self.n_launch_cycle = 0
        # Host upper bound on max(committed) over the slots, kept without device reads:
        # prefill sets it from the prompt length, a step adds at most gamma + 1 (qspec) or
        # 1 (greedy) committed positions per slot, poll() tightens it to the exact value.
        # The attention grid covers ceil(ctx_cap / chunk) key chunks; sizing ctx_cap from
        # this bound instead of the KV capacity drops the CTAs past every sequence's context
        # (at prompt 128, capacity 520: 9 chunk slots per (block, kv head), 3 in use).
        self._ctx_hi = 0
        self._chunk = _lib.load().qs_attention_chunk_len()   # keys per split-KV chunk

    def _setup_storage(self, model: TransformerModel, batch: int, gamma: int) -> None:
        """KV pool, workspace and the C model view the forwards run on (TP overrides)."""
        self.kv = KVCache(model.config, gamma_max=gamma, slots=batch)
        self.ws, self._ws_bufs = model.workspace(64)
        self.cm = model.c_model(self.kv)

    def _call_forward(self, b, mode: int, argmax_ptr: int, st: int) -> None:
        _lib.call("qs_forward", self.cm, b, mode, self.ws, None, argmax_ptr, st)

    def _prefill_argmax(self, prompt, slot: int, low: bool):
        """argmax of every prompt position (device int32 [n]) after the HIGH prefill."""
        _, argmax = run_forward_chunks(self.model, self.kv, prompt, 0, low, slot=slot)
        return argmax

    # ------------------------------------------------------------------ batches
    def _batches(self, per_seq: int, ctx_cap: int | None = None) -> list[tuple[_lib.Batch, int]]:
        """qs_batch_t descriptors: sequences grouped so each forward has <= 64 tokens.
        ``ctx_cap`` bounds every query's context (pos + 1) in the batch (default: the KV capacity)."""
        seqs_per = max(1, 64 // per_seq)
        out = []
        for s0 in range(0, self.B, seqs_per):
            ns = min(seqs_per, self.B - s0)
            off = s0 * per_seq * 4
            # uniform blocks (blk_tok0 = NULL): sequence i of the forward = tokens
            # [i * per_seq, (i + 1) * per_seq) -- the attention skips a block-table load
            b = _lib.Batch(T=ns * per_seq, tokens=self.t["tok"].data_ptr() + off,
                           positions=self.t["pos"].data_ptr() + off, slots=self.t["slot"].data_ptr() + off,
                           n_blk=ns, blk_tok0=None, blk_ntok=None, blk_qmax=per_seq,
                           ctx_cap=self.kv.capacity if ctx_cap is None else ctx_cap)
            out.append((b, off))
        return out

    def _forward(self, batches, low: bool) -> None:
        mode = _lib.QS_MODE_LOW if low else _lib.QS_MODE_HIGH
        st = _lib.stream_ptr()
        for b, off in batches:
            self._call_forward(b, mode, self.t["argmax"].data_ptr() + off, st)
            self._enq += _lib.load().qs_forward_launches()

    # ------------------------------------------------------------------ step bodies
    def _cycle_body(self) -> None:
        self._enq = 1 + self.gamma   # verify_prep + accept + gamma draft_preps, then forwards
        st = _lib.stream_ptr()
        for j in range(self.gamma):
            _lib.call("qs_draft_prep", self.seq, j, st)
            self._forward(self.draft_batches, self.draft_low)
        _lib.call("qs_verify_prep", self.seq, st)
        self._forward(self.verify_batches, False)
        _lib.call("qs_accept", self.seq, st)

    def _ar_body(self) -> None:
        self._enq = 2                # ar_prep + ar_commit, then the forward
        st = _lib.stream_ptr()
        _lib.call("qs_ar_prep", self.seq, st)
        self._forward(self.draft_batches, self.greedy_low)
        _lib.call("qs_ar_commit", self.seq, st)

    def launches_per_step(self) -> int:
        """Kernels one step launches (for the bench's gpu_launches claim), counted by the
        runtime while the step body was enqueued (qs_forward_launches)."""
        if getattr(self, "_enq", None) is None:
            self.step()
        return int(self._enq)

    def _advance(self) -> int:
        """Committed positions one step can add per slot (accept commits <= g_eff + 1)."""
        return self.gamma + 1 if self.algorithm == "qspec" else 1

    def _ctx_cap(self, ctx_hi: int) -> int:
        """Attention context bound of a step starting at max(committed) <= ctx_hi, rounded
        up to whole key chunks (one captured graph per chunk count)."""
        need = ctx_hi + self._advance()   # positions committed .. committed + gamma
        c = self._chunk
        return min(self.kv.capacity, -(-need // c) * c)

    def _set_ctx_cap(self, cap: int) -> None:
        for b, _ in self.draft_batches + self.verify_batches:
            b.ctx_cap = cap

    def _capture(self, cap: int, warm: bool) -> None:
        """Capture the step body for attention bound ``cap``.  Warm-up (sets kernel
        attributes outside capture) and capture run with every slot marked done: the
        accept/commit kernels skip done slots, so the only side effects are scratch
        buffers and KV rows past committed_len, which the next real cycle rewrites
        before reading."""
        import torch
        body = self._cycle_body if self.algorithm == "qspec" else self._ar_body
        self._set_ctx_cap(cap)
        done = self.t["done"].clone()
        self.t["done"].fill_(1)
        if warm:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                body()
            torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        torch.cuda.synchronize()
        self.t["done"].copy_(done)
        self.graphs[cap] = g

    def step(self) -> None:
        """One cycle (qspec) or one token (greedy) for every slot, replayed from a CUDA graph
        (one graph per attention context bound; the next few bounds are captured ahead so a
        run of steps does not stop to capture)."""
        body = self._cycle_body if self.algorithm == "qspec" else self._ar_body
        cap = self._ctx_cap(self._ctx_hi)
        self._ctx_hi += self._advance()
        if not self.use_graphs:
            self._set_ctx_cap(cap)
            body()
            return
        if cap not in self.graphs:
            self._capture(cap, warm=not self.graphs)
            nxt = cap
            for _ in range(3):
                nxt = self._ctx_cap(nxt)
                if nxt not in self.graphs:
                    self._capture(nxt, warm=False)
            self._set_ctx_cap(cap)
        self.graph = self.graphs[cap]
        self.graph.replay()

    def profile_step(self) -> list[tuple[float, int]]:
        """Replay one real step from a graph whose linear launches are bracketed by events.

        Returns [(ms, tag)] per linear launch (tag = mode*16 + kind, see qspec_b200.h).
        """
        import torch
        import ctypes as C
        body = self._cycle_body if self.algorithm == "qspec" else self._ar_body
        if self.graph is None:
            self.step()           # ensures warm-up happened (attributes set)
        self._set_ctx_cap(self._ctx_cap(self._ctx_hi))
        self._ctx_hi += self._advance()
        n_max = 8192
        _lib.call("qs_profile_enable", n_max)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        _lib.call("qs_profile_enable", 0)
        g.replay()
        torch.cuda.synchronize()
        ms = (C.c_float * n_max)()
        tags = (C.c_int32 * n_max)()
        n = _lib.i32()
        _lib.call("qs_profile_read", C.addressof(ms), C.addressof(tags), n_max, C.byref(n))
        self._prof_graph = g  # keep alive with its events
        return [(float(ms[i]), int(tags[i])) for i in range(n.value)]

    def ktrace_step(self):
        """Device timeline of one replayed step with PDL intact (qs_ktrace_*): per traced
        launch (linears, operand packs, attention) its tag and [first CTA entry, last CTA
        exit] in microseconds from the step's first entry."""
        import torch
        import ctypes as C
        body = self._cycle_body if self.algorithm == "qspec" else self._ar_body
        if self.graph is None:
            self.step()
        self._set_ctx_cap(self._ctx_cap(self._ctx_hi))
        self._ctx_hi += self._advance()
        cap = 16384
        buf = torch.zeros((cap, 2), dtype=torch.int64, device="cuda")
        _lib.call("qs_ktrace_enable", buf.data_ptr(), cap)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        tags = (C.c_int32 * cap)()
        n = _lib.i32()
        _lib.call("qs_ktrace_read", C.addressof(tags), cap, C.byref(n))
        _lib.call("qs_ktrace_enable", None, 0)
        n = n.value
        buf[:n, 0] = torch.iinfo(torch.int64).max
        buf[:n, 1] = 0
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        t = buf[:n].cpu().numpy().astype(np.float64)
        t0 = t[:, 0].min()
        self._kt_graph = g
        return [int(tags[i]) for i in range(n)], (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3

    # ------------------------------------------------------------------ admission
    def prefill(self, slot: int, prompt: list[int], max_new_tokens: int) -> None:
        """specdec.py:234-254: prompt through the HIGH path (greedy_mode for greedy), emit token 1."""
        import torch
        cfg = self.cfg
        if len(prompt) == 0:
            raise ShapeError("prompt must be non-empty")
        if len(prompt) + max_new_tokens > cfg.max_seq_len:
            raise SequenceOverflowError("prompt + max_new_tokens exceeds max_seq_len")
        if max_new_tokens > self.cap:
            raise ConfigError(f"max_new_tokens {max_new_tokens} exceeds engine capacity {self.cap}")
        if not torch.is_tensor(prompt):
            if min(prompt) < 0 or max(prompt) >= cfg.vocab_size:
                raise TokenIdError("prompt token out of vocab range")
            prompt = [int(t) for t in prompt]
        low = self.algorithm == "greedy" and self.greedy_low
        self._ctx_hi = max(self._ctx_hi, len(prompt))
        argmax = self._prefill_argmax(prompt, slot, low)
        first = argmax[len(prompt) - 1:len(prompt)]
        b = slot
        self.t["pending"][b:b + 1].copy_(first)
        self.t["out_tokens"][b * self.cap:b * self.cap + 1].copy_(first)
        vals = torch.tensor([len(prompt), 1, max_new_tokens], dtype=torch.int32)
        self.t["committed"][b] = int(vals[0])
        self.t["n_out"][b] = 1
        self.t["max_new"][b] = max_new_tokens
        for n in ("n_drafted", "n_accepted", "n_cycles", "dropped", "finish", "g_eff"):
            self.t[n][b] = 0
        f = int(first.item())
        if self.eos >= 0 and f == self.eos:
            self.t["done"][b], self.t["finish"][b] = 1, 1
        elif max_new_tokens <= 1:
            self.t["done"][b], self.t["finish"][b] = 1, 2
        else:
            self.t["done"][b] = 0

    def poll(self) -> bool:
        """Host read of the done flags (and committed lengths, which tighten the attention
        context bound): True when every slot is done."""
        import torch
        if getattr(self, "_poll_buf", None) is None:
            self._poll_buf = torch.empty(2 * self.B, dtype=torch.int32).pin_memory()
        h = self._poll_buf
        h[:self.B].copy_(self.t["done"], non_blocking=True)
        h[self.B:].copy_(self.t["committed"], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        self._ctx_hi = int(h[self.B:].max())
        return bool(h[:self.B].all())

    def all_done(self) -> bool:
        return self.poll()

    def run(self, max_steps: int = 1 << 30, poll: int = 1) -> int:
        steps = 0
        while steps < max_steps and not self.all_done():
            for _ in range(poll):
                self.step()
                steps += 1
        return steps

    def result(self, slot: int) -> SlotResult:
        t = {n: v.cpu().numpy() for n, v in self.t.items()}
        b = slot
        n = int(t["n_out"][b])
        cyc = int(t["n_cycles"][b])
        fin = {1: "eos", 2: "max_new_tokens"}.get(int(t["finish"][b]), "")
        return SlotResult(
            new_tokens=[int(x) for x in t["out_tokens"][b * self.cap: b * self.cap + n]],
            finish_reason=fin, n_drafted=int(t["n_drafted"][b]), n_accepted=int(t["n_accepted"][b]),
            n_cycles=cyc, dropped_after_eos=int(t["dropped"][b]),
            trace=t["trace"].reshape(self.B, self.cap, 4)[b, :cyc].copy(),
            trace_tok=t["trace_tok"].reshape(self.B, self.cap, self.gamma)[b, :cyc].copy())
