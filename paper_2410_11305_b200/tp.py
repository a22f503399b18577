"""Tensor parallelism for the 13B-shape config (BASELINE config 4).

One process per GPU; rank r holds a SHARD of every layer, cut out of the
device-layout stores (no re-quantisation, so the integer cores are unchanged):

* q/k/v: column split by heads (H/P query heads, KV/P kv heads per rank) -- whole
  128-row tiles of the fused q|k|v store;
* gate/up: column split of d_ff in whole quantisation groups (an uneven
  13/14-group split at TP8 for d_ff = 13824 = 108 groups); tiles of the
  interleaved gate/up store;
* o_proj, down_proj: row split along K = the rank's heads / d_ff groups -- whole
  128-wide chunks, so activation groups never straddle ranks and the per-group
  activation quantisation stays local;
* embedding, norms: replicated; lm_head replicated (``qs_forward_tp``) or VOCAB-SPLIT
  in whole 128-row tiles (``qs_forward_tp2``: each rank's (max, index) per token is
  all-gathered and reduced in rank order, lowest index winning ties -- numerics.py:81-86).

``qs_forward_tp`` runs the rank's forward and calls the all-reduce hook after
each row-split linear (2 per layer, [T, d_model] fp32 partial sums), then adds
the reduced sum into the residual stream.  ``qs_forward_tp2`` (the QSpec engine's
path, ``TPDecodeEngine``) runs the same collectives as ncclAllReduce / ncclAllGather
on the forward's stream from the C runtime -- no host callback, no sync -- so whole
draft/verify/accept cycles replay from one CUDA graph; with host hooks instead of a
communicator (gloo, the tests) it runs eagerly.  Results equal the single-GPU forward
up to fp32 summation order of the partials.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from types import SimpleNamespace

from . import _lib
from .engine import DecodeEngine
from .errors import ConfigError
from .model import ModelConfig, TransformerModel
from .quant import DeviceStore


@dataclass
class TPSplit:
    rank: int
    world: int
    heads: tuple[int, int]      # query heads [h0, h1)
    kv_heads: tuple[int, int]   # kv heads [k0, k1)
    ff: tuple[int, int]         # d_ff columns [f0, f1), group-aligned


def tp_split(cfg: ModelConfig, rank: int, world: int) -> TPSplit:
    """The rank's slice of heads / kv heads / d_ff (whole groups; remainder groups spread)."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} / world {world}")
    if cfg.n_heads % world or cfg.n_kv_heads % world:
        raise ConfigError(f"n_heads {cfg.n_heads} / n_kv_heads {cfg.n_kv_heads} not divisible by TP {world}")
    hd, g = cfg.head_dim, cfg.group_size
    if (hd * cfg.n_heads // world) % 128 or (hd * cfg.n_kv_heads // world) % 128 or hd % g:
        raise ConfigError("head shards must be whole 128-row tiles and whole groups")
    if g % 64 or cfg.d_ff % g:
        raise ConfigError("d_ff shards need group_size a multiple of 64 (128-row gate/up tiles)")
    hq, hk = cfg.n_heads // world, cfg.n_kv_heads // world
    G = cfg.d_ff // g
    g0, g1 = rank * G // world, (rank + 1) * G // world
    if (g1 - g0) * g * 2 % 128:
        raise ConfigError("gate/up shard is not whole tiles")
    return TPSplit(rank, world, (rank * hq, (rank + 1) * hq), (rank * hk, (rank + 1) * hk), (g0 * g, g1 * g))


def vocab_shard(vocab: int, rank: int, world: int) -> tuple[int, int]:
    """The rank's lm_head rows [v0, v1): whole 128-row tiles, remainder spread low-rank first."""
    tiles = -(-vocab // 128)
    t0, t1 = rank * tiles // world, (rank + 1) * tiles // world
    return t0 * 128, min(vocab, t1 * 128)


def _sub_store(src: DeviceStore, tiles, chunks, n: int, k: int) -> DeviceStore:
    """A new store holding tiles x chunks of src (device copies of whole 8 KiB blocks)."""
    import torch
    geo = src.geo
    codes = src.codes.view(geo.n_tiles, geo.n_chunks, 8192)[tiles][:, chunks].contiguous().view(-1)
    scales = src.scales[tiles][:, chunks].contiguous()
    ng = _lib.QWeight()
    _lib.call("qs_qweight_geometry", n, k, src.g, ng)
    if ng.n_tiles * ng.n_chunks * 8192 != codes.numel():
        raise ConfigError("shard does not match the device layout geometry")
    ng.codes, ng.scales = codes.data_ptr(), scales.data_ptr()
    return DeviceStore(n, k, src.g, codes, scales, ng)


class TPShard:
    """Rank-local weights + KV cache + workspace of a tensor-parallel model."""

    def __init__(self, model: TransformerModel, rank: int, world: int, *, slots: int = 1,
                 vocab_split: bool = False) -> None:
        import torch
        cfg = model.config
        self.model, self.cfg, self.split = model, cfg, tp_split(cfg, rank, world)
        sp = self.split
        H, KV, hd, g = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.group_size
        self.n_heads, self.n_kv_heads = sp.heads[1] - sp.heads[0], sp.kv_heads[1] - sp.kv_heads[0]
        self.d_ff = sp.ff[1] - sp.ff[0]
        t = lambda a, b: torch.arange(a, b, device="cuda")  # noqa: E731
        q_t = t(sp.heads[0] * hd // 128, sp.heads[1] * hd // 128)
        k_t = t((H * hd + sp.kv_heads[0] * hd) // 128, (H * hd + sp.kv_heads[1] * hd) // 128)
        v_t = t(((H + KV) * hd + sp.kv_heads[0] * hd) // 128, ((H + KV) * hd + sp.kv_heads[1] * hd) // 128)
        qkv_tiles = torch.cat([q_t, k_t, v_t])
        cpg = model.layers[0].o.geo.cpg
        o_chunks = t(sp.heads[0] * hd // g * cpg, sp.heads[1] * hd // g * cpg)
        gu_tiles = t(2 * sp.ff[0] // 128, 2 * sp.ff[1] // 128)
        dn_chunks = t(sp.ff[0] // g * cpg, sp.ff[1] // g * cpg)
        d = cfg.d_model
        allc = lambda s: torch.arange(s.geo.n_chunks, device="cuda")  # noqa: E731
        self.layers = []
        for lw in model.layers:
            allt = lambda s: torch.arange(s.geo.n_tiles, device="cuda")  # noqa: E731
            self.layers.append(dict(
                attn_norm=lw.attn_norm, ffn_norm=lw.ffn_norm,
                qkv=_sub_store(lw.qkv, qkv_tiles, allc(lw.qkv), (self.n_heads + 2 * self.n_kv_heads) * hd, d),
                o=_sub_store(lw.o, allt(lw.o), o_chunks, d, self.n_heads * hd),
                gate_up=_sub_store(lw.gate_up, gu_tiles, allc(lw.gate_up), 2 * self.d_ff, d),
                down=_sub_store(lw.down, allt(lw.down), dn_chunks, d, self.d_ff)))
        # lm_head: replicated, or this rank's vocab tiles (qs_forward_tp2)
        self.vocab_split = vocab_split
        head = model.lm_head.store
        if vocab_split:
            self.vocab = vocab_shard(cfg.vocab_size, rank, world)
            v0, v1 = self.vocab
            self.lm_head = _sub_store(head, t(v0 // 128, -(-v1 // 128)), allc(head), v1 - v0, d)
        else:
            self.vocab = (0, cfg.vocab_size)
            self.lm_head = head
        # rank-local paged KV cache (local kv heads), one block-table row per slot
        self.page = 16
        self.capacity = cfg.max_seq_len + 8
        pages = -(-self.capacity // self.page)
        self.block_table = torch.arange(slots * pages, dtype=torch.int32, device="cuda").reshape(slots, pages)
        shape = (slots * pages, self.n_kv_heads, self.page, hd)
        self.k = [torch.zeros(shape, device="cuda") for _ in range(cfg.n_layers)]
        self.v = [torch.zeros(shape, device="cuda") for _ in range(cfg.n_layers)]
        self._c_layers = (_lib.Layer * cfg.n_layers)()
        for i, sl in enumerate(self.layers):
            cl = self._c_layers[i]
            cl.attn_norm, cl.ffn_norm = sl["attn_norm"].data_ptr(), sl["ffn_norm"].data_ptr()
            cl.qkv, cl.o, cl.gate_up, cl.down = sl["qkv"].geo, sl["o"].geo, sl["gate_up"].geo, sl["down"].geo
            cl.k_cache, cl.v_cache = self.k[i].data_ptr(), self.v[i].data_ptr()
        self.cm = _lib.Model(n_layers=cfg.n_layers, d_model=d, n_heads=self.n_heads, n_kv_heads=self.n_kv_heads,
                             d_ff=self.d_ff, vocab=self.vocab[1] - self.vocab[0], group_size=g,
                             rope_len=model.rope_len,
                             norm_eps=cfg.norm_eps, tok_emb=model.token_embedding.data_ptr(),
                             final_norm=model.final_norm.data_ptr(), rope_cos=model.rope_cos.data_ptr(),
                             rope_sin=model.rope_sin.data_ptr(), lm_head=self.lm_head.geo,
                             layers=self._c_layers, block_table=self.block_table.data_ptr(),
                             bt_ld=self.block_table.shape[1], page=self.page, hadamard=int(cfg.hadamard))
        # workspace sized for the full model (a superset of the shard's needs)
        self.ws, self._bufs = model.workspace(64)
        import torch as _t
        self.partial = self._bufs["attn"].view(_t.float32)
        self._i32 = dict(dtype=torch.int32, device="cuda")

    def forward(self, tokens: list[int], positions: list[int], allreduce, mode: int = _lib.QS_MODE_HIGH,
                slot: int = 0):
        """One TP forward over T tokens of one sequence: returns (logits [T, V], argmax [T]) on the device."""
        import torch
        T = len(tokens)
        tok = torch.tensor(tokens, **self._i32)
        pos = torch.tensor(positions, **self._i32)
        sl = torch.full((T,), slot, **self._i32)
        z = torch.zeros(1, **self._i32)
        nt = torch.full((1,), T, **self._i32)
        b = _lib.Batch(T=T, tokens=tok.data_ptr(), positions=pos.data_ptr(), slots=sl.data_ptr(), n_blk=1,
                       blk_tok0=z.data_ptr(), blk_ntok=nt.data_ptr(), blk_qmax=T, ctx_cap=self.capacity)
        logits = torch.empty((T, self.cfg.vocab_size), device="cuda")
        arg = torch.empty(T, **self._i32)
        part = self.partial

        def hook(ptr, count, stream, user):
            try:
                if ptr != part.data_ptr():
                    return 1
                allreduce(part[:count])
                return 0
            except Exception:  # noqa: BLE001 - reported to the C side as a failure code
                return 1
        cb = _lib.ALLREDUCE_FN(hook)
        _lib.call("qs_forward_tp", self.cm, b, mode, self.ws, logits.data_ptr(), arg.data_ptr(), self.split.world,
                  C.cast(cb, C.c_void_p), None, _lib.stream_ptr())
        torch.cuda.synchronize()
        return logits, arg


def tp_generate_greedy(shard: TPShard, prompt: list[int], max_new_tokens: int, allreduce,
                       mode: int = _lib.QS_MODE_HIGH) -> list[int]:
    """Greedy decoding with the TP forward (prompt in chunks of <= 4, then one token per step)."""
    out: list[int] = []
    pos = 0
    nxt = None
    for s in range(0, len(prompt), 4):
        chunk = prompt[s:s + 4]
        _, arg = shard.forward(chunk, list(range(pos, pos + len(chunk))), allreduce, mode)
        pos += len(chunk)
        nxt = int(arg[-1].item())
    out.append(nxt)
    while len(out) < max_new_tokens:
        _, arg = shard.forward([out[-1]], [pos], allreduce, mode)
        pos += 1
        out.append(int(arg[0].item()))
    return out


class TPComm:
    """A TP group's collectives for ``qs_forward_tp2``: an NCCL communicator the C runtime
    drives on the forward's stream (``TPComm.nccl``), or host hooks (``TPComm.hooks``:
    gloo in the tests; eager only)."""

    def __init__(self, world: int, rank: int, *, nccl_comm=None, allreduce=None, allgather=None) -> None:
        import torch
        self.world, self.rank, self.nccl_comm = world, rank, nccl_comm
        self.scratch = torch.zeros(_lib.load().qs_tp_scratch_bytes(world), dtype=torch.uint8, device="cuda")
        self._ar, self._ag = allreduce, allgather
        self._bufs = {}

    @property
    def graphable(self) -> bool:
        return self.nccl_comm is not None

    @classmethod
    def nccl(cls, dist) -> "TPComm":
        """Communicator over the torch.distributed group's ranks (id broadcast from rank 0)."""
        world, rank = dist.get_world_size(), dist.get_rank()
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _lib.call("qs_tp_nccl_unique_id", uid)
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        comm = C.c_void_p()
        _lib.call("qs_tp_nccl_init", world, rank, uid, C.byref(comm))
        return cls(world, rank, nccl_comm=comm.value)

    @classmethod
    def hooks(cls, world: int, rank: int, allreduce, allgather) -> "TPComm":
        """allreduce(t): in-place fp32 sum of a device tensor; allgather(send, recv): recv[r] = send of rank r."""
        return cls(world, rank, allreduce=allreduce, allgather=allgather)

    def close(self) -> None:
        if self.nccl_comm is not None:
            _lib.call("qs_tp_nccl_destroy", self.nccl_comm)
            self.nccl_comm = None

    def c_struct(self, shard: "TPShard", partial) -> _lib.TP:
        """qs_tp_t for one shard (hooks bound to its all-reduce buffer and this scratch)."""
        import torch
        t = _lib.TP(world=self.world, rank=self.rank, vocab_off=shard.vocab[0], scratch=self.scratch.data_ptr())
        if self.nccl_comm is not None:
            t.nccl_comm = self.nccl_comm
            return t
        scratch = self.scratch.view(torch.int32)
        per = 64 * 2                     # int32 per rank record block (kTpMaxT int2)

        def ar(ptr, count, stream, user):
            try:
                if ptr != partial.data_ptr():
                    return 1
                self._ar(partial[:count])
                return 0
            except Exception:  # noqa: BLE001 - reported to the C side as a failure code
                return 1

        def ag(send, recv, nbytes, stream, user):
            try:
                if send != scratch.data_ptr() or nbytes != per * 4:
                    return 1
                self._ag(scratch[:per], scratch[per:per * (1 + self.world)].view(self.world, per))
                return 0
            except Exception:  # noqa: BLE001
                return 1
        self._bufs[id(shard)] = (_lib.ALLREDUCE_FN(ar), _lib.ALLGATHER_FN(ag))
        t.allreduce, t.allgather = self._bufs[id(shard)]
        return t


class TPDecodeEngine(DecodeEngine):
    """The batched QSpec / greedy engine (engine.DecodeEngine) over one rank's TP shard.

    Same device control kernels (draft_prep / verify_prep / accept), so the reference's
    cycle (specdec.py:258-317) runs unchanged; every forward is ``qs_forward_tp2``.  With
    an NCCL ``TPComm`` the whole cycle is captured into one CUDA graph."""

    def __init__(self, model: TransformerModel, comm: TPComm, batch: int, **kw) -> None:
        self.comm = comm
        self.shard = TPShard(model, comm.rank, comm.world, slots=batch, vocab_split=True)
        kw.setdefault("use_graphs", comm.graphable)
        super().__init__(model, batch, **kw)
        self.tp = comm.c_struct(self.shard, self.shard.partial)

    def _setup_storage(self, model, batch, gamma) -> None:
        sh = self.shard
        if gamma + 1 > sh.capacity - model.config.max_seq_len:
            raise ConfigError("gamma too large for the shard's KV capacity")
        self.kv = SimpleNamespace(capacity=sh.capacity)
        self.ws, self._ws_bufs = sh.ws, sh._bufs
        self.cm = sh.cm

    def _call_forward(self, b, mode: int, argmax_ptr: int, st: int) -> None:
        _lib.call("qs_forward_tp2", self.cm, b, mode, self.ws, None, argmax_ptr, C.byref(self.tp), st)

    def _prefill_argmax(self, prompt, slot: int, low: bool):
        import torch
        cfg = self.cfg
        hpk = cfg.n_heads // cfg.n_kv_heads
        tmax = min(64, max(1, 64 // hpk))
        ids = prompt if torch.is_tensor(prompt) else torch.tensor(prompt, dtype=torch.int32)
        ids = ids.to(device="cuda", dtype=torch.int32)
        n = ids.numel()
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        i32 = dict(dtype=torch.int32, device="cuda")
        mode = _lib.QS_MODE_LOW if low else _lib.QS_MODE_HIGH
        keep = []
        for s in range(0, n, tmax):
            T = min(tmax, n - s)
            pos = torch.arange(s, s + T, **i32)
            sl = torch.full((T,), slot, **i32)
            blk = torch.tensor([0, T], **i32)
            tok = ids[s:s + T].contiguous()
            keep += [pos, sl, blk, tok]
            b = _lib.Batch(T=T, tokens=tok.data_ptr(), positions=pos.data_ptr(), slots=sl.data_ptr(), n_blk=1,
                           blk_tok0=blk.data_ptr(), blk_ntok=blk[1:].data_ptr(), blk_qmax=T, ctx_cap=s + T)
            self._call_forward(b, mode, out[s:].data_ptr(), _lib.stream_ptr())
        torch.cuda.current_stream().synchronize()
        return out
