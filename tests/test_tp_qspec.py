"""Tensor-parallel QSpec (BASELINE config 4): the reference's draft/verify/
accept cycle (specdec.py:258-317) over TP shards with a vocab-split lm_head.

* world 1 over a real NCCL communicator: the whole cycle is captured into one CUDA graph
  (ncclAllReduce / ncclAllGather enqueued by the C runtime on the forward's stream) and
  must reproduce the single-GPU engine bit for bit -- tokens AND accept lengths.
* world 2 / 4 as processes sharing the one GPU with gloo host hooks (eager): QSpec
  tokens equal the single-GPU tokens (fp32 reassociation of the row-split partials
  only; the distributed argmax keeps the lowest-index tie rule).
"""

from __future__ import annotations

import ctypes as C
import os
import socket

import numpy as np
import pytest

import paper_2410_11305_b200 as Q

pytestmark = pytest.mark.gpu

C13 = dict(n_layers=2, d_model=5120, n_heads=40, n_kv_heads=40, d_ff=13824, vocab_size=32000, max_seq_len=128,
           group_size=128)
B, GAMMA, NEW = 2, 3, 12


def _prompts(vocab):
    rng = np.random.default_rng(42)
    return [[int(t) for t in rng.integers(0, vocab, 9 + 4 * b)] for b in range(B)]


def _single_gpu(model):
    from paper_2410_11305_b200.engine import DecodeEngine
    eng = DecodeEngine(model, B, gamma=GAMMA, max_new_cap=NEW + 4)
    for b, p in enumerate(_prompts(model.config.vocab_size)):
        eng.prefill(b, p, NEW)
    eng.run()
    return [eng.result(b) for b in range(B)]


def test_tp_world1_nccl_graph_matches_single_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2410_11305_b200 import _lib
    from paper_2410_11305_b200.tp import TPComm, TPDecodeEngine
    model = Q.random_init(Q.ModelConfig(**C13), 0)
    ref = _single_gpu(model)
    uid = (C.c_uint8 * 128)()
    _lib.call("qs_tp_nccl_unique_id", uid)
    comm = C.c_void_p()
    _lib.call("qs_tp_nccl_init", 1, 0, uid, C.byref(comm))
    tc = TPComm(1, 0, nccl_comm=comm.value)
    try:
        eng = TPDecodeEngine(model, tc, B, gamma=GAMMA, max_new_cap=NEW + 4)
        assert eng.use_graphs
        for b, p in enumerate(_prompts(model.config.vocab_size)):
            eng.prefill(b, p, NEW)
        eng.run()
        got = [eng.result(b) for b in range(B)]
    finally:
        tc.close()
    for g, r in zip(got, ref):
        assert g.new_tokens == r.new_tokens
        assert g.trace[:, 1].tolist() == r.trace[:, 1].tolist()   # per-cycle accept lengths
        assert (g.n_drafted, g.n_accepted) == (r.n_drafted, r.n_accepted)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2410_11305_b200.tp import TPComm, TPDecodeEngine

    def allreduce(t):
        h = t.cpu()
        dist.all_reduce(h)
        t.copy_(h)

    def allgather(send, recv):
        h = send.cpu()
        out = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(out, h)
        recv.copy_(torch.stack(out))

    model = Q.random_init(Q.ModelConfig(**C13), 0)
    eng = TPDecodeEngine(model, TPComm.hooks(world, rank, allreduce, allgather), B, gamma=GAMMA,
                         max_new_cap=NEW + 4)
    assert not eng.use_graphs
    for b, p in enumerate(_prompts(model.config.vocab_size)):
        eng.prefill(b, p, NEW)
    eng.run()
    res = [eng.result(b) for b in range(B)]
    if rank == 0:
        np.save(os.path.join(out_dir, "toks.npy"), np.array([r.new_tokens for r in res], dtype=object),
                allow_pickle=True)
        np.save(os.path.join(out_dir, "drafted.npy"), np.array([r.n_drafted for r in res]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_tp_qspec_gloo_matches_single_gpu(world, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    model = Q.random_init(Q.ModelConfig(**C13), 0)
    ref = _single_gpu(model)
    toks = np.load(tmp_path / "toks.npy", allow_pickle=True)
    assert [list(t) for t in toks] == [r.new_tokens for r in ref]
    assert all(d > 0 for d in np.load(tmp_path / "drafted.npy"))
