"""Tensor parallelism for the 13B-shape config: shard geometry on CPU, and
the sharded forward with its all-reduce hook against the single-GPU forward
(world_size ranks as processes sharing one GPU, gloo all-reduce)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import paper_2410_11305_b200 as Q
from paper_2410_11305_b200.tp import tp_split

C13 = dict(n_layers=40, d_model=5120, n_heads=40, n_kv_heads=40, d_ff=13824, vocab_size=32000, max_seq_len=512,
           group_size=128)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_tp_split_13b_covers_everything_group_aligned(world):
    cfg = Q.ModelConfig(**C13)
    sps = [tp_split(cfg, r, world) for r in range(world)]
    assert [s.heads for s in sps] == [(r * 40 // world, (r + 1) * 40 // world) for r in range(world)]
    ff = [s.ff for s in sps]
    assert ff[0][0] == 0 and ff[-1][1] == 13824 and all(a[1] == b[0] for a, b in zip(ff, ff[1:]))
    sizes = {b - a for a, b in ff}
    assert all(sz % 128 == 0 for sz in sizes)
    if world == 8:  # 108 groups over 8 ranks: 13 or 14 groups each
        assert sizes == {13 * 128, 14 * 128}


def test_tp_split_rejects_bad_shapes():
    with pytest.raises(Q.ConfigError):
        tp_split(Q.ModelConfig(**C13), 0, 3)   # 40 heads / 3
    with pytest.raises(Q.ConfigError):
        tp_split(Q.ModelConfig(**C13), 4, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tp_worker(rank, world, port, cfg_kw, prompt, n_new, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2410_11305_b200.tp import TPShard, tp_generate_greedy

    def allreduce(t):  # host-staged gloo all-reduce of a device buffer (NCCL on real TP ranks)
        h = t.cpu()
        dist.all_reduce(h)
        t.copy_(h)

    model = Q.random_init(Q.ModelConfig(**cfg_kw), 0)
    shard = TPShard(model, rank, world)
    logits, _ = shard.forward(prompt[:4], [0, 1, 2, 3], allreduce)
    shard2 = TPShard(model, rank, world)
    toks = tp_generate_greedy(shard2, prompt, n_new, allreduce)
    if rank == 0:
        np.save(os.path.join(out_dir, "logits.npy"), logits.cpu().numpy())
        np.save(os.path.join(out_dir, "toks.npy"), np.array(toks))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 8])
def test_tp_forward_matches_single_gpu(world, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    cfg_kw = dict(C13, n_layers=2, max_seq_len=128)
    prompt = [11, 2024, 7, 31999, 5, 100, 42]
    n_new = 8
    mp.spawn(_tp_worker, args=(world, _free_port(), cfg_kw, prompt, n_new, str(tmp_path)), nprocs=world, join=True)
    model = Q.random_init(Q.ModelConfig(**cfg_kw), 0)
    kv = Q.KVCache(model.config)
    full = Q.forward(model, prompt[:4], kv, Q.ExecutionMode.HIGH_PRECISION, Q.WriteTarget.VERIFY).numpy()
    tp_logits = np.load(tmp_path / "logits.npy")
    err = np.abs(tp_logits - full).max() / np.abs(full).max()
    assert err < 1e-4, err   # fp32 partial sums reassociated across ranks
    ref = Q.generate_greedy(model, prompt, Q.ExecutionMode.HIGH_PRECISION,
                            Q.GenerationConfig(max_new_tokens=n_new)).new_tokens
    assert list(np.load(tmp_path / "toks.npy")) == ref


def test_vocab_shard_tiles_cover_vocab():
    from paper_2410_11305_b200.tp import vocab_shard
    for V in (32000, 128256, 1024, 1000):
        for world in (1, 2, 4, 8):
            sh = [vocab_shard(V, r, world) for r in range(world)]
            assert sh[0][0] == 0 and sh[-1][1] == V
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            assert all(v0 % 128 == 0 for v0, _ in sh)
