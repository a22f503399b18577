"""Repro helper: one HIGH/LOW forward of T tokens on the tiny model (debugging)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2410_11305_b200 as Q
from paper_2410_11305_b200.model import run_forward_chunks
TINY = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, d_ff=768, vocab_size=1024, max_seq_len=400, group_size=128)
m = Q.random_init(Q.ModelConfig(**TINY), 0)
T = int(sys.argv[1]); base = int(sys.argv[2]) if len(sys.argv) > 2 else 0
low = len(sys.argv) > 3 and sys.argv[3] == "low"
kv = Q.KVCache(m.config)
ids = [int(t) for t in np.random.default_rng(1).integers(0, 1024, T)]
lg, am = run_forward_chunks(m, kv, ids, base, low)
torch.cuda.synchronize()
print("ok", T, base, am[:4].tolist())
