"""A few T-token forwards of a 2-layer 7B-shape model (ncu target for the in-forward linear
launches: chained or not, per QS_EMIT / QS_CHAIN_SPLIT).

    python scripts/prof_forward.py 16 low 3
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_11305_b200 as Q
from paper_2410_11305_b200.model import run_forward_chunks

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16
low = (sys.argv[2] if len(sys.argv) > 2 else "low") == "low"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = Q.ModelConfig(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=32, d_ff=11008, vocab_size=32000,
                    max_seq_len=256, group_size=128)
model = Q.random_init(cfg, 0)
ids = [int(t) for t in np.random.default_rng(T).integers(0, cfg.vocab_size, T)]
for _ in range(reps):
    kv = Q.KVCache(model.config)
    run_forward_chunks(model, kv, ids, 0, low)
torch.cuda.synchronize()
print("ok")
