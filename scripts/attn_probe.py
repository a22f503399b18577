"""Time the persistent kernel's attention phase alone (QS_MK_ATTN_ONLY) after a few real steps."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
import paper_2410_11305_b200 as Q
from paper_2410_11305_b200 import _lib
from paper_2410_11305_b200.engine import DecodeEngine
from bench import CFG7B
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = dict(CFG7B, n_layers=2)
model = Q.random_init(Q.ModelConfig(**cfg), 0)
eng = DecodeEngine(model, B, gamma=3, algorithm="greedy", use_graphs=False, persistent=True)
prompts = np.random.default_rng(42).integers(0, cfg["vocab_size"], size=(B, 128))
for b in range(B):
    eng.prefill(b, [int(t) for t in prompts[b]], 64)
for _ in range(3):
    eng.step()
torch.cuda.synchronize()
dbg = torch.zeros(8 * 64, dtype=torch.int64, device="cuda")
_lib.call("qs_debug_timeline", dbg.data_ptr())
os.environ["QS_MK_ATTN_ONLY"] = "1"
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    e0.record()
    eng.step()
    e1.record()
    torch.cuda.synchronize()
    print(f"ar_prep + attention-only + commit: {e0.elapsed_time(e1) * 1e3:.1f} us")
d = dbg.cpu().numpy().reshape(-1, 8).astype(np.float64)
t0 = d[0, 0]
for r in d[:4]:
    if r[0] == 0:
        break
    print(" ".join(f"{(v - t0) / 1e3:8.2f}" for v in r[:8]))
