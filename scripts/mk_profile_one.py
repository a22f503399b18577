"""One persistent forward (7B shape, LAYERS layers) inside an NVTX range for ncu capture."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
import paper_2410_11305_b200 as Q
from paper_2410_11305_b200.engine import DecodeEngine
from bench import CFG7B

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
algo = sys.argv[2] if len(sys.argv) > 2 else "greedy"
layers = int(os.environ.get("LAYERS", "32"))
cfg = dict(CFG7B, n_layers=layers)
model = Q.random_init(Q.ModelConfig(**cfg), 0)
eng = DecodeEngine(model, B, gamma=3, algorithm=algo, use_graphs=False, persistent=True)
prompts = np.random.default_rng(42).integers(0, cfg["vocab_size"], size=(B, 128))
for b in range(B):
    eng.prefill(b, [int(t) for t in prompts[b]], 64)
eng.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
eng.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
