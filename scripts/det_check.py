import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2410_11305_b200 as Q
from paper_2410_11305_b200.engine import DecodeEngine
from bench import CFG7B
from oracle import qspec_oracle as O
m = Q.random_init(Q.ModelConfig(**CFG7B), 0)
prompts = np.random.default_rng(42).integers(0, 32000, size=(16, 128))
res = []
for rep in range(3):
    for alg in ("qspec", "greedy"):
        eng = DecodeEngine(m, 1, gamma=3, max_new_cap=136, algorithm=alg)
        eng.prefill(0, [int(t) for t in prompts[0]], 128)
        for _ in range(20):
            eng.step()
        torch.cuda.synchronize()
        r = eng.result(0)
        print(rep, alg, len(r.new_tokens), r.new_tokens[:24], r.n_accepted, r.n_drafted, flush=True)
