"""One decode step of the bench workload inside an NVTX range "step" (for ncu --nvtx-include step/).

    ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --batch 16
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--gamma", type=int, default=3)
    ap.add_argument("--algorithm", default="qspec")
    ap.add_argument("--small", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2410_11305_b200 as Q
    from paper_2410_11305_b200.engine import DecodeEngine
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import CFG7B
    kw = dict(CFG7B) if not a.small else dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, d_ff=768,
                                              vocab_size=1024, max_seq_len=512, group_size=128)
    model = Q.random_init(Q.ModelConfig(**kw), 0)
    prompts = np.random.default_rng(42).integers(0, kw["vocab_size"], size=(a.batch, 128))
    eng = DecodeEngine(model, a.batch, gamma=a.gamma, max_new_cap=136, algorithm=a.algorithm, use_graphs=False)
    for b in range(a.batch):
        eng.prefill(b, [int(t) for t in prompts[b]], 128)
    eng.step()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("step")
    eng.step()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("profiled one", a.algorithm, "step, batch", a.batch)


if __name__ == "__main__":
    main()
