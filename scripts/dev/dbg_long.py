"""Repro helper: tiny model, long prompt, greedy HIGH / LOW and QSpec (debugging)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2410_11305_b200 as Q
TINY = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, d_ff=768, vocab_size=1024, max_seq_len=400, group_size=128)
m = Q.random_init(Q.ModelConfig(**TINY), 0)
P = int(sys.argv[1]) if len(sys.argv) > 1 else 270
p = [int(t) for t in np.random.default_rng(1).integers(0, 1024, P)]
for what in ("high", "low", "qspec"):
    try:
        if what == "qspec":
            r = Q.generate_qspec(m, p, Q.GenerationConfig(gamma=3, max_new_tokens=20))
            print(what, r.new_tokens[:10], "acc", r.acceptance_rate, flush=True)
        else:
            mode = Q.ExecutionMode.HIGH_PRECISION if what == "high" else Q.ExecutionMode.LOW_PRECISION
            r = Q.generate_greedy(m, p, mode, Q.GenerationConfig(max_new_tokens=20))
            print(what, r.new_tokens[:10], flush=True)
    except Exception as e:  # noqa
        print(what, "FAILED", str(e)[:200], flush=True)
        break
