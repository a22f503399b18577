"""Calibrate statistical draft-path parity: the reference's own algorithm with float64-accurate
linear sums (a faithful implementation that only rounds differently) vs the reference.  Research."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
from oracle import qspec_oracle as O

TINY = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, d_ff=768, vocab_size=1024, group_size=128)
orig = O.qlinear
def exact(lin, x, low):
    xq = O.fake_quant(x, lin.g) if low else x
    return (xq.astype(np.float64) @ lin.wt.astype(np.float64)).astype(np.float32)

def stats(m, prompts, n_new):
    out = []
    for p in prompts:
        p = [int(t) for t in p]
        lo = O.generate(m, p, max_new=n_new, qspec=False, low_greedy=True).new_tokens
        qs = O.generate(m, p, gamma=3, max_new=n_new)
        out.append((lo, [c[1] for c in qs.cycles], qs.acceptance_rate, sum(c[1] for c in qs.cycles), sum(len(c[0]) for c in qs.cycles)))
    return out

for name, cfgkw, P, n_new in (("tiny", dict(TINY, max_seq_len=160), 16, 64), ("ctx", dict(TINY, max_seq_len=400), 270, 40)):
    m = O.random_model(O.OracleConfig(**cfgkw), 0)
    prompts = np.random.default_rng(42).integers(0, 1024, size=(8, P))
    O.qlinear = orig; a = stats(m, prompts, n_new)
    O.qlinear = exact; b = stats(m, prompts, n_new)
    O.qlinear = orig
    div = []
    for (la, ta, *_), (lb, tb, *_) in zip(a, b):
        d = next((i for i, (x, y) in enumerate(zip(la, lb)) if x != y), len(la))
        div.append(d)
    same_tr = sum(ta == tb for (_, ta, *_), (_, tb, *_) in zip(a, b))
    acc_a = sum(x[3] for x in a) / sum(x[4] for x in a); acc_b = sum(x[3] for x in b) / sum(x[4] for x in b)
    print(name, "LOW first divergence per prompt", div, "| identical accept traces", same_tr, "/ 8",
          "| aggregate acceptance ref %.4f f64-sums %.4f" % (acc_a, acc_b), flush=True)
