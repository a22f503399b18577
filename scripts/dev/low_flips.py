"""Where do the W4A4 (LOW) forwards of two fp32 summation orders part ways?  Research script."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
from oracle import qspec_oracle as O

C7B = dict(d_model=4096, n_heads=32, n_kv_heads=32, d_ff=11008, vocab_size=32000, max_seq_len=512, group_size=128)
cfg = O.OracleConfig(n_layers=2, **C7B)
m = O.random_model(cfg, 0)
g = np.load(os.path.join(os.path.dirname(__file__), "..", "..", "tests", "golden", "large_7b2l.npz"))
toks = [int(x) for x in g["fwd_tokens"]]
orig = O.qlinear
log = []
def mk(exact):
    def f(lin, x, low):
        xq = O.fake_quant(x, lin.g) if low else x
        codes = O.quantize_rows(x, lin.g)[0] if low else None
        y = ((xq.astype(np.float64) @ lin.wt.astype(np.float64)).astype(np.float32) if exact
             else np.einsum("ik,kj->ij", xq, lin.wt, optimize=False))
        log.append((x.copy(), codes, y.copy()))
        return y
    return f
res = []
for ex in (False, True):
    log.clear()
    O.qlinear = mk(ex)
    lo4 = O.forward(m, toks, O.OracleKV(cfg), True, "verify")
    res.append((lo4, list(log)))
names = ["q", "k", "v", "o", "gate", "up", "down"] * 2 + ["lm_head"]
for i, ((xa, ca, ya), (xb, cb, yb)) in enumerate(zip(res[0][1], res[1][1])):
    dx = np.abs(xa - xb).max() / max(np.abs(xa).max(), 1e-30)
    nflip = int((ca != cb).sum())
    dy = np.abs(ya - yb).max(-1) / np.abs(ya).max(-1)
    print(f"{i:2d} {names[i]:8s} in rel {dx:.2e} code flips {nflip:5d} / {ca.size}  out rel per row {np.round(dy, 6)}")
