"""How sensitive is the reference's W4A4 (LOW) forward to fp32 summation order?

Runs the CPU oracle (bit-exact restatement of the reference) on a BASELINE-shape
2-layer model twice: once as is, once with every linear's fp32 sum computed in
float64 and rounded once (about what the device's exact-integer-core linear does),
and reports how far the LOW logits and the activation codes move.  Research script.
"""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
from oracle import qspec_oracle as O

case = sys.argv[1] if len(sys.argv) > 1 else "7b2l"
C7B = dict(d_model=4096, n_heads=32, n_kv_heads=32, d_ff=11008, vocab_size=32000, max_seq_len=512, group_size=128)
C8B = dict(d_model=4096, n_heads=32, n_kv_heads=8, d_ff=14336, vocab_size=128256, max_seq_len=512,
           rope_theta=500000.0, group_size=128)
cfg = O.OracleConfig(n_layers=2, **(C7B if case == "7b2l" else C8B))
t = time.time()
m = O.random_model(cfg, 0)
print("init", time.time() - t, flush=True)
g = np.load(os.path.join(os.path.dirname(__file__), "..", "..", "tests", "golden", f"large_{case}.npz"))
toks = [int(x) for x in g["fwd_tokens"]]

orig = O.qlinear
flips = {"n": 0, "tot": 0}
def exact_qlinear(lin, x, low):
    if low:
        x = O.fake_quant(x, lin.g)
    return (x.astype(np.float64) @ lin.wt.astype(np.float64)).astype(np.float32)

def run(fn):
    O.qlinear = fn
    kv = O.OracleKV(cfg)
    hi = O.forward(m, toks, kv, False, "verify")
    kv.commit(3)
    nxt = int(g["fwd.low1_token"][0])
    lo1 = O.forward(m, [nxt], kv, True, "draft")
    lo4 = O.forward(m, toks, O.OracleKV(cfg), True, "verify")
    return hi, lo1, lo4

ref = run(orig)
alt = run(exact_qlinear)
O.qlinear = orig
for name, a, b in zip(("high4", "low1", "low4"), ref, alt):
    key = f"fwd.{name}"
    am = g[f"{key}.absmax"]
    print(name, "oracle==golden argmax", list(np.argmax(a, -1)) == list(g[f"{key}.argmax"]),
          "| exact-sum vs oracle: max rel", (np.abs(a - b).max(-1) / np.abs(a).max(-1)).round(5),
          "argmax eq", list(np.argmax(a, -1)) == list(np.argmax(b, -1)))
