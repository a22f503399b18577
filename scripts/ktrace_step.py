"""Device timeline of one replayed decode step (qs_ktrace_*): every forward-path launch's
[first CTA entry, last CTA exit] from %globaltimer, inside the real CUDA graph (PDL intact).

    python scripts/ktrace_step.py --batch 16 [--algorithm qspec|greedy] [--model 7b|8b] [--dump f.json]

Prints per-kind busy time, the idle gaps between consecutive launches (no kernel of
ours running), and the step span; ``--dump`` writes the raw launch list.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

KINDS = {0: "qkv", 1: "o", 2: "gate_up", 3: "down", 4: "lm_head", 5: "pack", 6: "attention", 15: "linear"}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--algorithm", default="qspec")
    ap.add_argument("--model", default="7b")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dump", default=None)
    a = ap.parse_args()
    import torch
    import paper_2410_11305_b200 as Q
    from paper_2410_11305_b200 import _lib
    from paper_2410_11305_b200.engine import DecodeEngine

    cfgs = {"7b": dict(d_model=4096, n_heads=32, n_kv_heads=32, d_ff=11008, vocab_size=32000, max_seq_len=512),
            "8b": dict(d_model=4096, n_heads=32, n_kv_heads=8, d_ff=14336, vocab_size=128256, max_seq_len=512,
                       rope_theta=500000.0)}
    model = Q.random_init(Q.ModelConfig(n_layers=a.layers, group_size=128, **cfgs[a.model]), 0)
    eng = DecodeEngine(model, a.batch, gamma=3, max_new_cap=256, algorithm=a.algorithm)
    rng = np.random.default_rng(42)
    for b in range(a.batch):
        eng.prefill(b, [int(t) for t in rng.integers(0, model.config.vocab_size, a.prompt)], 200)
    eng.step()  # warm-up + the normal graph
    body = eng._cycle_body if a.algorithm == "qspec" else eng._ar_body
    cap = 16384
    buf = torch.zeros((cap, 2), dtype=torch.int64, device="cuda")
    _lib.call("qs_ktrace_enable", buf.data_ptr(), cap)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    tags = (C.c_int32 * cap)()
    n = _lib.i32()
    _lib.call("qs_ktrace_read", C.addressof(tags), cap, C.byref(n))
    _lib.call("qs_ktrace_enable", None, 0)
    n = n.value
    spans = []
    for _ in range(a.reps):
        buf[:, 0] = np.iinfo(np.int64).max
        buf[:, 1] = 0
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        spans.append(buf[:n].cpu().numpy().astype(np.float64))
    t = spans[-1]
    t0 = t[:, 0].min()
    st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3  # us
    tg = [tags[i] for i in range(n)]
    per: dict[str, list[float]] = {}
    for i in range(n):
        key = ("draft." if tg[i] // 16 == 1 else "verify.") + KINDS.get(tg[i] % 16, str(tg[i] % 16))
        d = per.setdefault(key, [0, 0.0])
        d[0] += 1
        d[1] += en[i] - st[i]
    # idle = time covered by no launch
    order = np.argsort(st)
    idle, cur = 0.0, 0.0
    for i in order:
        if st[i] > cur:
            idle += st[i] - cur
        cur = max(cur, en[i])
    span = en.max()
    print(f"launches {n}  span {span:.1f} us  idle (no kernel of ours running) {idle:.1f} us  "
          f"replays {[round(float((s[:, 1].max() - s[:, 0].min()) / 1e3), 1) for s in spans]}")
    for k, (cnt, tot) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:18s} n={cnt:5d}  sum dur {tot:9.1f} us  avg {tot / cnt:7.2f} us")
    # one layer's chain in detail (the 2nd layer of the first forward)
    print("first 24 launches: tag start end dur gap_from_prev_end")
    prev = 0.0
    for i in range(min(n, 24)):
        print(f"  {KINDS.get(tg[i] % 16, tg[i] % 16):10s} {st[i]:9.2f} {en[i]:9.2f} {en[i] - st[i]:7.2f} {st[i] - prev:7.2f}")
        prev = en[i]
    if a.dump:
        json.dump({"tags": tg, "start_us": st.tolist(), "end_us": en.tolist()}, open(a.dump, "w"))


if __name__ == "__main__":
    main()
