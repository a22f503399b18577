"""%globaltimer timeline of one persistent forward (CTA 0's view of every phase).

    python scripts/mk_timeline.py [batch] [low|high]
Columns: phase kind, worker start (after the previous phase), dependency satisfied,
done (CTA 0's share published), operand producer's dependency satisfied (linears),
weight producer starting that linear's weights -- all in us from the first record.
"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
import paper_2410_11305_b200 as Q
from paper_2410_11305_b200 import _lib
from paper_2410_11305_b200.engine import DecodeEngine
from bench import CFG7B

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
low = len(sys.argv) > 2 and sys.argv[2] == "low"
layers = int(os.environ.get("LAYERS", "32"))
cfg = dict(CFG7B, n_layers=layers)
if os.environ.get("DMODEL"):  # shrink the model (TLB / L2 experiments): d, ff scaled, 32 heads of 128 kept if possible
    d = int(os.environ["DMODEL"])
    cfg.update(d_model=d, n_heads=max(1, d // 128), n_kv_heads=max(1, d // 128), d_ff=int(os.environ.get("DFF", 2 * d)),
               vocab_size=int(os.environ.get("VOCAB", 4096)))
model = Q.random_init(Q.ModelConfig(**cfg), 0)
eng = DecodeEngine(model, B, gamma=3, algorithm="greedy", greedy_low=low, use_graphs=False, persistent=True)
prompts = np.random.default_rng(42).integers(0, cfg["vocab_size"], size=(B, 128))
for b in range(B):
    eng.prefill(b, [int(t) for t in prompts[b]], 64)
for _ in range(3):
    eng.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    e0.record()
    eng.step()
    e1.record()
    torch.cuda.synchronize()
print(f"step without instrumentation: {e0.elapsed_time(e1) * 1e3:.1f} us")
dbg = torch.zeros(8192 + 400 * 148, dtype=torch.int64, device="cuda")
_lib.call("qs_debug_timeline", dbg.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng.step()
e1.record()
torch.cuda.synchronize()
_lib.call("qs_debug_timeline", None)
print(f"step (ar_prep + forward + commit): {e0.elapsed_time(e1) * 1e3:.1f} us, B={B}, {'LOW' if low else 'HIGH'}")
d = dbg.cpu().numpy().reshape(-1, 4).astype(np.float64)
n = 9 * layers + 2
d = d[:n]
t0 = d[d > 0].min()
rel = np.where(d > 0, (d - t0) / 1e3, np.nan)
kinds = (["pack_qkv", "qkv", "attn", "pack_o", "o", "pack_gu", "gate_up", "pack_down", "down"] * layers
         + ["pack_head", "lm_head"])
agg = {}
prev_done = 0.0
for p in range(n):
    k = kinds[p]
    st, dep, done, wprod = rel[p]
    if p < 20 or p > n - 4:
        print(f"{p:4d} {k:10s} start {st:8.1f} dep {dep:8.1f} done {done:8.1f} wprod {wprod:8.1f}")
    a = agg.setdefault(k, [])
    a.append(done - prev_done if not np.isnan(done) else np.nan)
    if not np.isnan(done):
        prev_done = done
print("mean time from previous phase done to this phase done (CTA 0), us:")
for k, v in agg.items():
    print(f"  {k:10s} {np.nanmean(v):8.2f}")
print("total", np.nanmax(rel))
sd = dbg.cpu().numpy()[4 * 512: 4 * 512 + 10 * 256].reshape(10, 256).astype(np.float64)
sd = np.where(sd > 0, (sd - t0) / 1e3, np.nan)
print("per-stage (CTA 0): stage  wprod  unpack  aprod  mma  epi  mma:accempty  mma:afull  mma:tfull  aprod:aempty  mma:issued")
for i in range(int(os.environ.get('S0', 0)), min(int(os.environ.get('S0', 0)) + 40, 256)):
    if np.all(np.isnan(sd[:, i])):
        break
    print(f"{i:4d} " + " ".join(f"{v:8.1f}" for v in sd[:, i]))
ad = dbg.cpu().numpy()[4 * 512 + 10 * 256: 4 * 512 + 11 * 256].reshape(-1, 8).astype(np.float64)
ad = np.where(ad > 0, (ad - t0) / 1e3, np.nan)
print("attention items of CTA 0 warp 0 (layer 1): start, after-setup, after-scores, after-softmax, end, kbatch0, kbatch1, kbatch2")
for r in ad[:8]:
    if np.all(np.isnan(r)):
        break
    print(" ".join(f"{v:8.2f}" for v in r[:8]))
raw = dbg.cpu().numpy()[4 * 512 + 10 * 256: 4 * 512 + 11 * 256].reshape(-1, 8)
print("in-kernel latency probe rounds (us):", [round(float(x) / 1e3, 2) for x in raw[1, 1:5]])
print("2048 dependent FMA us:", raw[1, 5] / 1e3, " 256 dependent shfl+add us:", raw[1, 6] / 1e3)

# per-CTA completion of every phase: when the phase is complete (max over CTAs) and the spread
ct = dbg.cpu().numpy()[8192: 8192 + n * 148].reshape(n, 148).astype(np.float64)
ct = np.where(ct > 0, (ct - t0) / 1e3, np.nan)
done = np.nanmax(ct, axis=1)
first = np.nanmin(ct, axis=1)
agg2 = {}
prev = 0.0
for p in range(n):
    agg2.setdefault(kinds[p], []).append((done[p] - prev, done[p] - first[p], int(np.nanargmax(ct[p]))))
    prev = done[p]
print("phase completion (all CTAs): mean duration from previous phase complete, mean spread first->last CTA, slowest CTAs")
for k, v in agg2.items():
    a = np.array([x[:2] for x in v])
    print(f"  {k:10s} {a[:, 0].mean():8.2f} {a[:, 1].mean():8.2f}   slowest {[x[2] for x in v[:4]]}")
print("forward total (last phase complete):", done[-1])
# hop latency: CTA 0 sees phase p's dependency satisfied vs the dependency's last publisher
hops = {}
for p in range(1, n):
    dep_done = done[p - 1]
    seen = rel[p][1]
    if not np.isnan(seen) and not np.isnan(dep_done):
        hops.setdefault(kinds[p], []).append(seen - dep_done)
print("hop latency (CTA 0 sees dependency - last CTA published it), us:")
for k, v in hops.items():
    print(f"  {k:10s} {np.mean(v):7.2f}")
# work after the hop: CTA 0 phase done - dependency seen
print("CTA 0 work after dependency seen, us:")
w = {}
for p in range(1, n):
    if not np.isnan(rel[p][1]) and not np.isnan(ct[p][0]):
        w.setdefault(kinds[p], []).append(ct[p][0] - rel[p][1])
for k, v in w.items():
    print(f"  {k:10s} {np.mean(v):7.2f}")
