"""CTA timeline of ONE linear launch inside a real decode forward (needs a build with
QS_NVCC_EXTRA=-DQS_LIN_TIMELINE=1): which part of a linear's span is ramp, operand wait,
stages, stream-K fixup and exit.

    python scripts/lin_step_trace.py --batch 1 --layers 4 --which o [--mode high|low]
Times are ns relative to the earliest CTA entry of that launch.
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_11305_b200 as Q
from paper_2410_11305_b200 import _lib
from paper_2410_11305_b200.model import run_forward_chunks

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--which", default="o")
ap.add_argument("--layer", type=int, default=2)
ap.add_argument("--mode", default="high")
a = ap.parse_args()
cfg = Q.ModelConfig(n_layers=a.layers, d_model=4096, n_heads=32, n_kv_heads=32, d_ff=11008, vocab_size=32000,
                    max_seq_len=512, group_size=128)
model = Q.random_init(cfg, 0)
kv = Q.KVCache(cfg, gamma_max=3, slots=1)
ids = [int(t) for t in np.random.default_rng(42).integers(0, 32000, a.batch)]
low = a.mode == "low"
run_forward_chunks(model, kv, ids * 4, 0, low)       # warm (attributes, context)
torch.cuda.synchronize()
idx = 1 + 4 * a.layer + {"qkv": 0, "o": 1, "gate_up": 2, "down": 3}[a.which]
dbg = torch.zeros(8192, dtype=torch.int64, device="cuda")
_lib.call("qs_debug_timeline", dbg.data_ptr())
_lib.call("qs_debug_select", idx)
run_forward_chunks(model, kv, ids, 200, low)
torch.cuda.synchronize()
_lib.call("qs_debug_select", 0)
_lib.call("qs_debug_timeline", None)
d = dbg.cpu().numpy().astype(np.int64)
names = {1024: "entry", 4096: "pdl_wait_ret", 3072: "first_w_data", 4608: "first_act_mma", 3584: "last_seg_fixup",
         5120: "owner_got_parts", 6144: "parts_summed", 6656: "postop_done", 7168: "rms_barrier",
         7936: "rms_inv", 7680: "rms_quantised", 5632: "epi_done", 2048: "exit"}
ent = d[1024:1024 + 148]
t0 = ent[ent > 0].min()
print(f"{a.which} layer {a.layer} T={a.batch} mode={a.mode}")
for off, nm in sorted(names.items(), key=lambda kv: np.median(d[kv[0]:kv[0] + 148][d[kv[0]:kv[0] + 148] > 0] - t0)
                      if (d[kv[0]:kv[0] + 148] > 0).any() else 1e18):
    v = d[off:off + 148]
    v = v[v > 0] - t0
    if len(v) == 0:
        print(f"  {nm:16s} (none)")
        continue
    p = np.percentile(v, [0, 10, 50, 90, 100]).astype(int)
    print(f"  {nm:16s} n={len(v):3d}  min {p[0]:6d}  p10 {p[1]:6d}  med {p[2]:6d}  p90 {p[3]:6d}  max {p[4]:6d}")
# per-owner step durations (owners = CTAs that waited for contributor partials)
own = np.nonzero(d[5120:5120 + 148] > 0)[0]
if len(own):
    steps = [(3584, 5120, "own seg end -> partials ready"), (5120, 6144, "partials summed"),
             (6144, 6656, "post-op"), (6656, 7168, "leaves + owner barrier"), (7168, 7936, "1/rms"),
             (7936, 7680, "quantise"), (7680, 2048, "-> exit")]
    print(f"  owners n={len(own)} (median / max ns per step)")
    for s0, s1, nm in steps:
        x, y = d[s0 + own], d[s1 + own]
        ok = (x > 0) & (y > 0)
        if ok.any():
            dd = (y - x)[ok]
            print(f"    {nm:28s} {int(np.median(dd)):6d} {int(dd.max()):6d}")
