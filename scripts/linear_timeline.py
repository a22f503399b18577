"""%globaltimer timeline of one tensor-core linear launch (pipeline diagnosis).

Per-CTA entry / exit times for all CTAs and per-stage role events for CTA 0.
The stamps are compiled out by default: build with
QS_NVCC_EXTRA=-DQS_LIN_TIMELINE=1 python -c "from paper_2410_11305_b200 import build as b; b.build(force=True)"
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_11305_b200 as Q
from paper_2410_11305_b200 import _lib
from paper_2410_11305_b200.quant import _ws

n, k, M = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (11008, 4096, 1)))
mode = sys.argv[4] if len(sys.argv) > 4 else "w4a4"
w = torch.randn(n, k, device="cuda") * 0.02
stores = [Q.quantize_groupwise(w, 128) for _ in range(12)]
x = torch.randn(M, k, device="cuda")
y = torch.empty(M, n, device="cuda")
ws = _ws.get(n, k, 128)
fn = "qs_w4a4_linear" if mode == "w4a4" else "qs_w4a16_linear"
md = 1 if mode == "w4a4" else 0
st = _lib.stream_ptr()
_lib.call(fn, stores[0].store.geo, x.data_ptr(), M, y.data_ptr(), ws, st)
dbg = torch.zeros(8192, dtype=torch.int64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(4):
    _lib.call("qs_debug_timeline", dbg.data_ptr() if rep == 3 else None)
    if rep == 3:
        e0.record()
    _lib.call("qs_linear_prepacked", stores[1 + rep].store.geo, M, md, y.data_ptr(), ws, st)
    if rep == 3:
        e1.record()
_lib.call("qs_debug_timeline", None)
torch.cuda.synchronize()
d = dbg.cpu().numpy()
ent = d[1024:1024 + 148]
ext = d[2048:2048 + 148]
ent, ext = ent[ent > 0], ext[ext > 0]
t0 = ent.min()
print(f"event time {e0.elapsed_time(e1)*1e3:.1f} us; CTAs {len(ent)}; entry spread {ent.max()-t0} ns; "
      f"exit min {ext.min()-t0} max {ext.max()-t0} ns; median dur {np.median(ext-ent):.0f} ns")
fd = d[3072:3072 + 148] - t0
fx = d[3584:3584 + 148] - t0
ex = d[2048:2048 + 148] - t0
order = np.argsort(ex)
print("slowest CTAs (cta, first_data, last_segment_fixup, exit):", [(int(c), int(fd[c]), int(fx[c]), int(ex[c])) for c in order[-8:]])
print("fastest CTAs:", [(int(c), int(fd[c]), int(fx[c]), int(ex[c])) for c in order[:4]])
print("first-data percentiles (ns):", np.percentile(fd, [0, 50, 90, 100]).astype(int))
print(" i  prod_issue  unpack_done  mma_issued  epi_done   (ns from first CTA entry)")
for i in range(64):
    if d[i] == 0:
        break
    print(f"{i:3d} " + " ".join(f"{(d[r * 64 + i] - t0) if d[r * 64 + i] else -1:10d}" for r in range(4)))

print(" i  mma_top  acc_ok  full_ok  tfull_ok  mmas_issued | unpack_start | epi_start")
for i in range(64):
    if d[i] == 0:
        break
    print(f"{i:3d} " + " ".join(f"{(d[r * 64 + i] - t0) if d[r * 64 + i] else -1:8d}" for r in (4, 5, 6, 7, 8, 9, 10)))

print(" i  epi_top  sfull_ok  acc_ok(epi_start)  ld_done  epi_done")
for i in range(64):
    if d[i] == 0:
        break
    print(f"{i:3d} " + " ".join(f"{(d[r * 64 + i] - t0) if d[r * 64 + i] else -1:8d}" for r in (11, 12, 10, 13, 3)))
