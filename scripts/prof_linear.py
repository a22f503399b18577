"""One store, one operand: pack+linear once, then the prepacked linear twice (ncu target:
-k regex:linear_tc --launch-skip 2 -c 1 captures the last one).

    python scripts/prof_linear.py 28672x8192 64 w4a16
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_11305_b200 as Q
from paper_2410_11305_b200 import _lib
from paper_2410_11305_b200.quant import _ws

n, k = map(int, sys.argv[1].split("x"))
M = int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "w4a16"
w = torch.randn(n, k, device="cuda") * 0.02
st = Q.quantize_groupwise(w, 128)
x = torch.randn(M, k, device="cuda")
y = torch.empty(M, n, device="cuda")
ws = _ws.get(n, k, 128)
s = _lib.stream_ptr()
_lib.call("qs_w4a16_linear" if mode == "w4a16" else "qs_w4a4_linear", st.store.geo, x.data_ptr(), M, y.data_ptr(), ws, s)
md = 0 if mode == "w4a16" else 1
for _ in range(2):
    _lib.call("qs_linear_prepacked", st.store.geo, M, md, y.data_ptr(), ws, s)
torch.cuda.synchronize()
print("ok")
