"""Per-launch time of the per-step operand pack (qs_act_quant path of act_pack_kernel) and linear."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2410_11305_b200 import _lib
st = _lib.stream_ptr()
for T in (1, 16, 64):
    K = 4096
    x = torch.randn(T, K, device="cuda")
    codes = torch.empty(T, K, dtype=torch.int8, device="cuda")
    sc = torch.empty(T, K // 128, device="cuda")
    fq = torch.empty(T, K, device="cuda")
    for _ in range(3):
        _lib.call("qs_act_quant", x.data_ptr(), T, K, 128, codes.data_ptr(), sc.data_ptr(), fq.data_ptr(), st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(200):
        _lib.call("qs_act_quant", x.data_ptr(), T, K, 128, codes.data_ptr(), sc.data_ptr(), fq.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    print(f"act_pack T={T}: {e0.elapsed_time(e1) * 1e3 / 200:.2f} us per launch (stream, PDL)")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g):
            for _ in range(50):
                _lib.call("qs_act_quant", x.data_ptr(), T, K, 128, codes.data_ptr(), sc.data_ptr(), fq.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
    g.replay(); torch.cuda.synchronize()
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    print(f"act_pack T={T}: {e0.elapsed_time(e1) * 1e3 / 50:.2f} us per launch (graph)")
