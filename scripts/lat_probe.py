"""Memory round-trip latency probe (qs_debug_latency): idle GPU, 8 x 512 B loads per round."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2410_11305_b200 import _lib
lib = _lib.load()
lib.qs_debug_latency.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
buf = torch.randn(1 << 28, device="cuda")  # 1 GiB
out = torch.zeros(65, dtype=torch.int64, device="cuda")
n_rows = buf.numel() // 128
for cg in (0, 1):
    for stride in (1, 16, 4096):
        for nb in (1, 32, 148):
            lib.qs_debug_latency(buf.data_ptr(), n_rows, 64, stride, nb, out.data_ptr(), cg, torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            v = out[:64].cpu().numpy()
            print(f"cg={cg} stride={stride:5d} blocks={nb:4d}: round us median {sorted(v)[32] / 1e3:.2f} min {v.min() / 1e3:.2f} max {v.max() / 1e3:.2f}")
