"""Measured dense int8 tensor-core throughput (torch._int_mm -> cuBLASLt IMMA) on this B200:
the denominator for the W4A4 linear's tensor-pipe fraction (SURVEY 8d asks for it; it is not in
MEASURED_PEAKS.json)."""
import json, os, sys
import torch

res = {}
for n in (4096, 8192, 16384):
    a = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[n] = 2 * n ** 3 / (ms / 1e3) / 1e12
    print(f"int8 GEMM {n}^3: {ms:.3f} ms, {res[n]:.0f} TOPS", flush=True)
out = {"int8_tops_measured": round(max(res.values()), 1), "per_size": {str(k): round(v, 1) for k, v in res.items()},
       "method": "torch._int_mm (cuBLASLt int8 IMMA), square n^3, CUDA events, 20 reps"}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/int8_peak.json", "w"), indent=1)
print(json.dumps(out))
