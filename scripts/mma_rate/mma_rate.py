"""Time per tcgen05.mma.kind::i8 (A in TMEM): 1-SM M=128 vs 2-SM M=256, for several N.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o scripts/mma_rate/libmma_rate.so scripts/mma_rate/mma_rate.cu
    python scripts/mma_rate/mma_rate.py
"""
import ctypes as C, os, sys
import torch
lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmma_rate.so"))
lib.mma_rate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
out = torch.zeros(148 + 148 * 4, dtype=torch.int64, device="cuda")
stop = torch.zeros(1, dtype=torch.int32, device="cuda")
src = torch.zeros(64 * 32768, dtype=torch.uint8, device="cuda")
lib.mma_set_src.argtypes = [C.c_void_p]
lib.mma_set_src(src.data_ptr())
reps = 2000
for st, cg, n in [(0, 1, 8), (0, 1, 16), (0, 1, 32), (0, 1, 64), (0, 1, 128), (0, 1, 192), (0, 1, 256),
                  (0, 2, 32), (0, 2, 64), (0, 2, 192), (1, 1, 8), (1, 1, 16), (1, 1, 192), (2, 1, 8), (2, 1, 16)]:
    if True:
        grid = 148
        out.zero_(); stop.zero_()
        rc = lib.mma_rate(n, cg, reps, out.data_ptr(), grid, st, stop.data_ptr())
        if rc != 0:
            print(f"cg={cg} N={n}: error {rc}", flush=True)
            continue
        allv = out.cpu().numpy()
        v = allv[:148]
        v = v[v > 0]
        ns = float(v.mean()) / (reps * 4)
        rows_per_sm = 128  # per SM: M=256 pair covers 128 rows on each SM
        extra = ""
        if st == 2:
            nb = allv[148:148 + 148 * 4].reshape(148, 4)[:, 0]
            extra = f"; concurrent bulk copies: {nb[nb > 0].mean() * 32768 / float(v.mean()):.1f} B/ns per SM"
        elif st:
            sts = allv[148:148 + 148 * 4].reshape(148, 4)
            iters = sts[sts > 0].mean()
            t_ns = float(v.mean())
            extra = f"; concurrent tcgen05.st: {iters * 4 * 4096 * 4 / t_ns:.1f} B/ns per SM (4 warps)"
        print(f"st={st} cg={cg} M={128 * cg} N={n:3d}: {ns:6.1f} ns per MMA instruction; "
              f"{rows_per_sm * 32 / ns:6.1f} int8 A bytes/ns per SM{extra}", flush=True)

lib.mma_turnaround.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p]
for sl, ch in ((2, 1), (4, 1), (8, 1), (2, 4), (3, 4)):
    out.zero_()
    rc = lib.mma_turnaround(sl, ch, reps, out.data_ptr())
    v = out.cpu().numpy()[:148]
    v = v[v > 0]
    per = float(v.mean()) / reps
    print(f"turnaround N=8 slots={sl} chunks/slot={ch}: {per:7.1f} ns per slot, {per / (4 * ch):5.1f} ns per MMA "
          f"({8192 * ch / per:6.1f} packed-weight B/ns per SM); rc={rc}", flush=True)
