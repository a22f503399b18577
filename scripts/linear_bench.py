"""Microbench (BASELINE config C4): W4A4 / W4A16 linear, M tokens, vs the HBM roofline.

Rotates over enough distinct weight stores that every call streams from HBM
(working set > 126 MB L2).  Times pack+linear (what qlinear_forward launches)
with CUDA events; bytes = N*K/2 + 4*N*K/g + 4*M*K + 4*M*N.
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="11008x4096,4096x11008,28672x8192,8192x28672")
    ap.add_argument("--ms", default="1,4,16,64")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch
    import paper_2410_11305_b200 as Q
    from paper_2410_11305_b200 import _lib
    from paper_2410_11305_b200.quant import _ws
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"]
    i8 = os.path.join(root, "profiles", "int8_peak.json")   # scripts/int8_peak.py (cuBLASLt int8)
    int8_tops = json.load(open(i8))["int8_tops_measured"] if os.path.exists(i8) else None
    out = []
    for shp in a.shapes.split(","):
        n, k = map(int, shp.split("x"))
        wbytes = n * k // 2 + 4 * n * (k // 128)
        copies = max(2, int(400e6 // wbytes) + 1)
        w = torch.randn(n, k, device="cuda") * 0.02
        stores = [Q.quantize_groupwise(w, 128) for _ in range(copies)]
        for M in map(int, a.ms.split(",")):
            x = torch.randn(M, k, device="cuda")
            y = torch.empty(M, n, device="cuda")
            # the C ABI takes <= 64 tokens per call (qs_linear_max_tokens); larger M runs as
            # 64-token calls, each streaming the weights again (what qlinear_forward does)
            chunks = [(m0, min(64, M - m0)) for m0 in range(0, M, 64)]
            for mode, fn in (("w4a4", "qs_w4a4_linear"), ("w4a16", "qs_w4a16_linear")):
                ws = _ws.get(n, k, 128)
                st = _lib.stream_ptr()
                def call(i):
                    for m0, mm in chunks:
                        _lib.call(fn, stores[i % copies].store.geo, x[m0:].data_ptr(), mm, y[m0:].data_ptr(), ws, st)

                for i in range(3):
                    call(i)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for i in range(a.reps):
                    call(i)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / a.reps
                # linear kernel alone on the packed operand
                md = 1 if mode == "w4a4" else 0
                e0.record()
                for i in range(a.reps):
                    for m0, mm in chunks:
                        _lib.call("qs_linear_prepacked", stores[i % copies].store.geo, mm, md, y[m0:].data_ptr(), ws, st)
                e1.record()
                torch.cuda.synchronize()
                us_lin = e0.elapsed_time(e1) * 1e3 / a.reps
                byts = wbytes + 4 * M * k + 4 * M * n
                r = {"shape": shp, "M": M, "mode": mode, "us": round(us, 2), "us_linear_only": round(us_lin, 2),
                     "GBps_linear_only": round(byts / us_lin / 1e3, 1), "GBps": round(byts / us / 1e3, 1),
                     "frac_hbm": round(byts / us / 1e3 / peak, 3),
                     "TOPS": round(2 * M * n * k * (3 if mode == "w4a16" else 1) / us / 1e6, 2)}
                if int8_tops:  # tensor-pipe fraction of the int8 MACs the kernel actually issues
                    r["frac_int8_tensor"] = round(r["TOPS"] / int8_tops, 4)
                out.append(r)
                print(json.dumps(r), flush=True)
        del stores
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
