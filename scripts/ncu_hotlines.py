"""Top CUDA source lines by warp-stall samples / instructions (ncu --import-source capture, -lineinfo build).

    python scripts/ncu_hotlines.py rep.ncu-rep [top] [samples|inst]
"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
by = sys.argv[3] if len(sys.argv) > 3 else "samples"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0, "", collections.Counter()])
cur_file, h = "", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) < 8:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    key = (cur_file, ln)
    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    agg[key][0] += f(r[4])
    agg[key][1] += f(r[7])
    agg[key][2] = r[1].strip()[:80]
    for ci, name in enumerate(h):
        if name.startswith("stall_") and "Not Issued" not in name and ci < len(r):
            agg[key][3][name[6:]] += f(r[ci])
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot_s:.0f}, instructions {tot_i:.0f}")
k = 0 if by == "samples" else 1
for (fn, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][k])[:top]:
    top3 = ", ".join(f"{k}={int(c)}" for k, c in v[3].most_common(3) if c > 0)
    print(f"{v[0]:8.0f} {v[0] / tot_s:6.3f} {v[1] / tot_i:6.3f}  {fn}:{ln}: {v[2][:60]}  [{top3}]")
