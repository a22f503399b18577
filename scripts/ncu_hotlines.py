"""Summarise an .ncu-rep source page: warp-stall samples per CUDA source line (and top SASS)."""
import csv, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
lines, sass = [], []
cur = None
for r in rows:
    if len(r) > 5 and r[0].isdigit():
        cur = (int(r[0]), r[1][:110])
        try:
            lines.append((int(r[4]), cur[0], cur[1]))
        except ValueError:
            pass
    elif len(r) > 5 and r[0] == "" and r[2].startswith("0x"):
        try:
            sass.append((int(r[4]), r[3][:90], cur[0] if cur else -1))
        except ValueError:
            pass
tot = sum(x[0] for x in lines) or 1
print("total stall samples", tot)
for s, l, src in sorted(lines, reverse=True)[:n]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  L{l}: {src}")
print("--- top SASS")
for s, ins, l in sorted(sass, reverse=True)[:n]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  L{l}: {ins}")
