"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel name."""
import collections, csv, sys

for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    agg = collections.OrderedDict()
    tot = 0.0
    for r in rows[hi + 1:]:
        name = r[ki].split('(')[0]
        v = float(r[vi].replace(',', '')) / 1000
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    print(f, 'total us', round(tot, 1))
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k[:60]:60s} n={n:5d} total={t:9.1f}us avg={t / n:8.2f}us share={t / tot:.3f}")
