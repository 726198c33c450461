"""Summarise an ncu --csv launch list: per-kernel-kind total/mean time."""
import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, vi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
gi = h.index('Grid Size') if 'Grid Size' in h else None
agg = collections.OrderedDict()
tot = 0
for r in rows[hi + 1:]:
    if r[mi] != 'gpu__time_duration.sum':
        continue
    name = re.sub(r'\(.*', '', r[ki]).replace('void ', '').replace('(anonymous namespace)::', '')
    key = name + (f" grid={r[gi]}" if gi is not None else "")
    t = float(r[vi].replace(',', ''))
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1; a[1] += t; tot += t
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t/1e3:10.1f} us {100*t/tot:5.1f}%  n={n:4d}  mean={t/n/1e3:8.2f} us  {k}")
print(f"total {tot/1e3:.1f} us over {sum(n for n,_ in agg.values())} launches")
