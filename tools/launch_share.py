"""Kernel time shares from an `ncu --metrics gpu__time_duration.sum --csv` launch list.
Only the launches of the LAST solve are kept (bench runs warm-up + timed steps)."""
import collections
import csv
import re
import sys

path = sys.argv[1]
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
r = csv.reader(lines)
h = next(r)
ik, iv, im = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Name')
for row in r:
    if row[im] != 'gpu__time_duration.sum':
        continue
    name = re.sub(r'\(.*', '', row[ik]).replace('bseg::', '')
    name = re.sub(r'<.*>', '<..>', name)
    rows.append((name, float(row[iv].replace(',', ''))))
# split solves at the first kernel of each solve (zaddsub)
starts = [i for i, (n, _) in enumerate(rows) if n.startswith('zaddsub')]
last = rows[starts[-1]:] if starts else rows
unit = 'ns'
tot = sum(v for _, v in last)
agg = collections.defaultdict(lambda: [0, 0.0])
for n, v in last:
    agg[n][0] += 1
    agg[n][1] += v
print(f'launches in the last solve: {len(last)}; summed kernel time {tot / 1e6:.2f} ms '
      f'(cold-cache, serialised by ncu)')
print(f'{"kernel":40s} {"launches":>8s} {"ms":>9s} {"share":>7s}')
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f'{n:40s} {c:8d} {v / 1e6:9.3f} {100 * v / tot:6.1f}%')
