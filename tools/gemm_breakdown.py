"""Join the BSE_GEMM_LOG shape log (stderr of the last solve) with an ncu launch list of the
same command: per-shape GEMM time and achieved TFLOP/s (dev tool).
Usage: python tools/gemm_breakdown.py launches.csv shapes.log"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
r = csv.reader(lines)
h = next(r)
ik, iv, im = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Name')
durs = [float(x[iv].replace(',', '')) for x in r
        if len(x) > iv and x[im] == 'gpu__time_duration.sum' and 'zgemm_dmma' in x[ik]]
shapes = [l.split() for l in open(sys.argv[2]) if l.startswith('zgemm ')]
n = min(len(durs), len(shapes))
durs, shapes = durs[-n:], shapes[-n:]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d, sh in zip(durs, shapes):
    key = ' '.join(sh[1:-2])
    agg[key][0] += 1
    agg[key][1] += d
    agg[key][2] += float(sh[-1])
tot = sum(v[1] for v in agg.values())
print(f'{n} zgemm launches, {tot / 1e6:.2f} ms')
for k, (c, d, gf) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f'{k:50s} x{c:4d} {d / 1e6:8.3f} ms  {gf / (d * 1e-9) / 1e3 if d else 0:6.1f} TF/s')
