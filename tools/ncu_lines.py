"""Per-CUDA-source-line warp stall samples from an ncu report (needs -lineinfo)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
fname = None
agg = []
tot = 0
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == 'File Path':
        fname = row[1].split('/')[-1]
        continue
    if row[0] in ('Function Name', 'Line No'):
        continue
    if row[0] and row[0].isdigit() and len(row) > 4 and row[4].isdigit():
        v = int(row[4])
        tot += v
        agg.append((v, f'{fname}:{row[0]}', row[1].strip()[:90]))
agg.sort(reverse=True)
print('total samples', tot)
for v, loc, src in agg[:top]:
    print(f'{100 * v / max(tot, 1):5.1f}%  {loc:18s} {src}')
