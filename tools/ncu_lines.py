"""Per-CUDA-source-line warp stall samples from an ncu report (needs -lineinfo).
Usage: python tools/ncu_lines.py report.ncu-rep [top] [--reasons]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 25
reasons = '--reasons' in sys.argv
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
fname = None
hdr = None
agg = []
tot = 0
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == 'File Path':
        fname = row[1].split('/')[-1]
        continue
    if row[0] == 'Function Name':
        continue
    if row[0] == 'Line No':
        hdr = row
        continue
    if hdr and row[0].isdigit() and len(row) > 4 and row[4].isdigit():
        v = int(row[4])
        tot += v
        st = {}
        if reasons:
            for i, h in enumerate(hdr):
                if h.startswith('stall_') and '(Not Issued)' not in h and i < len(row) and row[i].isdigit():
                    if int(row[i]):
                        st[h[6:]] = int(row[i])
        agg.append((v, f'{fname}:{row[0]}', row[1].strip()[:80], st))
agg.sort(key=lambda x: -x[0])
print('total samples', tot)
for v, loc, src, st in agg[:top]:
    extra = ''
    if st:
        extra = '  [' + ', '.join(f'{k}:{100 * c / max(v, 1):.0f}%' for k, c in sorted(st.items(), key=lambda x: -x[1])[:3]) + ']'
    print(f'{100 * v / max(tot, 1):5.1f}%  {loc:18s} {src}{extra}')
