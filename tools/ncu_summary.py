"""Summarise an ncu report: key throughput metrics + top stall instructions (dev tool)."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ('Duration', 'DRAM Throughput', 'Memory Throughput', 'L2 Cache Throughput',
        'Compute (SM) Throughput', 'Registers Per Thread', 'Achieved Occupancy', 'Grid Size',
        'Block Size', 'L2 Hit Rate', 'Warp Cycles Per Issued Instruction', 'Issue Slots Busy',
        'DRAM Frequency', 'SM Frequency')


def details(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True,
                         text=True).stdout
    r = csv.reader(io.StringIO(out))
    h = next(r)
    res = collections.OrderedDict()
    for row in r:
        d = dict(zip(h, row))
        k = (d.get('Kernel Name', '')[:40], d['Metric Name'])
        if d['Metric Name'] in KEYS:
            res[k] = f"{d['Metric Value']} {d['Metric Unit']}"
    return res


def raw(rep, names):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(h, row))
        res.append({n: d.get(n) for n in names if n in d})
    return res


def stalls(rep, top=15):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    start = 2 if rows and rows[0] and rows[0][0] == 'Kernel Name' else 1
    h = rows[start - 1]
    if 'Warp Stall Sampling (All Samples)' not in h:
        return []
    i_s, i_src = h.index('Warp Stall Sampling (All Samples)'), h.index('Source')
    body = rows[start:]
    tot = sum(int(r[i_s]) for r in body if r[i_s].isdigit())
    items = sorted(((int(r[i_s]), k) for k, r in enumerate(body) if r[i_s].isdigit()), reverse=True)
    res = []
    for v, k in items[:top]:
        prev = ' | '.join(body[j][i_src].strip()[:40] for j in range(max(0, k - 2), k))
        res.append(f"{100 * v / tot:5.1f}%  {body[k][i_src].strip()[:60]:60s}  <- {prev}")
    return res


if __name__ == '__main__':
    for rep in sys.argv[1:]:
        print('==', rep)
        for k, v in details(rep).items():
            print(f'  {k[1]:40s} {v}')
        for r in raw(rep, ['dram__bytes_read.sum', 'dram__bytes_write.sum',
                           'lts__t_bytes.sum', 'gpu__time_duration.sum']):
            print('  ', r)
        for s in stalls(rep):
            print('  ', s)
