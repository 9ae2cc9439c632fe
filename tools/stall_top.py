"""Top SASS instructions for one stall reason: python tools/stall_top.py <source.csv.gz> <reason> [n]"""
import csv, gzip, sys
f, reason = sys.argv[1], sys.argv[2]
op = gzip.open if f.endswith('.gz') else open
rows = list(csv.reader(op(f, 'rt')))
hdr = rows[1]
col = hdr.index('stall_' + reason)
data = [r for r in rows[2:] if len(r) >= len(hdr)]
tot = sum(float(r[col] or 0) for r in data) or 1
idx = sorted(range(len(data)), key=lambda i: -float(data[i][col] or 0))
for i in idx[:int(sys.argv[3]) if len(sys.argv) > 3 else 15]:
    prev = data[i - 1][1].strip()[:40] if i else ''
    print(f"{100 * float(data[i][col] or 0) / tot:5.1f}%  {data[i][1].strip()[:60]:60s} | prev: {prev}")
