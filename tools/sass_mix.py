"""Instruction mix of an `ncu --page source --csv` SASS export: executed warp
instructions per opcode (top N), so instruction overhead can be attributed."""
import collections, csv, gzip, sys
f = sys.argv[1]
op = gzip.open if f.endswith('.gz') else open
rows = list(csv.reader(op(f, 'rt')))
hdr = rows[1]
ie = hdr.index('Instructions Executed')
cnt = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[1].strip()
    opc = src.split()[0] if src else '?'
    if opc.startswith('@'):
        opc = src.split()[1]
    try:
        cnt[opc.split('.')[0]] += int(r[ie] or 0)
    except ValueError:
        pass
tot = sum(cnt.values()) or 1
print(f'total warp instrs {tot:,}')
for k, v in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f'{k:10s} {v:14,} {100*v/tot:5.1f}%')
