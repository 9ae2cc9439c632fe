"""Summarise an `ncu --page source --csv` export (SASS view): stall totals and top instructions."""
import csv, gzip, sys
f = sys.argv[1]
op = gzip.open if f.endswith('.gz') else open
rows = list(csv.reader(op(f, 'rt')))
hdr = rows[1]
data = rows[2:]
st = [c for c in hdr if c.startswith('stall_') and '(Not Issued)' not in c]
tot = {c: 0 for c in st}
samp_i = hdr.index('Warp Stall Sampling (All Samples)')
lines = []
for r in data:
    if len(r) < len(hdr):
        continue
    for c in st:
        try:
            tot[c] += float(r[hdr.index(c)] or 0)
        except ValueError:
            pass
    try:
        lines.append((float(r[samp_i] or 0), r[1].strip()))
    except ValueError:
        pass
s = sum(tot.values()) or 1
print('stall share:', ', '.join(f'{k[6:]}={100*v/s:.1f}%' for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]))
lines.sort(reverse=True)
tot_s = sum(l[0] for l in lines) or 1
for smp, src in lines[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f'{100*smp/tot_s:5.1f}%  {src}')
