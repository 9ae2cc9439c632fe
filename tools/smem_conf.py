"""Shared-memory instructions with excess wavefronts (bank conflicts) from an
`ncu --page source --csv` SASS export."""
import csv, gzip, sys
f = sys.argv[1]
op = gzip.open if f.endswith('.gz') else open
rows = list(csv.reader(op(f, 'rt')))
hdr = rows[1]
ix = {k: hdr.index(k) for k in ('Instructions Executed', 'L1 Wavefronts Shared Excessive', 'L1 Wavefronts Shared',
                                'L1 Wavefronts Shared Ideal', 'Warp Stall Sampling (All Samples)')}
out = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        ex = float(r[ix['L1 Wavefronts Shared Excessive']] or 0)
    except ValueError:
        continue
    if ex > 0:
        out.append((ex, r[0], r[1].strip(), r[ix['Instructions Executed']], r[ix['L1 Wavefronts Shared']],
                    r[ix['L1 Wavefronts Shared Ideal']]))
out.sort(reverse=True)
tot = sum(o[0] for o in out)
print(f'excess wavefronts total {tot:,.0f}')
for o in out[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f'{o[0]:12,.0f}  exec={o[3]:>10} wf={o[4]:>10} ideal={o[5]:>10}  {o[2][:70]}')
