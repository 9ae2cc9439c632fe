"""Tabulate gpurun_out/abi.log (tools/ab_interleave.sh): min ms over rounds per lib."""
import collections
d = collections.defaultdict(lambda: collections.defaultdict(list))
libs = []
for l in open('gpurun_out/abi.log'):
    f = l.split()
    if len(f) < 5 or not f[3].startswith('2^'):
        continue
    if f[0] not in libs:
        libs.append(f[0])
    d[(f[2], f[3])][f[0]].append(float(f[4]))
print('prec   N     ' + ' '.join(f'{c:>16s}' for c in libs))
for k in sorted(d, key=lambda k: (k[0], int(k[1][2:]))):
    print(f"{k[0]:6s} {k[1]:5s} " + ' '.join(
        f"{min(d[k][c]):8.4f}/{max(d[k][c]):7.4f}" if d[k][c] else ' ' * 16 for c in libs))
