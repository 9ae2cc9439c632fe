"""Tabulate gpurun_out/sched.log (tools/k7_sched_sweep.sh): ms per 1 GiB transform, one column per schedule."""
import collections
d = collections.defaultdict(dict)
cfgs = []
for l in open('gpurun_out/sched.log'):
    f = l.split()
    if len(f) < 6 or not f[4].startswith('2^'):
        continue
    cfg = '/'.join(f[:3])
    if cfg not in cfgs:
        cfgs.append(cfg)
    d[(f[3], f[4])][cfg] = float(f[5])
print('prec   N     ' + ' '.join(f'{c:>9s}' for c in cfgs))
for k in sorted(d, key=lambda k: (k[0], int(k[1][2:]))):
    print(f"{k[0]:6s} {k[1]:5s} " + ' '.join(f"{d[k].get(c, 0):9.4f}" for c in cfgs))
