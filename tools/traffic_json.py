"""profiles/traffic.json: DRAM bytes (read + write) per launch of the C2 kernels,
from ncu --set full captures (gpurun_out/prof_<tag>_fp64_n<N>.raw.csv, 1 GiB
input = the bench's per-N workload). bench.py reports it as roofline.traffic."""
import csv, glob, json, os, re, sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic.json"
out = json.load(open(dst)) if os.path.exists(dst) else {}
names = {"1m": 1 << 20, "256k": 1 << 18}
for f in glob.glob(os.path.join(src, "prof_k*_fp64_n*.raw.csv")):
    m = re.search(r"prof_(k\d)_fp64_n(\w+)\.raw\.csv", f)
    if not m:
        continue
    n = names.get(m.group(2)) or int(m.group(2))
    rows = list(csv.reader(open(f)))
    hdr, units = rows[0], rows[1]
    tot = 0.0
    for r in rows[2:]:
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            v = float(r[i])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[i], 1)
            tot += v * scale
    out[str(n)] = {"bytes": round(tot), "kernel": m.group(1), "source": os.path.basename(f)}
json.dump(out, open(dst, "w"), indent=1, sort_keys=True)
print(json.dumps(out, indent=1))
