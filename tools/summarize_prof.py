"""Summarise ncu captures (gpurun_out/prof_*.raw.csv) and the launch list into
a markdown table under profiles/.

    python tools/summarize_prof.py gpurun_out profiles/<tag>.md
"""
import csv
import glob
import os
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "smem/CTA"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem conflicts"),
    ("smsp__inst_executed.sum", "warp instrs"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def main(src, dst):
    out = []
    for f in sorted(glob.glob(os.path.join(src, "prof_*.raw.csv"))):
        rows = list(csv.reader(open(f)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        out.append(f"### {os.path.basename(f)[5:-8]}\n")
        out.append("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
        out.append("|---" * (len(KEYS) + 1) + "|")
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")].split("(")[0]
            vals = []
            for k, _ in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    vals.append(f"{r[i]} {units[i]}".strip())
                else:
                    vals.append("-")
            out.append(f"| `{name}` | " + " | ".join(vals) + " |")
        out.append("")
    lf = os.path.join(src, "launches.csv")
    if os.path.exists(lf):
        lines = [l for l in open(lf) if not l.startswith("==")]
        rows = list(csv.reader(lines))
        if rows:
            hdr = rows[0]
            tot = {}
            for r in rows[1:]:
                try:
                    name = r[hdr.index("Kernel Name")].split("(")[0]
                    if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
                        continue
                    v = float(r[hdr.index("Metric Value")].replace(",", ""))
                    unit = r[hdr.index("Metric Unit")]
                    v = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
                except (ValueError, IndexError):
                    continue
                c, t = tot.get(name, (0, 0.0))
                tot[name] = (c + 1, t + v)
            s = sum(t for _, t in tot.values()) or 1.0
            out.append("### launch list (ncu gpu__time_duration.sum, cold-cache serialised)\n")
            out.append("| kernel | launches | total us | share |")
            out.append("|---|---|---|---|")
            for name, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
                out.append(f"| `{name}` | {c} | {t:.1f} | {100 * t / s:.1f}% |")
    open(dst, "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
