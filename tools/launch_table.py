"""Print kernel name + duration (us) from an ncu --metrics gpu__time_duration.sum --csv log."""
import csv
import sys

for f in sys.argv[1:]:
    print("==", f)
    for r in csv.reader(open(f)):
        if len(r) > 10 and r[-3] == "gpu__time_duration.sum":
            unit = r[-2]
            v = float(r[-1].replace(",", ""))
            us = v / 1e3 if unit == "nsecond" else (v if unit == "usecond" else v * 1e3)
            print(f"  {us:10.1f} us  {r[4][:90]}")
