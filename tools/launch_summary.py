"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv
--log-file X.csv) per kernel: launches, total ms (cold-cache, serialised),
share of the listed device time.

    python tools/launch_summary.py gpurun_out/x_launches.csv "header line" > profiles/rNN_x_launches_summary.txt
"""
import csv
import sys
from collections import defaultdict


def main(path, header=""):
    n = defaultdict(int)
    t = defaultdict(float)
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3, "second": 1e3}
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        n[name] += 1
        t[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot = sum(t.values()) or 1.0
    if header:
        print(header)
    for k in sorted(t, key=lambda k: -t[k]):
        print(f"{n[k]:5d} {t[k]:12.3f} ms {100 * t[k] / tot:6.2f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
