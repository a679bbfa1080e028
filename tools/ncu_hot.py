"""Summarise an ncu report: top SASS instructions by warp-stall samples for one kernel.
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kern,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
hdr = rows[hi]
si, wi = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
ai = hdr.index("Address")
data = []
for k, r in enumerate(rows[hi + 1:]):
    try:
        data.append((int(r[wi]), k, r[ai], r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot}, instructions {len(data)}")
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0]:7d} {100 * d[0] / tot:5.1f}%  #{d[1]:5d} {d[3][:100]}")
