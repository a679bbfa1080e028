"""Aggregate ncu warp-stall samples and executed instructions by CUDA source line.
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kern,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
fname = "?"
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            res.append((int(r[4] or 0), int(r[7] or 0), fname, r[0], r[1][:95]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
toti = sum(x[1] for x in res) or 1
print(f"total stall samples {tot}, warp instructions executed {toti}")
for x in sorted(res, reverse=True)[:n]:
    print(f"{x[0]:7d} {100 * x[0] / tot:5.1f}%  inst {100 * x[1] / toti:5.1f}%  {x[2]}:{x[3]} {x[4]}")
