"""Summarise an ncu --set full report (one entry per kernel launch) into JSON.
usage: python tools/ncu_summary.py report.ncu-rep out.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_tensor.sum",
        "launch__shared_mem_per_block_dynamic"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
res = []
for r in rows[2:]:
    d = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            v = r[i]
            try:
                v = float(v.replace(",", ""))
            except ValueError:
                pass
            d[k] = v
    d["units"] = {k: units[hdr.index(k)] for k in KEYS if k in hdr}
    res.append(d)
json.dump(res, open(sys.argv[2], "w"), indent=1)
for d in res:
    print(d.get("Kernel Name", "?")[:60], d.get("gpu__time_duration.sum"), d["units"].get("gpu__time_duration.sum"),
          "DRAM r/w", d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum"), d["units"].get("dram__bytes_read.sum"))
