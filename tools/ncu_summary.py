"""Summarise an ncu --set full report: per kernel duration, DRAM bytes, throughputs, occupancy."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "warp_inst",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_cycles_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
}
idx = {h: i for i, h in enumerate(hdr)}
out = []
for r in rows[2:]:
    d = {"kernel": r[idx["Kernel Name"]].split("(")[0].replace("<unnamed>::", "")}
    for k, name in want.items():
        if k in idx:
            v = r[idx[k]].replace(",", "")
            try:
                d[name] = float(v)
            except ValueError:
                d[name] = v
            d[name + "_unit"] = units[idx[k]]
    out.append(d)
for d in out:
    print(json.dumps(d))
