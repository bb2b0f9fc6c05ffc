"""Steady-state DRAM traffic per config-4 step from an ncu application-replay CSV of
tools/prof_rsd.py (PF_NF=2: 2 frequencies x all planes; the engine runs 3 times, K1 twice):
  python tools/traffic_summary.py gpurun_out/<dir>/traffic_app.csv > profiles/r2_traffic_steady.json
Per-step figures scale the per-run sums by F / 2 (K1: per launch)."""
import collections
import csv
import json
import re
import sys

path = sys.argv[1]
F, NF, ENGINE_RUNS, K1_RUNS = 32, 2, 3, 2
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
acc = collections.defaultdict(lambda: collections.defaultdict(float))
ids = collections.defaultdict(set)
for r in rows[1:]:
    name = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).replace("void ", "").replace("<unnamed>::", "")
    acc[name][r[ix["Metric Name"]]] += float(r[ix["Metric Value"]].replace(",", ""))
    ids[name].add(r[ix["ID"]])
out = {"source": "ncu --replay-mode application --cache-control none --clock-control none, "
                 "tools/prof_rsd.py (config 4, 2 frequencies x all 256 planes, engine run 3 times, "
                 "K1 run 2 times), kernels serialised by the profiler; per-step figures scale the "
                 "per-run sums by F/2 = 16 (K1: per launch); " + path,
       "kernels": {}}
prop = 0.0
for name, m in acc.items():
    n = len(ids[name])
    k1 = "temporal" in name
    scale = (1.0 / n) if k1 else (F / NF) / ENGINE_RUNS
    d = {"launches_per_step": 1 if k1 else n * scale,
         "dram_read_bytes_per_step": m.get("dram__bytes_read.sum", 0.0) * scale,
         "dram_write_bytes_per_step": m.get("dram__bytes_write.sum", 0.0) * scale,
         "l2_bytes_per_step": m.get("lts__t_bytes.sum", 0.0) * scale,
         "time_ms_per_step_serialised": m.get("gpu__time_duration.sum", 0.0) * scale / 1e6}
    out["kernels"][name] = d
    if re.match(r"k_p(a|b12|c_h)", name):
        prop += d["dram_read_bytes_per_step"] + d["dram_write_bytes_per_step"]
out["propagation_dram_bytes_per_step"] = prop
out["compulsory_bytes_per_step"] = 32 * 512 * 512 * 8 + 256 * 512 * 512 * 8
out["ratio_to_compulsory"] = prop / out["compulsory_bytes_per_step"]
print(json.dumps(out, indent=1))
