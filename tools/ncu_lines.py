"""Aggregate an ncu --page source --csv (cuda,sass) dump per source line: instructions and stall samples."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
cur_file, hdr, out = None, None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    try:
        inst = int(r[hdr.index("Instructions Executed")] or 0)
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    stalls = {h: int(v) for h, v in zip(hdr, r) if h.startswith("stall_") and "Not Issued" not in h
              and v.isdigit() and int(v) > 0}
    top_st = sorted(stalls.items(), key=lambda x: -x[1])[:3]
    out.append((samp, inst, f"{cur_file}:{r[0]}", r[1].strip()[:70], top_st))
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"total samples {tot_s}  instructions {tot_i}")
for s, i, loc, src, st in sorted(out, key=lambda x: -x[0])[:top]:
    print(f"{s/tot_s*100:5.1f}%smp {i/tot_i*100:5.1f}%ins {loc:26s} {src:70s} {st}")
