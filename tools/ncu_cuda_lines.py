"""Per-CUDA-line stall breakdown from `ncu -i REP --page source --csv --print-source cuda,sass -k K`.
Usage: python tools/ncu_cuda_lines.py CSV [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
cols = {c: h.index(c) for c in ("Warp Stall Sampling (All Samples)", "stall_long_sb", "stall_wait", "stall_lg",
                                "stall_short_sb", "Instructions Executed")}
out, tot = [], 0
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) < len(h) or not r[0].isdigit():
        continue
    v = {c: float(r[i]) if r[i].replace(".", "", 1).isdigit() else 0.0 for c, i in cols.items()}
    tot += v["Warp Stall Sampling (All Samples)"]
    out.append((v["Warp Stall Sampling (All Samples)"], fname, int(r[0]), r[1].strip()[:70], v))
out.sort(key=lambda x: -x[0])
print("total samples", tot)
for s, f, ln, src, v in out[:top]:
    print("%6.1f%% %s:%d lsb=%d wait=%d lg=%d ssb=%d inst=%d  %s" % (100 * s / tot, f, ln, v["stall_long_sb"], v["stall_wait"],
          v["stall_lg"], v["stall_short_sb"], v["Instructions Executed"], src))
