"""Aggregate an ncu SASS source-page CSV by CUDA source line (via nvdisasm -g)."""
import csv, re, sys, collections
sass, csvf, kern = sys.argv[1], sys.argv[2], sys.argv[3]
lines = open(sass).read().split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text.") and kern in l][0]
off2line = {}
cur = None
for l in lines[start:]:
    if l.startswith("//---") and kern not in l and off2line:
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
h = rows[1]
ai, ei, si = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = rows[2:]
base = int(data[0][ai], 16)
agg = collections.defaultdict(lambda: [0, 0])
tot_e = tot_s = 0
for r in data:
    off = int(r[ai], 16) - base
    e, s = int(r[ei] or 0), int(r[si] or 0)
    agg[off2line.get(off, ("?", 0))][0] += e
    agg[off2line.get(off, ("?", 0))][1] += s
    tot_e += e; tot_s += s
src = {}
for k, (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:45]:
    print(f"{k[0]}:{k[1]:5d}  inst {e/1e6:8.2f}M ({100*e/tot_e:5.1f}%)  stall-samples {100*s/max(tot_s,1):5.1f}%")
print("total inst", tot_e / 1e6, "M")
