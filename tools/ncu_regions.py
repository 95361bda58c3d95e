"""Per-source-region instruction and stall breakdown of one kernel from an ncu SASS
source page (CSV) and nvdisasm -g of the same cubin.
Usage: python tools/ncu_regions.py SASS CSV KERNEL_SUBSTR file:lo:hi:name ..."""
import collections
import csv
import re
import sys

sass, csvf, kern = sys.argv[1], sys.argv[2], sys.argv[3]
lines = open(sass).read().split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text.") and kern in l][0]
off2line, cur = {}, None
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
ai, ei = h.index("Address"), h.index("Instructions Executed")
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
data = rows[2:]
base = int(data[0][ai], 16)
regions = [(a.split(":")[0], int(a.split(":")[1]), int(a.split(":")[2]), a.split(":")[3]) for a in sys.argv[4:]]


def region(k):
    for f, lo, hi, nm in regions:
        if k[0] == f and lo <= k[1] <= hi:
            return nm
    return "other"


inst = collections.Counter()
st = collections.defaultdict(collections.Counter)
for r in data:
    k = off2line.get(int(r[ai], 16) - base, ("?", 0))
    g = region(k)
    inst[g] += int(r[ei] or 0)
    for c in stall_cols:
        st[g][c] += int(r[h.index(c)] or 0)
te = sum(inst.values())
ts = sum(sum(v.values()) for v in st.values())
print(f"total inst {te/1e6:.1f}M  stall samples {ts}")
for g in [x[3] for x in regions] + ["other"]:
    tot = sum(st[g].values())
    top = ", ".join(f"{c[6:]} {100*v/ts:.1f}" for c, v in st[g].most_common(4) if v)
    print(f"{g:22s} inst {inst[g]/1e6:7.2f}M {100*inst[g]/te:5.1f}%  samples {100*tot/ts:5.1f}%  [{top}]")
