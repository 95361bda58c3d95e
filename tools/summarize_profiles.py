"""Writes the judged profile summaries under profiles/ from a tools/profile_round.sh run.

usage: python tools/summarize_profiles.py [round_tag]   (default r01; reads gpurun_out/<tag>_*)
Runs here (no GPU): it only parses the CSV launch list and `ncu -i` of the .ncu-rep.
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")

# ---- launch list (one prof_step run: a sizing frame + 3 timed-shape frames)
rows = [r for r in csv.reader(open(os.path.join(src, f"{tag}_launches.csv"))) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    k = r[ki].split("(")[0].split("::")[-1].strip()
    agg.setdefault(k, []).append(float(r[vi].replace(",", "")))
frames = max(1, len(next((v for k, v in agg.items() if k.startswith("k_render")), [1])))
shutil.copy(os.path.join(src, f"{tag}_launches.csv"), os.path.join(dst, f"{tag}_launches_c3.csv"))
tot = sum(sum(v) for k, v in agg.items() if k != "k_validate") / frames
out = [f"# Round {tag[1:]} -- kernel launch list of one C3 frame (ncu gpu__time_duration, --clock-control none)", "",
       f"Source: `profiles/{tag}_launches_c3.csv` (`ncu --metrics gpu__time_duration.sum --clock-control none --csv "
       "python tools/prof_step.py`), averaged over the profiled frames.",
       "Cold-cache, serialised launches (K1b normally overlaps K2-K4 on its side stream): use the SHARES; "
       "live in-graph timings are in bench.py `stages_ms`.", "",
       "| kernel | launches / frame | ns / frame | share |", "|---|---|---|---|"]
for k, v in agg.items():
    if k == "k_validate":
        continue
    ns = sum(v) / frames
    out.append(f"| {k} | {len(v) / frames:g} | {ns:.0f} | {100 * ns / tot:.1f}% |")
out.append(f"| total | | {tot:.0f} | 100% |")
open(os.path.join(dst, f"{tag}_launch_summary.md"), "w").write("\n".join(out) + "\n")

# ---- K5 full capture
rep = os.path.join(src, f"{tag}_k_render.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hh, units, vals = r[0], r[1], r[2]
get = lambda m: (float(vals[hh.index(m)].replace(",", "")), units[hh.index(m)]) if m in hh else (None, "")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second"]
lines = [f"# Round {tag[1:]} -- k_render (K5) ncu --set full capture, C3 (300k primitives, 1245x825)", "",
         "Command: `ncu --set full --clock-control none --import-source on -k regex:k_render -s 1 -c 1 "
         "python tools/prof_step.py` (cold caches, serialised; compare shares, not absolutes).", "",
         "| metric | value | unit |", "|---|---|---|"]
for m in want:
    v, u = get(m)
    if v is not None:
        lines.append(f"| {m} | {v:g} | {u} |")
rd, ru = get("dram__bytes_read.sum")
wr, wu = get("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
traffic = rd * scale.get(ru, 1) + wr * scale.get(wu, 1)
lines.append(f"| DRAM traffic (read+write) | {traffic:.4g} | bytes |")
stalls = []
for i, m in enumerate(hh):
    if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio"):
        try:
            stalls.append((float(vals[i]), m[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
lines += ["", "Issue-stall reasons (warps per issue-active cycle):", ""]
lines += [f"- {n}: {v:.2f}" for v, n in sorted(stalls, reverse=True)[:10]]
open(os.path.join(dst, f"{tag}_k_render_summary.md"), "w").write("\n".join(lines) + "\n")
json.dump({"kernel": "k_render", "config": "C3", "bytes_per_launch": traffic,
           "source": f"profiles/{tag}_k_render_summary.md (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)"},
          open(os.path.join(dst, "render_traffic_bytes.json"), "w"), indent=1)
# ---- every kernel of one frame: DRAM traffic and duration (cold, serialised)
km = os.path.join(src, f"{tag}_kernel_metrics.csv")
if os.path.exists(km):
    rows = [r for r in csv.reader(open(km)) if len(r) > 10]
    h = rows[0]
    ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    idi = h.index("ID")
    per = collections.OrderedDict()
    for r in rows[1:]:
        key = (r[idi], r[ki].split("(")[0].split("::")[-1].strip())
        v = float(r[vi].replace(",", ""))
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
              "nsecond": 1e-9, "msecond": 1e-3}.get(r[ui], 1)
        per.setdefault(key, {})[r[mi]] = v
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks.get("hbm_gbs", 6536.0))
    lines = [f"# Round {tag[1:]} -- DRAM traffic and duration of every kernel of one C3 frame", "",
             "Command: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
             "smsp__issue_active...,sm__warps_active... --clock-control none --csv python tools/prof_step.py "
             "--frames 1` (the last profiled frame; cold caches, serialised).",
             f"HBM peak = {hbm:.0f} GB/s (MEASURED_PEAKS.json).  Only K1a/K1b move enough bytes to approach it;",
             "K2-K4 are latency-bound (short chains of dependent partitions), K5 is ALU/latency-bound (bench.py roofline).", "",
             "| kernel | µs | DRAM read MB | DRAM write MB | GB/s | frac of HBM peak | issue active % | warps active % |",
             "|---|---|---|---|---|---|---|---|"]
    ids = sorted({k[0] for k in per}, key=lambda x: int(x))
    last = {}
    for i in ids:
        for (id_, name), m in per.items():
            if id_ == i:
                last.setdefault(name, []).append(m)
    for name, ms in last.items():
        m = ms[-1]
        t = m.get("gpu__time_duration.sum", 0.0)
        rd = m.get("dram__bytes_read.sum", 0.0)
        wr = m.get("dram__bytes_write.sum", 0.0)
        bw = (rd + wr) / t / 1e9 if t else 0.0
        lines.append(f"| {name} | {t * 1e6:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {bw:.0f} | {bw / hbm:.2f} | "
                     f"{m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.0f} | "
                     f"{m.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.0f} |")
    open(os.path.join(dst, f"{tag}_kernel_rooflines.md"), "w").write("\n".join(lines) + "\n")
    print("wrote", f"{tag}_kernel_rooflines.md")
for f in (f"{tag}_bench.json", f"{tag}_reference.json"):
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f))
print("wrote", f"{tag}_launch_summary.md", f"{tag}_k_render_summary.md", "render_traffic_bytes.json")
