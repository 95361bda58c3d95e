"""Reads the SNP_INSTRUMENT per-warp clock accounting of K5 (A/B tool)."""
import os, sys, types
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2510_08491_b200 import snp
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
scene, cams, bg = synth.make_config(cfg)
ns = types.SimpleNamespace(omega=scene.omega, sh_degree=scene.sh_degree)
for f in snp.FIELDS:
    setattr(ns, f, torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).cuda())
h = snp.create_scene(ns, 0)
out = torch.empty((1, cams[0].height, cams[0].width, 4), device="cuda")
snp.render_views(h, cams, snp.make_opts(bg, sync_check=1), out)
opts = snp.make_opts(bg, sync_check=0)
snp.get_debug_counters(h)   # clears the instrumented slots
snp.render_views(h, cams, opts, out)
torch.cuda.synchronize()
ci = snp.get_debug_counters(h, 48)
c = ci.astype(np.float64)
tot = c[21]
names = {16: "wait", 17: "rounds", 18: "emit", 22: "fill", 23: "pre", 24: "setup", 25: "finish"}
parts = "  ".join("%s %.1f%%" % (nm, 100 * c[k] / tot) for k, nm in names.items())
other = tot - sum(c[k] for k in names)
print(cfg, "consumer-warp cycles:", parts, " other %.1f%%" % (100 * other / tot),
      " rounds=%d avg_lanes=%.1f total=%.3g" % (c[19], c[20] / max(c[19], 1), tot))
print(cfg, "producer: waiting on free slots %.1f%% of its time" % (100 * c[26] / max(c[27], 1)))
print(cfg, "touching (warp, record) pairs %.3g, with no candidate lane %.1f%%; emit calls (lane) %.3g, with empty list %.1f%%" % (
    c[37], 100 * c[38] / max(c[37], 1), c[39], 100 * c[40] / max(c[39], 1)))
print(cfg, "insertion steps per round %.2f" % (c[36] / max(c[19], 1)))
t0 = int(~np.uint64(ci[32])); tmax = int(ci[33]); tmean = int(ci[34]) * 1024.0 / max(int(ci[35]), 1)
print(cfg, "CTA end times after the first start: mean %.1f us, last %.1f us (tail %.1f us)" % (
    (tmean - t0) / 1e3, (tmax - t0) / 1e3, (tmax - tmean) / 1e3))
print(cfg, "insertion share of the rounds %.1f%%" % (100 * c[41] / max(c[17], 1)))
