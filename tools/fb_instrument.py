"""Reads the SNP_INSTRUMENT phase accounting of K6 (A/B tool)."""
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
c0 = snp.get_debug_counters(h).astype(np.float64)
snp.render_views(h, cams, snp.make_opts(bg, sync_check=0), out)
torch.cuda.synchronize()
c = snp.get_debug_counters(h).astype(np.float64)
ov = snp.get_stats(h)["overflow_pixels"]
raw = int(c[31])
nh, nl = raw & 0xffffffff, raw >> 32
print(cfg, "K6 pixels %d: phaseA %.0f cyc/px, sort %.0f cyc/px, selection-path px %d, hits/px %.1f, list/px %.1f" % (
    ov, c[28] / max(ov, 1), c[29] / max(ov, 1), c[30], nh / max(ov, 1), nl / max(ov, 1)))
