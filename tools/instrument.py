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
snp.render_views(h, cams, opts, out)
torch.cuda.synchronize()
c = snp.get_debug_counters(h).astype(np.float64)
tot = c[21]
print(cfg, "consumer-warp cycles: wait %.1f%%  rounds %.1f%%  emit %.1f%%  fill %.1f%%  pre %.1f%%  other %.1f%%  rounds=%d avg_lanes=%.1f total=%.3g" % (
    100 * c[16] / tot, 100 * c[17] / tot, 100 * c[18] / tot, 100 * c[22] / tot, 100 * c[23] / tot,
    100 * (tot - c[16] - c[17] - c[18] - c[22] - c[23]) / tot, c[19], c[20] / max(c[19], 1), tot))
