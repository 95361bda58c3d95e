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
tot = c[28:32].sum()
print(cfg, "k_pass CTA cycles (sum over CTAs): start+load %.1f%% rank %.1f%% lookback %.1f%% scan+scatter %.1f%%  mean per CTA %.0f cycles" % tuple(
    [100 * c[28 + i] / tot for i in range(4)] + [tot / (4 * (int(snp.get_stats(h)['n_dup']) + 3071) // 3072)]))
