"""Profiling driver: a few non-graph frames of one config (default C3) so that
ncu sees every kernel launch of the hot path individually."""
import argparse
import os
import sys
import types

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2510_08491_b200 import snp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--frames", type=int, default=3)
ap.add_argument("--views", type=int, default=0)
args = ap.parse_args()

scene, cams, bg = synth.make_config(args.config, views=args.views or None)
ns = types.SimpleNamespace(omega=scene.omega, sh_degree=scene.sh_degree)
for f in snp.FIELDS:
    setattr(ns, f, torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).cuda())
h = snp.create_scene(ns, 0)
out = torch.empty((len(cams), cams[0].height, cams[0].width, 4), device="cuda")
snp.render_views(h, cams, snp.make_opts(bg, sync_check=1), out)
torch.cuda.synchronize()
opts = snp.make_opts(bg, sync_check=0)
for _ in range(args.frames):
    snp.render_views(h, cams, opts, out)
torch.cuda.synchronize()
print(snp.get_stats(h))
snp.destroy(h)
