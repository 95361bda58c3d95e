"""One small render (and a backward pass) of the hot path for compute-sanitizer runs:
  python tools/sanitize_run.py c1|c2|deep|graze
c1: config C1 (128x128, 256 primitives), forward + backward; c2: a C2-shaped frame
(3000 primitives, 400x400, white background); deep: 2600 overlapping primitives per
ray with a pending limit of 1 (every pixel through K6w -> the block-wide K6);
graze: dense primitives seen at grazing incidence (K5 hands pixels to K6w)."""
import os
import sys
import types

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2510_08491_b200 import snp  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c1"
limit = 0
if which == "c1":
    scene, cams, bg = synth.make_config("C1")
elif which == "c2":
    scene = synth.make_scene(1, 3000, scale_mult=1.5, box=1.0)
    cams, bg = synth.orbit_cameras(1, 4.0, 400, 400, 555.0), (1.0, 1.0, 1.0)
elif which == "deep":
    n = 2600
    scene = synth.make_scene(21, n, box=0.3)
    i = np.arange(n)
    scene.centers[:] = np.stack([5.0 + 0.01 * i, np.zeros(n), np.zeros(n)], 1).astype(np.float32)
    r = 1.2 + 0.035 * (i % 4)
    scene.scales[:] = np.stack([r, r, r], 1).astype(np.float32)
    scene.w2 *= np.float32(1e-4)
    scene.b2[:] = np.float32(3e-4)
    cams, bg, limit = [synth.look_at((0, 0, 0), (1, 0, 0), 32, 24, 1600.0)], (0, 0, 0), 1
else:
    rng = np.random.default_rng(31)
    scene = synth.make_scene(32, 150, box=0.6)
    scene.centers[:] = rng.uniform(-0.4, 0.4, (150, 3)).astype(np.float32)
    scene.scales[:] = rng.uniform(0.04, 0.1, (150, 3)).astype(np.float32)
    scene.w2[:] = 0.0
    scene.b2[:] = (50.0 / scene.scales.max(1)).astype(np.float32)
    cams, bg = [synth.look_at((0.3, -3.0, 0.4), (0.0, 0.0, 0.0), 160, 120, 600.0)], (0, 0, 0)
ns = types.SimpleNamespace(omega=scene.omega, sh_degree=scene.sh_degree)
for f in snp.FIELDS:
    setattr(ns, f, torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).cuda())
h = snp.create_scene(ns, 0)
if limit:
    snp.set_pending_limit(h, limit)
out = torch.empty((len(cams), cams[0].height, cams[0].width, 4), device="cuda")
snp.render_views(h, cams, snp.make_opts(bg, sync_check=1), out)
snp.render_views(h, cams, snp.make_opts(bg, sync_check=0), out)
if which == "c1":
    grads = {f: torch.zeros_like(getattr(ns, f)) for f in snp.FIELDS}
    snp.render_backward(h, snp.make_opts(bg), torch.ones_like(out), grads)
torch.cuda.synchronize()
print(which, snp.get_stats(h), "finite:", bool(torch.isfinite(out).all()))
snp.destroy(h)
