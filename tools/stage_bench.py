"""Times each stage (project / bin_sort / render) with CUDA events, median of N."""
import argparse, os, statistics, sys, types
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2510_08491_b200 import snp
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--views", type=int, default=0)
ap.add_argument("--plimit", type=int, default=0)
ap.add_argument("--n-hidden", type=int, default=8)
ap.add_argument("--bin-flags", type=int, default=0)   # snp_set_binning (tight binning, 8(f)3)
args = ap.parse_args()
scene, cams, bg = synth.make_config(args.config, views=args.views or None, n_hidden=args.n_hidden)
ns = types.SimpleNamespace(omega=scene.omega, sh_degree=scene.sh_degree)
for f in snp.FIELDS:
    setattr(ns, f, torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).cuda())
h = snp.create_scene(ns, 0)
if args.plimit:
    snp.set_pending_limit(h, args.plimit)
if args.bin_flags:
    snp.set_binning(h, args.bin_flags)
out = torch.empty((len(cams), cams[0].height, cams[0].width, 4), device="cuda")
snp.render_views(h, cams, snp.make_opts(bg, sync_check=1), out)
opts = snp.make_opts(bg, sync_check=0)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
cc = snp.make_cameras(cams)
t = {"project": [], "bin_sort": [], "render": []}
for _ in range(args.iters):
    flush.zero_()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(); snp.project(h, cc); e[1].record(); snp.bin_sort(h, opts); e[2].record(); snp.render(h, opts, out); e[3].record()
    torch.cuda.synchronize()
    for k, (a, b) in zip(t, zip(e[:-1], e[1:])):
        t[k].append(a.elapsed_time(b) * 1e3)
print(args.config, {k: round(statistics.median(v), 1) for k, v in t.items()}, "us", snp.get_stats(h))
