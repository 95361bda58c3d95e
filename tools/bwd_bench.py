"""Times K7 (snp_render_backward) on a config: forward frame, then the backward for a
random dL/d(out) (CUDA events, median of N)."""
import argparse, os, statistics, sys, types
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2510_08491_b200 import snp
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--record", action="store_true", help="snp_set_record: backward from the forward's recorded hits")
args = ap.parse_args()
scene, cams, bg = synth.make_config(args.config)
ns = types.SimpleNamespace(omega=scene.omega, sh_degree=scene.sh_degree)
for f in snp.FIELDS:
    setattr(ns, f, torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).cuda())
h = snp.create_scene(ns, 0)
if args.record:
    snp.set_record(h, True)
V, H, W = len(cams), cams[0].height, cams[0].width
out = torch.empty((V, H, W, 4), device="cuda")
opts = snp.make_opts(bg)
snp.render_views(h, cams, opts, out)
G = torch.randn((V, H, W, 4), device="cuda")
grads = {f: torch.zeros(getattr(scene, f).shape, device="cuda")
         for f in ("w1", "b1", "w2", "b2", "sh", "centers", "rotations", "scales")}
ts = []
for _ in range(args.iters):
    for v in grads.values():
        v.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); snp.render_backward(h, opts, G, grads, fwd_rgba=out); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
st = snp.get_stats(h)
skipped = int(snp.get_stats(h)["backward_skipped"])
print(args.config, "legacy" if os.environ.get("SNP_BWD_LEGACY") else ("recorded" if args.record else "k5-path"), "backward us median %.1f (forward render stage for comparison: see stage_bench)" % statistics.median(ts),
      "composited", st["composited"], "skipped pixels", skipped)
snp.destroy(h)
