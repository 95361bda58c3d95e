"""Per-phase CUDA-event breakdown of one Trainer step (forward / loss / backward / Adam)
at a config (default C4, 64 views)."""
import argparse, os, sys, types
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2510_08491_b200 import snp, train

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--views", type=int, default=64)
args = ap.parse_args()
scene, cams, bg = synth.make_config(args.config, views=args.views)
ns = types.SimpleNamespace(omega=scene.omega, sh_degree=scene.sh_degree)
for f in snp.FIELDS:
    setattr(ns, f, torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).cuda())
h = snp.create_scene(ns, 0)
H, W = cams[0].height, cams[0].width
target = torch.rand((len(cams), H, W, 3), device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
tr = train.Trainer(h, scene, len(cams), H, W, "cuda", opts=snp.make_opts(bg))
for _ in range(2):
    tr.step(cams, target)
torch.cuda.synchronize()
res = {k: [] for k in ("forward", "loss", "backward", "adam")}
B = train.CAMERA_BATCH
for _ in range(3):
    tr.flat.zero_(); tr.loss.zero_()
    t = {k: 0.0 for k in res}
    for v0 in range(0, len(cams), B):   # as Trainer.step: one camera batch at a time
        v1 = min(len(cams), v0 + B)
        out, gout = tr.out[v0:v1], tr.gout[v0:v1]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(); snp.render_views(h, cams[v0:v1], tr.opts, out)
        ev[1].record(); snp.loss_3dgs(h, out, target[v0:v1], gout, tr.loss, tr.dssim_lambda, step_views=len(cams))
        ev[2].record(); snp.render_backward(h, tr.opts, gout, tr.grads, fwd_rgba=out)
        ev[3].record(); torch.cuda.synchronize()
        for i, k in enumerate(("forward", "loss", "backward")):
            t[k] += ev[i].elapsed_time(ev[i + 1])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); tr.step_count += 1; snp.adam_step(h, tr.grads, tr.step_count, tr.lr); e1.record()
    torch.cuda.synchronize()
    t["adam"] = e0.elapsed_time(e1)
    for k in res:
        res[k].append(t[k])
print({k: round(float(np.median(v)), 2) for k, v in res.items()}, "ms (record mode:", h is not None, ")")
