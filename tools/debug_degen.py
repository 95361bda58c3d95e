"""Debug: the degenerate-primitives parity case -- worst pixels and their hits."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth, oracle
from gpu_util import gpu_render
rng = np.random.default_rng(11)
base = synth.make_scene(12, 240, box=0.8)
m = base.n
sc = base.subset(np.arange(m))
k = rng.permutation(m)
thin, sheet, zero, opaque = k[:30], k[30:60], k[60:90], k[90:120]
sc.scales[thin] = np.stack([np.full(30, 4e-4), np.full(30, 0.4), np.full(30, 3e-4)], 1).astype(np.float32)
sc.scales[sheet] = np.stack([np.full(30, 0.35), np.full(30, 0.3), np.full(30, 5e-4)], 1).astype(np.float32)
sc.w2[zero] = 0.0
sc.b2[zero] = 0.0
sc.b2[opaque] = (40.0 / sc.scales[opaque].max(1)).astype(np.float32)
big = synth.make_scene(13, 1, box=0.1)
big.centers[:] = 0.0
big.scales[:] = np.float32([[1.1, 0.9, 0.7]])
big.b2[:] = np.float32([0.05])
sc = synth.concat_scenes(sc, big)
kind = {int(i): "thin" for i in thin}
kind.update({int(i): "sheet" for i in sheet}); kind.update({int(i): "zero" for i in zero})
kind.update({int(i): "opaque" for i in opaque}); kind[m] = "big"
variants = {"all": (1.9, 3.3), "noclip": (0.01, 1e4)}
for name, (tn, tf) in variants.items():
    cam = synth.look_at((0.0, -2.6, 0.9), (0.1, 0.0, 0.0), 83, 61, 70.0, fy=55.0, cx=30.3, cy=35.7,
                        t_near=tn, t_far=tf)
    res = gpu_render(sc, [cam], (0.1, 0.2, 0.3))
    img_o, fl, _ = oracle.render_frame(sc, cam, (0.1, 0.2, 0.3))
    err = np.abs(res["img"][0].astype(np.float64) - img_o).max(-1)
    print(name, "max err", err.max(), "n>1e-4", int((err > 1e-4).sum()))
    for idx in np.argsort(err.ravel())[::-1][:4]:
        y, x = divmod(int(idx), cam.width)
        ids, ti, to = oracle.pixel_hits(sc, cam, x, y)
        print("  px", (x, y), "err %.2e" % err[y, x], "gpu", res["img"][0, y, x], "orc", img_o[y, x])
        for i, a, b in list(zip(ids, ti, to))[:8]:
            print("     hit", int(i), kind.get(int(i), "-"), "t_in %.6f t_out %.6f" % (a, b))
