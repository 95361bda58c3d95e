"""Debug: locate GPU-vs-oracle mismatches on a sampled C3 frame."""
import os, sys, types
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth, oracle
from gpu_util import gpu_render, sample_pixels, compare

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
scene, cams, bg = synth.make_config(cfg)
px, py = sample_pixels(cams[0], 2500, 6, seed=7)
out_o, fl, st = oracle.render_pixels(scene, cams[0], px, py, bg)
for lim in (8, 1):
    res = gpu_render(scene, cams, bg, pending_limit=lim)
    g = res["img"][0][py, px]
    err = np.abs(g - out_o).max(1)
    bad = np.nonzero((err > 1e-4) & (fl == 0))[0]
    print(f"SNP_DEBUG={os.environ.get('SNP_DEBUG')} limit={lim} bad={len(bad)} stats={res['stats']}")
    for i in bad[:12]:
        print("  px", px[i], py[i], "tile", px[i] // 16, py[i] // 16, "err", err[i], "gpu", g[i], "orc", out_o[i], "hits", st[i])
