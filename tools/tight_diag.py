"""Tight binning diagnostics: frame differences against the rect binning (per config)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth
from test_gpu_parity import _render_with_binning
for cfg in sys.argv[1:] or ["C2"]:
    scene, cams, bg = synth.make_config(cfg)
    ref, st0 = _render_with_binning(scene, cams, bg, 0)
    for f in (1, 3):
        out, st = _render_with_binning(scene, cams, bg, f)
        d = np.abs(out - ref).max(-1)
        bad = np.argwhere(d > 0)
        print(cfg, "flags", f, "max diff %.3g" % d.max(), "pixels differing", len(bad), ">1e-6:", int((d > 1e-6).sum()),
              ">1e-4:", int((d > 1e-4).sum()), "overflow", st0["overflow_pixels"], st["overflow_pixels"],
              "first", bad[:5].tolist())
