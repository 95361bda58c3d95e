"""Reads the SNP_SORT_INSTRUMENT accounting of K3 (A/B tool): per pass the wall span
(first CTA start -> last partition end, %globaltimer ns) and the phase split summed over
partitions."""
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
opts = snp.make_opts(bg, sync_check=1)
cc = snp.make_cameras(cams)
for it in range(3):
    if it == 2:
        snp.get_debug_counters(h)   # clears the instrumented slots
    snp.project(h, cc)
    snp.bin_sort(h, opts)
    torch.cuda.synchronize()
c = snp.get_debug_counters(h)
spans = []
for p in range(4):
    t0 = (~np.uint64(c[16 + 3 * p])) if c[16 + 3 * p] else 0
    spans.append((int(c[17 + 3 * p]) - int(t0)) / 1e3 if c[16 + 3 * p] else 0.0)
starts = [int(~np.uint64(c[16 + 3 * p])) for p in range(4)]
gaps = [(starts[p + 1] - int(c[17 + 3 * p])) / 1e3 for p in range(3)]
tot = float(sum(c[28:32]))
print(cfg, "k_pass spans us", [round(x, 2) for x in spans], "gaps us", [round(x, 2) for x in gaps],
      "phase split: load %.0f%% rank %.0f%% lookback %.0f%% scan+scatter %.0f%%" % tuple(100 * c[28 + i] / tot for i in range(4)))
