import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import synth
from test_gpu_parity import _deep_scene
from gpu_util import torch_scene
from paper_2510_08491_b200 import snp
for nh in (600, 2600):
    scene = _deep_scene(nh)
    cam = synth.look_at((0, 0, 0), (1, 0, 0), 32, 24, 1600.0)
    h = snp.create_scene(torch_scene(scene), 0)
    out = torch.zeros((1, 24, 32, 4), device="cuda")
    snp.render_views(h, [cam], snp.make_opts(), out)
    torch.cuda.synchronize()
    print(nh, "forward ok", snp.get_stats(h)["overflow_pixels"], flush=True)
    snp.destroy(h)
