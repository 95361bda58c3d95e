import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth, oracle
from gpu_util import gpu_render
scene, cams, bg = synth.make_config("C3")
cam = cams[0]
x, y = 1241, 693
ids, ti, to = oracle.pixel_hits(scene, cam, x, y)
print("oracle hits", ids, ti)
r, pr, d = oracle.bin_view(scene, cam)
for i in ids:
    print(i, "rect", r[i], "prect", pr[i], "L", d[i:i+1].view(np.float32))
tx, ty = oracle.tiles_of(cam)
k, iv, rg = oracle.bin_sort(r, d, scene.n, 1, tx, ty)
t = (y // 16) * tx + x // 16
lst = iv[rg[t, 0]:rg[t, 1]]
print("tile", t, "range", rg[t], "contains", [int(i) in set(lst.tolist()) for i in ids])
res = gpu_render(scene, cams, bg, binning=True)
rg_g, dg, kg, ig, rng_g = res["binning"]
print("gpu range", rng_g[t], "gpu list contains", [int(i) in set(ig[rng_g[t,0]:rng_g[t,1]].tolist()) for i in ids])
print("gpu px", res["img"][0, y, x])
