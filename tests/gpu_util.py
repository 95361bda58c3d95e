"""Helpers for the -m gpu parity tests: run the CUDA path through the C ABI."""
import types

import numpy as np

TOL = 1e-4   # BASELINE north_star: within 1e-4 absolute per RGB/opacity channel


def torch_scene(scene):
    import torch
    ns = types.SimpleNamespace(omega=scene.omega, sh_degree=scene.sh_degree)
    for f in ("centers", "rotations", "scales", "w1", "b1", "w2", "b2", "sh"):
        setattr(ns, f, torch.from_numpy(np.ascontiguousarray(getattr(scene, f), np.float32)).cuda())
    return ns


def gpu_render(scene, cams, bg=(0.0, 0.0, 0.0), t_floor=1e-4, stripe=(0, 1), pending_limit=0,
               device_scene=True, host_out=False, binning=False, sync_check=1, repeat=1, colour_mode=0):
    import torch
    from paper_2510_08491_b200 import snp
    src = torch_scene(scene) if device_scene else scene
    h = snp.create_scene(src, 0)
    try:
        if pending_limit:
            snp.set_pending_limit(h, pending_limit)
        V, H, W = len(cams), int(cams[0].height), int(cams[0].width)
        mem = snp.SNP_MEM_HOST if host_out else snp.SNP_MEM_DEVICE
        first = snp.make_opts(bg, t_floor, stripe[0], stripe[1], mem, 1, colour_mode)   # sizes the key buffer
        opts = snp.make_opts(bg, t_floor, stripe[0], stripe[1], mem, sync_check, colour_mode)
        if host_out:
            out = np.full((V, H, W, 4), np.nan, np.float32)
        else:
            out = torch.full((V, H, W, 4), float("nan"), device="cuda")
        for r in range(repeat):
            snp.render_views(h, cams, first if r == 0 else opts, out)
        torch.cuda.synchronize()
        stats = snp.get_stats(h)
        res = dict(img=out if host_out else out.cpu().numpy(), stats=stats)
        if binning:
            tiles = ((W + 15) // 16) * ((H + 15) // 16)
            res["binning"] = snp.get_binning(h, scene.n, V, tiles)
        return res
    finally:
        snp.destroy(h)


def compare(gpu_px, orc_px, flags, tol=TOL):
    """gpu_px [N,4] f32, orc_px [N,4] f64, flags [N]: max error over unflagged pixels."""
    err = np.abs(gpu_px.astype(np.float64) - orc_px).max(axis=1)
    ok = flags == 0
    return dict(max_unflagged=float(err[ok].max()) if ok.any() else 0.0,
                max_all=float(err.max()) if len(err) else 0.0,
                n_flagged=int((~ok).sum()), n=len(err),
                n_bad=int((err[ok] > tol).sum()))


def sample_pixels(cam, n_random, n_tiles, seed):
    rng = np.random.default_rng(seed)
    W, H = int(cam.width), int(cam.height)
    xs = list(rng.integers(0, W, n_random))
    ys = list(rng.integers(0, H, n_random))
    tx, ty = (W + 15) // 16, (H + 15) // 16
    for t in rng.choice(tx * ty, n_tiles, replace=False):
        x0, y0 = (t % tx) * 16, (t // tx) * 16
        for y in range(y0, min(y0 + 16, H)):
            for x in range(x0, min(x0 + 16, W)):
                xs.append(x)
                ys.append(y)
    return np.array(xs, np.int32), np.array(ys, np.int32)
