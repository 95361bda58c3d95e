"""GPU (sm_100a) parity against the CPU oracle, through the C ABI.

Bars (BASELINE north_star): bit-exact tile assignment, depth keys, sort order
and tile ranges; within 1e-4 absolute per RGB/opacity channel on rendered
pixels (on pixels the oracle does not flag as near-tie / grazing / T-floor
ambiguous, R23; the flagged count is bounded and reported)."""
import numpy as np
import pytest

import synth
from gpu_util import TOL, compare, gpu_render, sample_pixels

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_08491_b200 import build
    build.build()


def _check_binning(orc, scene, cams, res, stripe=(0, 1)):
    rects_g, depth_g, keys_g, ids_g, ranges_g = res["binning"]
    rs, ds = [], []
    for c in cams:
        r, _, d = orc.bin_view(scene, c)
        rs.append(r); ds.append(d)
    rects_o, depth_o = np.concatenate(rs), np.concatenate(ds)
    assert np.array_equal(rects_g, rects_o), np.argwhere((rects_g != rects_o).any(1))[:5]
    vis = rects_o[:, 0] >= 0
    assert np.array_equal(depth_g[vis], depth_o[vis])
    tx, ty = orc.tiles_of(cams[0])
    k, i, rg = orc.bin_sort(rects_o, depth_o, scene.n, len(cams), tx, ty, *stripe)
    assert len(keys_g) == len(k)
    assert np.array_equal(keys_g, k) and np.array_equal(ids_g, i)
    assert np.array_equal(ranges_g, rg)


@pytest.mark.parametrize("cfg,views", [("C1", 1), ("C2", 1), ("C3", 1), ("C1", 3), ("C5", 1)])
def test_binning_bit_exact(orc, cfg, views):
    scene, cams, bg = synth.make_config(cfg)
    if views > 1:
        c = cams[0]
        cams = synth.orbit_cameras(views, 4.0, c.width, c.height, c.fx, elev_deg=(10, 35))
    res = gpu_render(scene, cams, bg, binning=True)
    _check_binning(orc, scene, cams, res)


@pytest.mark.parametrize("stripe", [(1, 2), (0, 3), (2, 3)])
def test_binning_stripes_bit_exact(orc, stripe):
    scene, cams, bg = synth.make_config("C2")
    res = gpu_render(scene, cams, bg, binning=True, stripe=stripe)
    _check_binning(orc, scene, cams, res, stripe)


@pytest.mark.parametrize("variant", ["trained", "paper"])
def test_render_full_frame_C1(orc, variant):
    scene, cams, bg = synth.make_config("C1", variant=variant)
    res = gpu_render(scene, cams, bg)
    img_o, fl, _ = orc.render_frame(scene, cams[0], bg)
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    print(variant, c, res["stats"])
    assert c["max_unflagged"] <= TOL, c
    assert c["n_flagged"] <= 0.005 * c["n"]


@pytest.mark.parametrize("cfg,n_rand,n_tiles", [("C2", 3000, 6), ("C3", 2500, 6), ("C5", 600, 2)])
def test_render_sampled_full_size(orc, cfg, n_rand, n_tiles):
    """Full BASELINE sizes, in the launch configuration bench.py times
    (device-resident scene, no-sync binning after a sizing call)."""
    scene, cams, bg = synth.make_config(cfg)
    res = gpu_render(scene, cams, bg, sync_check=0, repeat=2)
    assert res["stats"]["capacity_overflow"] == 0
    px, py = sample_pixels(cams[0], n_rand, n_tiles, seed=7)
    out_o, fl, _ = orc.render_pixels(scene, cams[0], px, py, bg)
    g = res["img"][0][py, px]
    c = compare(g, out_o, fl)
    print(cfg, c, res["stats"])
    assert c["max_unflagged"] <= TOL, c
    assert c["n_flagged"] <= 0.02 * c["n"]


def test_multiview_batch_C4(orc):
    """C4 (64 orbit views in one call, two camera batches): every view, 150 random pixels
    plus one full tile each (9,984 + 64 x 256 pixels) against the oracle."""
    scene, cams, bg = synth.make_config("C4")
    res = gpu_render(scene, cams, bg)
    worst, flagged, n = 0.0, 0, 0
    for v in range(len(cams)):
        px, py = sample_pixels(cams[v], 150, 1, seed=v)
        out_o, fl, _ = orc.render_pixels(scene, cams[v], px, py, bg)
        c = compare(res["img"][v][py, px], out_o, fl)
        assert c["max_unflagged"] <= TOL, (v, c)
        worst, flagged, n = max(worst, c["max_unflagged"]), flagged + c["n_flagged"], n + c["n"]
    print("C4 all views:", worst, flagged, n)
    assert flagged <= 0.005 * n


def test_multiview_equals_single_view():
    """Batching views (view id in the key's top bits) changes nothing per view."""
    scene, cams, bg = synth.make_config("C2", n=3000)
    cams = synth.orbit_cameras(4, 4.0, 200, 120, 280.0)
    batch = gpu_render(scene, cams, bg)["img"]
    for v in range(4):
        one = gpu_render(scene, [cams[v]], bg)["img"][0]
        assert np.array_equal(batch[v], one)


@pytest.mark.parametrize("limit", [1, 2, 3])
def test_pending_overflow_fallback_exact(orc, limit):
    """Force the per-pixel pending buffer to overflow: K6 must keep parity."""
    scene, cams, bg = synth.make_config("C1")
    res = gpu_render(scene, cams, bg, pending_limit=limit)
    assert res["stats"]["overflow_pixels"] > 0
    img_o, fl, _ = orc.render_frame(scene, cams[0], bg)
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    assert c["max_unflagged"] <= TOL, c


def test_empty_scene_and_ragged_image(orc):
    cam = synth.orbit_cameras(1, 4.0, 37, 23, 40.0)[0]
    res = gpu_render(synth.empty_scene(), [cam], (0.2, 0.3, 0.4))
    img = res["img"][0]
    assert np.allclose(img[..., :3], np.float32([0.2, 0.3, 0.4])) and np.all(img[..., 3] == 0)
    scene = synth.make_scene(3, 300, box=0.7)
    res = gpu_render(scene, [cam], (0.2, 0.3, 0.4))
    img_o, fl, _ = orc.render_frame(scene, cam, (0.2, 0.3, 0.4))
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    assert c["max_unflagged"] <= TOL and not np.isnan(res["img"]).any()


def test_floor_zero_and_sh_degrees(orc):
    scene, cams, bg = synth.make_config("C1")
    for deg in (0, 1, 2, 3):
        scene.sh_degree = deg
        for fl_ in (0.0, 1e-4, 0.05):
            res = gpu_render(scene, cams, bg, t_floor=fl_)
            img_o, fl, _ = orc.render_frame(scene, cams[0], bg, t_floor=fl_)
            c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
            assert c["max_unflagged"] <= TOL, (deg, fl_, c)


def test_camera_inside_and_straddling_primitives(orc):
    """Camera inside big ellipsoids (t_in clipped to t_near) and primitives
    straddling the camera plane (full-image bbox, no conic pre-test)."""
    rng = np.random.default_rng(5)
    scene = synth.make_scene(6, 200, box=0.7)
    cam = synth.orbit_cameras(1, 2.0, 64, 48, 50.0)[0]
    big = synth.make_scene(7, 6, box=0.1, rmin=0.1, rmax=0.2)
    big.centers[:] = cam.C_w + rng.normal(size=(6, 3)).astype(np.float32) * 0.3
    big.scales[:] = rng.uniform(0.5, 1.2, (6, 3)).astype(np.float32)
    big.b2[:] = (0.3 / big.scales.max(1)).astype(np.float32)
    sc = synth.concat_scenes(scene, big)
    res = gpu_render(sc, [cam])
    img_o, fl, _ = orc.render_frame(sc, cam)
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    assert c["max_unflagged"] <= TOL, c


def test_determinism_host_paths_and_stripes():
    scene, cams, bg = synth.make_config("C2", n=4000)
    a = gpu_render(scene, cams, bg)["img"]
    b = gpu_render(scene, cams, bg, device_scene=False, host_out=True)["img"]
    assert np.array_equal(a, b)                       # host vs device input/output, bit-identical
    parts = [gpu_render(scene, cams, bg, stripe=(r, 3))["img"] for r in range(3)]
    H = cams[0].height
    for y in range(H):
        p = parts[(y // 16) % 3]
        assert np.array_equal(p[0, y], a[0, y])       # each stripe renders exactly its rows


def test_validation_errors_and_update_scene():
    """zero quaternion / non-positive scale / non-finite values are
    rejected with the primitive's index; snp_update_scene replaces values."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    sc = synth.make_scene(0, 64)
    for field, idx, val, word in (("rotations", (3,), 0.0, "quaternion"), ("scales", (5, 2), -1.0, "scale"),
                                  ("w1", (2, 3, 1), np.nan, "non-finite"), ("sh", (7, 4, 0), np.inf, "non-finite")):
        bad = sc.subset(np.arange(sc.n))
        getattr(bad, field)[idx] = val
        for src in (bad, torch_scene(bad)):
            with pytest.raises(snp.SnpError) as ei:
                snp.create_scene(src, 0)
            assert ei.value.status == 1 and word in str(ei.value)
    cams = synth.orbit_cameras(1, 4.0, 96, 64, 90.0)
    a = gpu_render(sc, cams)["img"]
    sc2 = synth.make_scene(9, 64)
    b = gpu_render(sc2, cams)["img"]
    h = snp.create_scene(sc, 0)
    out = torch.empty((1, 64, 96, 4), device="cuda")
    opts = snp.make_opts()
    snp.render_views(h, cams, opts, out)
    assert np.array_equal(out.cpu().numpy(), a)
    snp.update_scene(h, sc2)
    with pytest.raises(snp.SnpError):
        snp.render(h, opts, out)          # stale binning after an update: BAD_STATE
    snp.render_views(h, cams, opts, out)
    assert np.array_equal(out.cpu().numpy(), b)
    with pytest.raises(snp.SnpError):
        snp.update_scene(h, synth.make_scene(1, 10))   # n differs
    snp.destroy(h)


@pytest.mark.gpu
def test_stream_ordering_and_graph_capture():
    """K1b runs on the scene's side stream (forked after K1a, joined at the end of
    snp_bin_sort): project twice before binning, render twice after one binning,
    update the scene right after projecting, and replay the whole frame as a CUDA
    graph captured on a user stream -- every result bit-identical to a plain frame."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    scene, cams, bg = synth.make_config("C2", n=3000)
    V, H, W = len(cams), cams[0].height, cams[0].width
    ref = gpu_render(scene, cams, bg)["img"]
    cc = snp.make_cameras(cams)
    h = snp.create_scene(torch_scene(scene), 0)
    try:
        first = snp.make_opts(bg, sync_check=1)
        opts = snp.make_opts(bg, sync_check=0)
        out = torch.full((V, H, W, 4), float("nan"), device="cuda")
        other = synth.orbit_cameras(1, 3.0, W, H, 60.0)
        snp.project(h, snp.make_cameras(other))     # pending K1b, never binned
        snp.project(h, cc)                          # must wait for it
        snp.bin_sort(h, first)
        snp.render(h, opts, out)
        snp.render(h, opts, out)                    # second render of the same binning
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref)
        # update right after a projection (K1b still reading the old parameters)
        scene2, _, _ = synth.make_config("C2", n=3000)
        scene2.b2[:] = scene2.b2 * 0.5
        ref2 = gpu_render(scene2, cams, bg)["img"]
        snp.project(h, cc)
        snp.update_scene(h, torch_scene(scene2))
        snp.render_views(h, cams, first, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref2)
        # whole frame captured on a user stream, replayed
        st = torch.cuda.Stream()
        out.fill_(float("nan"))
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            snp.project(h, cc, st)
            snp.bin_sort(h, opts, st)
            snp.render(h, opts, out, st)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref2)
        s = snp.get_stats(h)
        assert s["composited"] > 0 and s["capacity_overflow"] == 0
    finally:
        snp.destroy(h)


def test_async_host_output():
    """SNP_MEM_HOST_ASYNC: the frame lands in (pinned) host memory once the stream is
    synchronised, bit-identical to the device output; SNP_MEM_HOST and stripes write 0
    outside the stripe."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    scene, cams, bg = synth.make_config("C2", n=2000)
    V, H, W = len(cams), cams[0].height, cams[0].width
    ref = gpu_render(scene, cams, bg)["img"]
    h = snp.create_scene(torch_scene(scene), 0)
    try:
        st = torch.cuda.Stream()
        out = torch.full((V, H, W, 4), float("nan")).pin_memory()
        snp.render_views(h, cams, snp.make_opts(bg, out_memory=snp.SNP_MEM_HOST_ASYNC), out, st)
        st.synchronize()
        assert np.array_equal(out.numpy(), ref)
        part = np.full((V, H, W, 4), np.nan, np.float32)
        snp.render_views(h, cams, snp.make_opts(bg, tile_row_begin=1, tile_row_stride=2,
                                                out_memory=snp.SNP_MEM_HOST), part)
        rows = np.array([(y // 16) % 2 == 1 for y in range(H)])
        assert np.array_equal(part[:, rows], ref[:, rows]) and not part[:, ~rows].any()
    finally:
        snp.destroy(h)


def test_degenerate_primitives_and_clipping(orc):
    """Needle- and sheet-like ellipsoids (axis ratios up to 1e3), a primitive covering
    most of the image, zero-density and near-opaque primitives, primitives cut by
    t_near and by t_far, an off-centre principal point and fx != fy: every pixel
    against the oracle (P:298-299 clipping, Eq. 9 clamp, Eq. 4 termination)."""
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
    cam = synth.look_at((0.0, -2.6, 0.9), (0.1, 0.0, 0.0), 83, 61, 70.0, fy=55.0, cx=30.3, cy=35.7,
                        t_near=1.9, t_far=3.3)
    res = gpu_render(sc, [cam], (0.1, 0.2, 0.3))
    img_o, fl, _ = orc.render_frame(sc, cam, (0.1, 0.2, 0.3))
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    assert c["max_unflagged"] <= TOL and c["n_flagged"] <= 0.02 * c["n"], c
    assert res["stats"]["composited"] > 0


@pytest.mark.parametrize("omega", [1.0, 10.0])
def test_other_omega(orc, omega):
    """omega is a scene parameter (P:394 uses 30; P:664-675 studies 1 and 10): the
    phase scaling of K1b's units and the oracle's Eq. 8 agree for other values."""
    scene, cams, bg = synth.make_config("C1")
    scene.omega = omega
    res = gpu_render(scene, cams, bg)
    img_o, fl, _ = orc.render_frame(scene, cams[0], bg)
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    assert c["max_unflagged"] <= TOL, c


def test_subpixel_primitives_far_away(orc):
    """Primitives smaller than a pixel at large depth: the pixel-centre rect (1/256 px
    slack) and the conic margin must not drop their hits."""
    rng = np.random.default_rng(21)
    sc = synth.make_scene(22, 400, box=0.8)
    d = np.stack([rng.uniform(-0.13, 0.13, 400), -np.ones(400), rng.uniform(-0.11, 0.11, 400)], 1)
    sc.centers[:] = (d * rng.uniform(20, 60, (400, 1))).astype(np.float32)
    sc.scales[:] = rng.uniform(0.005, 0.04, (400, 3)).astype(np.float32)
    sc.b2[:] = (2.0 / sc.scales.max(1)).astype(np.float32)
    cam = synth.look_at((0.0, 0.0, 0.0), (0.0, -1.0, 0.0), 96, 80, 400.0)
    res = gpu_render(sc, [cam])
    img_o, fl, _ = orc.render_frame(sc, cam)
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    assert c["max_unflagged"] <= TOL, c
    assert (img_o[..., 3] > 1e-3).sum() > 50   # the test does see primitives


def test_fallback_pixels_full_size_C5(orc, monkeypatch):
    """The pixels K5 hands to K6 at full C5 size (found by rendering once with K6
    disabled: they stay unwritten), checked one by one against the oracle."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    scene, cams, bg = synth.make_config("C5")
    V, H, W = 1, cams[0].height, cams[0].width
    h = snp.create_scene(torch_scene(scene), 0)
    try:
        out = torch.full((V, H, W, 4), float("nan"), device="cuda")
        monkeypatch.setenv("SNP_DEBUG", "2")          # skip K6
        snp.render_views(h, cams, snp.make_opts(bg), out)
        torch.cuda.synchronize()
        miss = torch.isnan(out[0, ..., 3]).nonzero().cpu().numpy()
        n_ovf = snp.get_stats(h)["overflow_pixels"]
        assert len(miss) == n_ovf > 0
        monkeypatch.delenv("SNP_DEBUG")
        out.fill_(float("nan"))
        snp.render_views(h, cams, snp.make_opts(bg, sync_check=0), out)
        torch.cuda.synchronize()
        img = out[0].cpu().numpy()
    finally:
        snp.destroy(h)
    assert not np.isnan(img).any()
    sel = miss[np.random.default_rng(3).permutation(len(miss))[:200]]
    py, px = sel[:, 0].astype(np.int64), sel[:, 1].astype(np.int64)
    out_o, fl, _ = orc.render_pixels(scene, cams[0], px, py, bg)
    c = compare(img[py, px], out_o, fl)
    assert c["max_unflagged"] <= TOL and c["n_flagged"] <= 0.1 * c["n"], c


def _deep_scene(n=2600):
    """n faint spheres strung along the view axis, 0.01 apart, radii cycling through
    four values: every ray hits all n (t_in order = a fixed permutation of the centre
    order, consecutive gaps >= ~1e-3, so no near-tie flags) and T stays ~0.1."""
    scene = synth.make_scene(21, n, box=0.3)
    i = np.arange(n)
    scene.centers[:] = np.stack([5.0 + 0.01 * i, np.zeros(n), np.zeros(n)], 1).astype(np.float32)
    r = 1.2 + 0.035 * (i % 4)
    scene.scales[:] = np.stack([r, r, r], 1).astype(np.float32)
    scene.w2 *= np.float32(1e-4)
    scene.b2[:] = np.float32(3e-4)
    return scene


@pytest.mark.parametrize("limit", [0, 1])
def test_deep_overlap_long_lists(orc, limit):
    """2600 hits on every ray of a 2x2-tile image: 2600-key tile lists (sort, ranges),
    long pending lists in K5 and, with a pending limit of 1, every pixel in K6 with
    more hits than its shared-memory capacity (kFbHits = 2048: the repeated-selection
    path)."""
    scene = _deep_scene()
    cam = synth.look_at((0, 0, 0), (1, 0, 0), 32, 24, 1600.0)
    res = gpu_render(scene, [cam], pending_limit=limit, binning=True)
    _check_binning(orc, scene, [cam], res)
    img_o, fl, st = orc.render_frame(scene, cam)
    assert st[..., 1].min() == 2600 and fl.sum() == 0
    if limit == 1:
        assert res["stats"]["overflow_pixels"] == 32 * 24
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    assert c["max_unflagged"] <= TOL, c


@pytest.mark.parametrize("n_hidden", [4, 16, 32])
def test_hidden_widths(orc, n_hidden):
    """N_sigma in {4, 16, 32} -- records of 6 + N + N/4 float4, K1b, K5
    and K6 instantiated per N -- against the oracle on a full C1-sized frame, also with
    pending overflow (K6), and on sampled pixels of a C2-sized view."""
    _, cams, bg = synth.make_config("C1")
    scene = synth.make_scene(31 + n_hidden, 400, n_hidden=n_hidden)
    assert scene.w1.shape[1] == n_hidden
    img_o, fl, _ = orc.render_frame(scene, cams[0], bg)
    for limit in (0, 2):
        res = gpu_render(scene, cams, bg, pending_limit=limit)
        assert limit == 0 or res["stats"]["overflow_pixels"] > 0
        c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
        assert c["max_unflagged"] <= TOL and c["n_flagged"] <= 0.01 * c["n"], (limit, c)
    big, cams2, bg2 = synth.make_config("C2")
    scene2 = synth.make_scene(41 + n_hidden, 10000, n_hidden=n_hidden)
    res = gpu_render(scene2, cams2, bg2)
    px, py = sample_pixels(cams2[0], 1500, 3, seed=n_hidden)
    out_o, fl2, _ = orc.render_pixels(scene2, cams2[0], px, py, bg2)
    c = compare(res["img"][0][py, px], out_o, fl2)
    assert c["max_unflagged"] <= TOL and c["n_flagged"] <= 0.02 * c["n"], c


@pytest.mark.parametrize("n_hidden", [8, 16])
def test_colour_per_ray(orc, n_hidden):
    """SNP_COLOUR_RAY: SH colour at each pixel's ray direction, in K5's
    blend and in K6 (forced pending overflow), against the oracle's per-ray mode; a C1
    frame at every SH degree and sampled pixels of the full C3 view."""
    from paper_2510_08491_b200 import snp
    _, cams, bg = synth.make_config("C1")
    scene = synth.make_scene(51, 400, n_hidden=n_hidden)
    for deg in (3, 1, 0):
        scene.sh_degree = deg
        img_o, fl, _ = orc.render_frame(scene, cams[0], bg, colour_per_ray=True)
        for limit in (0, 2):
            res = gpu_render(scene, cams, bg, pending_limit=limit, colour_mode=snp.SNP_COLOUR_RAY)
            c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
            assert c["max_unflagged"] <= TOL and c["n_flagged"] <= 0.01 * c["n"], (deg, limit, c)
    prim = gpu_render(scene, cams, bg, pending_limit=2)["img"][0]   # degree 0: the two modes coincide
    assert np.abs(prim - res["img"][0]).max() <= 1e-6
    if n_hidden == 8:
        scene3, cams3, bg3 = synth.make_config("C3")
        res = gpu_render(scene3, cams3, bg3, colour_mode=snp.SNP_COLOUR_RAY)
        px, py = sample_pixels(cams3[0], 1500, 3, seed=5)
        out_o, fl3, _ = orc.render_pixels(scene3, cams3[0], px, py, bg3, colour_per_ray=True)
        c = compare(res["img"][0][py, px], out_o, fl3)
        assert c["max_unflagged"] <= TOL and c["n_flagged"] <= 0.02 * c["n"], c


def test_temporal_views(orc):
    """Temporal scenes: one timestamp per view folded into K1b's
    records (omega (b1 + xi_t W_t)); a 3-view batch at xi_t = 0, 0.4, 1 against the
    oracle, detaching the weights restores the static image, non-finite weights are
    rejected with the primitive's index."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    scene, cams, bg = synth.make_config("C1")
    rng = np.random.default_rng(17)
    scene.w_t = rng.uniform(-1, 1, (scene.n, scene.n_hidden)).astype(np.float32)
    c = cams[0]
    cams = synth.orbit_cameras(3, 4.0, c.width, c.height, c.fx, elev_deg=(10, 35))
    times = [0.0, 0.4, 1.0]
    h = snp.create_scene(torch_scene(scene), 0)
    try:
        snp.set_temporal(h, scene.w_t)
        out = torch.full((3, c.height, c.width, 4), float("nan"), device="cuda")
        snp.render_views(h, cams, snp.make_opts(bg), out, xi_t=times)
        img = out.cpu().numpy()
        snp.set_temporal(h, None)
        snp.render_views(h, cams, snp.make_opts(bg), out)
        static = out.cpu().numpy()
        bad = scene.w_t.copy()
        bad[37, 2] = np.inf
        with pytest.raises(snp.SnpError, match="primitive 37"):
            snp.set_temporal(h, bad)
    finally:
        snp.destroy(h)
    for v, t in enumerate(times):
        cams[v].xi_t = t
        img_o, fl, _ = orc.render_frame(scene, cams[v], bg)
        cmp_ = compare(img[v].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
        assert cmp_["max_unflagged"] <= TOL and cmp_["n_flagged"] <= 0.01 * cmp_["n"], (v, cmp_)
    assert np.array_equal(static[0], img[0]) and np.abs(static[2] - img[2]).max() > 1e-3


@pytest.mark.parametrize("colour_mode,n_hidden", [(0, 8), (1, 8), (0, 16)])
def test_backward_mlp_and_sh_vs_finite_differences(orc, colour_mode, n_hidden):
    """K7 (snp_render_backward, SURVEY §8(f) rank 1 first part): dL/d{W1, b1, W2, b2, SH}
    for L = sum(G * out_rgba), against central differences of the fp64 oracle's forward
    on sampled parameters of hit primitives (geometry fixed)."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    scene = synth.make_scene(61, 150, box=0.6, n_hidden=n_hidden)
    # semi-transparent (no pixel reaches the T floor, whose stop rule makes L jump) and a
    # density bounded away from 0 (b2 > sum |W2|: no I <= 0 kink of Eq. 9), so that L is
    # smooth around the sampled parameters and finite differences see the derivative
    scene.w2 *= np.float32(0.8 / n_hidden)
    scene.b2[:] = (1.2 * np.abs(scene.w2).sum(1)).astype(np.float32)
    cam = synth.orbit_cameras(1, 3.0, 64, 48, 60.0)[0]
    bg = (0.1, 0.2, 0.3)
    rng = np.random.default_rng(62 + colour_mode + n_hidden)
    G = rng.normal(size=(1, 48, 64, 4)).astype(np.float32)
    h = snp.create_scene(torch_scene(scene), 0)
    try:
        opts = snp.make_opts(bg, colour_mode=colour_mode)
        out = torch.zeros((1, 48, 64, 4), device="cuda")
        snp.render_views(h, [cam], opts, out)
        grads = {f: torch.zeros(getattr(scene, f).shape, device="cuda")
                 for f in ("w1", "b1", "w2", "b2", "sh", "centers", "rotations", "scales")}
        snp.render_backward(h, opts, torch.from_numpy(G).cuda(), grads)
        torch.cuda.synchronize()
        assert snp.get_stats(h)["backward_skipped"] == 0
        assert out[..., 3].max().item() < 0.999
        g = {f: v.cpu().numpy().astype(np.float64) for f, v in grads.items()}
    finally:
        snp.destroy(h)
    ray = colour_mode == 1

    def loss(sc):
        img, _, _ = orc.render_frame(sc, cam, bg, colour_per_ray=ray)
        return float((img * G[0].astype(np.float64)).sum())

    hit = np.nonzero(np.abs(g["b2"]) > 0)[0]
    assert len(hit) > 20
    checks = []
    geo = ("centers", "rotations", "scales")
    skipped = []
    for f in ("w1", "b1", "w2", "b2", "sh") + geo:
        for _ in range(8):
            i = int(rng.choice(hit))
            idx = (i,) + tuple(int(rng.integers(0, s)) for s in getattr(scene, f).shape[1:])
            if f == "sh":
                idx = (i, int(rng.integers(0, 4)), int(rng.integers(0, 3)))   # low bands
            arr = getattr(scene, f)
            base = float(arr[idx])
            # geometry: steps far below the primitive size (the chord is sqrt-shaped at
            # the silhouette); the fp64 oracle resolves them
            step = np.float32(2e-3 * (abs(base) + 0.05)) if f not in geo else \
                np.float32(2e-4 * float(scene.scales[i].min()))
            fds = []
            for st in ((step, step / 4) if f in geo else (step,)):
                st = np.float32(st)
                vals = []
                for sgn in (1, -1):
                    arr[idx] = np.float32(base + sgn * st)
                    vals.append(loss(scene))
                arr[idx] = np.float32(base)
                hp, hm = float(np.float32(base + st)) - base, base - float(np.float32(base - st))
                fds.append((vals[0] - vals[1]) / (hp + hm))
            # a geometry parameter whose finite differences change with the step sits on a
            # pixel where the chord's sqrt-shaped silhouette edge is within reach: skipped
            if len(fds) == 2 and abs(fds[0] - fds[1]) > 1e-3 * max(abs(fds[0]), abs(fds[1]), 1e-3):
                skipped.append((f, idx, float(g[f][idx]), fds))
                continue
            checks.append((f, idx, float(g[f][idx]), fds[-1]))
    assert len(skipped) <= 6, skipped
    for group, tol in (("mlp+sh", 2e-3), ("geometry", 5e-3)):
        cs = [c for c in checks if (c[0] in geo) == (group == "geometry")]
        scale = max(abs(c[3]) for c in cs)
        worst = max(abs(c[2] - c[3]) / (abs(c[3]) + 1e-3 * scale) for c in cs)
        print("backward vs FD (%s): worst relative error %.2e over %d parameters (scale %.3g; %d skipped)"
              % (group, worst, len(cs), scale, len(skipped) if group == "geometry" else 0))
        for c in sorted(cs, key=lambda c: -abs(c[2] - c[3]) / (abs(c[3]) + 1e-3 * scale))[:4]:
            print("   ", c)
        bad = [c for c in cs if abs(c[2] - c[3]) > tol * abs(c[3]) + 0.1 * tol * scale]
        assert not bad, (group, bad, scale)


@pytest.mark.parametrize("colour_mode", [0, 1])
def test_backward_k5_path_matches_per_pixel_k7(monkeypatch, colour_mode):
    """The backward through K5's gradient mode (+ K7f, + the per-pixel K7 for the pixels
    K5 hands to its fallbacks, with their skip counts) equals the per-pixel K7 on every
    pixel (SNP_BWD_LEGACY=1), for all parameters, on a C2-shaped frame with forced
    pending overflow on some pixels (pending limit 3) and the dense grazing scene."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    rng = np.random.default_rng(81)
    cases = [(synth.make_scene(1, 2000, scale_mult=1.5, box=1.0), synth.orbit_cameras(2, 4.0, 160, 120, 220.0), 3)]
    n = 150
    sc = synth.make_scene(32, n, box=0.6)
    sc.centers[:] = rng.uniform(-0.4, 0.4, (n, 3)).astype(np.float32)
    sc.scales[:] = rng.uniform(0.04, 0.1, (n, 3)).astype(np.float32)
    sc.w2[:] = 0.0
    sc.b2[:] = (50.0 / sc.scales.max(1)).astype(np.float32)
    cases.append((sc, [synth.look_at((0.3, -3.0, 0.4), (0.0, 0.0, 0.0), 200, 150, 750.0)], 0))
    for scene, cams, limit in cases:
        V, H, W = len(cams), cams[0].height, cams[0].width
        G = torch.from_numpy(rng.normal(size=(V, H, W, 4)).astype(np.float32)).cuda()
        res = {}
        for legacy in (0, 1):
            monkeypatch.setenv("SNP_BWD_LEGACY", str(legacy))
            h = snp.create_scene(torch_scene(scene), 0)
            try:
                if limit:
                    snp.set_pending_limit(h, limit)
                opts = snp.make_opts((0.2, 0.3, 0.4), colour_mode=colour_mode)
                out = torch.zeros((V, H, W, 4), device="cuda")
                snp.render_views(h, cams, opts, out)
                grads = {f: torch.zeros(getattr(scene, f).shape, device="cuda") for f in snp.FIELDS}
                snp.render_backward(h, opts, G, grads, fwd_rgba=out if legacy == 0 else None)
                torch.cuda.synchronize()
                res[legacy] = {f: v.cpu().numpy().astype(np.float64) for f, v in grads.items()}
                if limit:
                    assert snp.get_stats(h)["overflow_pixels"] > 0
            finally:
                snp.destroy(h)
        for f in snp.FIELDS:
            a, b = res[0][f], res[1][f]
            scale = np.abs(b).max()
            assert np.abs(a - b).max() <= 2e-4 * scale + 1e-7, (f, np.abs(a - b).max(), scale)


def test_backward_two_camera_batches(monkeypatch):
    """34 views (two camera batches of at most 32): the K5-path backward, batch by batch
    (entry buffer, fallback queues and skip counts reset per batch), equals the per-pixel
    K7 on every parameter."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    scene = synth.make_scene(5, 600, box=0.7)
    cams = synth.orbit_cameras(34, 3.0, 40, 28, 50.0, elev_deg=(5, 60))
    G = torch.from_numpy(np.random.default_rng(7).normal(size=(34, 28, 40, 4)).astype(np.float32)).cuda()
    res = {}
    for legacy in (0, 1):
        monkeypatch.setenv("SNP_BWD_LEGACY", str(legacy))
        h = snp.create_scene(torch_scene(scene), 0)
        try:
            snp.set_pending_limit(h, 4)
            opts = snp.make_opts((0.1, 0.1, 0.1))
            out = torch.zeros((34, 28, 40, 4), device="cuda")
            snp.render_views(h, cams, opts, out)
            grads = {f: torch.zeros(getattr(scene, f).shape, device="cuda") for f in snp.FIELDS}
            snp.render_backward(h, opts, G, grads, fwd_rgba=out if legacy == 0 else None)
            torch.cuda.synchronize()
            res[legacy] = {f: v.cpu().numpy().astype(np.float64) for f, v in grads.items()}
        finally:
            snp.destroy(h)
    for f in snp.FIELDS:
        a, b = res[0][f], res[1][f]
        scale = np.abs(b).max()
        assert scale > 0 and np.abs(a - b).max() <= 2e-4 * scale + 1e-7, (f, np.abs(a - b).max(), scale)


def test_adam_and_l1_kernels():
    """snp_loss_l1 and snp_adam_step against their plain definitions (numpy, float64)."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    rng = np.random.default_rng(71)
    out = rng.uniform(0, 1, (5, 7, 4)).astype(np.float32)
    tgt = rng.uniform(0, 1, (5, 7, 3)).astype(np.float32)
    g = torch.zeros((5, 7, 4), device="cuda")
    loss = torch.zeros(1, device="cuda")
    snp.loss_l1(torch.from_numpy(out).cuda(), torch.from_numpy(tgt).cuda(), g, loss)
    d = out[..., :3].astype(np.float64) - tgt
    assert abs(loss.item() - np.abs(d).mean()) < 1e-6
    ref = np.concatenate([np.sign(d) / d.size, np.zeros((5, 7, 1))], -1)
    assert np.allclose(g.cpu().numpy(), ref, rtol=1e-6, atol=1e-9)
    scene = synth.make_scene(72, 50)
    h = snp.create_scene(torch_scene(scene), 0)
    try:
        grads = {f: torch.from_numpy(rng.normal(size=getattr(scene, f).shape).astype(np.float32)).cuda()
                 for f in snp.FIELDS}
        lr = {f: 1e-2 for f in snp.FIELDS}
        b1, b2, eps = 0.9, 0.999, 1e-8
        snp.adam_step(h, grads, 1, lr, b1, b2, eps)
        snp.adam_step(h, grads, 2, lr, b1, b2, eps)
        # read the updated parameters back through the binning-independent update path
        got = {}
        for f in snp.FIELDS:
            dev = torch.zeros(getattr(scene, f).shape, device="cuda")
            got[f] = dev
        snp.copy_params(h, got)
    finally:
        snp.destroy(h)
    for f in snp.FIELDS:
        p = getattr(scene, f).astype(np.float64)
        gg = grads[f].cpu().numpy().astype(np.float64)
        m = np.zeros_like(p); v = np.zeros_like(p)
        for t in (1, 2):
            gt = gg * p if f == "scales" else gg          # scales: Adam on log s
            m = b1 * m + (1 - b1) * gt
            v = b2 * v + (1 - b2) * gt * gt
            stp = lr[f] * (m / (1 - b1 ** t)) / (np.sqrt(v / (1 - b2 ** t)) + eps)
            p = p * np.exp(-stp) if f == "scales" else p - stp
        assert np.allclose(got[f].cpu().numpy(), p, rtol=2e-5, atol=2e-6), f


def _ssim_loss_torch(out, tgt, lam):
    """3DGS's loss, written with torch CPU ops in float64 (the plain reference of the op):
    (1 - lam) mean|x - y| + lam (1 - mean SSIM), SSIM from an 11x11 Gaussian window
    (sigma 1.5) by conv2d with zero padding, C1 = 0.01^2, C2 = 0.03^2, per channel."""
    import torch
    import torch.nn.functional as F
    x = out[..., :3].permute(0, 3, 1, 2)
    y = tgt.permute(0, 3, 1, 2)
    k = torch.arange(11, dtype=torch.float64) - 5
    g1 = torch.exp(-k * k / (2 * 1.5 ** 2))
    g1 = g1 / g1.sum()
    win = (g1[:, None] * g1[None, :]).expand(3, 1, 11, 11).contiguous()
    conv = lambda z: F.conv2d(z, win, padding=5, groups=3)  # noqa: E731
    mx, my = conv(x), conv(y)
    sxx, syy, sxy = conv(x * x) - mx * mx, conv(y * y) - my * my, conv(x * y) - mx * my
    C1, C2 = 0.01 ** 2, 0.03 ** 2
    ssim = ((2 * mx * my + C1) * (2 * sxy + C2)) / ((mx * mx + my * my + C1) * (sxx + syy + C2))
    return (1 - lam) * (x - y).abs().mean() + lam * (1 - ssim.mean())


@pytest.mark.parametrize("lam,shape", [(0.2, (2, 29, 37)), (0.0, (2, 29, 37)), (1.0, (2, 29, 37)),
                                       (0.2, (3, 70, 101)), (1.0, (1, 5, 7))])
def test_loss_3dgs_against_torch(lam, shape):
    """snp_loss_3dgs (the 3DGS loss, R25) against the torch float64 definition:
    loss and dL/d(out) by autograd, on views of a ragged 37x29 image (one 32x16 tile
    plus ragged ones), a 101x70 image (many tiles, ragged right/bottom edges) and a 7x5
    image (the 5-pixel halo wider than the image)."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    V, H, W = shape
    rng = np.random.default_rng(77 + H)
    out = rng.uniform(0, 1, (V, H, W, 4)).astype(np.float32)
    tgt = np.clip(out[..., :3] + rng.normal(0, 0.15, (V, H, W, 3)), 0, 1).astype(np.float32)
    h = snp.create_scene(torch_scene(synth.make_scene(1, 4)), 0)
    try:
        g = torch.zeros((V, H, W, 4), device="cuda")
        loss = torch.zeros(1, device="cuda")
        snp.loss_3dgs(h, torch.from_numpy(out).cuda(), torch.from_numpy(tgt).cuda(), g, loss, lam)
        torch.cuda.synchronize()
    finally:
        snp.destroy(h)
    xo = torch.from_numpy(out.astype(np.float64)).requires_grad_(True)
    ref = _ssim_loss_torch(xo, torch.from_numpy(tgt.astype(np.float64)), lam)
    ref.backward()
    assert abs(loss.item() - ref.item()) < 2e-6 * max(1.0, abs(ref.item())), (loss.item(), ref.item())
    gr = xo.grad.numpy()
    gg = g.cpu().numpy()
    scale = np.abs(gr).max()
    assert np.abs(gg - gr).max() <= 2e-4 * scale, (np.abs(gg - gr).max(), scale)


def test_scale_regularizer_kernel():
    """snp_scale_regularizer (P:416's std(s) penalty): R = w mean_i std(s_i) and dR/ds
    against the numpy definition and central differences of it."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    scene = synth.make_scene(73, 200)
    scene.scales[7] = np.float32([0.3, 0.3, 0.3])        # std 0: zero gradient
    w = 0.37
    h = snp.create_scene(torch_scene(scene), 0)
    try:
        gs = torch.zeros((200, 3), device="cuda")
        loss = torch.zeros(1, device="cuda")
        snp.scale_regularizer(h, w, gs, loss)
        torch.cuda.synchronize()
    finally:
        snp.destroy(h)
    s = scene.scales.astype(np.float64)

    def R(s):
        return w * np.std(s, axis=1).mean()
    assert abs(loss.item() - R(s)) < 1e-6 * max(1.0, R(s))
    g = gs.cpu().numpy()
    assert np.all(g[7] == 0)
    for i, j in ((0, 0), (3, 2), (150, 1), (199, 0)):
        e = 1e-6
        sp, sm = s.copy(), s.copy()
        sp[i, j] += e
        sm[i, j] -= e
        fd = (R(sp) - R(sm)) / (2 * e)
        assert abs(g[i, j] - fd) <= 1e-4 * abs(fd) + 1e-9, (i, j, g[i, j], fd)


@pytest.mark.parametrize("dssim_lambda", [0.0, 0.2])
def test_training_step_reduces_loss(dssim_lambda):
    """SURVEY §8(f) rank 4 on one GPU: render 4 views, L1 or 3DGS's L1 + D-SSIM vs
    target images of a reference scene, K7 gradients, Adam (P:735 rates, x5) -- the loss
    falls over 40 steps."""
    import torch
    from paper_2510_08491_b200 import snp, train
    from gpu_util import torch_scene
    true, cams, bg = synth.make_config("C1")
    cams = synth.orbit_cameras(4, 4.0, 96, 72, 90.0, elev_deg=(10, 40))
    h0 = snp.create_scene(torch_scene(true), 0)
    try:
        tgt = torch.zeros((4, 72, 96, 4), device="cuda")
        snp.render_views(h0, cams, snp.make_opts(bg), tgt)
        target = tgt[..., :3].contiguous()
    finally:
        snp.destroy(h0)
    rng = np.random.default_rng(73)
    init = synth.Scene(*(np.array(getattr(true, f)) for f in synth.scenes._FIELDS), omega=true.omega)
    init.sh[:, 0] += rng.normal(0, 0.4, init.sh[:, 0].shape).astype(np.float32)
    init.b2 *= np.float32(0.6)
    init.centers += rng.normal(0, 0.01, init.centers.shape).astype(np.float32)
    h = snp.create_scene(torch_scene(init), 0)
    try:
        tr = train.Trainer(h, init, 4, 72, 96, "cuda", lr={f: 5 * v for f, v in snp.PAPER_LR.items()},
                           opts=snp.make_opts(bg), dssim_lambda=dssim_lambda)
        losses = [tr.step(cams, target).item() for _ in range(40)]
    finally:
        snp.destroy(h)
    print("training losses", [round(l, 4) for l in losses[::8]], round(losses[-1], 4))
    assert np.all(np.isfinite(losses)) and losses[-1] < 0.6 * losses[0], losses


def test_backward_temporal_weights_vs_finite_differences(orc):
    """K7 on a temporal scene (R24): dL/dW_t = xi_t omega dI/d(omega b1) per hit, and b1's
    gradient, against central differences of the oracle at a view timestamp xi_t = 0.6."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    scene = synth.make_scene(81, 150, box=0.6)
    scene.w2 *= np.float32(0.1)
    scene.b2[:] = (1.2 * np.abs(scene.w2).sum(1)).astype(np.float32)
    rng = np.random.default_rng(82)
    scene.w_t = rng.uniform(-1, 1, (scene.n, scene.n_hidden)).astype(np.float32)
    cam = synth.orbit_cameras(1, 3.0, 64, 48, 60.0)[0]
    cam.xi_t = 0.6
    bg = (0.1, 0.2, 0.3)
    G = rng.normal(size=(1, 48, 64, 4)).astype(np.float32)
    h = snp.create_scene(torch_scene(scene), 0)
    try:
        snp.set_temporal(h, scene.w_t)
        gwt = torch.zeros(scene.w_t.shape, device="cuda")
        snp.set_temporal_grad(h, gwt)
        opts = snp.make_opts(bg)
        out = torch.zeros((1, 48, 64, 4), device="cuda")
        snp.render_views(h, [cam], opts, out, xi_t=[0.6])
        grads = {f: torch.zeros(getattr(scene, f).shape, device="cuda") for f in ("w1", "b1", "w2", "b2", "sh")}
        snp.render_backward(h, opts, torch.from_numpy(G).cuda(), grads)
        torch.cuda.synchronize()
        g = {"w_t": gwt.cpu().numpy().astype(np.float64), "b1": grads["b1"].cpu().numpy().astype(np.float64)}
    finally:
        snp.destroy(h)

    def loss(sc):
        img, _, _ = orc.render_frame(sc, cam, bg)
        return float((img * G[0].astype(np.float64)).sum())

    hit = np.nonzero(np.abs(grads["b2"].cpu().numpy()) > 0)[0]
    checks = []
    for f in ("w_t", "b1"):
        arr = getattr(scene, f)
        for _ in range(10):
            idx = (int(rng.choice(hit)), int(rng.integers(0, scene.n_hidden)))
            base = float(arr[idx])
            step = np.float32(2e-3 * (abs(base) + 0.05))
            vals = []
            for sgn in (1, -1):
                arr[idx] = np.float32(base + sgn * step)
                vals.append(loss(scene))
            arr[idx] = np.float32(base)
            hp, hm = float(np.float32(base + step)) - base, base - float(np.float32(base - step))
            checks.append((f, idx, float(g[f][idx]), (vals[0] - vals[1]) / (hp + hm)))
    scale = max(abs(c[3]) for c in checks)
    bad = [c for c in checks if abs(c[2] - c[3]) > 2e-3 * abs(c[3]) + 2e-4 * scale]
    assert not bad, (bad, scale)
    for c in checks:       # dL/dW_t = xi_t dL/db1 for the same unit (one view): exact per hit;
        if c[0] == "w_t":  # the two sums differ only in their fp32 atomic summation order
            assert abs(c[2] - 0.6 * g["b1"][c[1]]) <= 1e-4 * max(abs(c[2]), 1e-2 * scale)


def test_eager_emission_rule(orc, monkeypatch):
    """K5's eager mid-batch emission (kEager) is chosen from the binning alone (mean keys
    per tile > 150, or keys per visible primitive > 2.5): on for C5 (221; 2.9), off for
    C3 (90; 1.9); on C5 it hands fewer pixels to K6 than the forced default mode, on C3
    nothing changes, and the C5 fallback pixels keep parity."""
    scene5, cams5, bg5 = synth.make_config("C5")
    eager = gpu_render(scene5, cams5, bg5)
    monkeypatch.setenv("SNP_EAGER_EMIT", "0")
    forced = gpu_render(scene5, cams5, bg5)
    monkeypatch.delenv("SNP_EAGER_EMIT")
    assert eager["stats"]["overflow_pixels"] < 0.6 * forced["stats"]["overflow_pixels"]
    scene3, cams3, bg3 = synth.make_config("C3")
    a = gpu_render(scene3, cams3, bg3)
    monkeypatch.setenv("SNP_EAGER_EMIT", "0")
    b = gpu_render(scene3, cams3, bg3)
    assert np.array_equal(a["img"], b["img"]) and a["stats"] == b["stats"]
    px, py = sample_pixels(cams5[0], 600, 2, seed=11)
    out_o, fl, _ = orc.render_pixels(scene5, cams5[0], px, py, bg5)
    c = compare(eager["img"][0][py, px], out_o, fl)
    assert c["max_unflagged"] <= TOL and c["n_flagged"] <= 0.02 * c["n"], c


@pytest.mark.parametrize("n_hits,legacy", [(600, 1), (2600, 1), (2600, 0)])
def test_backward_long_hit_lists(orc, monkeypatch, n_hits, legacy):
    """K7's big-capacity passes (legacy = 1: the per-pixel K7 on every pixel): every pixel
    of the deep-overlap scene has 600 hits (more than the first pass holds: the 2048-hit
    shared-memory pass) or 2600 (more than that: the global-memory pass), none is skipped,
    and sampled W2/b2/centre gradients match central differences of the oracle; legacy =
    0: the same through K5's gradient mode (2600 entries per pixel) and K7f."""
    import torch
    monkeypatch.setenv("SNP_BWD_LEGACY", str(legacy))
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    scene = _deep_scene(n_hits)
    cam = synth.look_at((0, 0, 0), (1, 0, 0), 32, 24, 1600.0)
    rng = np.random.default_rng(91)
    G = rng.normal(size=(1, 24, 32, 4)).astype(np.float32)
    h = snp.create_scene(torch_scene(scene), 0)
    try:
        opts = snp.make_opts()
        out = torch.zeros((1, 24, 32, 4), device="cuda")
        snp.render_views(h, [cam], opts, out)
        grads = {f: torch.zeros(getattr(scene, f).shape, device="cuda") for f in snp.FIELDS}
        snp.render_backward(h, opts, torch.from_numpy(G).cuda(), grads)
        torch.cuda.synchronize()
        dc = snp.get_debug_counters(h, 56)
        if legacy:
            # the per-pixel K7 differentiates every pixel past its first (256-hit) pass,
            # and for 2600 hits past its second (2048)
            assert dc[49] == 32 * 24, dc[49]
            assert dc[50] == (32 * 24 if n_hits > 2048 else 0), dc[50]
        else:   # all through K5 + K7f: no entry overflow, no per-pixel K7 pass
            assert dc[52] == 0 and dc[49] == 0 and dc[51] * 1024 >= 32 * 24 * n_hits, (dc[52], dc[49], dc[51])
        assert snp.get_stats(h)["backward_skipped"] == 0              # none skipped
        g = {f: v.cpu().numpy().astype(np.float64) for f, v in grads.items()}
    finally:
        snp.destroy(h)

    def loss(sc):
        img, _, _ = orc.render_frame(sc, cam)
        return float((img * G[0].astype(np.float64)).sum())

    checks = []
    for f, idx in (("w2", (100, 3)), ("w2", (433, 0)), ("b2", (7,)), ("b2", (590,)), ("centers", (250, 1)),
                   ("scales", (321, 0))):
        arr = getattr(scene, f)
        base = float(arr[idx])
        # steps relative to the (tiny) density parameters of this scene
        step = np.float32(1e-3 * abs(base) + 1e-8) if f in ("w2", "b2") else np.float32(1e-4)
        vals = []
        for sgn in (1, -1):
            arr[idx] = np.float32(base + sgn * step)
            vals.append(loss(scene))
        arr[idx] = np.float32(base)
        hp, hm = float(np.float32(base + step)) - base, base - float(np.float32(base - step))
        checks.append((f, idx, float(g[f][idx]), (vals[0] - vals[1]) / (hp + hm)))
    scale = max(abs(c[3]) for c in checks)
    bad = [c for c in checks if abs(c[2] - c[3]) > 5e-3 * abs(c[3]) + 1e-3 * scale]
    assert not bad, (bad, checks)


def _grazing_q(scene, cam, px, py):
    """Q = 1 - min_t |S^-1 R^T (C + t d - mu)|^2 of every (pixel, primitive) in double
    (independent numpy geometry, for the test's coverage statement only)."""
    R = cam.R_wc.astype(np.float64)
    u = (px + 0.5 - cam.cx) / cam.fx
    v = (py + 0.5 - cam.cy) / cam.fy
    d = np.stack([u, v, np.ones_like(u)], 1) @ R.T
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    from scipy.spatial.transform import Rotation
    q = scene.rotations.astype(np.float64)
    Rp = Rotation.from_quat(np.concatenate([q[:, 1:], q[:, :1]], 1)).as_matrix()   # (x,y,z,w)
    W = np.transpose(Rp, (0, 2, 1)) / scene.scales.astype(np.float64)[:, :, None]
    o = cam.C_w.astype(np.float64)[None, :] - scene.centers.astype(np.float64)
    a = np.einsum("nij,pj->pni", W, d)
    b = np.einsum("nij,nj->ni", W, o)[None, :, :]
    A = (a * a).sum(-1)
    ts = -(a * b).sum(-1) / A
    bp = b + ts[..., None] * a
    return 1.0 - (bp * bp).sum(-1), np.sqrt(np.maximum(1.0 - (bp * bp).sum(-1), 0) / A) * 2


def test_grazing_rays_through_dense_primitives(orc):
    """SURVEY H2 / DESIGN R23: rays grazing near-opaque primitives (constant density
    rho = 50 / s_max, i.e. ~10^3 per unit length for s ~ 0.05; P:298-299 chord,
    Eq. 9) at 1 - q_min from 1e-5 up: the fp32 chord's relative error ~2e-7 / Q
    would put ~2e-4 on kappa at Q = 1e-4 -- the kernel's FP64 branch must keep
    every unflagged pixel within 1e-4."""
    rng = np.random.default_rng(31)
    n = 150
    sc = synth.make_scene(32, n, box=0.6)
    sc.centers[:] = rng.uniform(-0.4, 0.4, (n, 3)).astype(np.float32)
    sc.scales[:] = rng.uniform(0.04, 0.1, (n, 3)).astype(np.float32)
    sc.w2[:] = 0.0
    sc.b2[:] = (50.0 / sc.scales.max(1)).astype(np.float32)
    cam = synth.look_at((0.3, -3.0, 0.4), (0.0, 0.0, 0.0), 400, 300, 1500.0)
    yy, xx = np.mgrid[0:cam.height, 0:cam.width]
    Q, chord = _grazing_q(sc, cam, xx.ravel().astype(np.float64), yy.ravel().astype(np.float64))
    I = chord * sc.b2.astype(np.float64)[None, :]
    sel = (Q > 1e-5) & (Q < 1e-3) & (I > 0.2) & (I < 5.0)
    assert sel.sum() >= 100, sel.sum()          # the scene does exercise the window
    res = gpu_render(sc, [cam])
    img_o, fl, _ = orc.render_frame(sc, cam)
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    print(c, int(sel.sum()), res["stats"])
    assert c["max_unflagged"] <= TOL, c
    assert c["n_flagged"] <= 0.02 * c["n"], c


def test_render_full_frame_C3(orc):
    """The headline configuration, every pixel: the full 1245x825 C3 frame (300k
    primitives) in the launch configuration bench.py times, against the oracle's full
    frame (~1 min on the GPU box's host cores).  The flagged fraction is reported."""
    from paper_2510_08491_b200 import snp  # noqa: F401
    scene, cams, bg = synth.make_config("C3")
    res = gpu_render(scene, cams, bg, sync_check=0, repeat=2)
    img_o, fl, _ = orc.render_frame(scene, cams[0], bg)
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    print("C3 full frame", c, "flag kinds", np.bincount(fl.ravel(), minlength=8).tolist(), res["stats"])
    assert c["max_unflagged"] <= TOL, c
    assert c["n_flagged"] <= 1e-3 * c["n"], c


def test_render_full_frame_C2(orc):
    """Config C2 (10k primitives, 800x800, white background), every pixel against the
    oracle's full frame."""
    scene, cams, bg = synth.make_config("C2")
    res = gpu_render(scene, cams, bg, sync_check=0, repeat=2)
    img_o, fl, _ = orc.render_frame(scene, cams[0], bg)
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    print("C2 full frame", c)
    assert c["max_unflagged"] <= TOL, c
    assert c["n_flagged"] <= 1e-3 * c["n"], c


@pytest.mark.skipif(not __import__("os").environ.get("SNP_SLOW_TESTS"),
                    reason="8 min of oracle time on 16 cores: set SNP_SLOW_TESTS=1 (result in profiles/r02_full_frames.md)")
def test_render_full_frame_C5(orc):
    """Config C5 (1M large-footprint primitives, 1920x1080; K6w busy), every pixel against
    the oracle's full frame (~8 min on the GPU box's 16 host cores)."""
    scene, cams, bg = synth.make_config("C5")
    res = gpu_render(scene, cams, bg, sync_check=0, repeat=2)
    img_o, fl, _ = orc.render_frame(scene, cams[0], bg)
    c = compare(res["img"][0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    print("C5 full frame", c, "flag kinds", np.bincount(fl.ravel(), minlength=8).tolist(), res["stats"])
    assert c["max_unflagged"] <= TOL, c
    assert c["n_flagged"] <= 3e-3 * c["n"], c


def test_repeated_renders_bit_identical():
    """Races in K5's rings, the K5 -> K6w queue or the sort would show as frame-to-frame
    differences: 8 renders of the C3 frame and 3 of C5 (K6w busy) are bit-identical."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    for cfg, reps in (("C3", 8), ("C5", 3)):
        scene, cams, bg = synth.make_config(cfg)
        h = snp.create_scene(torch_scene(scene), 0)
        try:
            out = torch.empty((1, cams[0].height, cams[0].width, 4), device="cuda")
            snp.render_views(h, cams, snp.make_opts(bg, sync_check=1), out)
            ref = out.clone()
            for _ in range(reps):
                out.fill_(float("nan"))
                snp.render_views(h, cams, snp.make_opts(bg, sync_check=0), out)
                torch.cuda.synchronize()
                assert torch.equal(out, ref), cfg
        finally:
            snp.destroy(h)


def _render_with_binning(scene, cams, bg, flags, colour_mode=0):
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    h = snp.create_scene(torch_scene(scene), 0)
    try:
        snp.set_binning(h, flags)
        V, H, W = len(cams), cams[0].height, cams[0].width
        out = torch.zeros((V, H, W, 4), device="cuda")
        snp.render_views(h, cams, snp.make_opts(bg, colour_mode=colour_mode), out)
        torch.cuda.synchronize()
        return out.cpu().numpy(), snp.get_stats(h)
    finally:
        snp.destroy(h)


@pytest.mark.parametrize("cfg", ["C1", "C2", "elongated"])
def test_tight_binning(orc, cfg):
    """§8(f)3 tight binning (snp_set_binning).  SNP_BIN_CONIC_TILES drops only tiles whose
    pixel centres the silhouette ellipse misses: the frame equals the rect binning's (up to
    an ulp on pixels that moved between K5 and K6), with fewer tested pairs.  With
    SNP_BIN_TILE_DEPTH as well (per-tile depth bounds: the per-ray order is unchanged, only
    when hits are emitted) the frame stays within the parity tolerance of the oracle."""
    if cfg == "elongated":   # thin diagonal primitives: their rects are mostly empty
        rng = np.random.default_rng(12)
        scene = synth.make_scene(12, 3000, box=0.8)
        s = rng.uniform(0.004, 0.01, (3000, 3)).astype(np.float32)
        s[:, 0] = rng.uniform(0.08, 0.25, 3000).astype(np.float32)
        scene.scales[:] = s
        cams = synth.orbit_cameras(2, 3.0, 320, 240, 300.0)
        bg = (0.1, 0.2, 0.3)
    else:
        scene, cams, bg = synth.make_config(cfg)
    ref, st0 = _render_with_binning(scene, cams, bg, 0)
    con, st1 = _render_with_binning(scene, cams, bg, 1)
    both, st3 = _render_with_binning(scene, cams, bg, 3)
    print(cfg, "dead keys", st1["dead_keys"], "of", st1["n_dup"], "tested", st0["tested_pairs"], "->",
          st1["tested_pairs"], "overflow", st0["overflow_pixels"], st1["overflow_pixels"], st3["overflow_pixels"])
    assert st0["dead_keys"] == 0 and st1["dead_keys"] > 0 and st1["n_dup"] == st0["n_dup"]
    # No hit is lost: the frame equals the rect binning's except for pixels that moved
    # between K5 and K6 (fewer records per batch move K5's emission points, and with them
    # which pixels overflow; the two paths may round the blend an ulp apart) -- and so do
    # K5's counters, which count an overflowing pixel's hits twice
    d = np.abs(con - ref)
    assert d.max() <= 2.5e-7 and (d.max(-1) > 0).sum() <= 4 * max(st0["overflow_pixels"], st1["overflow_pixels"]), \
        (d.max(), (d.max(-1) > 0).sum())
    assert st1["tested_pairs"] < st0["tested_pairs"]
    assert st3["dead_keys"] == st1["dead_keys"]
    assert np.abs(both - ref).max() <= 1e-5, np.abs(both - ref).max()
    # (and the oracle on the first view)
    img_o, fl, _ = orc.render_frame(scene, cams[0], bg)
    cmp_ = compare(both[0].reshape(-1, 4), img_o.reshape(-1, 4), fl.ravel())
    assert cmp_["max_unflagged"] <= TOL, cmp_


def test_tight_binning_deep_overlap(orc):
    """Tight binning on the deep-overlap scene (600 hits per pixel, K6 and the long pending
    lists): the per-tile depth bounds change when hits are emitted, never which or in
    what order, so the frame matches the rect binning's within 1e-5."""
    scene = _deep_scene(600)
    cam = synth.look_at((0, 0, 0), (1, 0, 0), 32, 24, 1600.0)
    ref, st0 = _render_with_binning(scene, [cam], (0.0, 0.0, 0.0), 0)
    both, st3 = _render_with_binning(scene, [cam], (0.0, 0.0, 0.0), 3)
    assert np.abs(both - ref).max() <= 1e-5


@pytest.mark.parametrize("colour_mode", [0, 1])
def test_backward_from_recorded_forward(colour_mode):
    """snp_set_record: the forward render records its composited hits and the backward
    forms dL/dI, dL/dc from them (no second traversal).  Same frame as without recording
    (bit-identical), and the same gradients as the gradient-mode traversal on every
    parameter (up to atomic order), on a C2-shaped 2-view frame with forced pending
    overflow (limit 3: K6 / the per-pixel K7 take those pixels from their recorded hits on)
    and on the dense grazing scene."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    rng = np.random.default_rng(93)
    cases = [(synth.make_scene(1, 2000, scale_mult=1.5, box=1.0), synth.orbit_cameras(2, 4.0, 160, 120, 220.0), 3)]
    n = 150
    sc = synth.make_scene(32, n, box=0.6)
    sc.centers[:] = rng.uniform(-0.4, 0.4, (n, 3)).astype(np.float32)
    sc.scales[:] = rng.uniform(0.04, 0.1, (n, 3)).astype(np.float32)
    sc.w2[:] = 0.0
    sc.b2[:] = (50.0 / sc.scales.max(1)).astype(np.float32)
    cases.append((sc, [synth.look_at((0.3, -3.0, 0.4), (0.0, 0.0, 0.0), 200, 150, 750.0)], 0))
    for scene, cams, limit in cases:
        V, H, W = len(cams), cams[0].height, cams[0].width
        G = torch.from_numpy(rng.normal(size=(V, H, W, 4)).astype(np.float32)).cuda()
        res, frames = {}, {}
        for record in (0, 1):
            h = snp.create_scene(torch_scene(scene), 0)
            try:
                snp.set_record(h, record)
                if limit:
                    snp.set_pending_limit(h, limit)
                opts = snp.make_opts((0.2, 0.3, 0.4), colour_mode=colour_mode)
                out = torch.zeros((V, H, W, 4), device="cuda")
                snp.render_views(h, cams, opts, out)
                grads = {f: torch.zeros(getattr(scene, f).shape, device="cuda") for f in snp.FIELDS}
                snp.render_backward(h, opts, G, grads, fwd_rgba=out)
                torch.cuda.synchronize()
                frames[record] = out.cpu().numpy()
                res[record] = {f: v.cpu().numpy().astype(np.float64) for f, v in grads.items()}
                if limit:
                    assert snp.get_stats(h)["overflow_pixels"] > 0
            finally:
                snp.destroy(h)
        assert np.array_equal(frames[0], frames[1])
        for f in snp.FIELDS:
            a, b = res[1][f], res[0][f]
            scale = np.abs(b).max()
            assert np.abs(a - b).max() <= 2e-4 * scale + 1e-7, (f, np.abs(a - b).max(), scale)


def test_loss_3dgs_parts_add_up():
    """snp_loss_3dgs_part: a step's views taken in two parts (as Trainer.step does per
    camera batch) give the loss and dL/d(out) of snp_loss_3dgs over the whole step."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    rng = np.random.default_rng(78)
    V, H, W = 5, 40, 52
    out = torch.from_numpy(rng.uniform(0, 1, (V, H, W, 4)).astype(np.float32)).cuda()
    tgt = torch.from_numpy(rng.uniform(0, 1, (V, H, W, 3)).astype(np.float32)).cuda()
    h = snp.create_scene(torch_scene(synth.make_scene(1, 4)), 0)
    try:
        g_all, l_all = torch.zeros_like(out), torch.zeros(1, device="cuda")
        snp.loss_3dgs(h, out, tgt, g_all, l_all, 0.2)
        g_p, l_p = torch.zeros_like(out), torch.zeros(1, device="cuda")
        for v0, v1 in ((0, 2), (2, 5)):
            snp.loss_3dgs(h, out[v0:v1], tgt[v0:v1], g_p[v0:v1], l_p, 0.2, step_views=V)
        torch.cuda.synchronize()
    finally:
        snp.destroy(h)
    assert abs(l_p.item() - l_all.item()) <= 1e-6 * abs(l_all.item())
    assert torch.equal(g_p, g_all)


def test_record_reuse_guards():
    """A record is used only by a backward of the same projection (and colour mode and
    transmittance floor): after a new projection the backward takes the gradient-mode
    traversal and gives that path's gradients."""
    import torch
    from paper_2510_08491_b200 import snp
    from gpu_util import torch_scene
    scene = synth.make_scene(3, 800, box=0.7)
    cams = synth.orbit_cameras(2, 3.0, 96, 72, 120.0)
    G = torch.from_numpy(np.random.default_rng(5).normal(size=(2, 72, 96, 4)).astype(np.float32)).cuda()
    opts = snp.make_opts((0.1, 0.1, 0.1))

    def grads_of(record, reproject):
        h = snp.create_scene(torch_scene(scene), 0)
        try:
            snp.set_record(h, record)
            out = torch.zeros((2, 72, 96, 4), device="cuda")
            snp.render_views(h, cams, opts, out)
            if reproject:   # a new projection (same cameras) drops the record
                snp.project(h, snp.make_cameras(cams))
                snp.bin_sort(h, opts)
            gr = {f: torch.zeros(getattr(scene, f).shape, device="cuda") for f in snp.FIELDS}
            snp.render_backward(h, opts, G, gr, fwd_rgba=out)
            torch.cuda.synchronize()
            return {f: v.cpu().numpy().astype(np.float64) for f, v in gr.items()}
        finally:
            snp.destroy(h)

    ref = grads_of(0, False)
    for record, reproject in ((1, True), (1, False)):
        got = grads_of(record, reproject)
        for f in snp.FIELDS:
            scale = np.abs(ref[f]).max()
            assert np.abs(got[f] - ref[f]).max() <= 2e-4 * scale + 1e-7, (record, reproject, f)
