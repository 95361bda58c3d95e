"""Pins for the oracle's binning definition (DESIGN.md "Binning definition",
SURVEY 8(c) step 11; readings R18, R19).

The paper has no tiles; what must hold is that binning never loses a hit and
that the depth key is a lower bound of every ray's entry depth:
  * conservativeness: every (pixel, primitive) hit found by brute-force exact
    intersection lies inside the primitive's pixel-centre rect (and tile rect);
  * tightness: the rect is within ~1 px of the true hit extent (in-frame prims);
  * L <= t_in for every hit;
  * emission/sort/ranges equal an independent Python construction with a
    stable library sort (np.argsort kind='stable').
"""
import numpy as np
import pytest

import synth


def _all_hits(orc, scene, cam, pixels):
    out = []
    for (x, y) in pixels:
        ids, ti, to = orc.pixel_hits(scene, cam, x, y)
        out.append((x, y, ids, ti))
    return out


@pytest.mark.parametrize("cfg", ["C1"])
def test_conservative_and_lower_bound_full_frame(orc, cfg):
    sc, cams, _ = synth.make_config(cfg)
    cam = cams[0]
    rects, prects, depth = orc.bin_view(sc, cam)
    L = depth.view(np.float32).astype(np.float64)
    W, H = cam.width, cam.height
    seen_x = {}
    for y in range(H):
        for x in range(W):
            ids, ti, _ = orc.pixel_hits(sc, cam, x, y)
            for i, t in zip(ids, ti):
                r = prects[i]
                assert r[0] >= 0, f"hit primitive {i} was culled"
                assert r[0] <= x <= r[2] and r[1] <= y <= r[3], (i, x, y, r)
                tr = rects[i]
                assert tr[0] <= x // 16 <= tr[2] and tr[1] <= y // 16 <= tr[3]
                assert L[i] <= t, (i, L[i], t)
                lo, hi = seen_x.get(i, (x, x))
                seen_x[i] = (min(lo, x), max(hi, x))
    assert len(seen_x) > 100


def test_bbox_is_the_exact_silhouette_extent(orc):
    """The pixel-centre rect equals the one implied by the true silhouette extent,
    measured by projecting dense samples of the ellipsoid surface (pinhole, no
    oracle code): ceil(x_min - 1/2 - eps) within the sampling error."""
    from scipy.spatial.transform import Rotation
    sc, cams, _ = synth.make_config("C1")
    cam = cams[0]
    _, prects, _ = orc.bin_view(sc, cam)
    Rw = cam.R_wc.astype(np.float64)
    Cw = cam.C_w.astype(np.float64)
    th, ph = np.meshgrid(np.linspace(0, np.pi, 300), np.linspace(0, 2 * np.pi, 600))
    u = np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], -1).reshape(-1, 3)
    fx, fy, cx, cy = (float(np.float32(v)) for v in (cam.fx, cam.fy, cam.cx, cam.cy))
    checked = 0
    for i in range(0, sc.n, 2):
        if prects[i, 0] <= 0 or prects[i, 2] >= cam.width - 1 or prects[i, 1] <= 0 or prects[i, 3] >= cam.height - 1:
            continue
        q = sc.rotations[i].astype(np.float64)
        R = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
        pts = sc.centers[i].astype(np.float64) + (u * sc.scales[i].astype(np.float64)) @ R.T
        pc = np.linalg.solve(Rw, (pts - Cw).T).T
        xs = fx * pc[:, 0] / pc[:, 2] + cx
        ys = fy * pc[:, 1] / pc[:, 2] + cy
        eps = 1.0 / 256
        for lo, hi, (a, b) in ((xs.min(), xs.max(), prects[i, [0, 2]]), (ys.min(), ys.max(), prects[i, [1, 3]])):
            assert np.ceil(lo - 0.5 - eps - 0.01) <= a <= np.ceil(lo - 0.5 - eps), (i, lo, a)
            assert np.floor(hi - 0.5 + eps) <= b <= np.floor(hi - 0.5 + eps + 0.01), (i, hi, b)
        checked += 1
    assert checked > 50


def test_conservative_sampled_360_scene(orc):
    """C3-shaped scene (reduced count so brute force stays cheap), random pixels."""
    sc, cams, _ = synth.make_config("C3", n=20000)
    cam = cams[0]
    rects, prects, depth = orc.bin_view(sc, cam)
    L = depth.view(np.float32).astype(np.float64)
    rng = np.random.default_rng(41)
    nh = 0
    for _ in range(60):
        x, y = int(rng.integers(cam.width)), int(rng.integers(cam.height))
        ids, ti, _ = orc.pixel_hits(sc, cam, x, y)
        for i, t in zip(ids, ti):
            r = prects[i]
            assert r[0] <= x <= r[2] and r[1] <= y <= r[3]
            assert L[i] <= t
            nh += 1
    assert nh > 20


def test_culled_primitives_never_hit(orc):
    """Primitives behind the camera / outside the frustum are culled and indeed never hit."""
    cam = synth.orbit_cameras(1, 4.0, 32, 24, 30.0)[0]
    sc = synth.make_scene(42, 400, box=6.0, rmin=0.5, rmax=1.5)   # scattered all around the camera
    rects, prects, depth = orc.bin_view(sc, cam)
    culled = set(np.nonzero(rects[:, 0] < 0)[0].tolist())
    assert len(culled) > 20
    for y in range(0, 24, 3):
        for x in range(0, 32, 3):
            ids, _, _ = orc.pixel_hits(sc, cam, x, y)
            assert not (set(ids.tolist()) & culled)


def _python_bin_sort(rects, depth, n, n_views, tx, ty, row_begin=0, row_stride=1):
    T = tx * ty
    tb = 0
    while (1 << tb) < T:
        tb += 1
    keys, ids = [], []
    for v in range(n_views):
        for i in range(n):
            r = rects[v * n + i]
            if r[0] < 0:
                continue
            for y in range(r[1], r[3] + 1):
                if y < row_begin or (y - row_begin) % row_stride:
                    continue
                for x in range(r[0], r[2] + 1):
                    keys.append((v << (tb + 19)) | ((y * tx + x) << 19) | (int(depth[v * n + i]) >> 12))
                    ids.append(i)
    keys = np.array(keys, np.uint64)
    ids = np.array(ids, np.uint32)
    o = np.argsort(keys, kind="stable")
    keys, ids = keys[o], ids[o]
    ranges = np.zeros((n_views * T, 2), np.uint32)
    slot = (keys >> np.uint64(19 + tb)) * np.uint64(T) + ((keys >> np.uint64(19)) & np.uint64((1 << tb) - 1))
    for s in np.unique(slot):
        w = np.nonzero(slot == s)[0]
        ranges[int(s)] = (w[0], w[-1] + 1)
    return keys, ids, ranges


@pytest.mark.parametrize("stripe", [(0, 1), (1, 2), (0, 3)])
def test_bin_sort_matches_python_stable_sort(orc, stripe):
    sc, cams, _ = synth.make_config("C1")
    cams = synth.orbit_cameras(3, 4.0, 128, 96, 150.0)
    rects, depth = [], []
    for c in cams:
        r, _, d = orc.bin_view(sc, c)
        rects.append(r); depth.append(d)
    rects = np.concatenate(rects); depth = np.concatenate(depth)
    tx, ty = orc.tiles_of(cams[0])
    k, i, rg = orc.bin_sort(rects, depth, sc.n, 3, tx, ty, *stripe)
    k2, i2, rg2 = _python_bin_sort(rects, depth, sc.n, 3, tx, ty, *stripe)
    assert np.array_equal(k, k2) and np.array_equal(i, i2) and np.array_equal(rg, rg2)
    assert np.all(np.diff(k.astype(np.uint64)) >= 0)


def test_stripes_partition_the_tiles(orc):
    sc, cams, _ = synth.make_config("C1")
    cam = cams[0]
    r, _, d = orc.bin_view(sc, cam)
    tx, ty = orc.tiles_of(cam)
    k, i, rg = orc.bin_sort(r, d, sc.n, 1, tx, ty)
    parts = [orc.bin_sort(r, d, sc.n, 1, tx, ty, b, 3) for b in range(3)]
    assert sum(len(p[0]) for p in parts) == len(k)
    for t in range(tx * ty):
        row = t // tx
        p = parts[row % 3]
        a = i[rg[t, 0]:rg[t, 1]]
        b = p[1][p[2][t, 0]:p[2][t, 1]]
        assert np.array_equal(a, b)


def test_tile_bits(orc):
    assert orc.tile_bits(1) == 0 and orc.tile_bits(2) == 1 and orc.tile_bits(64) == 6
    assert orc.tile_bits(65) == 7 and orc.tile_bits(4056) == 12


def test_empty_scene_bins_nothing(orc):
    cam = synth.orbit_cameras(1, 4.0, 32, 32, 30.0)[0]
    r, _, d = orc.bin_view(synth.empty_scene(), cam)
    k, i, rg = orc.bin_sort(r, d, 0, 1, 2, 2)
    assert len(k) == 0 and not rg.any()
