"""Pins for the oracle renderer: ordering + compositing (Eq. 4, P:169-180,
P:364) around the per-ray kernel.

References: SPEC's closed-form blends, a T-floor stop case worked by
hand, Eq. 2 ray-marching (reading R20) with 10^5
samples per segment on per-ray-disjoint scenes (north_star: "within 1e-6"),
zero density outside the ellipsoid (north_star), alpha in [0,1] and
non-increasing transmittance (north_star), occlusion monotonicity and energy
bound, determinism across thread counts, and exact
translation equivariance."""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import synth

C0 = 0.28209479177387814
LN2 = math.log(2.0)


def _prims(specs, N=8):
    """specs: list of dict(mu, s, q=(1,0,0,0), W1, b1, W2, b2, rgb or sh)."""
    n = len(specs)
    sc = synth.empty_scene(N)
    if n == 0:
        return sc
    f = lambda k, shape, default: np.array([np.asarray(p.get(k, default), np.float64).reshape(shape)  # noqa
                                            for p in specs], np.float32)
    sh = np.zeros((n, 16, 3), np.float32)
    for i, p in enumerate(specs):
        if "sh" in p:
            sh[i] = p["sh"]
        else:
            sh[i, 0] = (np.asarray(p.get("rgb", (0.5, 0.5, 0.5))) - 0.5) / C0
    return synth.Scene(f("mu", (3,), 0), f("q", (4,), (1, 0, 0, 0)), f("s", (3,), 1),
                       f("W1", (N, 3), np.zeros((N, 3))), f("b1", (N,), np.zeros(N)),
                       f("W2", (N,), np.zeros(N)), f("b2", (), 0.0), sh)


def _colour(sc, i):
    return C0 * sc.sh[i, 0].astype(np.float64) + 0.5


def _axis_cam(W=1, H=1, fx=100.0):
    return synth.Camera(np.eye(3, dtype=np.float32), np.zeros(3, np.float32), fx, fx,
                        W / 2.0, H / 2.0, W, H)


def _px(orc, sc, cam, bg=(0, 0, 0), **kw):
    out, fl, st = orc.render_pixels(sc, cam, [0], [0], bg, **kw)
    return out[0], fl[0], st[0]


def test_empty_scene_is_background(orc):
    cam = _axis_cam(4, 3)
    img, fl, st = orc.render_frame(synth.empty_scene(), cam, bg=(0.25, 0.5, 1.0))
    assert np.all(img[..., :3] == np.array([0.25, 0.5, 1.0])) and np.all(img[..., 3] == 0)


def test_single_and_two_primitive_blends(orc):
    r = 1.0
    beta = LN2 / (2 * r)    # chord 2r through the centre -> I = ln 2 -> kappa = 0.5
    a = dict(mu=(0, 0, 5), s=(r, r, r), b2=beta, rgb=(0.9, 0.2, 0.1))
    b = dict(mu=(0, 0, 10), s=(r, r, r), b2=beta, rgb=(0.1, 0.8, 0.3))
    cam = _axis_cam()
    bg = np.array([0.0, 0.0, 1.0])
    sc = _prims([a])
    out, _, _ = _px(orc, sc, cam, bg=(0, 0, 0))
    assert np.allclose(out[:3], 0.5 * _colour(sc, 0), atol=1e-7)
    assert abs(out[3] - 0.5) < 1e-7
    for order in ([a, b], [b, a]):   # primitive index order must not matter
        sc = _prims(order)
        ia, ib = (0, 1) if order[0] is a else (1, 0)
        out, _, st = _px(orc, sc, cam, bg=tuple(bg))
        want = 0.5 * _colour(sc, ia) + 0.25 * _colour(sc, ib) + 0.25 * bg
        assert np.allclose(out[:3], want, atol=1e-7), (out, want)
        assert abs(out[3] - 0.75) < 1e-7 and st[0] == 2 and st[1] == 2


def test_transmittance_floor_stop(orc):
    """kappa = 0.95 layers: T = 0.05^k; T after 3 = 1.25e-4 >= 1e-4, after 4 < 1e-4 -> stop."""
    r = 0.5
    beta = -math.log(0.05) / (2 * r)
    rgbs = [(0.9, 0.1, 0.1), (0.1, 0.9, 0.1), (0.1, 0.1, 0.9), (0.6, 0.6, 0.1), (1.0, 1.0, 1.0), (1, 1, 1)]
    specs = [dict(mu=(0, 0, 3 + 2 * i), s=(r, r, r), b2=beta, rgb=c) for i, c in enumerate(rgbs)]
    sc = _prims(specs[::-1])           # reversed index order
    cam = _axis_cam()
    bg = np.array([0.3, 0.3, 0.3])
    out, fl, st = _px(orc, sc, cam, bg=tuple(bg))
    n = len(specs)
    kap = 1 - math.exp(-2 * r * np.float32(beta))
    T, C = 1.0, np.zeros(3)
    for i in range(4):
        C += T * kap * _colour(sc, n - 1 - i)
        T *= 1 - kap
    assert np.allclose(out[:3], C + T * bg, atol=1e-7)
    assert st[1] == 4 and st[0] == 6


def _bisect_segment(o, d, mu, R, s, t_lo, t_hi, iters=200):
    """Boundaries of the ellipsoid along the ray by sign-change bisection (no quadratic solve)."""
    def f(t):
        y = (R.T @ (o + t * d - mu)) / s
        return y @ y - 1.0
    ts = np.linspace(t_lo, t_hi, 4001)
    vals = np.array([f(t) for t in ts])
    idx = np.nonzero(np.sign(vals[:-1]) != np.sign(vals[1:]))[0]
    out = []
    for i in idx:
        a, b = ts[i], ts[i + 1]
        fa = f(a)
        for _ in range(iters):
            m = 0.5 * (a + b)
            fm = f(m)
            if np.sign(fm) == np.sign(fa):
                a, fa = m, fm
            else:
                b = m
        out.append(0.5 * (a + b))
    return out


def _density(x, p, omega=30.0):
    y = (x - p["mu"]) / p["smax"]
    return np.cos(omega * (y @ p["W1"].T + p["b1"])) @ p["W2"] + p["b2"]


def _raymarch_pixel(o, d, prims, bg, nsamp=100_000):
    """Eq. 2 over the hit segments (empty space skipped), per-sample colour = the
    containing primitive's colour.  Segments are per-ray disjoint by construction."""
    segs = []
    for p in prims:
        tc = (p["mu"] - o) @ d
        b = _bisect_segment(o, d, p["mu"], p["R"], p["s"], max(0.0, tc - 1.5 * p["smax"]), tc + 1.5 * p["smax"])
        if len(b) == 2:
            segs.append((b[0], b[1], p))
    segs.sort(key=lambda z: z[0])
    logT, C = 0.0, np.zeros(3)
    for a, b, p in segs:
        h = (b - a) / nsamp
        t = a + (np.arange(nsamp) + 0.5) * h
        sig = _density(o[None] + t[:, None] * d[None], p)
        x = sig * h
        cum = np.concatenate([[0.0], np.cumsum(x)[:-1]])
        C += p["rgb"] * np.sum(np.exp(-(logT + cum)) * (1 - np.exp(-x)))   # Eq. 2 (R20)
        logT += x.sum()
    T = math.exp(-logT)
    return C + T * np.asarray(bg), 1 - T, [s[2] for s in segs]


def test_disjoint_scene_matches_eq2_raymarch(orc):
    rng = np.random.default_rng(21)
    specs, plist = [], []
    for k in range(5):
        s = rng.uniform(0.3, 0.7, 3)
        mu = np.array([rng.uniform(-0.2, 0.2), rng.uniform(-0.2, 0.2), 3.0 + 2.0 * k])
        q = rng.normal(size=4); q /= np.linalg.norm(q)
        W1 = rng.uniform(-1 / 3, 1 / 3, (8, 3)); b1 = rng.uniform(-1, 1, 8)
        W2 = rng.uniform(-1, 1, 8) * 0.5 / s.max(); b2 = rng.uniform(0.8, 2.0) / s.max()
        rgb = rng.uniform(0.05, 0.95, 3)
        specs.append(dict(mu=mu, s=s, q=q, W1=W1, b1=b1, W2=W2, b2=b2, rgb=rgb))
    sc = _prims(specs)
    for i in range(sc.n):    # use the exact fp32 values the oracle sees
        q = sc.rotations[i].astype(np.float64)
        plist.append(dict(mu=sc.centers[i].astype(np.float64), s=sc.scales[i].astype(np.float64),
                          smax=float(sc.scales[i].max()),
                          R=Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix(),
                          W1=sc.w1[i].astype(np.float64), b1=sc.b1[i].astype(np.float64),
                          W2=sc.w2[i].astype(np.float64), b2=float(sc.b2[i]), rgb=_colour(sc, i)))
    cam = _axis_cam(6, 6, fx=60.0)
    bg = (0.2, 0.4, 0.6)
    img, fl, st = orc.render_frame(sc, cam, bg=bg, t_floor=1e-30)
    checked = 0
    for y in range(6):
        for x in range(6):
            o, d = orc.pixel_ray(cam, x, y)
            rgb, op, hit = _raymarch_pixel(o, d, plist, bg)
            # Eq. 4 == Eq. 2 only when every primitive integral is >= 0 (no clamp)
            ok = all(orc.integral(o, d, *_seg(orc, o, d, p), p["mu"], p["smax"], p["W1"], p["b1"],
                                  p["W2"], p["b2"]) >= 0 for p in hit)
            if not ok:
                continue
            checked += 1
            assert np.max(np.abs(img[y, x, :3] - rgb)) < 1e-6, (x, y)
            assert abs(img[y, x, 3] - op) < 1e-6
    assert checked >= 20


def _seg(orc, o, d, p):
    q = Rotation.from_matrix(p["R"]).as_quat()
    hit, ti, to, _ = orc.intersect(o, d, 0.0, 1e4, p["mu"], [q[3], q[0], q[1], q[2]], p["s"])
    assert hit
    return ti, to


def test_zero_density_outside_ellipsoid(orc):
    """north_star: marching the WHOLE ray with sigma := 0 outside E reproduces the
    closed form over [t_in, t_out]; rays that miss E get kappa = 0 whatever the MLP."""
    rng = np.random.default_rng(22)
    mu = np.array([0.1, -0.2, 4.0]); s = np.array([0.6, 0.3, 0.45])
    q = rng.normal(size=4); q /= np.linalg.norm(q)
    R = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
    W1 = rng.uniform(-1 / 3, 1 / 3, (8, 3)); b1 = rng.uniform(-1, 1, 8)
    W2 = rng.uniform(-1, 1, 8) * 0.5 / 0.6; b2 = 1.5 / 0.6
    p = dict(mu=mu, smax=0.6, W1=W1, b1=b1, W2=W2, b2=b2)
    o = np.zeros(3)
    for _ in range(10):
        d = np.array([rng.uniform(-0.1, 0.1), rng.uniform(-0.1, 0.1), 1.0]); d /= np.linalg.norm(d)
        hit, ti, to, _ = orc.intersect(o, d, 0.01, 1e4, mu, q, s)
        n = 400_000
        t = 0.01 + (np.arange(n) + 0.5) * (8.0 - 0.01) / n
        x = o[None] + t[:, None] * d[None]
        y = ((x - mu) @ R) / s
        inside = np.einsum("ij,ij->i", y, y) < 1.0
        Iq = np.sum(np.where(inside, _density(x, p), 0.0)) * (8.0 - 0.01) / n
        if hit:
            I = orc.integral(o, d, ti, to, mu, 0.6, W1, b1, W2, b2)
            # boundary discontinuities cost O(h sigma) each with the midpoint rule
            assert abs(I - Iq) < 4 * (8.0 / n) * (abs(b2) + np.abs(W2).sum()), (I, Iq)
        else:
            assert not inside.any()
    # a miss contributes nothing: the pixel is exactly background
    sc = _prims([dict(mu=(5, 5, 4), s=(0.5, 0.5, 0.5), W1=W1, b1=b1, W2=W2 * 100, b2=100.0)])
    out, _, st = _px(orc, sc, _axis_cam(), bg=(0.1, 0.2, 0.3))
    bg32 = np.array([0.1, 0.2, 0.3], np.float32).astype(np.float64)   # the ABI carries fp32
    assert np.all(out[:3] == bg32) and out[3] == 0.0 and st[0] == 0


def _random_scene(seed, n=40, dc_only=False):
    sc = synth.make_scene(seed, n, box=0.6)
    if dc_only:
        rng = np.random.default_rng(seed)
        sc.sh[:] = 0
        sc.sh[:, 0, :] = ((rng.uniform(0, 1, (n, 3)) - 0.5) / C0).astype(np.float32)
    return sc


def test_alpha_range_and_transmittance_non_increasing(orc):
    sc = _random_scene(31, 60)
    cams = synth.orbit_cameras(1, 4.0, 24, 24, 40.0)
    rng = np.random.default_rng(32)
    base, _, _ = orc.render_frame(sc, cams[0], t_floor=1e-300)
    assert np.all(base[..., 3] >= 0) and np.all(base[..., 3] <= 1)
    for _ in range(5):
        keep = np.sort(rng.choice(sc.n, sc.n // 2, replace=False))
        sub, _, _ = orc.render_frame(sc.subset(keep), cams[0], t_floor=1e-300)
        assert np.all(sub[..., 3] <= base[..., 3] + 1e-12)   # more primitives -> T never rises


def test_energy_bound_and_occlusion(orc):
    sc = _random_scene(33, 60, dc_only=True)
    cam = synth.orbit_cameras(1, 4.0, 24, 24, 40.0)[0]
    img, _, _ = orc.render_frame(sc, cam, bg=(1.0, 0.5, 0.0))
    assert img[..., :3].min() >= 0 and img[..., :3].max() <= 1 + 1e-12
    # occluder: huge opaque sphere between camera and scene, colour c -> every pixel == c
    C = np.asarray(cam.C_w, np.float64)
    mu = C * 0.6
    occ = _prims([dict(mu=mu, s=(2.5, 2.5, 2.5), b2=200.0, rgb=(0.3, 0.7, 0.2))])
    both = synth.concat_scenes(sc, occ)
    img2, _, _ = orc.render_frame(both, cam, bg=(1.0, 0.5, 0.0))
    c = _colour(occ, 0)
    assert np.max(np.abs(img2[..., :3] - c)) < 1e-6


def test_determinism_across_threads(orc):
    sc, cams, bg = synth.make_config("C1")
    a, fa, sa = orc.render_frame(sc, cams[0], bg, nthreads=1)
    b, fb, sb = orc.render_frame(sc, cams[0], bg, nthreads=4)
    assert np.array_equal(a, b) and np.array_equal(fa, fb) and np.array_equal(sa, sb)


def test_translation_equivariance_exact(orc):
    """Centres and camera on a 2^-12 grid, shift by a dyadic vector: fp32 inputs stay
    exact, so the double oracle must give the same image."""
    sc = _random_scene(34, 50)
    sc.centers = (np.round(sc.centers * 4096) / 4096).astype(np.float32)
    cam = synth.orbit_cameras(1, 4.0, 16, 16, 25.0)[0]
    cam.C_w = (np.round(cam.C_w.astype(np.float64) * 4096) / 4096).astype(np.float32)
    a, _, _ = orc.render_frame(sc, cam)
    c = np.array([0.5, -1.25, 2.0], np.float32)
    sc2 = sc.subset(np.arange(sc.n))
    sc2.centers = sc.centers + c
    cam.C_w = cam.C_w + c
    b, _, _ = orc.render_frame(sc2, cam)
    assert np.max(np.abs(a - b)) < 1e-12


@pytest.mark.parametrize("bad", ["q", "s"])
def test_invalid_scene_rejected(orc, bad):
    sc = _random_scene(35, 4)
    if bad == "q":
        sc.rotations[1] = 0
    else:
        sc.scales[2, 1] = 0
    with pytest.raises(ValueError):
        orc.render_pixels(sc, _axis_cam(), [0], [0])


def test_colour_per_ray(orc):
    """with colour_per_ray the SH colour is taken at each pixel's own
    ray direction.  One primitive of constant density in front of an axis camera:
    out_rgb / alpha is the colour, which must equal SH(d) for d built here from the
    pinhole model (x + 0.5 - cx) / fx, (y + 0.5 - cy) / fy, 1 (SH basis pinned against
    scipy in test_oracle_colour); at the pixel whose ray passes through mu the two modes
    agree, elsewhere they differ; at SH degree 0 the modes give identical images."""
    rng = np.random.default_rng(12)
    sh = rng.normal(0, 0.3, (16, 3))
    W, H, fx = 9, 7, 20.0
    cam = _axis_cam(W, H, fx)
    px0, py0 = 6, 2                     # mu on this pixel's ray
    d0 = np.array([(px0 + 0.5 - W / 2.0) / fx, (py0 + 0.5 - H / 2.0) / fx, 1.0])
    sc = _prims([dict(mu=5.0 * d0, s=(1.5, 1.5, 1.5), b2=0.4, sh=sh)])
    sc.sh_degree = 3
    ray, fl, _ = orc.render_frame(sc, cam, colour_per_ray=True)
    prim, _, _ = orc.render_frame(sc, cam)
    assert not fl.any()
    yy, xx = np.mgrid[0:H, 0:W]
    hit = ray[..., 3] > 0
    assert hit.sum() > 20
    for y, x in zip(yy[hit], xx[hit]):
        d = np.array([(x + 0.5 - W / 2.0) / fx, (y + 0.5 - H / 2.0) / fx, 1.0])
        d /= np.linalg.norm(d)
        c = orc.sh_color(sh, d, 3)
        assert np.allclose(ray[y, x, :3] / ray[y, x, 3], c, rtol=1e-12, atol=1e-12), (x, y)
    assert np.allclose(ray[py0, px0], prim[py0, px0], rtol=1e-12, atol=1e-14)
    assert np.abs(ray - prim)[hit].max() > 1e-3
    sc.sh_degree = 0
    a, _, _ = orc.render_frame(sc, cam, colour_per_ray=True)
    b, _, _ = orc.render_frame(sc, cam)
    assert np.array_equal(a, b)


def test_temporal_density(orc):
    """Temporal scenes (appendix "Dynamic scenes"; P:289 time as an extra network input,
    reading R24): at a view's timestamp xi_t the phase of unit k is
    omega (W1_k . x^ + xi_t W_t,k + b1_k).  Pins: xi_t = 0 reproduces the static image
    bit for bit; a single primitive's alpha equals 1 - exp(-I) with I from midpoint
    quadrature of that density along the pixel ray (10^5 samples, 1e-6)."""
    rng = np.random.default_rng(13)
    N = 8
    W1 = rng.uniform(-1 / 3, 1 / 3, (N, 3))
    b1 = rng.uniform(-1, 1, N)
    W2 = rng.uniform(-1, 1, N) * 0.3
    sc = _prims([dict(mu=(0.1, -0.05, 4.0), s=(0.8, 0.5, 0.6), q=(0.9, 0.2, -0.3, 0.1), W1=W1, b1=b1,
                      W2=W2, b2=0.6)])
    sc.w_t = rng.uniform(-1, 1, (1, N)).astype(np.float32)
    cam = _axis_cam(5, 5, 12.0)
    static = synth.Scene(*(getattr(sc, f) for f in synth.scenes._FIELDS), omega=sc.omega)
    a, _, _ = orc.render_frame(static, cam)
    b, _, _ = orc.render_frame(sc, cam)
    assert np.array_equal(a, b)
    cam.xi_t = 0.75
    img, fl, st = orc.render_frame(sc, cam)
    assert not fl.any() and np.abs(img - a).max() > 1e-3
    xi = float(np.float32(0.75))
    smax = float(np.float32(0.8))
    mu = np.array([0.1, -0.05, 4.0], np.float32).astype(np.float64)
    W1f, b1f, W2f = (np.asarray(v, np.float32).astype(np.float64) for v in (W1, b1, W2))
    wt = sc.w_t[0].astype(np.float64)
    checked = 0
    for y in range(5):
        for x in range(5):
            ids, ti, to = orc.pixel_hits(sc, cam, x, y)
            if len(ids) == 0:
                assert img[y, x, 3] == 0.0
                continue
            o, d = orc.pixel_ray(cam, x, y)
            n = 100_000
            t = ti[0] + (np.arange(n) + 0.5) * (to[0] - ti[0]) / n
            xh = (o[None] + t[:, None] * d[None] - mu) / smax
            sig = np.cos(OMEGA_ * (xh @ W1f.T + b1f + xi * wt)) @ W2f + float(np.float32(0.6))
            I = sig.sum() * (to[0] - ti[0]) / n
            assert abs(img[y, x, 3] - (1.0 - math.exp(-max(I, 0.0)))) < 1e-6, (x, y)
            checked += 1
    assert checked >= 9


OMEGA_ = 30.0
