"""Pins for the oracle's geometry: quaternion rotation, pixel rays and the
analytic line-ellipsoid intersection.  Each check is against
something other than the oracle's own formula: SPEC worked examples,
scipy's Rotation, sign-change bisection of the implicit function, and
equivariance properties."""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def test_quat_identity_and_axis(orc):
    assert np.allclose(orc.quat_to_rot([1, 0, 0, 0]), np.eye(3), atol=0)
    R = orc.quat_to_rot([math.sqrt(0.5), 0, 0, math.sqrt(0.5)])   # 90 deg about z
    assert np.allclose(R @ [1, 0, 0], [0, 1, 0], atol=1e-15)


def test_quat_matches_scipy_and_normalises(orc):
    rng = np.random.default_rng(1)
    for _ in range(200):
        q = rng.normal(size=4) * rng.uniform(0.1, 10)
        R = orc.quat_to_rot(q)
        Rs = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()  # scipy is scalar-last
        assert np.max(np.abs(R - Rs)) < 1e-14
    with pytest.raises(ValueError):
        orc.quat_to_rot([0, 0, 0, 0])


def _cam(W=64, H=48, fx=50.0, fy=55.0, cx=None, cy=None, R=None, C=(0, 0, 0)):
    R = np.eye(3, dtype=np.float32) if R is None else np.asarray(R, np.float32)
    return synth.Camera(R, np.asarray(C, np.float32), fx, fy, W / 2 if cx is None else cx,
                        H / 2 if cy is None else cy, W, H)


def test_pixel_ray_examples(orc):
    cam = _cam(cx=10.5, cy=20.5)           # pixel (10,20) centre sits on the principal point
    o, d = orc.pixel_ray(cam, 10, 20)
    assert np.allclose(d, [0, 0, 1], atol=0) and np.allclose(o, 0)
    cam = _cam(fx=50.0, cx=10.5 - 50.0, cy=20.5)   # cx offset by fx -> (1,0,1)/sqrt2
    _, d = orc.pixel_ray(cam, 10, 20)
    assert np.allclose(d, np.array([1, 0, 1]) / math.sqrt(2), atol=1e-15)


def test_pixel_ray_reprojection(orc):
    """A point at depth z on the ray projects back to the pixel centre (pinhole)."""
    rng = np.random.default_rng(2)
    Rw = Rotation.random(random_state=3).as_matrix().astype(np.float32)
    cam = _cam(W=200, H=100, fx=120.0, fy=130.0, cx=97.3, cy=51.1, R=Rw, C=(1.0, -2.0, 0.5))
    Rw64 = Rw.astype(np.float64)
    for _ in range(50):
        x, y = rng.integers(0, 200), rng.integers(0, 100)
        o, d = orc.pixel_ray(cam, x, y)
        assert abs(np.linalg.norm(d) - 1) < 1e-15
        p = o + 3.7 * d
        # the fp32 R_wc is the linear map the ray goes through; invert it exactly
        pc = np.linalg.solve(Rw64, p - np.asarray(cam.C_w, np.float64))
        u = np.float32(cam.fx) * pc[0] / pc[2] + np.float32(cam.cx)
        v = np.float32(cam.fy) * pc[1] / pc[2] + np.float32(cam.cy)
        assert abs(u - (x + 0.5)) < 1e-9 and abs(v - (y + 0.5)) < 1e-9


def test_intersect_spec_examples(orc):
    I4 = [1, 0, 0, 0]
    hit, ti, to, _ = orc.intersect([-2, 0, 0], [1, 0, 0], 0, 100, [0, 0, 0], I4, [1, 1, 1])
    assert hit and ti == 1.0 and to == 3.0
    hit, *_ = orc.intersect([-2, 2, 0], [1, 0, 0], 0, 100, [0, 0, 0], I4, [1, 1, 1])
    assert not hit
    qz = [math.sqrt(0.5), 0, 0, math.sqrt(0.5)]
    hit, ti, to, _ = orc.intersect([0, -5, 0], [0, 1, 0], 0, 100, [0, 0, 0], qz, [2, 1, 1])
    assert hit and abs(ti - 3) < 1e-14 and abs(to - 7) < 1e-14
    hit, ti, to, _ = orc.intersect([0, 0, 0], [1, 0, 0], 0, 100, [0, 0, 0], I4, [1, 1, 1])
    assert hit and ti == 0.0 and to == 1.0                                  # S:74 (clipped entry)
    hit, *_ = orc.intersect([-2, 0, 0], [1, 0, 0], 0, 0.5, [0, 0, 0], I4, [1, 1, 1])
    assert not hit                                                          # segment ends before entry


def _implicit(x, mu, R, s):
    y = (R.T @ (x - mu)) / s
    return y @ y - 1.0


def _bisect_boundaries(o, d, mu, R, s, tmax, n=20000):
    ts = np.linspace(0.0, tmax, n)
    pts = o[None] + ts[:, None] * d[None]
    y = ((pts - mu) @ R) / s
    f = np.einsum("ij,ij->i", y, y) - 1.0
    out = []
    for i in np.nonzero(np.sign(f[:-1]) != np.sign(f[1:]))[0]:
        a, b = ts[i], ts[i + 1]
        fa = _implicit(o + a * d, mu, R, s)
        for _ in range(100):
            m = 0.5 * (a + b)
            fm = _implicit(o + m * d, mu, R, s)
            if np.sign(fm) == np.sign(fa):
                a, fa = m, fm
            else:
                b = m
        out.append(0.5 * (a + b))
    return out


def test_intersect_vs_sign_change_bisection(orc):
    """analytic roots agree with sign changes of the implicit function."""
    rng = np.random.default_rng(4)
    n_hit = 0
    for _ in range(300):
        mu = rng.uniform(-1, 1, 3)
        s = np.exp(rng.uniform(np.log(0.1), np.log(2.0), 3))
        q = rng.normal(size=4)
        R = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
        o = mu + rng.normal(size=3) * 6.0
        if rng.uniform() < 0.7:   # aim at a point inside E (mostly hits)
            u = rng.normal(size=3); u *= rng.uniform(0, 0.95) / np.linalg.norm(u)
            target = mu + R @ (s * u)
        else:
            target = mu + rng.normal(size=3) * s.max()
        d = target - o
        d /= np.linalg.norm(d)
        tmax = np.linalg.norm(target - o) + 3 * s.max()
        hit, ti, to, _ = orc.intersect(o, d, 0.0, 1e4, mu, q, s)
        roots = _bisect_boundaries(o, d, mu, R, s, tmax)
        if len(roots) == 2 and roots[1] - roots[0] > 1e-3 * s.max():
            n_hit += 1
            assert hit
            tol = 1e-7 * (1 + tmax)
            assert abs(ti - roots[0]) < tol and abs(to - roots[1]) < tol
            mid = o + 0.5 * (ti + to) * d
            assert _implicit(mid, mu, R, s) < 0          # S:77 midpoint strictly inside
        elif len(roots) == 0:
            assert not hit
    assert n_hit > 100


def test_intersect_equivariance(orc):
    """translating / rotating ellipsoid and ray together leaves (t_in, t_out) unchanged."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        mu = rng.uniform(-1, 1, 3)
        s = np.exp(rng.uniform(np.log(0.2), np.log(2.0), 3))
        q = rng.normal(size=4)
        o = mu + rng.normal(size=3) * 4
        d = (mu + rng.normal(size=3) * 0.5 * s.max()) - o
        d /= np.linalg.norm(d)
        base = orc.intersect(o, d, 0.0, 1e4, mu, q, s)
        c = rng.normal(size=3) * 10
        sh = orc.intersect(o + c, d, 0.0, 1e4, mu + c, q, s)
        assert base[0] == sh[0]
        if base[0]:
            assert abs(base[1] - sh[1]) < 1e-9 and abs(base[2] - sh[2]) < 1e-9
        Rr = Rotation.random(random_state=int(rng.integers(1 << 30)))
        qr = Rr.as_quat()                      # (x,y,z,w)
        qn = q / np.linalg.norm(q)
        qc = (Rr * Rotation.from_quat([qn[1], qn[2], qn[3], qn[0]])).as_quat()
        rot = orc.intersect(Rr.apply(o), Rr.apply(d), 0.0, 1e4, Rr.apply(mu),
                            [qc[3], qc[0], qc[1], qc[2]], s)
        assert base[0] == rot[0]
        if base[0]:
            assert abs(base[1] - rot[1]) < 1e-7 and abs(base[2] - rot[2]) < 1e-7
        del qr
