"""Pins for the oracle's view-dependent colour ("Spherical Harmonics",
P:394 "four bands ... Similar to 3DGS").  References: SPEC's printed values
(S:239-241), scipy's complex spherical harmonics (library routine), and exact
Gram orthonormality on a Gauss-Legendre x uniform-azimuth product rule."""
import math

import numpy as np
from scipy.special import sph_harm_y


def _real_sh_scipy(l, m, d):
    theta = math.acos(max(-1.0, min(1.0, d[2])))
    phi = math.atan2(d[1], d[0])
    if m == 0:
        return sph_harm_y(l, 0, theta, phi).real
    if m > 0:
        return math.sqrt(2) * sph_harm_y(l, m, theta, phi).real
    return math.sqrt(2) * sph_harm_y(l, -m, theta, phi).imag


def test_sh_basis_matches_scipy(orc):
    rng = np.random.default_rng(11)
    for _ in range(100):
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        Y = orc.sh_basis(d)
        i = 0
        for l in range(4):
            for m in range(-l, l + 1):
                assert abs(Y[i] - _real_sh_scipy(l, m, d)) < 1e-12, (l, m)
                i += 1


def test_sh_gram_orthonormal(orc):
    x, w = np.polynomial.legendre.leggauss(16)
    nphi = 32
    G = np.zeros((16, 16))
    for ct, wt in zip(x, w):
        st = math.sqrt(1 - ct * ct)
        for k in range(nphi):
            ph = 2 * math.pi * k / nphi
            Y = orc.sh_basis([st * math.cos(ph), st * math.sin(ph), ct])
            G += np.outer(Y, Y) * wt * (2 * math.pi / nphi)
    assert np.max(np.abs(G - np.eye(16))) < 1e-12


def test_sh_color_spec_examples(orc):
    sh = np.zeros((16, 3), np.float32)
    sh[0] = 1.0
    c = orc.sh_color(sh, [0.3, -0.4, math.sqrt(1 - 0.25)])
    assert np.allclose(c, 0.28209479177387814 + 0.5, atol=1e-15)        # S:239 "0.7820948"
    assert np.allclose(orc.sh_color(np.zeros((16, 3), np.float32), [0, 0, 1]), 0.5)
    sh = np.zeros((16, 3), np.float32)
    sh[2] = 0.25                                                          # degree-1, along z
    up, dn = orc.sh_color(sh, [0, 0, 1]), orc.sh_color(sh, [0, 0, -1])
    assert np.allclose(up - dn, 2 * 0.4886025119029199 * 0.25, atol=1e-15)
    sh = np.zeros((16, 3), np.float32)
    sh[0] = -5.0
    assert np.all(orc.sh_color(sh, [1, 0, 0]) == 0.0)                     # max(0, .) clamp (R15)


def test_sh_degree_truncation(orc):
    rng = np.random.default_rng(12)
    sh = rng.normal(size=(16, 3)).astype(np.float32)
    d = rng.normal(size=3); d /= np.linalg.norm(d)
    Y = orc.sh_basis(d)
    for deg in range(4):
        nc = (deg + 1) ** 2
        want = np.maximum(0.0, Y[:nc] @ sh[:nc].astype(np.float64) + 0.5)
        assert np.allclose(orc.sh_color(sh, d, degree=deg), want, atol=1e-14)
