"""Pins for the oracle's closed-form line integral (Eq. 7-8) and
kernel (Eq. 9).

Independent references: brute-force midpoint quadrature of the pointwise
density of Eq. 5-6 (10^5..2x10^5 samples; BASELINE north_star "brute-force
ray-marching quadrature ... within 1e-6"), the constant-density closed form
(density x chord, north_star), the h -> 0 limit, additivity and
origin-shift invariance, the literal Eq. 8 difference form,
and the printed kernel values."""
import math

import numpy as np
import pytest

OMEGA = 30.0


def _density_np(x, mu, smax, W1, b1, W2, b2, omega=OMEGA):
    """Eq. 5-6 evaluated pointwise (vectorised over x[...,3])."""
    y = (x - mu) / smax
    z = y @ W1.T + b1
    return np.cos(omega * z) @ W2 + b2


def _rand_prim(rng, trained=True, N=8):
    mu = rng.uniform(-1, 1, 3)
    s = np.exp(rng.uniform(np.log(0.1), np.log(10.0), 3))
    smax = s.max()
    W1 = rng.uniform(-1 / 3, 1 / 3, (N, 3))
    b1 = rng.uniform(-1, 1, N)
    W2 = rng.uniform(-1, 1, N) * (0.5 / smax if trained else math.sqrt(6 / N) / OMEGA)
    b2 = rng.uniform(0.2, 2.0) / smax
    return mu, s, smax, W1, b1, W2, b2


def test_density_spec_examples(orc):
    # S:140 "W2 = 0, b2 = 5 -> density 5"; S:141 single unit at x^ = 0 -> cos(0) = 1
    W1 = np.zeros((8, 3)); b1 = np.zeros(8); W2 = np.zeros(8)
    assert orc.density([0.3, -0.2, 0.1], [0, 0, 0], 1.0, W1, b1, W2, 5.0) == 5.0
    W1 = np.array([[1.0, 0, 0]]); b1 = np.zeros(1); W2 = np.ones(1)
    assert orc.density([0.0, 0.7, -0.4], [0, 0, 0], 2.0, W1, b1, W2, 0.0, omega=30.0) == 1.0
    # Eq. 5 uses ||s||_inf with no rotation: x = mu + (2,0,0), s=(2,1,.5) -> x^ = (1,0,0)
    W1 = np.array([[1.0, 0, 0]]); W2 = np.ones(1)
    v = orc.density([2.0, 0, 0], [0, 0, 0], 2.0, W1, np.zeros(1), W2, 0.0, omega=1.0)
    assert abs(v - math.cos(1.0)) < 1e-15


@pytest.mark.parametrize("N", [8, 4, 16, 32])
def test_integral_vs_bruteforce_quadrature(orc, N):
    """Eq. 8 closed form vs midpoint quadrature of Eq. 6, for the paper's width and the
    other supported widths N_sigma."""
    rng = np.random.default_rng(7 + N)
    worst = 0.0
    for case in range(60 if N == 8 else 20):
        mu, s, smax, W1, b1, W2, b2 = _rand_prim(rng, trained=case % 2 == 0, N=N)
        o = mu + rng.normal(size=3) * 5 * smax
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        t_in = rng.uniform(0, 3 * smax)
        t_out = t_in + rng.uniform(0.01, 2.0) * smax
        I = orc.integral(o, d, t_in, t_out, mu, smax, W1, b1, W2, b2)
        n = 200_000
        t = t_in + (np.arange(n) + 0.5) * (t_out - t_in) / n
        Iq = _density_np(o[None] + t[:, None] * d[None], mu, smax, W1, b1, W2, b2).sum() * (t_out - t_in) / n
        err = abs(I - Iq) / (1 + abs(Iq))
        worst = max(worst, err)
    assert worst < 1e-6, worst


def test_constant_density_chord(orc):
    """W2 = 0: I = b2 * chord, chord of a sphere = 2 sqrt(r^2 - b^2)."""
    rng = np.random.default_rng(8)
    for _ in range(50):
        r = rng.uniform(0.1, 3)
        bimp = rng.uniform(0, 0.95) * r
        o = np.array([-10.0, bimp, 0.0]); d = np.array([1.0, 0, 0]); mu = np.zeros(3)
        hit, ti, to, _ = orc.intersect(o, d, 0.0, 1e4, mu, [1, 0, 0, 0], [r, r, r])
        chord = 2 * math.sqrt(r * r - bimp * bimp)
        assert hit and abs((to - ti) - chord) < 1e-12 * (1 + r)
        beta = rng.uniform(0.1, 5)
        W1 = rng.uniform(-1 / 3, 1 / 3, (8, 3))
        I = orc.integral(o, d, ti, to, mu, r, W1, rng.uniform(-1, 1, 8), np.zeros(8), beta)
        assert abs(I - beta * chord) < 1e-12 * (1 + beta * chord)


def test_h_zero_limit(orc):
    """W1 row (0,0,1), ray along x -> h = 0, I = dt (W2 cos(w(W1.o^ + b1)) + b2)."""
    W1 = np.array([[0.0, 0.0, 1.0]]); b1 = np.array([0.3]); W2 = np.array([0.7]); b2 = 0.2
    o = np.array([-3.0, 0.1, 0.4]); d = np.array([1.0, 0, 0]); mu = np.array([0.0, 0.0, 0.1])
    smax = 1.5
    I = orc.integral(o, d, 2.0, 4.0, mu, smax, W1, b1, W2, b2)
    ah = OMEGA * ((o[2] - mu[2]) / smax + b1[0])
    assert abs(I - 2.0 * (W2[0] * math.cos(ah) + b2)) < 1e-13


def test_additivity_and_origin_shift(orc):
    rng = np.random.default_rng(9)
    for _ in range(100):
        mu, s, smax, W1, b1, W2, b2 = _rand_prim(rng)
        o = mu + rng.normal(size=3) * 3 * smax
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        a, b = sorted(rng.uniform(0, 6 * smax, 2))
        m = rng.uniform(a, b)
        whole = orc.integral(o, d, a, b, mu, smax, W1, b1, W2, b2)
        parts = orc.integral(o, d, a, m, mu, smax, W1, b1, W2, b2) + \
            orc.integral(o, d, m, b, mu, smax, W1, b1, W2, b2)
        assert abs(whole - parts) < 1e-10 * (1 + abs(whole))
        c = rng.uniform(-2, 2) * smax   # o' = o + c d, bounds shifted by -c
        shifted = orc.integral(o + c * d, d, a - c, b - c, mu, smax, W1, b1, W2, b2)
        assert abs(whole - shifted) < 1e-9 * (1 + abs(whole))


def test_product_form_equals_eq8_difference_form(orc):
    """R3/R4: the product (sinc) form equals Eq. 8's F(t_out) - F(t_in) where h is not tiny."""
    rng = np.random.default_rng(10)
    for _ in range(300):
        mu, s, smax, W1, b1, W2, b2 = _rand_prim(rng)
        o = mu + rng.normal(size=3) * 2 * smax
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        a = rng.uniform(0, 2 * smax); b = a + rng.uniform(0.05, 1.0) * smax
        h = OMEGA * (W1 @ (d / smax))
        if np.min(np.abs(h * (b - a))) < 1e-3:
            continue
        p = orc.integral(o, d, a, b, mu, smax, W1, b1, W2, b2)
        q = orc.integral_eq8(o, d, a, b, mu, smax, W1, b1, W2, b2)
        assert abs(p - q) < 1e-7 * (1 + abs(q))


def test_kernel_values(orc):
    assert abs(orc.kernel(math.log(2.0)) - 0.5) < 1e-15
    assert orc.kernel(-3.2) == 0.0                           # S:164, Eq. 9 clamp
    assert orc.kernel(0.0) == 0.0
    for I in np.linspace(0, 50, 101):
        k = orc.kernel(I)
        assert 0.0 <= k <= 1.0
