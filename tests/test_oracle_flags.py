"""Pins for the oracle's condition flags (R23 = SURVEY A23), which decide
the pixels excluded from the 1e-4 parity bar.  Each case is built so that the
quantity the flag measures is known from the construction, not from the oracle:

  near-tie  consecutive hits in (t_in, id) order, up to the first hit after the
            stop, with t_in gap < 1e-7 max(1, t_in) -- protects the per-ray
            "depth-sorted" order of Eq. 4
  grazing   |1 - q_min| < 1e-5 (q_min = the ray's smallest value of the unit-sphere
            implicit |b + t a|^2: for a sphere of radius r whose centre is at
            distance x0 from the ray, 1 - q_min = 1 - (x0/r)^2), before the stop
  T-floor   |T/floor - 1| < 1e-3 after a composite -- the stop rule (R13)

Spheres on the optical axis of a 1x1 camera (ray d = (0, 0, 1) exactly), so
t_in = z - r and the gaps are fixed by fp32 parameter values chosen here.
"""
import math

import numpy as np

import synth
from test_oracle_render import _axis_cam, _prims

TIE, GRAZE, TFL = 1, 2, 4


def _flag(orc, specs, **kw):
    out, fl, st = orc.render_pixels(_prims(specs), _axis_cam(), [0], [0], (0, 0, 0), **kw)
    return int(fl[0]), st[0]


def _beta(I, r):
    """constant density giving I over a central chord 2r (kappa = 1 - exp(-I))"""
    return I / (2.0 * r)


def _tie_pair(t0, gap, r=0.25, I=0.5):
    """Two concentric spheres on the axis (z = t0 + r, exact in fp32 for the t0, r used
    here) with radii r and fp32(r - gap): entry depths t0 and t0 + (r - fp32(r - gap))."""
    z = np.float32(t0 + r)
    assert float(z) == t0 + r
    rb = np.float32(r - gap)
    a = dict(mu=(0, 0, z), s=(r, r, r), b2=_beta(I, r))
    b = dict(mu=(0, 0, z), s=(rb, rb, rb), b2=_beta(I, float(rb)))
    return [a, b], r - float(rb)


def test_near_tie_flag_threshold_relative_and_absolute():
    import oracle as orc
    # t ~ 10: the window is 1e-7 * 10 = 1e-6
    specs, g = _tie_pair(10.0, 5e-7)          # 5e-8 relative: must be flagged
    assert 4e-7 < g < 6e-7
    fl, st = _flag(orc, specs)
    assert fl & TIE and st[1] == 2
    specs, g = _tie_pair(10.0, 5e-6)          # 5e-7 relative: must not be flagged
    assert 4.5e-6 < g < 5.5e-6
    fl, st = _flag(orc, specs)
    assert not fl & TIE and st[1] == 2
    # t < 1: the window is absolute, 1e-7
    specs, g = _tie_pair(0.5, 5e-8, r=0.125)
    assert 3e-8 < g < 7e-8
    assert _flag(orc, specs)[0] & TIE
    specs, g = _tie_pair(0.5, 3e-7, r=0.125)
    assert 2.5e-7 < g < 3.5e-7
    assert not _flag(orc, specs)[0] & TIE
    # the old 1e-6 (1 + t) window would have flagged this one; A23's does not
    specs, g = _tie_pair(10.0, 2e-6)
    assert not _flag(orc, specs)[0] & TIE


def test_near_tie_only_up_to_the_stop():
    """A tie among hits the ray never reaches (behind the first hit after the stop)
    does not change the pixel and is not flagged; the same tie in front is."""
    import oracle as orc
    opaque = dict(mu=(0, 0, 3.5), s=(0.5, 0.5, 0.5), b2=_beta(12.0, 0.5))   # T = 6e-6 < floor
    pair, _ = _tie_pair(20.0, 5e-7)
    blocker2 = dict(mu=(0, 0, 6.0), s=(0.5, 0.5, 0.5), b2=_beta(0.5, 0.5))
    fl, st = _flag(orc, [opaque, blocker2] + pair)
    assert st[2] == 0 and not fl & TIE            # stop at the first hit, tie after the next one
    fl, st = _flag(orc, pair)
    assert fl & TIE


def _graze(q, r=1.0, z=10.0, I=1.0):
    """sphere of radius r whose centre is x0 = r sqrt(1 - q) off the axis: 1 - q_min = q
    (q < 0: a near miss)."""
    x0 = np.float32(r * math.sqrt(1.0 - q))
    got = 1.0 - (float(x0) / r) ** 2
    return dict(mu=(x0, 0, z), s=(r, r, r), b2=_beta(I, r)), got


def test_grazing_flag_threshold():
    import oracle as orc
    p, got = _graze(5e-6)
    assert abs(got - 5e-6) < 3e-7
    assert _flag(orc, [p])[0] & GRAZE               # grazing hit: flagged
    p, got = _graze(5e-5)
    assert abs(got - 5e-5) < 3e-7
    fl, st = _flag(orc, [p])
    assert not fl & GRAZE and st[0] == 1            # a hit, outside the window
    p, got = _graze(-5e-6)                          # near miss inside the window
    fl, st = _flag(orc, [p])
    assert fl & GRAZE and st[0] == 0
    p, got = _graze(-5e-5)
    fl, st = _flag(orc, [p])
    assert not fl and st[0] == 0


def test_grazing_behind_the_stop_not_flagged():
    import oracle as orc
    opaque = dict(mu=(0, 0, 3.5), s=(0.5, 0.5, 0.5), b2=_beta(12.0, 0.5))
    p, _ = _graze(5e-6, z=30.0)
    fl, st = _flag(orc, [opaque, p])
    assert st[2] == 0 and not fl & GRAZE
    p, _ = _graze(5e-6, z=1.8, r=0.3)               # in front of the opaque one: flagged
    assert _flag(orc, [opaque, p])[0] & GRAZE


def test_t_floor_flag():
    """One constant-density sphere: T = exp(-I) after it; I chosen so that T lands
    5e-4 (relative) above / below the 1e-4 floor (flagged) or 5e-3 above (not)."""
    import oracle as orc
    r = 0.5
    for rel, want in ((5e-4, True), (-5e-4, True), (5e-3, False), (-5e-3, False)):
        I = -math.log(1e-4 * (1.0 + rel))
        fl, st = _flag(orc, [dict(mu=(0, 0, 5), s=(r, r, r), b2=_beta(I, r))])
        assert bool(fl & TFL) == want, (rel, fl)
        assert st[2] == (0 if rel < 0 else -1)     # the stop index (stop iff T < floor)
    # a second hit after T crossed the floor band is never reached
    I = -math.log(1e-4 * (1.0 - 5e-3))
    fl, st = _flag(orc, [dict(mu=(0, 0, 5), s=(r, r, r), b2=_beta(I, r)),
                         dict(mu=(0, 0, 9), s=(r, r, r), b2=_beta(0.5, r))])
    assert fl == 0 and st[1] == 1 and st[0] == 2


def test_flags_do_not_fire_on_a_plain_scene():
    """No flag on well separated, non-grazing, semi-transparent hits."""
    import oracle as orc
    specs = [dict(mu=(0.1 * i, 0, 3 + 2 * i), s=(0.5, 0.5, 0.5), b2=_beta(0.7, 0.5)) for i in range(4)]
    fl, st = _flag(orc, specs)
    assert fl == 0 and st[1] == 4
