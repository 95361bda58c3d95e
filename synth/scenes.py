"""Seeded synthetic scenes and cameras shaped like the paper's workloads.

Holds no arithmetic of the method: it only draws parameters (the SIREN-style
ranges of P:393-394 "Primitives" paragraph, §3.3) and builds pinhole cameras.
Shapes follow BASELINE.json ``configs`` and SURVEY.md §8(d):

  C1  256 primitives, one 128x128 view (oracle renders the full frame in seconds)
  C2  10k primitives, Blender-synthetic-shaped object, one 800x800 view, white bg
  C3  300k primitives, Mip-NeRF360-shaped (60 % object surfaces + 40 % background
      shell at radius log-U(6, 40)), one 1245x825 view
  C4  C3's scene, 64 orbit views
  C5  1M large-footprint primitives (scale x3), 1920x1080

Conventions (readings R6-R8): quaternion (w, x, y, z); ``scales`` are
ellipsoid semi-axes in world units; camera looks along +z, x right, y down;
``R_wc`` is the world-from-camera rotation (row-major), ``C_w`` the camera centre.
"""
from __future__ import annotations

import dataclasses
import struct
from typing import Optional, List, Tuple

import numpy as np

N_HIDDEN = 8          # P:394 "number of hidden neurons N_sigma to 8"
OMEGA = 30.0          # P:394 "frequency multiplier omega to 30"
SH_COEFFS = 16        # P:394 "four bands of Spherical Harmonics" -> 16 coeffs x RGB
PARAMS_PER_PRIM = 3 + 3 + 4 + N_HIDDEN * 3 + N_HIDDEN + N_HIDDEN + 1 + SH_COEFFS * 3  # = 99


@dataclasses.dataclass
class Scene:
    centers: np.ndarray    # [n,3] f32  mu
    rotations: np.ndarray  # [n,4] f32  q = (w,x,y,z), any nonzero norm
    scales: np.ndarray     # [n,3] f32  s, semi-axes > 0
    w1: np.ndarray         # [n,N,3] f32
    b1: np.ndarray         # [n,N] f32
    w2: np.ndarray         # [n,N] f32
    b2: np.ndarray         # [n] f32
    sh: np.ndarray         # [n,16,3] f32, coefficient-major, RGB innermost
    omega: float = OMEGA
    sh_degree: int = 3
    w_t: Optional[np.ndarray] = None   # [n,N] f32 temporal weights W_t (appendix "Dynamic scenes"), or None

    @property
    def n(self) -> int:
        return int(self.centers.shape[0])

    @property
    def n_hidden(self) -> int:
        return int(self.w1.shape[1])

    def subset(self, idx) -> "Scene":
        idx = np.asarray(idx)
        return Scene(*(np.ascontiguousarray(getattr(self, f)[idx]) for f in _FIELDS),
                     omega=self.omega, sh_degree=self.sh_degree)

    def contiguous(self) -> "Scene":
        for f in _FIELDS:
            setattr(self, f, np.ascontiguousarray(getattr(self, f), dtype=np.float32))
        return self

    def records(self) -> np.ndarray:
        """[n, 99] flat records in NSPL order (center, scale, quat, W1, b1, W2, b2, SH)."""
        n = self.n
        return np.concatenate([
            self.centers.reshape(n, -1), self.scales.reshape(n, -1),
            self.rotations.reshape(n, -1), self.w1.reshape(n, -1),
            self.b1.reshape(n, -1), self.w2.reshape(n, -1),
            self.b2.reshape(n, 1), self.sh.reshape(n, -1)], axis=1).astype(np.float32)


_FIELDS = ("centers", "rotations", "scales", "w1", "b1", "w2", "b2", "sh")


@dataclasses.dataclass
class Camera:
    R_wc: np.ndarray       # [3,3] f32 world-from-camera rotation, row-major
    C_w: np.ndarray        # [3] f32 camera centre = ray origin o
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    t_near: float = 0.01   # S:295 defaults
    t_far: float = 1e4
    xi_t: float = 0.0      # timestamp of this view (temporal scenes only)


def empty_scene(n_hidden: int = N_HIDDEN) -> Scene:
    z = lambda *s: np.zeros(s, np.float32)  # noqa: E731
    return Scene(z(0, 3), z(0, 4), z(0, 3), z(0, n_hidden, 3), z(0, n_hidden),
                 z(0, n_hidden), z(0), z(0, SH_COEFFS, 3))


def concat_scenes(a: Scene, b: Scene) -> Scene:
    return Scene(*(np.concatenate([getattr(a, f), getattr(b, f)]) for f in _FIELDS),
                 omega=a.omega, sh_degree=a.sh_degree).contiguous()


# ----------------------------------------------------------------------------- cameras

def look_at(eye, target, width, height, fx, fy=None, cx=None, cy=None,
            up=(0.0, 0.0, 1.0), t_near=0.01, t_far=1e4) -> Camera:
    eye = np.asarray(eye, np.float64)
    f = np.asarray(target, np.float64) - eye
    f /= np.linalg.norm(f)
    x = np.cross(f, np.asarray(up, np.float64))
    x /= np.linalg.norm(x)
    y = np.cross(f, x)
    R = np.stack([x, y, f], axis=1)  # columns = camera axes in world coordinates
    fy = fx if fy is None else fy
    cx = width / 2.0 if cx is None else cx
    cy = height / 2.0 if cy is None else cy
    return Camera(R.astype(np.float32), eye.astype(np.float32), float(fx), float(fy),
                  float(cx), float(cy), int(width), int(height), float(t_near), float(t_far))


def orbit_cameras(n_views, radius, width, height, fx, elev_deg=(20.0, 20.0),
                  az0_deg=0.0, target=(0.0, 0.0, 0.0)) -> List[Camera]:
    cams = []
    for k in range(n_views):
        az = np.deg2rad(az0_deg + 360.0 * k / n_views)
        e0, e1 = elev_deg
        el = np.deg2rad(e0 + (e1 - e0) * (k / max(1, n_views - 1)))
        eye = np.asarray(target) + radius * np.array(
            [np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.sin(el)])
        cams.append(look_at(eye, target, width, height, fx))
    return cams


# ----------------------------------------------------------------------------- primitives

def _unit_vectors(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _sphere_surface_points(rng, n, n_spheres, box, rmin, rmax):
    c = rng.uniform(-box, box, size=(n_spheres, 3))
    r = rng.uniform(rmin, rmax, size=n_spheres)
    area = 4.0 * np.pi * r ** 2
    which = rng.choice(n_spheres, size=n, p=area / area.sum())
    pts = c[which] + r[which, None] * _unit_vectors(rng, n)
    return pts, float(area.sum())


def _log_uniform(rng, lo, hi, size):
    return np.exp(rng.uniform(np.log(lo), np.log(hi), size=size))


def _network_and_colour(rng, scales, variant, n_hidden=N_HIDDEN):
    n = scales.shape[0]
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w1 = rng.uniform(-1.0 / 3.0, 1.0 / 3.0, size=(n, n_hidden, 3))
    b1 = rng.uniform(-1.0, 1.0, size=(n, n_hidden))                       # reading R17
    smax = scales.max(axis=1)
    beta = rng.uniform(0.2, 2.0, size=n)
    b2 = beta / smax                                                      # reading R17
    if variant == "paper":
        bound = np.sqrt(6.0 / n_hidden) / OMEGA
        w2 = rng.uniform(-bound, bound, size=(n, n_hidden))
    elif variant == "trained":
        w2 = rng.uniform(-1.0, 1.0, size=(n, n_hidden)) * (0.5 / smax)[:, None]
    else:
        raise ValueError(variant)
    sh = rng.normal(0.0, 0.3, size=(n, SH_COEFFS, 3))
    sh[:, 1:, :] *= 0.1
    return q, w1, b1, w2, b2, sh


def make_scene(seed, n, kind="object", variant="trained", scale_mult=1.0,
               n_spheres=8, box=0.7, rmin=0.2, rmax=0.5, bg_fraction=0.0,
               bg_radius=(6.0, 40.0), n_hidden=N_HIDDEN) -> Scene:
    """Primitive cloud: ``(1-bg_fraction)`` on random sphere surfaces (object),
    ``bg_fraction`` in a background shell at log-uniform radius (360-degree scene)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n_bg = int(round(n * bg_fraction))
    n_obj = n - n_bg
    pts, area = _sphere_surface_points(rng, n_obj, n_spheres, box, rmin, rmax)
    spacing = np.sqrt(area / max(1, n_obj))
    s_obj = spacing * scale_mult * _log_uniform(rng, 0.3, 1.0, (n_obj, 3))
    if n_bg:
        rad = _log_uniform(rng, bg_radius[0], bg_radius[1], n_bg)
        pbg = rad[:, None] * _unit_vectors(rng, n_bg)
        theta = np.sqrt(4.0 * np.pi / n_bg)         # angular spacing of the shell
        s_bg = (rad * theta * scale_mult)[:, None] * _log_uniform(rng, 0.3, 1.0, (n_bg, 3))
        pts = np.concatenate([pts, pbg])
        s = np.concatenate([s_obj, s_bg])
        perm = rng.permutation(n)
        pts, s = pts[perm], s[perm]
    else:
        s = s_obj
    q, w1, b1, w2, b2, sh = _network_and_colour(rng, s, variant, n_hidden)
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    return Scene(f(pts), f(q), f(s), f(w1), f(b1), f(w2), f(b2), f(sh))


# ----------------------------------------------------------------------------- configs

CONFIGS = {
    "C1": dict(n=256, width=128, height=128, fx=177.8, views=1, seed=0,
               scene=dict(kind="object", scale_mult=1.0, n_spheres=8, box=0.7), bg=(0, 0, 0)),
    "C2": dict(n=10_000, width=800, height=800, fx=1111.11, views=1, seed=1,
               scene=dict(kind="object", scale_mult=1.5, n_spheres=8, box=1.0), bg=(1, 1, 1)),
    "C3": dict(n=300_000, width=1245, height=825, fx=0.93 * 1245, views=1, seed=2,
               scene=dict(kind="360", scale_mult=1.5, n_spheres=24, box=0.8, rmin=0.2,
                          rmax=0.4, bg_fraction=0.4), bg=(0, 0, 0)),
    "C4": dict(n=300_000, width=1245, height=825, fx=0.93 * 1245, views=64, seed=2,
               scene=dict(kind="360", scale_mult=1.5, n_spheres=24, box=0.8, rmin=0.2,
                          rmax=0.4, bg_fraction=0.4), bg=(0, 0, 0)),
    "C5": dict(n=1_000_000, width=1920, height=1080, fx=0.93 * 1920, views=1, seed=4,
               scene=dict(kind="360", scale_mult=3.0, n_spheres=24, box=0.8, rmin=0.2,
                          rmax=0.4, bg_fraction=0.4), bg=(0, 0, 0)),
}


def make_config(name, variant="trained", n=None, views=None,
                n_hidden=N_HIDDEN) -> Tuple[Scene, List[Camera], Tuple]:
    """Returns (scene, cameras, background) for a BASELINE config name (n_hidden: the
    MLP width N_sigma; the configs are quoted at the paper's 8)."""
    cfg = CONFIGS[name]
    n = cfg["n"] if n is None else n
    views = cfg["views"] if views is None else views
    sc = dict(cfg["scene"])
    sc.pop("kind")
    scene = make_scene(cfg["seed"], n, variant=variant, n_hidden=n_hidden, **sc)
    if views == 1:
        cams = orbit_cameras(1, 4.0, cfg["width"], cfg["height"], cfg["fx"],
                             elev_deg=(20.0, 20.0), az0_deg=30.0)
    else:
        cams = orbit_cameras(views, 4.0, cfg["width"], cfg["height"], cfg["fx"],
                             elev_deg=(15.0, 30.0), az0_deg=30.0)
    return scene, cams, tuple(float(c) for c in cfg["bg"])


# ----------------------------------------------------------------------------- NSPL file

_NSPL_MAGIC = b"NSPL"
_NSPL_VERSION = 1
_HDR = struct.Struct("<4sIIIfIQ")   # magic, version, n_hidden, sh_coeffs, omega, record_len, count


def save_nspl(scene: Scene, path) -> None:
    """Checkpoint interchange format: 32-byte header + 99 f32 per primitive."""
    rec = scene.records()
    with open(path, "wb") as fh:
        fh.write(_HDR.pack(_NSPL_MAGIC, _NSPL_VERSION, scene.n_hidden, SH_COEFFS,
                           float(scene.omega), rec.shape[1], scene.n))
        fh.write(rec.astype("<f4").tobytes())


def load_nspl(path) -> Scene:
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _HDR.size:
        raise ValueError(f"NSPL truncated at byte {len(raw)} (header needs {_HDR.size})")
    magic, ver, nh, shc, omega, rlen, count = _HDR.unpack_from(raw, 0)
    if magic != _NSPL_MAGIC:
        raise ValueError("NSPL bad magic at byte 0")
    if ver != _NSPL_VERSION:
        raise ValueError(f"NSPL unsupported version {ver} at byte 4")
    expect = 3 + 3 + 4 + nh * 3 + nh + nh + 1 + shc * 3
    if rlen != expect:
        raise ValueError(f"NSPL record length {rlen} != {expect} at byte 20")
    need = _HDR.size + 4 * rlen * count
    if len(raw) < need:
        raise ValueError(f"NSPL truncated at byte {len(raw)} (need {need})")
    rec = np.frombuffer(raw, "<f4", count * rlen, _HDR.size).reshape(count, rlen)
    o = 0

    def take(k, shape):
        nonlocal o
        a = np.ascontiguousarray(rec[:, o:o + k].reshape((count,) + shape), dtype=np.float32)
        o += k
        return a
    centers = take(3, (3,)); scales = take(3, (3,)); rot = take(4, (4,))
    w1 = take(nh * 3, (nh, 3)); b1 = take(nh, (nh,)); w2 = take(nh, (nh,))
    b2 = take(1, ()); sh = take(shc * 3, (shc, 3))
    return Scene(centers, rot, scales, w1, b1, w2, b2, sh, omega=float(omega))
