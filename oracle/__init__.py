"""CPU oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

ctypes wrapper around ``oracle/snp_oracle.c`` (plain C, double precision,
``-ffp-contract=off``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this module.
It shares no code with ``paper_2510_08491_b200`` and does not import it; the
only shared module is ``synth`` (seeded inputs, no method arithmetic).

Parity status of each function:
  quat_to_rot, pixel_ray, intersect, density, integral, integral_eq8, kernel,
  sh_basis, sh_color, render_pixels, bin_view, bin_sort   -- pinned
  (tests/test_oracle_*.py).  Images of trained scenes: parity unpinned (no
  datasets or weights exist in the reference).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "snp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

FLAG_NEAR_TIE = 1
FLAG_GRAZING = 2
FLAG_TFLOOR = 4
TIE_EPS = 1e-7      # DESIGN.md R23 = SURVEY A23: gap < 1e-7 max(1, t_in)
GRAZE_EPS = 1e-5    # DESIGN.md R23 = SURVEY A23: |1 - q_min| < 1e-5
T_FLOOR = 1e-4


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11, FP64, no FP contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-D_DEFAULT_SOURCE", "-ffp-contract=off", "-fno-fast-math",
               "-fopenmp", "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Scene(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_hidden", C.c_int32), ("sh_degree", C.c_int32),
                ("omega", C.c_double)] + [(f, C.c_void_p) for f in
                                          ("centers", "rotations", "scales", "w1", "b1", "w2", "b2", "sh",
                                           "w_t")]


class _Camera(C.Structure):
    _fields_ = [("R_wc", C.c_double * 9), ("C_w", C.c_double * 3), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("t_near", C.c_double),
                ("t_far", C.c_double), ("xi_t", C.c_double)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            dp = C.POINTER(C.c_double)
            L.orc_render_pixels.restype = C.c_int
            L.orc_render_pixels_ex.restype = C.c_int
            L.orc_render_frame.restype = C.c_int
            L.orc_bin_sort.restype = C.c_int64
            L.orc_pixel_hits.restype = C.c_int64
            L.orc_integral.restype = C.c_double
            L.orc_integral_eq8.restype = C.c_double
            L.orc_density.restype = C.c_double
            L.orc_kernel.restype = C.c_double
            L.orc_kernel.argtypes = [C.c_double]
            L.orc_intersect.restype = C.c_int
            L.orc_intersect.argtypes = [dp, dp, C.c_double, C.c_double, dp, dp, dp, dp, dp, dp]
            L.orc_integral.argtypes = [dp, dp, C.c_double, C.c_double, dp, C.c_double, C.c_int,
                                       C.c_double, dp, dp, dp, C.c_double]
            L.orc_integral_eq8.argtypes = L.orc_integral.argtypes
            L.orc_density.argtypes = [dp, dp, C.c_double, C.c_int, C.c_double, dp, dp, dp, C.c_double]
            L.orc_tile_bits.restype = C.c_int
            L.orc_tile_bits.argtypes = [C.c_int64]
            _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _dp(a):
    return np.ascontiguousarray(a, np.float64).ctypes.data_as(C.POINTER(C.c_double))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class _SceneRef:
    """Keeps the numpy buffers alive while C holds pointers into them."""

    def __init__(self, scene):
        self.arrs = [_f32(getattr(scene, f)) for f in
                     ("centers", "rotations", "scales", "w1", "b1", "w2", "b2", "sh")]
        w_t = getattr(scene, "w_t", None)   # temporal weights [n, N] (R24) or None
        if w_t is not None:
            self.arrs.append(_f32(w_t))
        self.s = _Scene(scene.n, int(scene.w1.shape[1]), int(scene.sh_degree), float(scene.omega),
                        *[a.ctypes.data for a in self.arrs[:8]],
                        self.arrs[8].ctypes.data if w_t is not None else None)


def _camera(cam) -> _Camera:
    c = _Camera()
    R = np.asarray(cam.R_wc, np.float32).astype(np.float64).reshape(9)
    for i in range(9):
        c.R_wc[i] = R[i]
    Cw = np.asarray(cam.C_w, np.float32).astype(np.float64)
    for i in range(3):
        c.C_w[i] = Cw[i]
    f32 = lambda v: float(np.float32(v))  # noqa: E731  -- the GPU receives fp32 camera values
    c.fx, c.fy, c.cx, c.cy = f32(cam.fx), f32(cam.fy), f32(cam.cx), f32(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    c.t_near, c.t_far = f32(cam.t_near), f32(cam.t_far)
    c.xi_t = f32(getattr(cam, "xi_t", 0.0))
    return c


# ------------------------------------------------------------------- renderer

def render_pixels(scene, cam, px, py, bg=(0.0, 0.0, 0.0), t_floor=T_FLOOR, nthreads=0,
                  tie_eps=TIE_EPS, graze_eps=GRAZE_EPS, colour_per_ray=False):
    """Oracle RGBA (float64) for the listed pixels plus flags and per-pixel stats
    (hits, composited, stop index).  colour_per_ray: SH colour at each pixel's ray
    direction instead of at normalize(mu - o)."""
    L = lib()
    px = np.ascontiguousarray(px, np.int32)
    py = np.ascontiguousarray(py, np.int32)
    n = px.shape[0]
    out = np.zeros((n, 4), np.float64)
    flags = np.zeros(n, np.int32)
    stats = np.zeros((n, 3), np.int32)
    sref = _SceneRef(scene)
    cam_c = _camera(cam)
    bgv = np.asarray([float(np.float32(b)) for b in bg], np.float64)
    r = L.orc_render_pixels_ex(C.byref(sref.s), C.byref(cam_c), _p(bgv), C.c_double(float(np.float32(t_floor))),
                               C.c_int64(n), _p(px), _p(py), _p(out), _p(flags), _p(stats),
                               C.c_int(nthreads), C.c_double(tie_eps), C.c_double(graze_eps),
                               C.c_int(1 if colour_per_ray else 0))
    if r != 0:
        raise ValueError(f"oracle render failed ({r}): invalid scene or out of memory")
    return out, flags, stats


def render_frame(scene, cam, bg=(0.0, 0.0, 0.0), t_floor=T_FLOOR, nthreads=0,
                 tie_eps=TIE_EPS, graze_eps=GRAZE_EPS, colour_per_ray=False):
    H, W = int(cam.height), int(cam.width)
    yy, xx = np.mgrid[0:H, 0:W]
    out, flags, stats = render_pixels(scene, cam, xx.ravel(), yy.ravel(), bg, t_floor, nthreads,
                                      tie_eps, graze_eps, colour_per_ray)
    return out.reshape(H, W, 4), flags.reshape(H, W), stats.reshape(H, W, 3)


def pixel_hits(scene, cam, px, py, cap=4096):
    """Brute-force (ids, t_in, t_out) of every primitive hit by pixel (px, py)."""
    ids = np.zeros(cap, np.int64)
    ti = np.zeros(cap)
    to = np.zeros(cap)
    sref = _SceneRef(scene)
    cam_c = _camera(cam)
    n = lib().orc_pixel_hits(C.byref(sref.s), C.byref(cam_c), C.c_int32(px), C.c_int32(py),
                             _p(ids), _p(ti), _p(to), C.c_int64(cap))
    if n > cap:
        return pixel_hits(scene, cam, px, py, cap=int(n))
    return ids[:n], ti[:n], to[:n]


# ------------------------------------------------------------- per-ray pieces

def quat_to_rot(q):
    R = np.zeros(9)
    r = lib().orc_quat_to_rot(_p(np.asarray(q, np.float64)), _p(R))
    if r != 0:
        raise ValueError("zero quaternion")
    return R.reshape(3, 3)


def pixel_ray(cam, px, py):
    o, d = np.zeros(3), np.zeros(3)
    cam_c = _camera(cam)
    lib().orc_pixel_ray(C.byref(cam_c), C.c_double(px), C.c_double(py), _p(o), _p(d))
    return o, d


def intersect(o, d, t_near, t_far, mu, q, s):
    """(hit, t_in, t_out, qmin) for one ray and one ellipsoid."""
    R = quat_to_rot(q).reshape(9)
    ti, to, qm = C.c_double(0), C.c_double(0), C.c_double(0)
    hit = lib().orc_intersect(_dp(o), _dp(d), t_near, t_far, _dp(mu), _dp(R), _dp(s),
                              C.byref(ti), C.byref(to), C.byref(qm))
    return bool(hit), ti.value, to.value, qm.value


def density(x, mu, smax, W1, b1, W2, b2, omega=30.0):
    W1 = np.asarray(W1, np.float64).reshape(-1, 3)
    return lib().orc_density(_dp(x), _dp(mu), smax, W1.shape[0], omega, _dp(W1), _dp(b1), _dp(W2), b2)


def integral(o, d, t_in, t_out, mu, smax, W1, b1, W2, b2, omega=30.0):
    W1 = np.asarray(W1, np.float64).reshape(-1, 3)
    return lib().orc_integral(_dp(o), _dp(d), t_in, t_out, _dp(mu), smax, W1.shape[0], omega,
                              _dp(W1), _dp(b1), _dp(W2), b2)


def integral_eq8(o, d, t_in, t_out, mu, smax, W1, b1, W2, b2, omega=30.0):
    W1 = np.asarray(W1, np.float64).reshape(-1, 3)
    return lib().orc_integral_eq8(_dp(o), _dp(d), t_in, t_out, _dp(mu), smax, W1.shape[0], omega,
                                  _dp(W1), _dp(b1), _dp(W2), b2)


def kernel(I):
    return lib().orc_kernel(float(I))


def sh_basis(d):
    out = np.zeros(16)
    lib().orc_sh_basis(_p(np.asarray(d, np.float64)), _p(out))
    return out


def sh_color(sh, d, degree=3):
    out = np.zeros(3)
    lib().orc_sh_color(C.c_int(degree), _p(_f32(sh)), _p(np.asarray(d, np.float64)), _p(out))
    return out


# -------------------------------------------------------------------- binning

TILE = 16


def tiles_of(cam):
    return (int(cam.width) + TILE - 1) // TILE, (int(cam.height) + TILE - 1) // TILE


def tile_bits(n_tiles):
    return int(lib().orc_tile_bits(C.c_int64(n_tiles)))


def bin_view(scene, cam):
    """Per-primitive (tile rect [n,4] or -1, pixel-centre rect [n,4] or -1, depth key bits [n])."""
    n = scene.n
    rects = np.zeros((n, 4), np.int32)
    prects = np.zeros((n, 4), np.int32)
    depth = np.zeros(n, np.uint32)
    sref = _SceneRef(scene)
    cam_c = _camera(cam)
    lib().orc_bin_view(C.byref(sref.s), C.byref(cam_c), _p(rects), _p(prects), _p(depth))
    return rects, prects, depth


def bin_sort(rects, depth, n, n_views, tiles_x, tiles_y, row_begin=0, row_stride=1):
    """Keys (u64), values (u32) in stable-sorted order and ranges [views*tiles, 2]."""
    L = lib()
    rects = np.ascontiguousarray(rects, np.int32)
    depth = np.ascontiguousarray(depth, np.uint32)
    T = tiles_x * tiles_y
    ranges = np.zeros((n_views * T, 2), np.uint32)
    empty_k = np.zeros(1, np.uint64)
    empty_i = np.zeros(1, np.uint32)
    ndup = L.orc_bin_sort(C.c_int64(n), C.c_int32(n_views), _p(rects), _p(depth), C.c_int32(tiles_x),
                          C.c_int32(tiles_y), C.c_int32(row_begin), C.c_int32(row_stride),
                          _p(empty_k), _p(empty_i), C.c_int64(0), _p(ranges))
    if ndup < 0:
        raise MemoryError("oracle bin_sort")
    keys = np.zeros(max(ndup, 1), np.uint64)
    ids = np.zeros(max(ndup, 1), np.uint32)
    r = L.orc_bin_sort(C.c_int64(n), C.c_int32(n_views), _p(rects), _p(depth), C.c_int32(tiles_x),
                       C.c_int32(tiles_y), C.c_int32(row_begin), C.c_int32(row_stride),
                       _p(keys), _p(ids), C.c_int64(ndup), _p(ranges))
    if r != ndup:
        raise RuntimeError("oracle bin_sort inconsistent")
    return keys[:ndup], ids[:ndup], ranges
