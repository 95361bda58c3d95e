"""Thin ctypes binding of ``include/snp.h`` (argument marshalling only).

Every step of the hot path runs in ``libsnp.so`` (hand-written CUDA for
sm_100a); this module only converts arrays/tensors to pointers, cameras and
options to the C structs, and statuses to exceptions.  There is no CPU
fallback: if the library is missing or no CUDA device is present the calls
raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SNP_LIB_PATH") or os.path.join(_HERE, "libsnp.so")   # override: A/B experiments only

SNP_OK = 0
STATUS = {0: "SNP_OK", 1: "SNP_ERR_INVALID_ARGUMENT", 2: "SNP_ERR_OUT_OF_MEMORY", 3: "SNP_ERR_CUDA",
          4: "SNP_ERR_UNSUPPORTED", 5: "SNP_ERR_BAD_STATE", 6: "SNP_ERR_CAPACITY"}
SNP_MEM_HOST = 0
SNP_MEM_DEVICE = 1
SNP_MEM_HOST_ASYNC = 2   # snp_render output only: copy enqueued on the stream, no synchronisation
SNP_COLOUR_PRIMITIVE = 0  # colour_mode: SH at normalize(mu - C) per primitive and view (default)
SNP_COLOUR_RAY = 1        # colour_mode: SH at each pixel's ray direction
SNP_BIN_CONIC_TILES = 1   # snp_set_binning: drop rect tiles the silhouette ellipse misses
SNP_BIN_TILE_DEPTH = 2    # snp_set_binning: per-tile depth lower bounds in the keys

EXPORTS = ("snp_version", "snp_create_scene", "snp_update_scene", "snp_project", "snp_bin_sort", "snp_render",
           "snp_render_views", "snp_destroy", "snp_last_error", "snp_get_binning", "snp_get_stats",
           "snp_set_pending_limit", "snp_get_debug_counters", "snp_set_temporal", "snp_project_at",
           "snp_render_backward", "snp_loss_l1", "snp_scale_regularizer", "snp_adam_step", "snp_get_params",
           "snp_set_temporal_grad", "snp_loss_3dgs", "snp_render_backward_ex", "snp_set_binning", "snp_set_record",
           "snp_loss_3dgs_part")


class SnpError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class SceneDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_hidden", C.c_int32), ("sh_degree", C.c_int32),
                ("omega", C.c_float), ("memory", C.c_int32)] + \
               [(f, C.c_void_p) for f in ("centers", "rotations", "scales", "w1", "b1", "w2", "b2", "sh")]


class Camera(C.Structure):
    _fields_ = [("R_wc", C.c_float * 9), ("C_w", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("t_near", C.c_float), ("t_far", C.c_float)]


class RenderOpts(C.Structure):
    _fields_ = [("background", C.c_float * 3), ("transmittance_floor", C.c_float),
                ("tile_row_begin", C.c_int32), ("tile_row_stride", C.c_int32),
                ("out_memory", C.c_int32), ("sync_check", C.c_int32), ("colour_mode", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in ("n_visible", "n_dup", "key_capacity", "tested_pairs",
                                          "candidate_pairs", "hit_pairs", "composited",
                                          "overflow_pixels", "capacity_overflow", "backward_skipped",
                                          "dead_keys")]


_lock = threading.Lock()
_lib = None


def lib():
    """Loads libsnp.so; raises if it has not been built (no fallback exists)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                                  "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            vp = C.c_void_p
            L.snp_version.restype = C.c_char_p
            L.snp_last_error.restype = C.c_char_p
            L.snp_create_scene.argtypes = [C.POINTER(SceneDesc), C.c_int, vp, C.POINTER(vp)]
            L.snp_update_scene.argtypes = [vp, C.POINTER(SceneDesc), vp]
            L.snp_project.argtypes = [vp, C.POINTER(Camera), C.c_int32, vp]
            L.snp_bin_sort.argtypes = [vp, C.POINTER(RenderOpts), vp]
            L.snp_render.argtypes = [vp, C.POINTER(RenderOpts), vp, vp]
            L.snp_render_views.argtypes = [vp, C.POINTER(Camera), C.c_int32, C.POINTER(RenderOpts), vp, vp]
            L.snp_destroy.argtypes = [vp]
            L.snp_get_binning.argtypes = [vp, vp, vp, vp, vp, C.c_int64, C.POINTER(C.c_int64), vp, vp]
            L.snp_get_stats.argtypes = [vp, C.POINTER(Stats), vp]
            L.snp_set_pending_limit.argtypes = [vp, C.c_int32]
            L.snp_set_binning.argtypes = [vp, C.c_int32]
            L.snp_set_record.argtypes = [vp, C.c_int32]
            L.snp_set_temporal.argtypes = [vp, vp, C.c_int32, vp]
            L.snp_render_backward.argtypes = [vp, C.POINTER(RenderOpts), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
            L.snp_render_backward_ex.argtypes = [vp, C.POINTER(RenderOpts), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                                 vp]
            L.snp_loss_l1.argtypes = [vp, vp, C.c_int64, vp, vp, vp]
            L.snp_get_params.argtypes = [vp, C.POINTER(vp), C.c_int32, vp]
            L.snp_set_temporal_grad.argtypes = [vp, vp]
            L.snp_scale_regularizer.argtypes = [vp, C.c_float, vp, vp, vp]
            L.snp_loss_3dgs.argtypes = [vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_float, vp, vp, vp]
            L.snp_loss_3dgs_part.argtypes = [vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_float, vp, vp,
                                             vp]
            L.snp_adam_step.argtypes = [vp, C.POINTER(vp), C.POINTER(C.c_float), C.c_float, C.c_float, C.c_float,
                                        C.c_int32, vp]
            L.snp_project_at.argtypes = [vp, C.POINTER(Camera), C.c_int32, vp, vp]
            L.snp_get_debug_counters.argtypes = [vp, vp, C.c_int32, vp]
            for f in EXPORTS:
                if f not in ("snp_version", "snp_last_error"):
                    getattr(L, f).restype = C.c_int
            _lib = L
    return _lib


def _check(status):
    if status != SNP_OK:
        raise SnpError(status, lib().snp_last_error().decode())


def _ptr(x):
    """Pointer of a numpy array (host) or a torch tensor (host or device)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


def _stream(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _is_device(x):
    return hasattr(x, "is_cuda") and x.is_cuda


FIELDS = ("centers", "rotations", "scales", "w1", "b1", "w2", "b2", "sh")


def _desc(scene, n_hidden=None, sh_degree=None, omega=None):
    arrs = []
    for f in FIELDS:
        a = getattr(scene, f)
        if not _is_device(a):
            a = np.ascontiguousarray(a, dtype=np.float32)
        else:
            a = a.contiguous().float()
        arrs.append(a)
    mem = SNP_MEM_DEVICE if _is_device(arrs[0]) else SNP_MEM_HOST
    n = int(arrs[0].shape[0])
    if n_hidden is None:   # w1 is [n, N, 3]
        n_hidden = int(arrs[3].shape[1]) if len(arrs[3].shape) == 3 else 8
    desc = SceneDesc(n, n_hidden, int(getattr(scene, "sh_degree", 3) if sh_degree is None else sh_degree),
                     float(getattr(scene, "omega", 30.0) if omega is None else omega), mem,
                     *[_ptr(a) for a in arrs])
    return desc, arrs


def create_scene(scene, device=0, stream=None, n_hidden=None, sh_degree=None, omega=None):
    """``scene`` has float32 C-contiguous arrays ``centers [n,3] ... sh [n,16,3]``
    (numpy = host memory, torch CUDA tensors = device memory)."""
    desc, keep = _desc(scene, n_hidden, sh_degree, omega)
    h = C.c_void_p()
    _check(lib().snp_create_scene(C.byref(desc), int(device), _stream(stream), C.byref(h)))
    del keep
    return h.value


def update_scene(h, scene, stream=None, n_hidden=None, sh_degree=None, omega=None):
    desc, keep = _desc(scene, n_hidden, sh_degree, omega)
    _check(lib().snp_update_scene(h, C.byref(desc), _stream(stream)))
    del keep


def make_cameras(cams):
    arr = (Camera * len(cams))()
    for i, c in enumerate(cams):
        R = np.asarray(c.R_wc, np.float32).reshape(9)
        Cw = np.asarray(c.C_w, np.float32).reshape(3)
        arr[i] = Camera((C.c_float * 9)(*R.tolist()), (C.c_float * 3)(*Cw.tolist()), float(c.fx), float(c.fy),
                        float(c.cx), float(c.cy), int(c.width), int(c.height), float(c.t_near), float(c.t_far))
    return arr


def make_opts(background=(0.0, 0.0, 0.0), transmittance_floor=1e-4, tile_row_begin=0, tile_row_stride=1,
              out_memory=SNP_MEM_DEVICE, sync_check=1, colour_mode=0):
    return RenderOpts((C.c_float * 3)(*[float(b) for b in background]), float(transmittance_floor),
                      int(tile_row_begin), int(tile_row_stride), int(out_memory), int(sync_check),
                      int(colour_mode))


def _times(xi_t, n):
    if xi_t is None:
        return None
    t = np.ascontiguousarray(np.broadcast_to(np.asarray(xi_t, np.float32), (n,)))
    return t


def project(h, cams, stream=None, xi_t=None):
    """K1 for the cameras; xi_t (temporal scenes): one timestamp per view, or None."""
    arr = cams if isinstance(cams, C.Array) else make_cameras(cams)
    t = _times(xi_t, len(arr))
    if t is None:
        _check(lib().snp_project(h, arr, len(arr), _stream(stream)))
    else:
        _check(lib().snp_project_at(h, arr, len(arr), t.ctypes.data_as(C.c_void_p), _stream(stream)))


def set_temporal_grad(h, grad_w_t):
    """Where snp_render_backward adds dL/dW_t (a zeroed CUDA tensor [n, N]) or None."""
    _check(lib().snp_set_temporal_grad(h, _ptr(grad_w_t)))


def set_temporal(h, w_t, stream=None):
    """Attach temporal weights w_t [n, N] (numpy = host, torch CUDA = device), or None."""
    if w_t is None:
        _check(lib().snp_set_temporal(h, None, SNP_MEM_HOST, _stream(stream)))
        return
    if _is_device(w_t):
        w = w_t.contiguous().float()
        _check(lib().snp_set_temporal(h, _ptr(w), SNP_MEM_DEVICE, _stream(stream)))
    else:
        w = np.ascontiguousarray(w_t, dtype=np.float32)
        _check(lib().snp_set_temporal(h, w.ctypes.data_as(C.c_void_p), SNP_MEM_HOST, _stream(stream)))


def bin_sort(h, opts, stream=None):
    _check(lib().snp_bin_sort(h, C.byref(opts), _stream(stream)))


def render(h, opts, out, stream=None):
    _check(lib().snp_render(h, C.byref(opts), _ptr(out), _stream(stream)))


def render_views(h, cams, opts, out, stream=None, xi_t=None):
    arr = cams if isinstance(cams, C.Array) else make_cameras(cams)
    if xi_t is None:
        _check(lib().snp_render_views(h, arr, len(arr), C.byref(opts), _ptr(out), _stream(stream)))
    else:
        project(h, arr, stream, xi_t)
        bin_sort(h, opts, stream)
        render(h, opts, out, stream)


def render_backward(h, opts, grad_rgba, grads, stream=None, fwd_rgba=None):
    """K7: adds dL/d{w1, b1, w2, b2, sh} and, when ``grads`` has "centers", "rotations" and
    "scales", the geometry gradients (dict of CUDA tensors shaped like the scene's arrays)
    for grad_rgba = dL/d(out RGBA) (CUDA tensor [V, H, W, 4]); fwd_rgba: the forward image
    the gradients refer to (the render's out), or None (rendered again)."""
    _check(lib().snp_render_backward_ex(h, C.byref(opts), _ptr(fwd_rgba), _ptr(grad_rgba), _ptr(grads["w1"]),
                                        _ptr(grads["b1"]), _ptr(grads["w2"]), _ptr(grads["b2"]), _ptr(grads["sh"]),
                                        _ptr(grads.get("centers")), _ptr(grads.get("rotations")),
                                        _ptr(grads.get("scales")), _stream(stream)))


# P:735 learning rates (MLP 1e-3, means 1.6e-4, scales 5e-3, quaternions 1e-3, SH 2.5e-3)
PAPER_LR = {"centers": 1.6e-4, "rotations": 1e-3, "scales": 5e-3, "w1": 1e-3, "b1": 1e-3, "w2": 1e-3, "b2": 1e-3,
            "sh": 2.5e-3}


def loss_l1(out_rgba, target_rgb, grad_rgba, loss, stream=None):
    """L1 photometric loss: writes dL/d(out) into grad_rgba and adds L to loss (CUDA
    tensors: out [..., 4], target [..., 3], loss a 1-element float tensor)."""
    n = out_rgba.numel() // 4
    _check(lib().snp_loss_l1(_ptr(out_rgba), _ptr(target_rgb), n, _ptr(grad_rgba), _ptr(loss), _stream(stream)))


def loss_3dgs(h, out_rgba, target_rgb, grad_rgba, loss, lambda_dssim=0.2, stream=None, step_views=None):
    """3DGS's loss (1 - lambda) L1 + lambda (1 - SSIM): out [V, H, W, 4], target
    [V, H, W, 3] CUDA tensors; writes dL/d(out) into grad_rgba, adds L to loss.  With
    step_views (snp_loss_3dgs_part) the means divide by that many views: parts of a
    step add up to the whole step's loss and gradient."""
    V, H, W = int(out_rgba.shape[0]), int(out_rgba.shape[1]), int(out_rgba.shape[2])
    if step_views is None:
        _check(lib().snp_loss_3dgs(h, _ptr(out_rgba), _ptr(target_rgb), V, H, W, float(lambda_dssim),
                                   _ptr(grad_rgba), _ptr(loss), _stream(stream)))
    else:
        _check(lib().snp_loss_3dgs_part(h, _ptr(out_rgba), _ptr(target_rgb), V, H, W, int(step_views),
                                        float(lambda_dssim), _ptr(grad_rgba), _ptr(loss), _stream(stream)))


def scale_regularizer(h, weight, grad_scales, loss, stream=None):
    _check(lib().snp_scale_regularizer(h, float(weight), _ptr(grad_scales), _ptr(loss), _stream(stream)))


def adam_step(h, grads, step, lr=None, beta1=0.9, beta2=0.999, eps=1e-15, stream=None):
    """One Adam step on the scene's parameters (grads: dict of CUDA tensors by FIELDS)."""
    lr = dict(PAPER_LR, **(lr or {}))
    ptrs = (C.c_void_p * 8)(*[_ptr(grads[f]) for f in FIELDS])
    lrs = (C.c_float * 8)(*[float(lr[f]) for f in FIELDS])
    _check(lib().snp_adam_step(h, ptrs, lrs, float(beta1), float(beta2), float(eps), int(step), _stream(stream)))


def copy_params(h, dst, stream=None):
    """Copies the scene's current parameters into dst (dict by FIELDS of CUDA tensors or
    numpy arrays, all on the same side)."""
    first = dst[FIELDS[0]]
    mem = SNP_MEM_DEVICE if _is_device(first) else SNP_MEM_HOST
    ptrs = (C.c_void_p * 8)(*[_ptr(dst[f]) for f in FIELDS])
    _check(lib().snp_get_params(h, ptrs, mem, _stream(stream)))


def destroy(h):
    if h:
        _check(lib().snp_destroy(h))


def set_pending_limit(h, k):
    _check(lib().snp_set_pending_limit(h, int(k)))


def set_record(h, on=True):
    """snp_set_record: renders of one camera batch also record their composited hits for
    the next backward (training)."""
    _check(lib().snp_set_record(h, 1 if on else 0))


def set_binning(h, flags):
    """snp_set_binning: SNP_BIN_CONIC_TILES | SNP_BIN_TILE_DEPTH (0 = rect binning)."""
    _check(lib().snp_set_binning(h, int(flags)))


def get_debug_counters(h, n=56, stream=None):
    out = np.zeros(n, np.uint64)
    _check(lib().snp_get_debug_counters(h, out.ctypes.data, int(n), _stream(stream)))
    return out


def get_stats(h, stream=None):
    s = Stats()
    _check(lib().snp_get_stats(h, C.byref(s), _stream(stream)))
    return {f: int(getattr(s, f)) for f, _ in Stats._fields_}


def get_binning(h, n, n_views, tiles, stream=None):
    """Host copies of (rects [V*n,4] int32, depth [V*n] u32, sorted keys, sorted ids, ranges [V*tiles,2])."""
    L = lib()
    rects = np.zeros((n_views * n, 4), np.int32)
    depth = np.zeros(n_views * n, np.uint32)
    ranges = np.zeros((n_views * tiles, 2), np.uint32)
    nd = C.c_int64(0)
    _check(L.snp_get_binning(h, rects.ctypes.data, depth.ctypes.data, None, None, 0, C.byref(nd),
                             ranges.ctypes.data, _stream(stream)))
    m = max(int(nd.value), 0)
    keys = np.zeros(max(m, 1), np.uint64)
    ids = np.zeros(max(m, 1), np.uint32)
    _check(L.snp_get_binning(h, None, None, keys.ctypes.data, ids.ctypes.data, m, C.byref(nd), None,
                             _stream(stream)))
    return rects, depth, keys[:m], ids[:m], ranges


class Renderer:
    """Convenience owner of one scene handle (torch tensors for device outputs)."""

    def __init__(self, scene, device=0, stream=None):
        self.h = create_scene(scene, device, stream)
        self.device = device

    def render(self, cams, out, background=(0, 0, 0), transmittance_floor=1e-4, stream=None, **kw):
        opts = make_opts(background, transmittance_floor, **kw)
        render_views(self.h, cams, opts, out, stream)
        return out

    def stats(self, stream=None):
        return get_stats(self.h, stream)

    def close(self):
        if self.h:
            destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
