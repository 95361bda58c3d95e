"""B200-native (sm_100a) forward splatting rasterizer for splattable neural
primitives (arXiv 2510.08491).

The product is ``libsnp.so`` (C ABI in ``include/snp.h``); ``snp`` is its thin
ctypes binding.  PyTorch, when used, only supplies device memory and streams.
"""
from . import snp  # noqa: F401
from .snp import (Renderer, SnpError, bin_sort, create_scene, destroy, get_binning,  # noqa: F401
                  get_stats, make_cameras, make_opts, project, render, render_views,
                  set_pending_limit, update_scene)

__all__ = ["snp", "Renderer", "SnpError", "create_scene", "project", "bin_sort", "render",
           "render_views", "destroy", "get_stats", "get_binning", "make_cameras", "make_opts",
           "set_pending_limit", "update_scene"]
